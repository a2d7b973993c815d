"""Generate tests/golden/geometry_fixtures.npz from the reference's OWN
geomio/voxel code (oracle/_ref), for the export formats either side of the
hot path (SURVEY.md §8 f, N4):

  extract_isosurface  geomio.hpp:45-108   vertices + triangles, in order
  export_mesh         geomio.hpp:272-316  binary STL and OBJ bytes
  VoxelMesh::write_raw voxel.hpp:105-114  r^3 occupancy bytes

Run in the dev container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_golden_geom.py

Small outputs are stored whole, larger ones as SHA-256 digests.
"""
from __future__ import annotations

import hashlib
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cases():
    rd = lambda sym, n, s: (lambda: O.random_design(sym, n, 2, -1, 1, s, use_ref=True))  # noqa: E731
    return [("seeded_3", rd("cubic_octant", 4, 3), (8, 16), (32,)),
            ("seeded_2024", rd("cubic_octant", 4, 2024), (), (32, 64)),
            ("c3_seed1", rd("cubic_octant", 8, 1), (), (64, 128)),
            ("none64_seed7", rd("none", 64, 7), (), (32,)),
            ("gyroid", O.gyroid_design, (), (32, 64)),
            ("plane_z", lambda: O.plane_design_z(0.5 / 32), (16,), ())]


def main() -> None:
    if O.ref() is None:
        raise SystemExit("oracle/_ref not built: make -C oracle ref (needs /root/reference)")
    arrays, keys, digests = {}, [], []
    tmp = tempfile.mkdtemp()
    for name, make, whole, digest in cases():
        d = make()
        arrays[f"{name}/positions"] = d.positions
        arrays[f"{name}/signs"] = d.signs
        arrays[f"{name}/weights"] = d.weights
        arrays[f"{name}/symmetry"] = np.array([O.SYM[d.symmetry]])
        for r in tuple(whole) + tuple(digest):
            g = O.sample_grid(d, r, use_ref=True)
            v, t = O.extract_isosurface(g, use_ref=True)
            raw_path = os.path.join(tmp, "m.raw")
            O.ref_write_raw(g, raw_path)
            raw = np.fromfile(raw_path, np.uint8)
            key = f"{name}/r{r}"
            arrays[f"{key}/counts"] = np.array([len(v), len(t)], np.int64)
            if r in whole:
                arrays[f"{key}/vertices"] = v
                arrays[f"{key}/triangles"] = t
                arrays[f"{key}/raw"] = raw
            keys.append(key)
            digests.append([sha(v), sha(t), sha(raw)])
    # export_mesh bytes of one small isosurface
    v = arrays["seeded_3/r8/vertices"]
    t = arrays["seeded_3/r8/triangles"]
    for fmt in ("stl", "obj"):
        path = os.path.join(tmp, f"m.{fmt}")
        O.ref_export_mesh(v, t, path, fmt)
        arrays[f"export/{fmt}"] = np.fromfile(path, np.uint8)
    arrays["digest/keys"] = np.array(keys)
    arrays["digest/values"] = np.array(digests)
    np.savez_compressed(os.path.join(HERE, "geometry_fixtures.npz"), **arrays)
    print(f"wrote {len(arrays)} arrays, {len(keys)} isosurface/raw digests")


if __name__ == "__main__":
    main()
