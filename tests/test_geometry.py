"""Export formats either side of the hot path (SURVEY.md §8 f, N4):
marching cubes (geomio.hpp:45-108), export_mesh (:272-316) and
VoxelMesh::write_raw (voxel.hpp:105-114).

Golden fixtures: tests/golden/geometry_fixtures.npz, generated from the
reference's own geomio/voxel code (oracle/_ref) by make_golden_geom.py.
CPU tests pin the oracle restatement and the host-side writers against them;
the GPU tests pin the device kernels (bit-exact vertices, identical triangle
lists and order, identical bytes).
"""
import hashlib
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "geometry_fixtures.npz")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gold():
    z = np.load(GOLD)
    g = {k: z[k] for k in z.files}
    g["_digest"] = dict(zip([str(k) for k in g["digest/keys"]], [list(v) for v in g["digest/values"]]))
    return g


def design_of(gold, name, mod):
    """Design from the fixture, as an oracle.Design or a product DesignParams."""
    sym = {0: "none", 1: "cubic_octant", 2: "tetrahedral"}[int(gold[f"{name}/symmetry"][0])]
    pos, sg, w = gold[f"{name}/positions"], gold[f"{name}/signs"], gold[f"{name}/weights"]
    if hasattr(mod, "Design"):
        return mod.Design(sym, 2, pos, sg, w)
    return mod.DesignParams(symmetry=sym, truncation=2, positions=pos, signs=sg, weights=w)


def keys(gold):
    return sorted(gold["_digest"])


# ------------------------------------------------------------------ CPU
def test_oracle_isosurface_matches_reference(O, gold):
    for key in keys(gold):
        name, rr = key.split("/")
        r = int(rr[1:])
        v, t = O.extract_isosurface(O.sample_grid(design_of(gold, name, O), r))
        dv, dt, _ = gold["_digest"][key]
        assert (len(v), len(t)) == tuple(gold[f"{key}/counts"]), key
        assert sha(v) == dv and sha(t) == dt, key
        if f"{key}/vertices" in gold:
            np.testing.assert_array_equal(v, gold[f"{key}/vertices"])
            np.testing.assert_array_equal(t, gold[f"{key}/triangles"])


def test_raw_bytes_host_writer_matches_reference(S, O, gold, tmp_path):
    """VoxelMesh.raw_bytes / write_raw (host) on the oracle's mesh == the reference file."""
    for key in keys(gold):
        name, rr = key.split("/")
        r = int(rr[1:])
        if r > 64:
            continue
        m = O.build_reduced_mesh(O.sample_grid(design_of(gold, name, O), r))
        el = np.flatnonzero(m.occupancy.reshape(-1))
        vm = S.api.VoxelMesh(r, el.astype(np.uint32), m.beta.reshape(-1)[el], m.full_fallback)
        raw = vm.raw_bytes()
        assert sha(raw) == gold["_digest"][key][2], key
        if f"{key}/raw" in gold:
            path = str(tmp_path / "m.raw")
            vm.write_raw(path)
            np.testing.assert_array_equal(np.fromfile(path, np.uint8), gold[f"{key}/raw"])


@pytest.mark.parametrize("fmt", ["stl", "obj"])
def test_export_mesh_bytes_match_reference(S, gold, tmp_path, fmt):
    mesh = S.api.TriMesh(gold["seeded_3/r8/vertices"], gold["seeded_3/r8/triangles"])
    path = str(tmp_path / f"m.{fmt}")
    S.api.export_mesh(mesh, path, fmt)
    np.testing.assert_array_equal(np.fromfile(path, np.uint8), gold[f"export/{fmt}"])


def test_export_mesh_errors(S, tmp_path):
    empty = S.api.TriMesh(np.zeros((0, 3)), np.zeros((0, 3), np.uint32))
    with pytest.raises(S.api.ValidationError):
        S.api.export_mesh(empty, str(tmp_path / "e.stl"))
    one = S.api.TriMesh(np.eye(3), np.array([[0, 1, 2]], np.uint32))
    with pytest.raises(S.api.IoError):
        S.api.export_mesh(one, str(tmp_path / "missing" / "e.stl"))


def test_mc_table_matches_reference():
    """The packed triangulation equals the reference's mc::kTriTable (dev container only)."""
    src = "/root/reference/proj/include/shellular/mc_tables.hpp"
    if not os.path.exists(src):
        pytest.skip("reference sources not present")
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen", os.path.join(HERE, "..", "tools", "gen_mc_table.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    table = gen.read_tri_table(src)
    hdr = open(os.path.join(HERE, "..", "paper_2511_04025_b200", "csrc", "mc_table.h")).read()
    words = [int(w, 16) for w in __import__("re").findall(r"0x([0-9a-f]{16})ull", hdr)]
    assert gen.unpack(words) == [[v for v in row if v != -1] for row in table]
    # the edge mask derived in the kernels == kEdgeTable
    text = open(src).read()
    body = text[text.index("kEdgeTable"):text.index("kTriTable")]
    edge_table = [int(x, 16) for x in __import__("re").findall(r"0x[0-9a-f]+", body)]
    ea = lambda k: k if k < 8 else k - 8  # noqa: E731
    eb = lambda k: (k + 1) % 4 if k < 4 else (4 + (k - 3) % 4 if k < 8 else k - 4)  # noqa: E731
    derived = [sum(1 << e for e in range(12) if ((c >> ea(e)) ^ (c >> eb(e))) & 1) for c in range(256)]
    assert derived == edge_table


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_device_isosurface_matches_reference(S, gold):
    for key in keys(gold):
        name, rr = key.split("/")
        r = int(rr[1:])
        m = S.extract_isosurface(S.sample_grid(design_of(gold, name, S), r))
        dv, dt, _ = gold["_digest"][key]
        assert (len(m.vertices), len(m.triangles)) == tuple(gold[f"{key}/counts"]), key
        assert sha(m.vertices) == dv and sha(m.triangles) == dt, key


@pytest.mark.gpu
def test_device_voxel_raw_matches_reference(S, gold):
    for key in keys(gold):
        name, rr = key.split("/")
        r = int(rr[1:])
        raw = S.api.voxel_raw(S.sample_grid(design_of(gold, name, S), r))
        assert sha(raw) == gold["_digest"][key][2], key


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2])
def test_device_isosurface_vs_oracle_c3(S, O, seed):
    """Paper setting (128^3, 64 charges): device MC == oracle MC, bit for bit."""
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), seed)
    od = O.random_design("cubic_octant", 8, 2, -1.0, 1.0, seed)
    m = S.extract_isosurface(S.sample_grid(d, 128))
    v, t = O.extract_isosurface(O.sample_grid(od, 128))
    np.testing.assert_array_equal(m.vertices, v)
    np.testing.assert_array_equal(m.triangles, t)


@pytest.mark.gpu
def test_device_isosurface_sphere_and_errors(S):
    R = 0.3
    g = S.sample_grid_fn(lambda x, y, z: (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2 - R * R, 64)
    m = S.extract_isosurface(g)
    assert abs(m.area() - 4 * np.pi * R * R) < 0.02 * 4 * np.pi * R * R
    assert m.triangles.max() < len(m.vertices)
    with pytest.raises(S.api.Error, match="no zero crossing"):
        S.extract_isosurface(S.sample_grid_fn(lambda x, y, z: 1.0 + 0 * x, 8))
    with pytest.raises(S.api.DegenerateDesignError):
        S.extract_isosurface(S.sample_grid_fn(lambda x, y, z: 0.0 * x, 8))
