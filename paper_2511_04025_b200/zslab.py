"""Config C5: one large design (256^3) z-slab-decomposed across GPUs over NCCL.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        -m paper_2511_04025_b200.zslab --r 256 --seed 1

Rank 0 creates the NCCL unique id through the library (shl_nccl_unique_id),
torch.distributed (gloo) broadcasts the 128 bytes, and every rank calls
shl_homogenize_zslab for its slab; C^H is identical on every rank.  With one
process the same slab code runs emulated (`--emulate G`).  The default
preconditioner is multigrid: level 0 on the slabs (ghost exchange before every
sweep, restriction all-reduced), coarse levels replicated on every rank.
"""
from __future__ import annotations

import argparse
import json
import os

import numpy as np


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, default=256)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--precision", default="mixed")
    ap.add_argument("--emulate", type=int, default=0, help="G slabs on one device")
    ap.add_argument("--preconditioner", default="auto", choices=["auto", "gmg", "jacobi"])
    a = ap.parse_args(argv)
    from . import api as S
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), a.seed)
    opt = S.HomogenizeOptions(residual_tol=a.tol, precision=a.precision, preconditioner=a.preconditioner)
    ctx = S.Context(local)
    if world == 1:
        if a.emulate >= 2:
            res = S.homogenize_slabs(d, S.ShellParams(), S.BaseMaterial(), a.r, a.emulate, opt, ctx)
        else:
            res = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), a.r, opt, ctx)
    else:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        res = S.homogenize_zslab(d, S.ShellParams(), S.BaseMaterial(), a.r, obj[0], rank, world,
                                 opt, ctx)
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"r": a.r, "ranks": world, "emulated_slabs": a.emulate,
                          "C": np.round(res.tensor, 12).tolist(),
                          "iterations": [int(v) for v in res.iterations],
                          "timings_ms": res.timings, "nodes": res.stats.n_nodes}))


if __name__ == "__main__":
    main()
