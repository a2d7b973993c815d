"""Config C5: one large design (256^3) z-slab-decomposed across GPUs over NCCL.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        -m paper_2511_04025_b200.zslab --r 256 --seed 1

Rank 0 creates the NCCL unique id through the library (shl_nccl_unique_id),
torch.distributed (gloo) broadcasts the 128 bytes, and every rank calls
shl_homogenize_zslab for its slab; C^H is identical on every rank.  With one
process the same slab code runs emulated (`--emulate G`).  `--transport host`
runs the per-rank path over torch.distributed (gloo) through the host-staged
transport (TorchSlabTransport) instead of NCCL.  The default
preconditioner is multigrid: level 0 on the slabs (ghost exchange before every
sweep, restriction all-reduced), coarse levels replicated on every rank.
"""
from __future__ import annotations

import argparse
import json
import os

import numpy as np


class TorchSlabTransport:
    """Host-staged z-slab transport over torch.distributed (any backend that
    moves CPU tensors, e.g. gloo): the callbacks of shl_homogenize_zslab_host.
    Ring neighbours: rank-1 (lo) and rank+1 (hi), periodic; tag 1 carries the
    plane sent upward, tag 2 the plane sent downward, so two ranks (lo == hi)
    still pair every message."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce_sum(self, buf: np.ndarray) -> None:
        import torch
        t = torch.from_numpy(buf)  # shares memory with the staging buffer
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def ring_exchange(self, send_hi, send_lo, recv_lo, recv_hi) -> None:
        import torch
        lo, hi = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        reqs = []
        if send_hi.size:
            reqs.append(self.dist.isend(torch.from_numpy(send_hi), hi, group=self.group, tag=1))
        if send_lo.size:
            reqs.append(self.dist.isend(torch.from_numpy(send_lo), lo, group=self.group, tag=2))
        if recv_lo.size:
            reqs.append(self.dist.irecv(torch.from_numpy(recv_lo), lo, group=self.group, tag=1))
        if recv_hi.size:
            reqs.append(self.dist.irecv(torch.from_numpy(recv_hi), hi, group=self.group, tag=2))
        for q in reqs:
            q.wait()


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, default=256)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--precision", default="mixed")
    ap.add_argument("--emulate", type=int, default=0, help="G slabs on one device")
    ap.add_argument("--preconditioner", default="auto", choices=["auto", "gmg", "jacobi"])
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"])
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
        if a.transport == "host":
            res = S.homogenize_zslab_host(d, S.ShellParams(), S.BaseMaterial(), a.r, rank, world,
                                          TorchSlabTransport(), opt, ctx)
        else:
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
