"""Design-space sweep sharded across GPUs (BASELINE.json config C4; SPEC's
`sample_campaign`, which the reference specifies but does not implement).

One process per GPU (torchrun).  Designs are independent, so there is no
data-path collective: ranks pull chunks of design indices from a shared
atomic counter (a torch.distributed TCPStore -- a dynamic work queue, because
PCG iteration counts vary ~6x between designs), homogenize each chunk with
one `shl_homogenize_batch` call, append every result to a per-rank JSONL log
(checkpoint: a restarted sweep skips indices already logged), and gather the
rows to rank 0 at the end (`gather_object`), which writes the CSV of
`props.make_report` rows.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
        -m paper_2511_04025_b200.sweep --n 4096 --r 64 --out runs/c4
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import time
from typing import Callable, Iterable

import numpy as np

from . import props

DesignFn = Callable[[Iterable[int]], list]  # indices -> list of result dicts


def completed_indices(out_dir: str) -> set[int]:
    done = set()
    for path in glob.glob(os.path.join(out_dir, "rank*.jsonl")):
        with open(path) as f:
            for line in f:
                line = line.strip()
                if not line:
                    continue
                try:
                    done.add(int(json.loads(line)["index"]))
                except (ValueError, KeyError):
                    pass  # torn tail line of a killed run
    return done


def load_rows(out_dir: str) -> dict[int, dict]:
    rows = {}
    for path in sorted(glob.glob(os.path.join(out_dir, "rank*.jsonl"))):
        with open(path) as f:
            for line in f:
                try:
                    row = json.loads(line)
                    rows[int(row["index"])] = row
                except (ValueError, KeyError):
                    pass
    return rows


def run_sweep(n: int, out_dir: str, homogenize_chunk: DesignFn, rank: int = 0, world: int = 1,
              store=None, chunk: int = 8, run_id: str = "sweep", gather=None) -> dict:
    """Pull chunks from the shared counter until exhausted; returns this rank's stats.

    `store` is any object with an atomic `add(key, amount) -> new value`
    (torch.distributed.TCPStore); `gather` collects per-rank row lists on rank 0
    (dist.gather_object wrapper) or None for a single process."""
    os.makedirs(out_dir, exist_ok=True)
    done = completed_indices(out_dir)
    log_path = os.path.join(out_dir, f"rank{rank}.jsonl")
    my_rows, claimed, computed = [], 0, 0
    t0 = time.perf_counter()
    local_next = 0
    with open(log_path, "a") as log:
        while True:
            if store is not None:
                hi = int(store.add(f"{run_id}/next", chunk))
            else:
                local_next += chunk
                hi = local_next
            lo = hi - chunk
            if lo >= n:
                break
            claimed += 1
            todo = [i for i in range(lo, min(hi, n)) if i not in done]
            if not todo:
                continue
            for row in homogenize_chunk(todo):
                row["rank"] = rank
                log.write(json.dumps(row) + "\n")
                my_rows.append(row)
                computed += 1
            log.flush()
            os.fsync(log.fileno())
    wall = time.perf_counter() - t0
    stats = {"rank": rank, "chunks": claimed, "designs": computed, "wall_s": wall}
    if gather is not None:
        gather(stats)
    return stats


def write_csv(out_dir: str, n: int) -> str:
    rows = load_rows(out_dir)
    path = os.path.join(out_dir, "results.csv")
    with open(path, "w") as f:
        f.write("index,seed,status,iterations_max,t_fwd_ms," + props.CSV_HEADER + "\n")
        for i in range(n):
            row = rows.get(i)
            if row is None:
                f.write(f"{i},,missing,,," + props.csv_row(None) + "\n")
                continue
            rep = None
            if row["status"] == 0:
                try:
                    rep = props.make_report(np.array(row["C"]), row["volume_ratio"])
                except props.SingularTensorError:
                    rep = None
            f.write(f"{i},{row['seed']},{row['status']},{max(row['iterations'])},"
                    f"{row['t_fwd_ms']:.4f}," + props.csv_row(rep) + "\n")
    return path


def device_chunk_fn(r: int, tol: float, precision: str, device: int, seed0: int = 0,
                    symmetry: str = "cubic_octant", n_pre: int = 8, lanes: int = 4) -> DesignFn:
    """Chunk evaluator on the local GPU through shl_homogenize_batch, `lanes`
    designs of a chunk in flight at once."""
    from . import api as S
    ctx = S.Context(device)
    spec = S.RandomDesignSpec(symmetry, n_pre, 2, -1.0, 1.0)
    opt = S.HomogenizeOptions(residual_tol=tol, precision=precision)

    def fn(indices):
        idx = list(indices)
        designs = [S.random_design(spec, seed0 + i) for i in idx]
        Cs, status, stats = S.homogenize_batch(designs, S.ShellParams(), S.BaseMaterial(), r, opt,
                                               ctx=ctx, lanes=lanes)
        return [{"index": i, "seed": seed0 + i, "status": int(st), "C": C.tolist(),
                 "iterations": [int(v) for v in s.iterations], "volume_ratio": s.volume_ratio,
                 "t_fwd_ms": s.timings["t_fwd"], "n_elements": int(s.n_elements)}
                for i, C, st, s in zip(idx, Cs, status, stats)]
    return fn


def main(argv=None):
    import torch
    import torch.distributed as dist

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--r", type=int, default=64)
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--precision", default="mixed")
    ap.add_argument("--chunk", type=int, default=8)
    ap.add_argument("--seed0", type=int, default=0)
    ap.add_argument("--out", default="runs/sweep")
    ap.add_argument("--lanes", type=int, default=4, help="designs in flight per GPU")
    a = ap.parse_args(argv)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    store, gather = None, None
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        host = os.environ.get("MASTER_ADDR", "127.0.0.1")
        port = int(os.environ.get("MASTER_PORT", "29500")) + 1
        store = dist.TCPStore(host, port, world, rank == 0)

        def gather(stats):
            out = [None] * world if rank == 0 else None
            dist.gather_object(stats, out, dst=0)
            if rank == 0:
                print(json.dumps({"ranks": out}))
    fn = device_chunk_fn(a.r, a.tol, a.precision, local, a.seed0, lanes=a.lanes)
    stats = run_sweep(a.n, a.out, fn, rank, world, store, a.chunk, f"sweep-{a.r}-{a.n}", gather)
    if world > 1:
        dist.barrier()
    if rank == 0:
        path = write_csv(a.out, a.n)
        print(json.dumps({"csv": path, **stats}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
