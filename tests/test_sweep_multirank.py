"""Multi-rank sweep driver on CPU: world_size 2 over gloo (the N>1 host path).

The device evaluator is swapped for the CPU oracle at r=8 (tests may use the
oracle as the checker/stand-in; the product sweep uses shl_homogenize_batch),
so this exercises exactly the host logic that runs on the 8-GPU box: the
TCPStore work queue, per-rank JSONL checkpoints, resume, gather_object and
the props CSV.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_chunk_fn(indices):
    import oracle as O
    rows = []
    for i in indices:
        d = O.random_design("cubic_octant", 4, 2, -1.0, 1.0, i)
        try:
            res = O.homogenize(d, 8, tol=1e-8)
            rows.append({"index": i, "seed": i, "status": 0, "C": res.C.tolist(),
                         "iterations": [int(v) for v in res.iterations],
                         "volume_ratio": res.volume_ratio, "t_fwd_ms": res.timings["t_fwd"],
                         "n_elements": res.n_elements})
        except O.OracleError as e:
            rows.append({"index": i, "seed": i, "status": e.code, "C": [[0.0] * 6] * 6,
                         "iterations": [0] * 6, "volume_ratio": 0.0, "t_fwd_ms": 0.0,
                         "n_elements": 0})
    return rows


def worker(rank, world, port, out_dir, n, chunk, result_file):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2511_04025_b200 import sweep
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            init_method=f"tcp://127.0.0.1:{port}")
    store = dist.TCPStore("127.0.0.1", port + 1, world, rank == 0)

    def gather(stats):
        out = [None] * world if rank == 0 else None
        dist.gather_object(stats, out, dst=0)
        if rank == 0:
            with open(result_file, "w") as f:
                json.dump(out, f)

    sweep.run_sweep(n, out_dir, oracle_chunk_fn, rank, world, store, chunk, "t", gather)
    dist.barrier()
    if rank == 0:
        sweep.write_csv(out_dir, n)
    dist.destroy_process_group()


def run(world, out_dir, n, chunk, tmp_path):
    port = free_port()
    res = str(tmp_path / f"stats_{port}.json")
    mp.spawn(worker, args=(world, port, out_dir, n, chunk, res), nprocs=world, join=True)
    with open(res) as f:
        return json.load(f)


def test_two_rank_sweep_queue_gather_resume(tmp_path):
    out = str(tmp_path / "sweep")
    n = 10
    stats = run(2, out, n, 2, tmp_path)
    assert sum(s["designs"] for s in stats) == n
    assert all(s["chunks"] >= 1 for s in stats)
    # every index exactly once across the per-rank checkpoints
    seen = []
    for r in range(2):
        with open(os.path.join(out, f"rank{r}.jsonl")) as f:
            seen += [json.loads(l)["index"] for l in f if l.strip()]
    assert sorted(seen) == list(range(n))
    lines = open(os.path.join(out, "results.csv")).read().strip().splitlines()
    assert len(lines) == n + 1 and "missing" not in "".join(lines)
    # C^H rows equal a direct single-process evaluation
    import oracle as O
    rows = {}
    for r in range(2):
        for l in open(os.path.join(out, f"rank{r}.jsonl")):
            row = json.loads(l)
            rows[row["index"]] = row
    ref = oracle_chunk_fn([3])[0]
    assert np.allclose(np.array(rows[3]["C"]), np.array(ref["C"]), rtol=1e-12, atol=0)

    # resume: nothing left to do
    stats2 = run(2, out, n, 2, tmp_path)
    assert sum(s["designs"] for s in stats2) == 0

    # lose rank 1's checkpoint: exactly its indices are recomputed
    lost = {json.loads(l)["index"] for l in open(os.path.join(out, "rank1.jsonl")) if l.strip()}
    os.remove(os.path.join(out, "rank1.jsonl"))
    stats3 = run(2, out, n, 2, tmp_path)
    assert sum(s["designs"] for s in stats3) == len(lost)


def test_props_report_isotropic():
    from oracle import direct as D
    from paper_2511_04025_b200 import props
    C = D.isotropic(1.0, 0.3)
    rep = props.make_report(C, 1.0)
    K, G = 1.0 / (3 * 0.4), 1.0 / 2.6
    assert rep["K_V"] == pytest.approx(K) and rep["K_R"] == pytest.approx(K)
    assert rep["G_V"] == pytest.approx(G) and rep["G_R"] == pytest.approx(G)
    assert rep["E_x"] == pytest.approx(1.0) and abs(rep["uai"]) < 1e-12
    assert rep["K_HS_upper"] == pytest.approx(K)  # v = 1: the solid itself
    with pytest.raises(props.SingularTensorError):
        props.make_report(np.diag([1.0, 0.0, 1.0, 1.0, 0.0, 1.0]), 0.5)
