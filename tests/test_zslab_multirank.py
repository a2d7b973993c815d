"""Multi-rank z-slab path (config C5, SURVEY.md §8 e) through the host-staged
transport (shl_homogenize_zslab_host + zslab.TorchSlabTransport over gloo).

* CPU (world size 2 and 3, gloo): the transport's ring exchange and sums --
  the host logic every rank of the 8-GPU run executes between its kernels.
* GPU (world size 2, both ranks on cuda:0): shl_homogenize_zslab_host end to
  end.  No kernel waits on another rank (each exchange is stream sync -> D2H
  -> gloo -> H2D), so two ranks may share one GPU; C^H must equal the
  undecomposed solve and the in-process two-slab emulation.
"""
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


def _init(rank, world, port):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    return dist


def transport_worker(rank, world, port, q):
    dist = _init(rank, world, port)
    from paper_2511_04025_b200.zslab import TorchSlabTransport
    t = TorchSlabTransport()
    # plane sizes differ per rank (and one is empty), as ghost planes do
    n_up = [5, 0, 7][rank % 3]      # what I send to rank+1 (its recv_lo)
    n_down = [3, 4, 0][rank % 3]    # what I send to rank-1 (its recv_hi)
    lo, hi = (rank - 1) % world, (rank + 1) % world
    send_hi = np.full(n_up, 100.0 * rank + 1, np.float64)
    send_lo = np.full(n_down, 100.0 * rank + 2, np.float64)
    recv_lo = np.zeros([5, 0, 7][lo % 3], np.float64)
    recv_hi = np.zeros([3, 4, 0][hi % 3], np.float64)
    t.ring_exchange(send_hi, send_lo, recv_lo, recv_hi)
    buf = np.arange(4, dtype=np.float32) * (rank + 1)
    t.allreduce_sum(buf)
    q.put((rank, recv_lo.tolist(), recv_hi.tolist(), buf.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_transport_ring_and_sum(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=transport_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(world):
        rank, rlo, rhi, buf = q.get(timeout=120)
        out[rank] = (rlo, rhi, buf)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    tot = sum(range(1, world + 1))
    for rank in range(world):
        lo, hi = (rank - 1) % world, (rank + 1) % world
        rlo, rhi, buf = out[rank]
        assert rlo == [100.0 * lo + 1] * [5, 0, 7][lo % 3]   # lo's upward plane
        assert rhi == [100.0 * hi + 2] * [3, 4, 0][hi % 3]   # hi's downward plane
        assert buf == [float(i * tot) for i in range(4)]


def zslab_worker(rank, world, port, r, prec, q):
    dist = _init(rank, world, port)
    import paper_2511_04025_b200 as S
    from paper_2511_04025_b200.zslab import TorchSlabTransport
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), 1)
    opt = S.HomogenizeOptions(residual_tol=1e-6, precision=prec)
    ctx = S.Context(0)
    res = S.homogenize_zslab_host(d, S.ShellParams(), S.BaseMaterial(), r, rank, world, TorchSlabTransport(),
                                  opt, ctx)
    q.put((rank, res.tensor.tolist(), [int(v) for v in res.iterations]))
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("r,prec", [(32, "fp64"), (64, "mixed")])
def test_zslab_host_transport_two_ranks(S, r, prec):
    d = S.random_design(S.RandomDesignSpec("cubic_octant", 8, 2, -1.0, 1.0), 1)
    opt = S.HomogenizeOptions(residual_tol=1e-6, precision=prec)
    ref = S.homogenize(d, S.ShellParams(), S.BaseMaterial(), r, opt)
    emu = S.homogenize_slabs(d, S.ShellParams(), S.BaseMaterial(), r, 2, opt)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=zslab_worker, args=(k, 2, port, r, prec, q)) for k in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, C, its in res:
        C = np.array(C)
        assert np.array_equal(C, res[0][1] if rank else C)  # every rank holds the same C^H
        assert np.linalg.norm(C - emu.tensor) <= 1e-12 * np.linalg.norm(emu.tensor)
        assert np.linalg.norm(C - ref.tensor) <= 1e-6 * np.linalg.norm(ref.tensor)
        assert max(abs(a - b) for a, b in zip(its, emu.iterations)) <= 1
