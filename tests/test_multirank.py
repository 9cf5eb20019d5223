"""Multi-process (world_size 2, gloo, CPU) checks of bench.py's N>1 logic:
each rank draws its own sub-domain, the step time is the max over ranks and
the reported value is all ranks' particles over that time (weak scaling)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    ws_, rank_, _ = bench.dist_env()
    pos, h = bench.subdomain(2, 2000, rank_)
    ms = 10.0 + 5.0 * rank_           # rank 1 is the slow one
    mx = bench.max_over_ranks(ms)
    q.put((rank_, ws_, float(pos[0, 0]), float(h.sum()), mx, bench.weak_value(2000, ws_, mx)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, ws0, x0, hs0, m0, v0), (r1, ws1, x1, hs1, m1, v1) = res
    assert ws0 == ws1 == 2 and (r0, r1) == (0, 1)
    assert x0 != x1 and hs0 != hs1                 # independent sub-domains
    assert m0 == m1 == 15.0                        # max over ranks
    assert v0 == v1 == pytest.approx(2 * 2000 / 15e-3)


def _worker_replicated(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    _, rank_, _ = bench.dist_env()
    pos_np, h_np, pos, h = bench.replicated_inputs(2, 3000, rank_, "cpu")
    had_data = pos_np is not None
    bench.broadcast_inputs(pos, h)        # gloo stands in for NCCL here
    ms = bench.max_over_ranks(8.0 + rank_)
    cfg = bench.config_block(2, 3000, ws, "replicated")
    q.put((rank_, had_data, float(pos.sum()), float(h.sum()), ms, bench.strong_value(pos.shape[0], ms),
           cfg["parallelism"], cfg.get("N_total")))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_replicated_gloo():
    """--mode replicated: rank 0 alone draws the set, the broadcast gives every
    rank the same bits, the value is the one set over the max step time."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_replicated, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, d0, ps0, hs0, m0, v0, par0, n0), (r1, d1, ps1, hs1, m1, v1, par1, n1) = res
    assert d0 and not d1
    assert ps0 == ps1 and hs0 == hs1                  # identical particle sets after the broadcast
    assert m0 == m1 == 9.0 and v0 == v1 == pytest.approx(3000 / 9e-3)
    assert "replicated" in par0 and n0 == n1 == 3000


def test_single_process_identity():
    import bench
    assert bench.max_over_ranks(3.5) == 3.5
    a = bench.subdomain(1, None, 0)
    b = bench.subdomain(1, None, 1)
    assert a[0].shape == b[0].shape and not np.array_equal(a[0], b[0])
