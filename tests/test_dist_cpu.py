"""World-size-2 gloo tests (CPU) of the multi-process host logic: IPC-handle
exchange, max-over-ranks timing, and bench.py's aggregation helpers."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2110_04478_b200.dist import allgather_bytes, barrier, init_from_env, max_over_ranks
    r, w, local, group = init_from_env("gloo")
    try:
        handles = allgather_bytes(bytes([r]) * 64, group)
        m = max_over_ranks(1.5 + r, group)
        barrier(group)
        q.put((r, [h[0] for h in handles], len(handles[0]), m))
    finally:
        dist.destroy_process_group()


def test_gloo_handle_exchange_and_max():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for r, firsts, n, m in res:
        assert firsts == [0, 1] and n == 64 and m == 2.5


def _plan_worker(rank, world, port, q, same):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2110_04478_b200 import themis as th
    from paper_2110_04478_b200.dist import check_same_plan, init_from_env
    r, w, local, group = init_from_env("gloo")
    try:
        # e.g. a per-rank measured H2D rate leaking into chunk_release_ns
        release = 1000 if same else 1000 + r
        plan = th.Plan(th.Topology((2, 2), (100000, 50000)), th.ALLREDUCE, 1 << 24, 16, chunk_release_ns=release)
        try:
            check_same_plan(plan, group)
            q.put((r, "ok"))
        except ValueError as e:
            q.put((r, str(e)))
        plan.close()
    finally:
        dist.destroy_process_group()


def test_gloo_plan_consistency_check():
    """Plans must be identical on every rank (R22); the host-side check
    catches a rank-dependent input before any kernel runs."""
    for same in (True, False):
        port = _free_port()
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=_plan_worker, args=(r, 2, port, q, same)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(120)
            assert p.exitcode == 0
        res = dict(q.get() for _ in range(2))
        if same:
            assert res == {0: "ok", 1: "ok"}
        else:
            assert all("ranks [1]" in v for v in res.values())


def test_rank_layout_helpers():
    from bench import logical_layout
    lay = logical_layout((2, 2, 2), 4)
    assert lay["V"] == 2 and lay["cross_gpu_dims"] == [1, 2]
    lay = logical_layout((2, 2, 2), 2)
    assert lay["V"] == 4 and lay["cross_gpu_dims"] == [2]
    lay = logical_layout((2, 2, 2), 1)
    assert lay["V"] == 8 and lay["cross_gpu_dims"] == []


def _cal_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    from paper_2110_04478_b200.dist import init_from_env
    r, w, local, group = init_from_env("gloo")
    try:
        # each rank measured slightly different per-dim rates
        rates = [412.3 + 3 * r, 207.9 - r, 101.4 + 0.5 * r]
        q.put((r, bench.calibrated_bw(rates, group)))
    finally:
        dist.destroy_process_group()


def test_gloo_calibrated_bw_identical_on_every_rank():
    """bench's calibrated-BW plan input: min over ranks, quantised -- the same
    tuple on every rank (else the ranks would launch different plans, R22)."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_cal_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    assert res[0][1] == res[1][1]
    q_ = 412.3 / 32                                          # min over ranks, quantum = fastest / 32
    assert res[0][1] == tuple(round(x / q_) * round(q_ * 1000) for x in (412.3, 206.9, 101.4))
