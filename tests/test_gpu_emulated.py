"""GPU parity: the sm_100a executor vs the oracle, all logical ranks emulated
inside one B200's HBM (W = 1, V = P).  Calls go through the C ABI.

* int32: bit-exact vs the plain definition sum_r x_r (mod 2^32);
* f32 / bf16 / f16: bit-exact vs the oracle run step by step with the same
  schedule (same per-stage coordinate-order sums and rounding, R18), and
  within the north_star tolerance of the fp64 sum (1e-5 f32, 1e-2 bf16,
  relative to sum_r |x_r|, F10);
* RS / AG halves against their definitions;
* sizes span several TMA tiles per slice plus a ragged tail.
"""

import numpy as np
import pytest
import torch

from oracle import data as O, engine as E, scheduler as S, topology as T
from paper_2110_04478_b200 import themis as th
from synth import ELEM_SIZE, host_inputs, torch_dtype

pytestmark = pytest.mark.gpu

COLL = {S.AR: th.ALLREDUCE, "RS": th.REDUCE_SCATTER, "AG": th.ALL_GATHER}
TOL = {"f32": 1e-5, "bf16": 1e-2, "f16": 3 * 2.0 ** -11}   # f16: one RNE per RS stage, D = 3


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


KIND_O = {th.RING: T.RING, th.DIRECT: T.DIRECT, th.SWITCH: T.SWITCH}


def oracle_sched(sizes, bw, coll, nbytes, C, policy, intra=E.SCF, kinds=None):
    ok = [KIND_O[k] for k in kinds] if kinds else None
    o = T.Topology.make(sizes, [b for b in bw], ok)
    return S.schedule_collective(o, coll, nbytes, C, S.THEMIS if policy == th.THEMIS else S.BASELINE)


def run_case(sizes, bw, dtype, C, slice_elems, coll=S.AR, policy=th.THEMIS, engine="tma", ctas=None,
             intra=th.SCF, repeat=1, kinds=None, dist="recipe", min_cta_bytes=0, concurrency=1, rotate=1,
             lookahead=1, push=False, ll=False):
    topo = th.Topology(tuple(sizes), tuple(bw), tuple(kinds) if kinds else None)
    P = topo.P
    N = P * C * slice_elems
    esz = ELEM_SIZE[dtype]
    comm = th.Comm(topo, N * esz, ll_bytes=(4 * N * esz if ll else 0))
    if ll:
        comm.set_ll(N * esz)
    comm.set_engine(engine)
    comm.set_timeout(10.0)
    comm.set_min_cta_bytes(min_cta_bytes)
    comm.set_window_rotation(bool(rotate))
    comm.set_lookahead(lookahead)
    comm.set_push(push)
    plan = th.Plan(topo, COLL[coll], N * esz, C, policy, intra, concurrency=concurrency).bind(comm, ctas)
    if ll and not any(k == th.RING and s_ >= 3 for k, s_ in zip(kinds or (), sizes)):
        assert plan.bound_ll()
    try:
        xs = host_inputs(P, N, dtype, dist=dist)
        for it in range(repeat):
            for r in range(P):
                v = comm.rank_view(r, N, dtype)
                src = torch.from_numpy(xs[r].view(np.int16) if dtype == "bf16" else xs[r])
                if dtype == "bf16":
                    src = src.view(torch.bfloat16)
                v.copy_(src.to(v.device))
            th.run(COLL[coll], comm, plan, N, dtype)
            torch.cuda.synchronize()
            comm.status()
        outs = []
        for r in range(P):
            t = comm.rank_view(r, N, dtype).cpu()
            outs.append(t.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else t.numpy())
        return xs, outs
    finally:
        plan.close()
        comm.close()


def check_ar(sizes, bw, dtype, C, slice_elems, policy=th.THEMIS, **kw):
    xs, outs = run_case(sizes, bw, dtype, C, slice_elems, S.AR, policy, **kw)
    N = xs[0].shape[0]
    P = len(xs)
    if dtype == "i32":
        want = O.allreduce_definition(xs, "i32")
        for r in range(P):
            assert np.array_equal(outs[r], want), f"rank {r}"
        return
    sched = oracle_sched(sizes, bw, S.AR, N * ELEM_SIZE[dtype], C, policy, kinds=kw.get("kinds"))
    tree = O.run_schedule(xs, sched, dtype)
    ref = O.allreduce_definition(xs, dtype)
    scale = O.abs_sum(xs, dtype)
    # north_star tolerance on the recipe inputs; on the adversarial "wide"
    # inputs the F10 worst-case bound (one RNE per RS stage: D * 2^-8 for bf16)
    # (F10: one RNE per RS stage -> D * 2^-8 for bf16, D * 2^-11 for f16; a ring
    # dim of P_k >= 3 rounds at each of its P_k - 1 hops, R18)
    kinds_ = kw.get("kinds") or (th.DIRECT,) * len(sizes)
    rounds = sum(pk - 1 if kd == th.RING and pk >= 3 else 1 for pk, kd in zip(sizes, kinds_))
    wide = {"bf16": rounds * 2.0 ** -8, "f16": rounds * 2.0 ** -11, "f32": TOL["f32"]}
    tol = TOL[dtype] if kw.get("dist", "recipe") == "recipe" else max(TOL[dtype], wide[dtype])
    for r in range(P):
        assert np.array_equal(outs[r].view(np.uint8), tree[r].view(np.uint8)), f"rank {r} not bit-exact"
        err = np.abs(O.to_f64(outs[r], dtype) - ref)
        assert np.all(err <= tol * scale)


# slice_elems chosen so one slice spans several 32 KiB TMA tiles plus a ragged
# (non-tile-multiple) tail: 20484 f32 = 81936 B = 2.5 tiles + 16 B.
RAGGED = {"f32": 20484, "i32": 20484, "bf16": 40968, "f16": 40968}


@pytest.mark.parametrize("sizes,bw", [((2,), (1,)), ((4,), (1,)), ((8,), (1,)), ((2, 2), (2, 1)), ((2, 4), (4, 1)),
                                      ((4, 2), (1, 1)), ((2, 2, 2), (1, 1, 1)), ((2, 2, 2), (4, 2, 1)),
                                      ((3, 2), (1, 1)), ((2, 2, 2, 2), (1, 1, 1, 1))])
def test_allreduce_int32_exact(sizes, bw):
    check_ar(sizes, bw, "i32", 4, RAGGED["i32"] // 4 + 3)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("policy", [th.THEMIS, th.BASELINE])
def test_allreduce_float_bitexact_vs_oracle(dtype, policy):
    check_ar((2, 2, 2), (1, 1, 1), dtype, 8, RAGGED[dtype], policy)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_allreduce_wide_values_order_sensitive(dtype):
    """Magnitudes over 16 binades make every float sum inexact, so bit-exactness
    against the oracle checks the summation order (R18) itself."""
    check_ar((2, 2, 2), (1, 1, 1), dtype, 8, RAGGED[dtype], dist="wide")
    check_ar((4, 2), (1, 1), dtype, 4, RAGGED[dtype], dist="wide")


R, Dk = th.RING, th.DIRECT


@pytest.mark.parametrize("sizes,kinds", [((3,), (R,)), ((4,), (R,)), ((8,), (R,)), ((4, 2), (R, Dk)),
                                         ((2, 4), (Dk, R)), ((3, 2, 2), (R, Dk, R)), ((2, 3, 2), (Dk, R, Dk))])
def test_ring_dimensions(sizes, kinds):
    """Table 1 Ring dims run the ring algorithm (P_k - 1 neighbour steps,
    PAPER.md:214/:234/:477): int32 exact and f32 bit-exact against the oracle's
    ring summation order."""
    bw = (1,) * len(sizes)
    check_ar(sizes, bw, "i32", 4, 2052, kinds=kinds)
    check_ar(sizes, bw, "f32", 4, RAGGED["f32"], kinds=kinds, dist="wide")
    check_ar(sizes, bw, "f32", 2, 4100, kinds=kinds, dist="wide", ctas=[3] * len(sizes))


@pytest.mark.parametrize("sizes,kinds", [((2, 2, 2), (Dk, Dk, Dk)), ((4, 2), (R, Dk)), ((3, 2, 2), (R, Dk, R))])
def test_op_windows_several_ops_in_flight(sizes, kinds):
    """Op windows: small ops on CTA windows, several ops of
    a dimension in flight — results unchanged (int32 exact, f32 bit-exact)."""
    bw = (1,) * len(sizes)
    for mcb in (4096, 65536):
        for rot in (1, 0):          # consecutive windows / every narrow op from CTA 0
            check_ar(sizes, bw, "i32", 64, 516, kinds=kinds, min_cta_bytes=mcb, ctas=[12] * len(sizes), rotate=rot)
            check_ar(sizes, bw, "f32", 16, 2052, kinds=kinds, min_cta_bytes=mcb, dist="wide", rotate=rot)


@pytest.mark.parametrize("sizes,kinds", [((2, 2, 2), (Dk, Dk, Dk)), ((4, 2), (R, Dk)), ((3, 2, 2), (R, Dk, R))])
def test_concurrency_aware_plans(sizes, kinds):
    """Plans pre-simulated with k servers per dim run each server's ops on its
    CTA slice (several chunks per dimension in flight)."""
    bw = (1,) * len(sizes)
    for k in (2, 4):
        check_ar(sizes, bw, "i32", 64, 516, kinds=kinds, concurrency=k, ctas=[8] * len(sizes))
        check_ar(sizes, bw, "f32", 16, 2052, kinds=kinds, concurrency=k, dist="wide")


def test_ring_reduce_scatter_all_gather():
    sizes, kinds, C = (4, 2), (R, Dk), 4
    xs, outs = run_case(sizes, (1, 1), "f32", C, 4096, "RS", kinds=kinds, dist="wide")
    N, P = xs[0].shape[0], 8
    sched = oracle_sched(sizes, (1, 1), "RS", N * 4, C, th.THEMIS, kinds=kinds)
    tree = O.run_schedule(xs, sched, "f32")
    blk = N // P
    for r in range(P):
        assert np.array_equal(outs[r][r * blk:(r + 1) * blk], tree[r][r * blk:(r + 1) * blk])
    xs, outs = run_case(sizes, (1, 1), "i32", C, 4096, "AG", kinds=kinds)
    cat = O.all_gather_definition(xs, P)
    for r in range(P):
        assert np.array_equal(outs[r], cat)


def test_ring_needs_tma_engine():
    with pytest.raises(th.ThemisError) as e:
        run_case((3,), (1,), "i32", 2, 1024, kinds=(R,), engine="ldg")
    assert e.value.status == 1


@pytest.mark.parametrize("sizes", [(2, 2, 2), (4, 2), (3, 2, 2)])
def test_custom_orders_non_reversed_ag(sizes):
    """Any RS order x any AG order per chunk (PAPER.md:420-430 Observation 1:
    the AG order may differ from the RS order) executes correctly."""
    import itertools
    import random
    from fractions import Fraction
    rng = random.Random(len(sizes) * 7 + sizes[0])
    D, P, C = len(sizes), int(np.prod(sizes)), 8
    perms = list(itertools.permutations(range(D)))
    rs = [rng.choice(perms) for _ in range(C)]
    ag = [rng.choice(perms) for _ in range(C)]
    topo = th.Topology(tuple(sizes), (1,) * D)
    for dtype, slice_elems in (("i32", 2052), ("f32", 4100)):
        N = P * C * slice_elems
        comm = th.Comm(topo, N * 4)
        comm.set_timeout(10.0)
        plan = th.Plan(topo, th.ALLREDUCE, N * 4, C, rs_orders=rs, ag_orders=ag).bind(comm, [4] * D)
        xs = host_inputs(P, N, dtype, dist="wide")
        for r in range(P):
            comm.rank_view(r, N, dtype).copy_(torch.from_numpy(xs[r]).cuda())
        th.run(th.ALLREDUCE, comm, plan, N, dtype)
        torch.cuda.synchronize()
        comm.status()
        o = T.Topology.make(sizes, (1,) * D)
        sched = S.Schedule(o, S.AR, Fraction(N * 4), C, [S.ChunkSchedule(c, rs[c], ag[c]) for c in range(C)], [], 0)
        want = O.run_schedule(xs, sched, dtype)
        for r in range(P):
            assert np.array_equal(comm.rank_view(r, N, dtype).cpu().numpy(), want[r]), f"rank {r}"
        plan.close()
        comm.close()


def test_allreduce_ldg_engine():
    check_ar((2, 2, 2), (1, 1, 1), "f32", 8, RAGGED["f32"], engine="ldg")
    check_ar((4, 2), (1, 1), "bf16", 4, RAGGED["bf16"], engine="ldg")
    check_ar((8,), (1,), "i32", 2, 1028, engine="ldg")


def test_allreduce_many_chunks_and_fifo():
    check_ar((2, 4), (1, 1), "f32", 64, 256, intra=th.FIFO)
    check_ar((2, 2, 2), (2, 2, 1), "i32", 256, 4)


def test_single_chunk_single_cta_per_dim():
    check_ar((2, 2, 2), (1, 1, 1), "f32", 1, 4096, ctas=[1, 1, 1])


def test_repeated_calls_epochs():
    check_ar((2, 2), (1, 1), "i32", 4, 1024, repeat=3)


@pytest.mark.parametrize("sizes", [(2, 2, 2), (4, 2), (3, 2)])
def test_reduce_scatter_and_all_gather(sizes):
    bw = (1,) * len(sizes)
    C = 4
    xs, outs = run_case(sizes, bw, "i32", C, 2048, "RS")
    P = len(xs)
    want = O.reduce_scatter_definition(xs, "i32", P)
    blk = xs[0].shape[0] // P
    for r in range(P):
        assert np.array_equal(outs[r][r * blk:(r + 1) * blk], want[r])
    xs, outs = run_case(sizes, bw, "i32", C, 2048, "AG")
    cat = O.all_gather_definition(xs, P)
    for r in range(P):
        assert np.array_equal(outs[r], cat)


def test_bf16_reduce_scatter_bitexact():
    sizes, bw, C = (2, 2, 2), (1, 1, 1), 4
    xs, outs = run_case(sizes, bw, "bf16", C, 4096, "RS")
    N = xs[0].shape[0]
    sched = oracle_sched(sizes, bw, "RS", N * 2, C, th.THEMIS)
    tree = O.run_schedule(xs, sched, "bf16")
    blk = N // 8
    for r in range(8):
        assert np.array_equal(outs[r][r * blk:(r + 1) * blk], tree[r][r * blk:(r + 1) * blk])


def test_argument_errors():
    topo = th.Topology((2, 2), (1, 1))
    N = 4 * 4 * 64
    comm = th.Comm(topo, N * 4)
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, 4)
    try:
        with pytest.raises(th.ThemisError) as e:         # not bound
            th.run(th.ALLREDUCE, comm, plan, N, "f32")
        assert e.value.status == 6
        plan.bind(comm)
        with pytest.raises(th.ThemisError) as e:         # count != plan bytes
            th.run(th.ALLREDUCE, comm, plan, N // 2, "f32")
        assert e.value.status == 1
        with pytest.raises(th.ThemisError) as e:         # wrong collective for the plan
            th.run(th.REDUCE_SCATTER, comm, plan, N, "f32")
        assert e.value.status == 6
        with pytest.raises(th.ThemisError) as e:         # outside the heap
            th.themis_allreduce(comm.heap + 8, N, "f32", plan)
        assert e.value.status == 5
        bad = th.Plan(topo, th.ALLREDUCE, 4 * 4 * 3 * 4, 4)   # 48 elements: not a multiple of P*C*4
        bad.bind(comm)
        with pytest.raises(th.ThemisError) as e:
            th.run(th.ALLREDUCE, comm, bad, 48, "f32")
        assert e.value.status == 2
        bad.close()
        with pytest.raises(th.ThemisError):              # too many CTAs for co-residency
            plan.bind(comm, [1000, 1000])
    finally:
        plan.close()
        comm.close()


def test_watchdog_on_missing_peer():
    """Fault injection: a peer that never runs its kernel
    must not hang the GPU — the watchdog latches THEMIS_ERR_TIMEOUT."""
    import ctypes as C
    from paper_2110_04478_b200._lib import MAX_GPUS, check, lib
    topo = th.Topology((2,), (1,))
    N = 2 * 4 * 1024
    sig, stride, hb = th.heap_layout(2, 2, N * 4)
    h0, h1 = C.c_void_p(), C.c_void_p()
    check(lib().themis_heap_alloc(hb, C.byref(h0)))
    check(lib().themis_heap_alloc(hb, C.byref(h1)))        # the silent "peer"'s heap
    heaps = (C.c_void_p * MAX_GPUS)(h0.value, h1.value)
    comm = C.c_void_p()
    tc = topo.to_c()
    check(lib().themis_comm_create(0, 2, C.byref(tc), heaps, hb, stride, C.byref(comm)))
    check(lib().themis_comm_set_timeout(comm, int(0.3e9)))
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, 4)
    check(lib().themis_plan_bind(plan.h, comm, None))
    buf = h0.value + sig
    check(lib().themis_allreduce(buf, N, 0, plan.h, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    st = lib().themis_comm_status(comm)
    assert st == 8
    with pytest.raises(th.ThemisError) as e:                # latched: next call reports it
        check(lib().themis_allreduce(buf, N, 0, plan.h, torch.cuda.current_stream().cuda_stream))
    assert e.value.status == 8
    plan.close()
    lib().themis_comm_free(comm)
    lib().themis_heap_free(h0)
    lib().themis_heap_free(h1)


@pytest.mark.parametrize("ll", [False, True])
def test_watchdog_mid_collective(ll):
    """a peer that passes the entry barrier but never publishes a
    stage's ready flags must time out *after* other dimension groups started
    streaming (producers blocked on ring slots give up on the abort flag) and
    the launch must return with THEMIS_ERR_TIMEOUT latched, not hang.
    W = 2, P = 4 (2x2): GPU 0 is real (ranks 0, 1; dim1 local), "GPU 1" is a
    silent heap on the same device whose ranks 2, 3 are faked as having
    entered (entry epoch + launch hash written into our pads)."""
    import ctypes as C
    import time
    from paper_2110_04478_b200._lib import MAX_GPUS, check, lib
    topo = th.Topology((2, 2), (1, 1))
    P, C_ = 4, 16
    N = P * C_ * (1 << (14 if ll else 18))                  # 64 MiB fp32 per rank: dim1 streams for ms
    sig, stride, hb = th.heap_layout(P, 2, N * 4)
    inbox = (16 << 20) if ll else 0                        # R31 inboxes after the data regions
    hb += 2 * inbox
    h0, h1 = C.c_void_p(), C.c_void_p()
    check(lib().themis_heap_alloc(hb, C.byref(h0)))
    check(lib().themis_heap_alloc(hb, C.byref(h1)))
    heaps = (C.c_void_p * MAX_GPUS)(h0.value, h1.value)
    comm = C.c_void_p()
    tc = topo.to_c()
    check(lib().themis_comm_create(0, 2, C.byref(tc), heaps, hb, stride, C.byref(comm)))
    check(lib().themis_comm_set_timeout(comm, int(0.5e9)))
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, C_, th.THEMIS)
    if ll:   # R31: the silent peer never sends its LL packets
        check(lib().themis_comm_set_ll(comm, inbox, N * 4))
    check(lib().themis_plan_bind(plan.h, comm, None))
    if ll:
        n = C.c_int32()
        check(lib().themis_plan_bound_ll(plan.h, C.byref(n)))
        assert n.value == 1
    hsh = C.c_uint64()
    check(lib().themis_plan_launch_hash(plan.h, N, 0, C.byref(hsh)))
    # signal pad of local rank v: [entry u32 P][exit u32 P][ready u32 P x kMaxOps][ring u64 P x 8 x 160][hash u64 P]
    k_max_ops, ring_off = 1024 * 2 * 8, 4 * (2 * P + P * 1024 * 2 * 8)
    hash_off = ring_off + 8 * P * 8 * 160
    for v in range(2):
        pad = torch.as_tensor(th._CAI(h0.value + v * sig, sig // 4, "<i4"), device="cuda")
        s32 = lambda x: x - (1 << 32) if x >= (1 << 31) else x
        for src in (2, 3):                                  # the fake GPU's ranks entered epoch 1 ...
            pad[src] = 1
            pad[hash_off // 4 + 2 * src] = s32(hsh.value & 0xFFFFFFFF)    # ... with the identical plan
            pad[hash_off // 4 + 2 * src + 1] = s32(hsh.value >> 32)
    assert k_max_ops == 16384
    torch.cuda.synchronize()
    t0 = time.time()
    check(lib().themis_allreduce(h0.value + 2 * sig, N, 0, plan.h, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert time.time() - t0 < 10
    assert lib().themis_comm_status(comm) == 8
    plan.close()
    lib().themis_comm_free(comm)
    lib().themis_heap_free(h0)
    lib().themis_heap_free(h1)


def test_trace_follows_enforced_order():
    topo = th.Topology((2, 2, 2), (1, 1, 1))
    C_ = 8
    N = 8 * C_ * 4096
    comm = th.Comm(topo, N * 4)
    comm.enable_trace(True)
    comm.set_min_cta_bytes(0)   # full-width ops: one op at a time per dim group
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, C_).bind(comm, [4, 4, 4])
    try:
        th.run(th.ALLREDUCE, comm, plan, N, "f32")
        torch.cuda.synchronize()
        tr = comm.fetch_trace(plan).astype(np.int64)
        assert np.all(tr[:, :, 1] >= tr[:, :, 0]) and np.all(tr > 0)
        for k, ops in enumerate(plan.dim_ops()):
            starts = [tr[c, s, 0] for c, s in ops]
            assert starts == sorted(starts), f"dim {k} ran out of the enforced order"
        for c in range(C_):                             # chunk chains respected
            for s in range(1, 6):
                assert tr[c, s, 0] >= tr[c, s - 1, 1] - 2000   # globaltimer granularity slack
    finally:
        plan.close()
        comm.close()


@pytest.mark.parametrize("sizes,bw,C_,dtype,release", [((2, 2), (1, 1), 4, "i32", 0),
                                                       ((2, 2, 2), (1, 1, 1), 16, "f32", 0),
                                                       ((4, 2), (2, 1), 8, "i32", 0),
                                                       ((2, 2, 2), (4000, 2000, 1000), 64, "f32", 20_000)])
def test_host_buffer_entry_point(sizes, bw, C_, dtype, release):
    """themis_allreduce_host streams chunks host -> device -> host around the
    kernel (h2d / d2h flags); three back-to-back calls with fresh inputs, each
    checked: int32 exact, fp32 bit-exact vs the oracle's schedule."""
    topo = th.Topology(sizes, bw)
    P = topo.P
    N = P * C_ * (RAGGED[dtype] // 4 + 3)
    comm = th.Comm(topo, N * 4)
    comm.set_timeout(10.0)
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, C_, chunk_release_ns=release).bind(comm)
    try:
        outs = []
        for it in range(3):
            xs = host_inputs(P, N, dtype, seed=1000 + it)
            hin = torch.from_numpy(np.concatenate(xs)).pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            th.themis_allreduce_host(hin.data_ptr(), hout.data_ptr(), comm.data_ptr, N, dtype, plan)
            outs.append((xs, hin, hout))
        torch.cuda.synchronize()
        comm.status()
        for xs, _, hout in outs:
            if dtype == "i32":
                want = [O.allreduce_definition(xs, "i32")] * P
            else:
                want = O.run_schedule(xs, oracle_sched(sizes, bw, S.AR, N * 4, C_, th.THEMIS), dtype)
            for r in range(P):
                assert np.array_equal(hout.numpy()[r * N:(r + 1) * N].view(np.uint8), want[r].view(np.uint8)), r
    finally:
        plan.close()
        comm.close()


@pytest.mark.parametrize("n,dtype", [(1, "i32"), (12345, "i32"), (1 << 16, "f32"), (77777, "bf16")])
def test_tensor_all_reduce_any_numel(n, dtype):
    """Comm.all_reduce: user tensors of any numel (zero-padded to the granule,
    R17) reduce to the plain definition; int32 bit-exact, floats within the
    north_star tolerance of the fp64 sum."""
    topo = th.Topology((2, 2, 2), (1, 1, 1))
    comm = th.Comm(topo, 1 << 22)
    try:
        xs = host_inputs(8, n, dtype)
        ts = []
        for r in range(8):
            src = torch.from_numpy(xs[r].view(np.int16) if dtype == "bf16" else xs[r])
            ts.append((src.view(torch.bfloat16) if dtype == "bf16" else src).cuda())
        comm.all_reduce(ts, n_chunks=4)
        if dtype == "i32":
            comm.all_reduce(ts, n_chunks=4)             # second call reuses the cached plan
        torch.cuda.synchronize()
        comm.status()
        if dtype == "i32":
            once = O.allreduce_definition(xs, "i32")
            want = O.allreduce_definition([once] * 8, "i32")
            for r in range(8):
                assert np.array_equal(ts[r].cpu().numpy(), want)
            return
        ref = O.allreduce_definition(xs, dtype)
        scale = O.abs_sum(xs, dtype)
        for r in range(8):
            t = ts[r].cpu()
            out = t.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else t.numpy()
            assert np.all(np.abs(O.to_f64(out, dtype) - ref) <= TOL[dtype] * scale)
    finally:
        comm.close()


def test_cuda_graph_capture_and_replay():
    """Collectives captured in a CUDA graph replay correctly: the epoch lives
    on the device (a6), so each replay is a fresh collective.  int32 exact:
    two All-Reduces per graph, three replays = six All-Reduces in a row."""
    topo = th.Topology((2, 2, 2), (1, 1, 1))
    P, C_ = 8, 4
    N = P * C_ * 1024
    comm = th.Comm(topo, N * 4)
    comm.set_timeout(10.0)
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, C_).bind(comm)
    try:
        xs = host_inputs(P, N, "i32")
        for r in range(P):
            comm.rank_view(r, N, "i32").copy_(torch.from_numpy(xs[r]))
        th.run(th.ALLREDUCE, comm, plan, N, "i32")            # eager call first (epoch 1)
        torch.cuda.synchronize()
        want = O.allreduce_definition(xs, "i32")
        assert np.array_equal(comm.rank_view(3, N, "i32").cpu().numpy(), want)
        for r in range(P):                                     # restart from the inputs
            comm.rank_view(r, N, "i32").copy_(torch.from_numpy(xs[r]))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                th.run(th.ALLREDUCE, comm, plan, N, "i32")
                th.run(th.ALLREDUCE, comm, plan, N, "i32")
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        comm.status()
        want = xs
        for _ in range(6):
            want = [O.allreduce_definition(want, "i32")] * P
        for r in range(P):
            assert np.array_equal(comm.rank_view(r, N, "i32").cpu().numpy(), want[0]), f"rank {r}"
    finally:
        plan.close()
        comm.close()


@pytest.mark.parametrize("sizes,kinds", [((2, 2, 2), None), ((4, 2), None), ((2, 2, 2), (th.DIRECT, th.RING, th.DIRECT)),
                                         ((3, 4), (th.RING, th.DIRECT))])
@pytest.mark.parametrize("la", [2, 8, 32])
def test_runtime_intra_dim_order(sizes, kinds, la):
    """R28: producers pick the first ready op among the next L of the enforced
    list (direct dims; ring dims keep the static order) — results stay
    bit-exact against the oracle (every op's sum is order-independent), with
    repeated calls, windows and mixed ring/direct dims; int32 and f32."""
    P = int(np.prod(sizes))
    kw = dict(kinds=kinds, lookahead=la, repeat=2)
    check_ar(sizes, (1,) * len(sizes), "i32", 16, 4 * 300, **kw)
    check_ar(sizes, (4,) + (1,) * (len(sizes) - 1), "f32", 16, 4 * 301, dist="wide", **kw)
    check_ar(sizes, (1,) * len(sizes), "i32", 8, 4 * 64, min_cta_bytes=4096, ctas=[6] * len(sizes), **kw)
    assert P >= 8


@pytest.mark.parametrize("sizes,kinds", [((2, 2, 2), None), ((4, 2), None), ((2, 4), None), ((8,), None),
                                         ((2, 3, 2), (th.DIRECT, th.RING, th.DIRECT)), ((2, 2, 2, 2), None)])
@pytest.mark.parametrize("la", [1, 16])
def test_push_all_gather(sizes, kinds, la):
    """R30: direct AG ops executed as pushes (TMA bulk stores into the dim
    peers; the next stage waits for the k x k' plane) -- AR and AG-only
    bit-exact against the oracle, with ring dims mixed in (they stay pulls),
    repeated calls, op windows and the runtime order."""
    P = int(np.prod(sizes))
    kw = dict(kinds=kinds, lookahead=la, push=True, repeat=2)
    check_ar(sizes, (1,) * len(sizes), "i32", 16, 4 * 300, **kw)
    check_ar(sizes, (4,) + (1,) * (len(sizes) - 1), "f32", 8, 4 * 301, dist="wide", **kw)
    check_ar(sizes, (1,) * len(sizes), "bf16", 8, 8 * 257, dist="wide", min_cta_bytes=4096, ctas=[5] * len(sizes), **kw)
    xs, outs = run_case(sizes, (2,) * len(sizes), "i32", 8, 4 * 129, "AG", th.THEMIS, kinds=kinds, lookahead=la,
                        push=True)
    N = xs[0].shape[0]
    sched = oracle_sched(sizes, (2,) * len(sizes), "AG", N * 4, 8, th.THEMIS, kinds=kinds)
    want = O.run_schedule(xs, sched, "i32")
    for r in range(P):
        assert np.array_equal(outs[r], want[r]), f"AG rank {r}"


@pytest.mark.parametrize("sizes,kinds", [((2, 2, 2), None), ((4, 2), None), ((2, 4), None), ((8,), None),
                                         ((3, 2), None), ((2, 2, 2, 2), None), ((4, 4), (th.SWITCH, th.DIRECT))])
def test_ll_small_collectives(sizes, kinds):
    """R31: LL packets (payload + epoch in every 8-byte store, receivers poll
    the data) -- AR bit-exact against the oracle (same coordinate-order sums),
    int32 exact, repeated calls (epoch tags), op windows; RS / AG halves."""
    kw = dict(kinds=kinds, ll=True, repeat=3)
    check_ar(sizes, (1,) * len(sizes), "i32", 8, 4 * 100, **kw)
    check_ar(sizes, (4,) + (1,) * (len(sizes) - 1), "f32", 4, 4 * 101, dist="wide", **kw)
    check_ar(sizes, (1,) * len(sizes), "bf16", 8, 8 * 33, dist="wide", min_cta_bytes=2048, ctas=[3] * len(sizes), **kw)
    P = int(np.prod(sizes))
    for coll in ("RS", "AG"):
        xs, outs = run_case(sizes, (2,) * len(sizes), "i32", 4, 4 * 57, coll, th.THEMIS, kinds=kinds, ll=True)
        N = xs[0].shape[0]
        sched = oracle_sched(sizes, (2,) * len(sizes), coll, N * 4, 4, th.THEMIS, kinds=kinds)
        want = O.run_schedule(xs, sched, "i32")
        blk = N // P
        for r in range(P):
            got = outs[r][r * blk:(r + 1) * blk] if coll == "RS" else outs[r]
            exp = want[r][r * blk:(r + 1) * blk] if coll == "RS" else want[r]
            assert np.array_equal(got, exp), f"{coll} rank {r}"


def test_ll_falls_back_when_the_inbox_is_too_small():
    """A plan whose LL regions do not fit the inbox binds without LL (pull
    path) and stays exact; ring dims never run LL."""
    topo = th.Topology((2, 2), (1, 1))
    N = 4 * 8 * 256
    comm = th.Comm(topo, N * 4, ll_bytes=1 << 20)
    try:
        comm.set_ll(N * 4, 4096)                      # far too small for this plan's regions
        plan = th.Plan(topo, th.ALLREDUCE, N * 4, 8).bind(comm)
        assert not plan.bound_ll()
        plan.close()
        comm.set_ll(N * 4)
        plan = th.Plan(topo, th.ALLREDUCE, N * 4, 8).bind(comm)
        assert plan.bound_ll()
        plan.close()
        rt = th.Topology((3, 2), (1, 1), (th.RING, th.DIRECT))
        comm2 = th.Comm(rt, 6 * 8 * 256 * 4, ll_bytes=1 << 20)
        comm2.set_ll(1 << 20)
        plan = th.Plan(rt, th.ALLREDUCE, 6 * 8 * 256 * 4, 8).bind(comm2)
        assert not plan.bound_ll()
        plan.close()
        comm2.close()
    finally:
        comm.close()


def test_max_ranks_and_many_chunks():
    """Edge sizes on the executor: 64 logical ranks (2^6, the per-comm
    maximum) in one GPU, and 1024 chunks (THEMIS_MAX_CHUNKS) on 2x2x2 —
    int32 exact."""
    check_ar((2,) * 6, (1,) * 6, "i32", 4, 516, ctas=[8] * 6)
    check_ar((2, 2, 2), (1, 1, 1), "i32", 1024, 8, ctas=[16, 16, 16])


def test_tensor_all_reduce_empty():
    """numel = 0: nothing to reduce, nothing touched, no error."""
    comm = th.Comm(th.Topology((2, 2), (1, 1)), 1 << 20)
    try:
        ts = [torch.empty(0, dtype=torch.float32, device="cuda") for _ in range(4)]
        comm.all_reduce(ts, n_chunks=4)
        torch.cuda.synchronize()
        comm.status()
        assert all(t.numel() == 0 for t in ts)
    finally:
        comm.close()


def test_tensor_reduce_scatter_all_gather():
    """Comm.reduce_scatter / all_gather on user tensors: RS block r == block r
    of the sum, AG == the concatenation of all blocks, int32 exact; the
    granule is enforced."""
    topo = th.Topology((2, 4), (2, 1))
    P, C_ = 8, 4
    n = P * C_ * 4 * 33
    comm = th.Comm(topo, n * 4)
    try:
        xs = host_inputs(P, n, "i32")
        outs = comm.reduce_scatter([torch.from_numpy(x).cuda() for x in xs], n_chunks=C_)
        want = O.allreduce_definition(xs, "i32")
        blk = n // P
        for r in range(P):
            assert np.array_equal(outs[r].cpu().numpy(), want[r * blk:(r + 1) * blk])
        gathered = comm.all_gather(outs, n_chunks=C_)
        for r in range(P):
            assert np.array_equal(gathered[r].cpu().numpy(), want)
        with pytest.raises(th.ThemisError):
            comm.reduce_scatter([torch.zeros(n + 4, dtype=torch.int32, device="cuda")] * P, n_chunks=C_)
        comm.status()
    finally:
        comm.close()


def test_random_executor_configs():
    """Randomised executor parity (N = 1): 40 random (topology, kinds, BW,
    dtype, chunks, policy, intra, concurrency, op windows, CTA caps) — every
    output bit-exact against the oracle run with the same schedule (int32
    against the plain definition)."""
    import os
    import random
    rng = random.Random(int(os.environ.get("THEMIS_RANDOM_SEED", 4478)))
    for i in range(int(os.environ.get("THEMIS_RANDOM_CASES", 40))):
        D = rng.randint(1, 4)
        sizes = [rng.choice([2, 2, 3, 4]) for _ in range(D)]
        while int(np.prod(sizes)) > 32:
            sizes[rng.randrange(D)] = 2
        kinds = tuple(rng.choice([th.DIRECT, th.DIRECT, th.RING]) for _ in range(D))
        bw = tuple(rng.choice([1, 2, 3, 4, 8]) for _ in range(D))
        dtype = rng.choice(["i32", "f32", "bf16", "f16"])
        C_ = rng.choice([1, 2, 4, 8, 16])
        policy = rng.choice([th.THEMIS, th.BASELINE])
        intra = rng.choice([th.SCF, th.FIFO])
        conc = rng.choice([1, 1, 2])
        mcb = rng.choice([0, 0, 8192])
        vec = 16 // ELEM_SIZE[dtype]
        slice_elems = vec * rng.randint(1, 700)
        ctas = [rng.randint(max(2, conc), 24) for _ in range(D)]
        la = rng.choice([1, 1, 4, 16])
        push = rng.random() < 0.4
        kw = dict(kinds=kinds, ctas=ctas, intra=intra, concurrency=conc, min_cta_bytes=0 if conc > 1 else mcb,
                  dist="wide" if dtype != "i32" else "recipe", lookahead=la, push=push)
        try:
            check_ar(tuple(sizes), bw, dtype, C_, slice_elems, policy, **kw)
        except AssertionError as e:
            raise AssertionError(f"case {i}: sizes {sizes} kinds {kinds} bw {bw} {dtype} C {C_} policy {policy} "
                                 f"intra {intra} conc {conc} mcb {mcb} slice {slice_elems} ctas {ctas} "
                                 f"lookahead {la} push {push}: {e}")


def test_random_rs_ag_configs():
    """Randomised RS / AG halves (N = 1): 24 random (topology, kinds, BW,
    dtype, chunks, policy) — RS block r and the full AG buffer bit-exact
    against the oracle's schedule, int32 also against the plain definitions."""
    import os
    import random
    rng = random.Random(int(os.environ.get("THEMIS_RANDOM_SEED", 2110)))
    for i in range(int(os.environ.get("THEMIS_RANDOM_CASES", 24))):
        D = rng.randint(1, 3)
        sizes = tuple(rng.choice([2, 3, 4]) for _ in range(D))
        kinds = tuple(rng.choice([th.DIRECT, th.RING]) for _ in range(D))
        bw = tuple(rng.choice([1, 2, 4]) for _ in range(D))
        dtype = rng.choice(["i32", "f32", "bf16", "f16"])
        C_ = rng.choice([1, 2, 4, 8])
        policy = rng.choice([th.THEMIS, th.BASELINE])
        coll = rng.choice(["RS", "AG"])
        slice_elems = (16 // ELEM_SIZE[dtype]) * rng.randint(1, 500)
        la, push, mcb = rng.choice([1, 1, 8]), rng.random() < 0.4, rng.choice([0, 0, 4096])
        xs, outs = run_case(sizes, bw, dtype, C_, slice_elems, coll, policy, kinds=kinds,
                            dist="wide" if dtype != "i32" else "recipe", lookahead=la, push=push, min_cta_bytes=mcb)
        P, N = len(xs), xs[0].shape[0]
        sched = oracle_sched(sizes, bw, coll, N * ELEM_SIZE[dtype], C_, policy, kinds=kinds)
        tree = O.run_schedule(xs, sched, dtype)
        blk = N // P
        msg = f"case {i}: {coll} sizes {sizes} kinds {kinds} bw {bw} {dtype} C {C_} policy {policy} la {la} push {push} mcb {mcb}"
        for r in range(P):
            got = outs[r][r * blk:(r + 1) * blk] if coll == "RS" else outs[r]
            want = tree[r][r * blk:(r + 1) * blk] if coll == "RS" else tree[r]
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), msg + f" rank {r}"
        if dtype == "i32":
            if coll == "RS":
                d = O.reduce_scatter_definition(xs, "i32", P)
                assert all(np.array_equal(outs[r][r * blk:(r + 1) * blk], d[r]) for r in range(P)), msg
            else:
                cat = O.all_gather_definition(xs, P)
                assert all(np.array_equal(outs[r], cat) for r in range(P)), msg


def test_plan_outlives_comm():
    """A plan bound to a comm that is closed first is unbound (not dangling):
    running it reports PLAN_MISMATCH ("not bound"); rebinding to a new comm works."""
    topo = th.Topology((2, 2), (1, 1))
    N = 4 * 4 * 1024
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, 4)
    comm = th.Comm(topo, N * 4)
    plan.bind(comm)
    ptr = comm.data_ptr
    comm.close()
    with pytest.raises(th.ThemisError) as e:
        th.themis_allreduce(ptr, N, "i32", plan)
    assert e.value.status == 6
    comm2 = th.Comm(topo, N * 4)
    try:
        plan.bind(comm2)
        xs = host_inputs(4, N, "i32")
        for r in range(4):
            comm2.rank_view(r, N, "i32").copy_(torch.from_numpy(xs[r]))
        th.run(th.ALLREDUCE, comm2, plan, N, "i32")
        torch.cuda.synchronize()
        assert np.array_equal(comm2.rank_view(2, N, "i32").cpu().numpy(), O.allreduce_definition(xs, "i32"))
    finally:
        plan.close()
        comm2.close()
