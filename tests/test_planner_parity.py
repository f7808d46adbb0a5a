"""Bit-exact parity: C++ planner in libthemis (through the C ABI) vs the oracle.

The planner is host code, so these run without a GPU.  Compared exactly:
per-chunk RS/AG orders, per-dimension enforced op order, every op's
pre-simulated start/end time, makespan, busy_K, idle_K, N_K and the final Dim
Load Tracker, after converting the oracle's rationals with the plan's
time_scale / byte_scale.
"""

import random
from fractions import Fraction

import pytest

from oracle import engine as E, scheduler as S, topology as T
from paper_2110_04478_b200 import themis as th

KINDS = {T.RING: th.RING, T.DIRECT: th.DIRECT, T.SWITCH: th.SWITCH, T.NVLS: th.NVLS}
COLLS = {S.AR: th.ALLREDUCE, "RS": th.REDUCE_SCATTER, "AG": th.ALL_GATHER}
INTRA = {E.SCF: th.SCF, E.FIFO: th.FIFO, E.SCF_LITERAL: th.SCF_LITERAL}


def make_pair(sizes, bw_mbps, kinds=None, lat=None):
    kinds = kinds or [T.DIRECT] * len(sizes)
    lat = lat or [0] * len(sizes)
    o = T.Topology.make(sizes, [Fraction(b, 1000) for b in bw_mbps], kinds, lat)   # bytes/ns
    g = th.Topology(tuple(sizes), tuple(bw_mbps), tuple(KINDS[k] for k in kinds), tuple(lat))
    return o, g


def compare(o_topo, g_topo, coll, nbytes, C, policy, intra, div=16, charge=False, release=0):
    sched = S.schedule_collective(o_topo, coll, nbytes, C, policy, div)
    m = E.simulate(sched, intra, charge_latency=charge, release=release)
    plan = th.Plan(g_topo, COLLS[coll], nbytes, C, th.THEMIS if policy == S.THEMIS else th.BASELINE,
                   INTRA[intra], div, charge, chunk_release_ns=release)
    try:
        info = plan.info
        ts, bs = info["time_scale"], info["byte_scale"]
        rs, ag = plan.orders()
        D = o_topo.D
        for cs in sched.chunks:
            if cs.rs:
                assert tuple(int(x) for x in rs[cs.chunk]) == cs.rs
            if cs.ag:
                assert tuple(int(x) for x in ag[cs.chunk]) == cs.ag
        assert info["n_greedy"] == sched.n_greedy
        assert plan.dim_ops() == [list(x) for x in m.dim_order]
        assert Fraction(info["makespan"], ts) == m.makespan
        assert [Fraction(b, ts) for b in info["busy"]] == m.busy
        assert [Fraction(b, ts) for b in info["idle"]] == m.idle
        assert [Fraction(v, bs) for v in info["dim_volume"]] == m.volume
        assert [Fraction(v, ts) for v in info["final_load"]] == sched.loads
        st, en = plan.times()
        NS = info["n_stages"]
        for (c, s), t0 in m.start.items():
            assert Fraction(int(st[c * NS + s]), ts) == t0
            assert Fraction(int(en[c * NS + s]), ts) == m.end[(c, s)]
        assert D == info["ndims"]
    finally:
        plan.close()


def test_fig3_example():
    o, g = make_pair((4, 4), (2000, 1000))
    for pol in (S.BASELINE, S.THEMIS):
        for ip in (E.FIFO, E.SCF, E.SCF_LITERAL):
            compare(o, g, S.AR, 256 << 20, 4, pol, ip)


@pytest.mark.parametrize("ratio", [(4, 2, 1), (1, 1, 1), (2, 2, 1)])
def test_config2_2x2x2(ratio):
    o, g = make_pair((2, 2, 2), [r * 100000 for r in ratio])
    for pol in (S.BASELINE, S.THEMIS):
        compare(o, g, S.AR, 1 << 30, 64, pol, E.SCF)
        compare(o, g, S.AR, 1 << 30, 64, pol, E.FIFO)


def test_config1_2x4():
    o, g = make_pair((2, 4), (200000, 50000))
    for pol in (S.BASELINE, S.THEMIS):
        compare(o, g, S.AR, 64 * 1024, 4, pol, E.SCF)


@pytest.mark.parametrize("name", sorted(T.PRESETS))
def test_table2_topologies_1024_ranks(name):
    t = T.PRESETS[name]
    bw = [int(d.bw * 1000) for d in t.dims]
    assert all(Fraction(b, 1000) == d.bw for b, d in zip(bw, t.dims))
    o, g = make_pair(t.sizes, bw, [d.kind for d in t.dims], [int(d.step_latency) for d in t.dims])
    for mb in (100, 1000):
        for pol in (S.BASELINE, S.THEMIS):
            for ip in (E.SCF, E.FIFO):
                compare(o, g, S.AR, mb << 20, 64, pol, ip)
    compare(o, g, S.AR, 100 << 20, 64, S.THEMIS, E.SCF, charge=True)


def test_config5_2x8x8x8_rs_ag():
    o, g = make_pair((2, 8, 8, 8), (300000, 175000, 150000, 100000))
    for coll in ("RS", "AG", S.AR):
        for mb in (4, 64, 1024):
            compare(o, g, coll, mb << 20, 64, S.THEMIS, E.SCF)


BWS = [12500, 25000, 50000, 100000, 150000, 175000, 200000, 250000, 300000, 375000, 400000, 450000, 900000]


def test_random_configs():
    rng = random.Random(20211010)
    skipped = 0
    for _ in range(400):
        D = rng.randint(1, 4)
        sizes = [rng.choice([2, 3, 4, 5, 8, 16]) for _ in range(D)]
        kinds = [rng.choice([T.RING, T.DIRECT, T.SWITCH, T.NVLS]) if s & (s - 1) == 0 else
                 rng.choice([T.RING, T.DIRECT]) for s in sizes]
        bw = [rng.choice(BWS) if rng.random() < 0.7 else rng.randint(1, 12) for _ in range(D)]
        lat = [rng.choice([0, rng.randint(0, 3000)]) for _ in range(D)]
        o, g = make_pair(sizes, bw, kinds, lat)
        coll = rng.choice([S.AR, S.AR, "RS", "AG"])
        nbytes = rng.randint(1, 1 << 22) * rng.choice([1, 4096])
        try:
            compare(o, g, coll, nbytes, rng.randint(1, 48), rng.choice([S.BASELINE, S.THEMIS]),
                    rng.choice([E.SCF, E.FIFO, E.SCF_LITERAL]), rng.choice([16, 16, rng.randint(1, 100)]),
                    rng.random() < 0.2)
        except th.ThemisError as e:      # exact 64-bit outputs cannot hold this plan
            assert e.status == 4
            skipped += 1
    assert skipped < 40


@pytest.mark.parametrize("sizes", [(4,), (8,), (2, 4), (4, 2), (2, 2, 2), (2, 8, 8, 8), (4, 4, 8, 8)])
def test_nvls_algorithm_row(sizes):
    """R29: NVLS dims model each AR chunk's last-RS /
    first-AG pair as one in-switch op; the C++ planner matches the oracle bit
    for bit (orders, enforced op order, every op time, N_K, tracker), with and
    without per-op latency, for NVLS on every / some dims."""
    D = len(sizes)
    bw = [100000 * (D - k) for k in range(D)]
    for nv_dims in ({D - 1}, set(range(D))):
        kinds = [T.NVLS if k in nv_dims else T.SWITCH for k in range(D)]
        o, g = make_pair(sizes, bw, kinds, [700] * D)
        for pol in (S.BASELINE, S.THEMIS):
            for ip in (E.SCF, E.FIFO):
                compare(o, g, S.AR, 256 << 20, 64, pol, ip)
            compare(o, g, S.AR, 64 << 20, 16, pol, E.SCF, charge=True)
        compare(o, g, "RS", 64 << 20, 16, S.THEMIS, E.SCF)          # RS / AG-only: no fused pair
        compare(o, g, "AG", 64 << 20, 16, S.THEMIS, E.SCF)


def test_custom_orders_full_space():
    """themis_plan_custom: arbitrary RS x AG orders per chunk
    pre-simulated bit-exactly like the oracle's engine."""
    import itertools
    rng = random.Random(99)
    for _ in range(90):
        D = rng.randint(1, 3)
        sizes = [rng.choice([2, 3, 4]) for _ in range(D)]
        bw = [rng.choice(BWS) for _ in range(D)]
        # NVLS dims too (R29): a chunk's pair is fused only if its last RS dim is its first AG dim
        kinds = [rng.choice([T.DIRECT, T.NVLS]) if s_ & (s_ - 1) == 0 else T.DIRECT for s_ in sizes]
        o, g = make_pair(sizes, bw, kinds)
        C = rng.randint(1, 12)
        coll = rng.choice([S.AR, "RS", "AG"])
        perms = list(itertools.permutations(range(D)))
        rs = [rng.choice(perms) for _ in range(C)]
        ag = [rng.choice(perms) for _ in range(C)]
        chunks = [S.ChunkSchedule(c, rs[c] if coll != "AG" else (), ag[c] if coll != "RS" else ())
                  for c in range(C)]
        nbytes = rng.randint(1, 1 << 20) * 4096
        sched = S.Schedule(o, coll, Fraction(nbytes), C, chunks, [], 0)
        intra = rng.choice([E.SCF, E.FIFO])
        m = E.simulate(sched, intra)
        plan = th.Plan(g, COLLS[coll], nbytes, C, th.THEMIS, INTRA[intra],
                       rs_orders=rs if coll != "AG" else None, ag_orders=ag if coll != "RS" else None)
        try:
            ts = plan.info["time_scale"]
            assert plan.dim_ops() == [list(x) for x in m.dim_order]
            assert Fraction(plan.info["makespan"], ts) == m.makespan
            assert [Fraction(v, plan.info["byte_scale"]) for v in plan.info["dim_volume"]] == m.volume
        finally:
            plan.close()
    with pytest.raises(th.ThemisError):
        th.Plan(th.Topology((2, 2), (1, 1)), th.ALLREDUCE, 4096, 2, rs_orders=[(0, 0), (0, 1)],
                ag_orders=[(1, 0), (1, 0)])


def test_concurrency_servers_bit_exact():
    """Pre-simulation with k parallel servers per dim:
    per-dim op order, server of every op, times, busy / idle bit-exact."""
    rng = random.Random(515)
    for _ in range(80):
        D = rng.randint(1, 3)
        sizes = [rng.choice([2, 3, 4, 8]) for _ in range(D)]
        bw = [rng.choice(BWS) for _ in range(D)]
        lat = [rng.choice([0, rng.randint(0, 2000)]) for _ in range(D)]
        o, g = make_pair(sizes, bw, None, lat)
        sv = rng.choice([2, 3, 4, 8])
        coll = rng.choice([S.AR, S.AR, "RS", "AG"])
        C = rng.randint(1, 40)
        nbytes = rng.randint(1, 1 << 22) * 4096
        pol = rng.choice([S.BASELINE, S.THEMIS])
        intra = rng.choice([E.SCF, E.FIFO, E.SCF_LITERAL])
        charge = rng.random() < 0.3
        sched = S.schedule_collective(o, coll, nbytes, C, pol)
        m = E.simulate(sched, intra, charge_latency=charge, servers=sv)
        plan = th.Plan(g, COLLS[coll], nbytes, C, th.THEMIS if pol == S.THEMIS else th.BASELINE, INTRA[intra], 16,
                       charge, concurrency=sv)
        try:
            info = plan.info
            ts = info["time_scale"]
            assert plan.dim_ops() == [list(x) for x in m.dim_order]
            srv = plan.servers()
            NS = info["n_stages"]
            st, en = plan.times()
            for (c, s), t0 in m.start.items():
                assert int(srv[c, s]) == m.server[(c, s)]
                assert Fraction(int(st[c * NS + s]), ts) == t0
                assert Fraction(int(en[c * NS + s]), ts) == m.end[(c, s)]
            assert Fraction(info["makespan"], ts) == m.makespan
            assert [Fraction(b, ts) for b in info["busy"]] == m.busy
            assert [Fraction(b, ts) for b in info["idle"]] == m.idle
            assert [Fraction(v, ts) for v in info["final_load"]] == sched.loads
        finally:
            plan.close()


def test_plan_validation_errors():
    with pytest.raises(th.ThemisError) as e:
        th.Plan(th.Topology((1, 4), (1, 1)), th.ALLREDUCE, 1024, 4)
    assert e.value.status == 1
    with pytest.raises(th.ThemisError):
        th.Plan(th.Topology((6,), (1,), (th.SWITCH,)), th.ALLREDUCE, 1024, 4)
    with pytest.raises(th.ThemisError):
        th.Plan(th.Topology((2, 2), (1, 1)), th.ALLREDUCE, 0, 4)
    with pytest.raises(th.ThemisError):
        th.Plan(th.Topology((2, 2), (1, 1)), th.ALLREDUCE, 1024, -1)
    with pytest.raises(th.ThemisError):                       # n_chunks = 0 (auto) is custom-orders-free only
        th.Plan(th.Topology((2, 2), (1, 1)), th.ALLREDUCE, 1024, 0, rs_orders=[[0, 1]], ag_orders=[[1, 0]])
    with pytest.raises(th.ThemisError):
        th.Plan(th.Topology((2, 2), (1, 0)), th.ALLREDUCE, 1024, 4)


def test_overflow_is_reported():
    # pairwise-coprime bandwidths make lcm * P * C exceed the 64-bit outputs
    g = th.Topology((16, 16, 16, 16), (999983, 999979, 999961, 999959))
    with pytest.raises(th.ThemisError) as e:
        th.Plan(g, th.ALLREDUCE, 1 << 40, 1024)
    assert e.value.status == 4


def test_plan_hash_deterministic():
    g = th.Topology((2, 2, 2), (1, 1, 1))
    a = th.Plan(g, th.ALLREDUCE, 1 << 30, 64)
    b = th.Plan(g, th.ALLREDUCE, 1 << 30, 64)
    c = th.Plan(g, th.ALLREDUCE, 1 << 30, 64, policy=th.BASELINE)
    assert a.info["hash"] == b.info["hash"] != c.info["hash"]


@pytest.mark.parametrize("sizes,bw,lat,nbytes,pol", [
    ((2, 2, 2), (80000, 80000, 80000), (8000, 9000, 8500), 1 << 20, S.THEMIS),    # calibrated A_K (profiles/r01/calibration)
    ((2, 2, 2), (80000, 80000, 80000), (8000, 9000, 8500), 64 << 20, S.THEMIS),
    ((2, 2, 2), (80000, 80000, 80000), (8000, 9000, 8500), 1 << 30, S.BASELINE),
    ((4, 2), (200000, 50000), (500, 2000), 16 << 20, S.THEMIS),
    ((2, 4), (100000, 100000), (0, 0), 4 << 20, S.THEMIS),                          # A = 0: ties / pipelining
    ((8,), (300000,), (1000,), 1 << 24, S.THEMIS),
])
def test_auto_chunks_parity(sizes, bw, lat, nbytes, pol):
    """n_chunks = 0: the C++ planner picks the same C as the oracle's
    choose_chunks and the resulting plan is bit-identical."""
    o, g = make_pair(sizes, bw, lat=list(lat))
    want = E.choose_chunks(o, S.AR, nbytes, pol, E.SCF if pol == S.THEMIS else E.FIFO, charge_latency=True)
    plan = th.Plan(g, th.ALLREDUCE, nbytes, th.AUTO_CHUNKS, th.THEMIS if pol == S.THEMIS else th.BASELINE,
                   th.SCF if pol == S.THEMIS else th.FIFO, charge_latency=True)
    try:
        assert plan.n_chunks == want[0]
        assert Fraction(plan.info["makespan"], plan.info["time_scale"]) == want[2].makespan
    finally:
        plan.close()
    compare(o, g, S.AR, nbytes, want[0], pol, E.SCF if pol == S.THEMIS else E.FIFO, charge=True)


def test_auto_chunks_alignment_error():
    g = th.Topology((2, 2), (1000, 1000))
    with pytest.raises(th.ThemisError) as e:
        th.Plan(g, th.ALLREDUCE, 4 * 16 + 8, th.AUTO_CHUNKS)
    assert e.value.status == 2          # THEMIS_ERR_ALIGNMENT


@pytest.mark.parametrize("release", [1, 37, 2000, 250_000])
def test_chunk_release_parity(release):
    """Host streaming (R26): chunk c ready at (c+1)*release ns — per-dim order
    and every start/end time bit-exact against the oracle, both policies,
    with and without per-op latency, including ties between arrivals and
    completions."""
    o, g = make_pair((2, 2, 2), (100000, 100000, 100000), lat=[500, 700, 900])
    for pol in (S.BASELINE, S.THEMIS):
        for ip in (E.SCF, E.FIFO):
            for charge in (False, True):
                compare(o, g, S.AR, 64 << 20, 16, pol, ip, charge=charge, release=release)
    o, g = make_pair((4, 2), (200000, 50000))
    compare(o, g, S.AR, 16 << 20, 8, S.THEMIS, E.SCF, release=release)


def test_max_dims_and_chunks():
    """Edge sizes: THEMIS_MAX_DIMS = 8 dims (2^8 ranks) and 1024 chunks
    (THEMIS_MAX_CHUNKS), both policies, bit-exact against the oracle."""
    o, g = make_pair((2,) * 8, (8000, 7000, 6000, 5000, 4000, 3000, 2000, 1000))
    for pol in (S.BASELINE, S.THEMIS):
        compare(o, g, S.AR, 256 << 20, 8, pol, E.SCF)
    o, g = make_pair((2, 2, 2), (1000, 1000, 1000))
    compare(o, g, S.AR, 1 << 30, 1024, S.THEMIS, E.SCF)
    with pytest.raises(th.ThemisError):
        th.Plan(th.Topology((2,) * 9, (1,) * 9), th.ALLREDUCE, 1 << 20, 4)
    with pytest.raises(th.ThemisError):
        th.Plan(th.Topology((2, 2), (1, 1)), th.ALLREDUCE, 1 << 20, 1025)


def test_random_small_configs_10k():
    """SURVEY.md §4 tier 3: >= 10^4 random (topology, bytes, C, policy, intra)
    tuples, small enough to run in well under a minute, every field bit-exact."""
    rng = random.Random(2110_04478)
    skipped = 0
    for _ in range(10_000):
        D = rng.randint(1, 3)
        sizes = [rng.choice([2, 3, 4, 8]) for _ in range(D)]
        bw = [rng.choice([1, 2, 3, 4, 5, 7, 8, 16]) * rng.choice([1, 1000, 50000]) for _ in range(D)]
        lat = [rng.choice([0, 0, rng.randint(1, 5000)]) for _ in range(D)]
        o, g = make_pair(sizes, bw, None, lat)
        coll = rng.choice([S.AR, S.AR, "RS", "AG"])
        nbytes = rng.randint(1, 1 << 16) * rng.choice([1, 16, 4096])
        try:
            compare(o, g, coll, nbytes, rng.randint(1, 8), rng.choice([S.BASELINE, S.THEMIS]),
                    rng.choice([E.SCF, E.FIFO, E.SCF_LITERAL]), 16, rng.random() < 0.3,
                    release=rng.choice([0, 0, 0, rng.randint(1, 100_000)]))
        except th.ThemisError as e:
            assert e.status == 4
            skipped += 1
    assert skipped < 200


@pytest.mark.parametrize("coll", [S.AR, "RS", "AG"])
def test_csv_export_matches_oracle(coll):
    """Plan export is byte-identical to the oracle's export."""
    o, g = make_pair((2, 4, 2), (300000, 200000, 100000))
    for nbytes, C in ((1 << 24, 16), (1000, 3)):
        sched = S.schedule_collective(o, coll, nbytes, C, S.THEMIS)
        plan = th.Plan(g, COLLS[coll], nbytes, C, th.THEMIS)
        try:
            assert plan.to_csv() == S.export_csv(sched)
        finally:
            plan.close()


def test_table2_presets_in_the_binding():
    """The binding's TABLE2 presets equal the oracle's transcription of
    PAPER.md Table 2 (sizes, aggregate BW, kinds, latencies), and a Themis plan
    on each is bit-identical to the oracle's."""
    for name, g in th.TABLE2.items():
        o = T.PRESETS[name]
        assert g.sizes == tuple(d.size for d in o.dims)
        assert [Fraction(b, 1000) for b in g.bw_mbps] == [d.bw for d in o.dims]
        assert [KINDS[d.kind] for d in o.dims] == list(g.kinds)
        assert [Fraction(x) for x in g.latency_ns] == [d.step_latency for d in o.dims]
        compare(o, g, S.AR, 1 << 30, 16, S.THEMIS, E.SCF)


def test_plan_utilization_matches_oracle():
    """Plan.utilization() == the oracle's util (R14) exactly, both policies."""
    for sizes, bw in (((2, 2, 2), (100000, 100000, 100000)), ((4, 2), (200000, 50000)), ((16, 8, 8), (100000, 100000, 50000))):
        o, g = make_pair(sizes, bw)
        for pol in (S.BASELINE, S.THEMIS):
            m = E.simulate(S.schedule_collective(o, S.AR, 1 << 28, 32, pol), E.SCF if pol == S.THEMIS else E.FIFO)
            plan = th.Plan(g, th.ALLREDUCE, 1 << 28, 32, th.THEMIS if pol == S.THEMIS else th.BASELINE,
                           th.SCF if pol == S.THEMIS else th.FIFO)
            try:
                assert plan.utilization() == m.util
            finally:
                plan.close()
