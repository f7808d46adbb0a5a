"""Pins for the oracle's topology / latency model / Algorithm 1 / engine.

Each test pins the oracle to something other than itself: values printed in
PAPER.md (tests/golden/paper_values.json, each entry cited), closed forms,
invariants, special cases, or brute force.
"""

import itertools
import json
import math
import os
import random
from fractions import Fraction as F

import pytest

from oracle import brute, collectives as col, engine as E, scheduler as S, topology as T

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
MB = 2 ** 20


def fig3_topo():
    g = GOLD["fig3"]
    return T.Topology.make(g["sizes"], g["bw_ratio"])


def fig3_unit(topo):
    # "the 64MB RS ... takes 1 unit of time when running on dim1"
    return col.chunk_load(topo.dims[0], col.RS, 64 * MB)


# ---------------------------------------------------------------- topology
def test_table2_presets_match_paper():
    for name, bws in GOLD["table2_aggr_bw_gbps"].items():
        if name.startswith("_"):
            continue
        t = T.PRESETS[name]
        assert [d.bw * 8 for d in t.dims] == [F(b) for b in bws], name
        assert list(t.sizes) == GOLD["table2_sizes"][name]
        assert t.P == 1024


def test_topology_validation_and_coords():
    with pytest.raises(ValueError):
        T.Topology.make((6,), (1,), (T.SWITCH,))          # SPEC.md:39 power-of-two rule
    with pytest.raises(ValueError):
        T.Topology.make((6,), (1,), (T.NVLS,))            # R29: a switch that reduces, same rule
    with pytest.raises(ValueError):
        T.Topology.make((4,), (0,))                        # BW > 0
    with pytest.raises(ValueError):
        T.Topology.make((1, 4), (1, 1))
    t = T.Topology.make((2, 4, 3), (1, 1, 1))
    for r in range(t.P):
        assert t.rank_of(t.coords(r)) == r
    assert t.coords(1) == (1, 0, 0)                         # dim1 fastest
    assert t.coords(2) == (0, 1, 0)
    assert t.dim_peers(0, 1) == [0, 2, 4, 6]
    # dim peers by brute force: ranks whose coordinates differ from r only on dim k
    for r in range(t.P):
        for k in range(t.D):
            want = [q for q in range(t.P) if all(t.coords(q)[i] == t.coords(r)[i] for i in range(t.D) if i != k)]
            assert sorted(t.dim_peers(r, k)) == want


# ---------------------------------------------------------------- collectives
def test_footnote_nk_and_size_changes():
    g = GOLD["footnote_nk"]
    assert col.bytes_sent(col.RS, g["p"], g["chunk_mb"] * MB) == g["n_mb"] * MB
    # 64MB RS and 16MB AG on the same p=4 dim take the same time
    assert col.bytes_sent(col.RS, 4, 64 * MB) == col.bytes_sent(col.AG, 4, 16 * MB)
    # RS shrinks by P, AG multiplies by P
    assert col.size_after(col.RS, 4, 64 * MB) == 16 * MB
    assert col.size_after(col.AG, 4, 16 * MB) == 64 * MB


def test_step_counts():
    g = GOLD["ring_ar_steps"]
    p = g["p"]
    assert col.num_steps(col.RS, T.RING, p) + col.num_steps(col.AG, T.RING, p) == g["steps"]  # :477
    assert col.num_steps(col.RS, T.DIRECT, 8) == 1
    assert col.num_steps(col.RS, T.SWITCH, 8) == 3
    d = T.Dim(4, F(1), T.RING, F(20))
    assert col.fixed_delay(d, col.RS) == 60


def test_fig3_stage_times():
    """stage latencies 1, 0.5, 0.5, 1 units for a 64MB chunk."""
    t = fig3_topo()
    u = fig3_unit(t)
    sched = S.schedule_collective(t, S.AR, 256 * MB, 4, S.BASELINE)
    ops = E.chunk_ops(sched)[0]
    assert [op.duration / u for op in ops] == [F(x).limit_denominator() for x in GOLD["fig3"]["stage_time_units"]]


# ---------------------------------------------------------------- Algorithm 1
def test_fig6_schedule():
    """c1 baseline, c2 starts from dim2, c3/c4 start from dim1."""
    t = fig3_topo()
    s = S.schedule_collective(t, S.AR, 256 * MB, 4, S.THEMIS)
    assert [cs.rs[0] + 1 for cs in s.chunks] == GOLD["fig6"]["first_dim_per_chunk_1based"]
    for cs in s.chunks:
        assert cs.ag == tuple(reversed(cs.rs))              # Algorithm 1 line 8


def test_fig6_threshold_arithmetic():
    """Threshold = RS of chunk/16 on the min-load dim.  Before
    c1 loads are equal (0 < thr -> baseline, :392); before c2 the gap is
    1 unit (dim1 charged 1+1, dim2 0.5+0.5) and thr = (3/4)*4MB/BW2 = 1/8 unit."""
    t = fig3_topo()
    u = fig3_unit(t)
    chunk = 64 * MB
    loads0 = [F(0), F(0)]
    assert S.threshold(t, loads0, chunk, 16) / u == F(1, 16)
    inc, _ = S.walk_loads(t, col.RS, (0, 1), chunk)
    inc2, _ = S.walk_loads(t, col.AG, (1, 0), chunk / 16)
    loads1 = [a + b for a, b in zip(inc, inc2)]
    assert [x / u for x in loads1] == [2, 1]
    assert S.threshold(t, loads1, chunk, 16) / u == F(1, 8)


def test_themis_equals_baseline_when_stage_balanced():
    """PAPER.md:334/:338/:703-705 (Just Enough): BW(dim1) = P1 * BW(dim2) ...
    -> stage times equal -> loads stay within the threshold -> baseline order.
    The paper's condition drops the (P-1)/P factors (R20); with
    unequal sizes the exact balance is BW_k/BW_k+1 = (P_k-1) P_k+1 / (P_k+1 - 1),
    e.g. 8x4 balances at 28:3, not 8:1."""
    for sizes, bws in [((4, 4), (4, 1)), ((2, 2, 2), (4, 2, 1)), ((2, 2), (2, 1)), ((8, 8), (8, 1)),
                       ((8, 4), (28, 3))]:
        t = T.Topology.make(sizes, bws)
        s = S.schedule_collective(t, S.AR, 64 * MB, 64, S.THEMIS)
        assert s.n_greedy == 0
        m = E.simulate(s, E.SCF)
        # only the pipeline fill/drain is lost: 2 stage-times of ~2C per dim
        assert m.util >= F(98, 100) if t.D == 2 else m.util >= F(95, 100)


def test_under_provisioned_2d_keeps_baseline():
    """BW(dim1) > P1*BW(dim2) in 2D -> no better schedule;
    the greedy keeps dim1-first (dim1 always least loaded)."""
    t = T.Topology.make((2, 4), (200, 50))
    s = S.schedule_collective(t, S.AR, 64 * 1024, 4, S.THEMIS)
    assert all(cs.rs == (0, 1) for cs in s.chunks)


def test_d1_single_schedule():
    t = T.Topology.make((8,), (1,))
    s = S.schedule_collective(t, S.AR, 1 << 20, 16, S.THEMIS)
    assert all(cs.rs == (0,) and cs.ag == (0,) for cs in s.chunks)


def test_schedule_structure_random():
    rng = random.Random(7)
    for _ in range(40):
        D = rng.randint(1, 4)
        t = T.Topology.make([rng.choice([2, 3, 4, 8]) for _ in range(D)],
                            [rng.randint(1, 9) for _ in range(D)])
        for coll in (S.AR, "RS", "AG"):
            s = S.schedule_collective(t, coll, rng.randint(1, 10 ** 9), rng.randint(1, 40), S.THEMIS)
            for cs in s.chunks:
                for o in (cs.rs, cs.ag):
                    assert o == () or sorted(o) == list(range(D))
                if coll == S.AR:
                    assert cs.ag == tuple(reversed(cs.rs))
            s2 = S.schedule_collective(t, coll, s.total_bytes, s.n_chunks, S.THEMIS)
            assert s2.chunks == s.chunks                         # determinism (:500)


def test_threshold_divisor_limits():
    """Huge divisor -> threshold -> 0 -> greedy whenever loads differ;
    tiny divisor -> threshold above any gap -> baseline."""
    t = T.Topology.make((2, 2, 2), (1, 1, 1))
    s = S.schedule_collective(t, S.AR, 1 << 30, 64, S.THEMIS, threshold_div=F(1, 10 ** 6))
    assert s.n_greedy == 0
    s = S.schedule_collective(t, S.AR, 1 << 30, 64, S.THEMIS, threshold_div=10 ** 9)
    assert s.n_greedy == 63


def test_volume_closed_form():
    """N_K = sum_i n_K^i; the RS half telescopes to
    S(P-1)/P per NPU whatever the order, AG likewise."""
    rng = random.Random(3)
    for _ in range(60):
        D = rng.randint(1, 4)
        t = T.Topology.make([rng.choice([2, 3, 4, 8]) for _ in range(D)], [rng.randint(1, 5) for _ in range(D)])
        S_ = F(rng.randint(1, 10 ** 9))
        C = rng.randint(1, 8)
        perms = list(itertools.permutations(range(D)))
        chunks = []
        for c in range(C):
            rs = rng.choice(perms)
            chunks.append(S.ChunkSchedule(c, rs, tuple(reversed(rs))))
        sched = S.Schedule(t, S.AR, S_, C, chunks, [], 0)
        N = S.dim_volumes(sched)
        assert sum(N) == 2 * S_ * F(t.P - 1, t.P)
        # per-chunk formula: N_{pi_j} += 2 * (chunk / prod_{i<j} P_{pi_i}) * (P-1)/P
        want = [F(0)] * D
        for cs in chunks:
            b = S_ / C
            for d in cs.rs:
                p = t.dims[d].size
                want[d] += 2 * b * F(p - 1, p)
                b /= p
        assert N == want


# ---------------------------------------------------------------- engine
def test_fig3_baseline_makespan():
    """dim1 carries 4 RS + 4 AG stages of 1 unit each, so the
    makespan is >= 8 units; the FIFO pipeline attains it (Fig 3a)."""
    t = fig3_topo()
    u = fig3_unit(t)
    s = S.schedule_collective(t, S.AR, 256 * MB, 4, S.BASELINE)
    for pol in (E.FIFO, E.SCF, E.SCF_LITERAL):
        m = E.simulate(s, pol)
        assert m.makespan / u == 8
        assert m.busy[0] / u == 8 and m.busy[1] / u == 4


def test_fig3_themis_scf_is_optimal():
    """Fig 3b shows Themis reducing the time; with the SCF key
    on transfer volume it reaches the brute-force optimum over all 16
    reversed-AG assignments and over the full (2!2!)^4 space."""
    t = fig3_topo()
    u = fig3_unit(t)
    s = S.schedule_collective(t, S.AR, 256 * MB, 4, S.THEMIS)
    m = E.simulate(s, E.SCF)
    best, _, n = brute.exhaustive_best(t, S.AR, 256 * MB, 4, E.SCF)
    assert n == 16
    bestf, _, nf = brute.exhaustive_best(t, S.AR, 256 * MB, 4, E.SCF, full=True)
    assert nf == 256
    assert m.makespan == best == bestf
    assert m.makespan / u == 7
    assert m.makespan < E.simulate(S.schedule_collective(t, S.AR, 256 * MB, 4, S.BASELINE), E.FIFO).makespan


def test_space_size_formula_and_enumeration():
    g = GOLD["space_size"]
    assert brute.space_size(g["D"], g["C"], S.AR, full=True) == g["value"]
    t = T.Topology.make((2, 2, 2), (1, 1, 1))
    assert sum(1 for _ in brute.candidates(t, S.AR, 2, full=False)) == 36
    assert sum(1 for _ in brute.candidates(t, S.AR, 1, full=True)) == 36
    assert sum(1 for _ in brute.candidates(t, "RS", 3)) == 216


def test_engine_single_chunk_closed_form():
    """One chunk, D=1, ring p=4, latency L, BW X: makespan =
    2*(3L) + 2*(3S/4)/X."""
    t = T.Topology.make((4,), (5,), (T.RING,), (20,))
    Sz = 1000
    s = S.schedule_collective(t, S.AR, Sz, 1, S.THEMIS)
    m = E.simulate(s, E.FIFO, charge_latency=True)
    assert m.makespan == 2 * 3 * 20 + 2 * F(3 * Sz, 4) / 5


def test_engine_invariants_random():
    rng = random.Random(11)
    for _ in range(30):
        D = rng.randint(1, 3)
        t = T.Topology.make([rng.choice([2, 3, 4]) for _ in range(D)], [rng.randint(1, 6) for _ in range(D)])
        Sz = rng.randint(10 ** 3, 10 ** 9)
        C = rng.randint(1, 12)
        for pol in (S.BASELINE, S.THEMIS):
            s = S.schedule_collective(t, S.AR, Sz, C, pol)
            for ip in (E.FIFO, E.SCF, E.SCF_LITERAL):
                m = E.simulate(s, ip)
                assert m.makespan == max(m.finish)
                assert all(f == b + i for f, b, i in zip(m.finish, m.busy, m.idle))
                assert all(i >= 0 for i in m.idle)
                # lower bounds: every dim's load, and the Ideal (Table 3)
                assert all(m.makespan >= n / d.bw for n, d in zip(m.volume, t.dims))
                assert m.makespan >= E.ideal_time(s)
                assert m.volume == S.dim_volumes(s)
                assert 0 < m.util <= 1
                # replaying the recorded per-dim order reproduces the run (:530)
                r = E.simulate(s, ip, enforced=m.dim_order)
                assert r.makespan == m.makespan and r.start == m.start
            if pol == S.BASELINE:
                # equal chunks + identical schedules: FIFO == SCF
                assert E.simulate(s, E.FIFO).makespan == E.simulate(s, E.SCF).makespan


def test_parallel_servers_per_dim():
    """PAPER.md:461/:491 provision (several chunks per dimension in parallel):
    `servers` parallel servers with BW_K/servers each.  Work conservation gives
    the closed form 2*C*v/BW for a D = 1 All-Reduce whose C is a multiple of
    the server count; busy/volume are server-count invariant; replaying the
    recorded per-server orders reproduces the run."""
    t = T.Topology.make((4,), (3,))
    Sz, C = 1 << 20, 8
    s = S.schedule_collective(t, S.AR, Sz, C, S.THEMIS)
    v = col.bytes_sent(col.RS, 4, F(Sz, C))
    for sv in (1, 2, 4, 8):
        m = E.simulate(s, E.SCF, servers=sv)
        assert m.makespan == 2 * C * v / 3
        assert set(m.server.values()) == set(range(sv))
    rng = random.Random(21)
    for _ in range(20):
        D = rng.randint(1, 3)
        t = T.Topology.make([rng.choice([2, 3, 4]) for _ in range(D)], [rng.randint(1, 5) for _ in range(D)])
        s = S.schedule_collective(t, S.AR, rng.randint(1, 10 ** 8), rng.randint(1, 16), S.THEMIS)
        base = E.simulate(s, E.SCF)
        for sv in (2, 3):
            m = E.simulate(s, E.SCF, servers=sv)
            assert m.busy == base.busy and m.volume == base.volume
            assert all(m.makespan >= n / d.bw for n, d in zip(m.volume, t.dims))
            r = E.simulate(s, E.SCF, servers=sv, enforced=m.dim_order, enforced_server=m.server)
            assert r.start == m.start and r.makespan == m.makespan


def test_inconsistent_order_deadlocks():
    """NPUs/dims running chunk ops in inconsistent orders
    can deadlock.  Enforcing orders where dim1 wants c1's AG before c0's RS
    while c1's AG needs c1's RS on dim0 ... forms a cycle."""
    t = T.Topology.make((2, 2), (1, 1))
    chunks = [S.ChunkSchedule(0, (0, 1), (1, 0)), S.ChunkSchedule(1, (1, 0), (0, 1))]
    s = S.Schedule(t, S.AR, F(1024), 2, chunks, [], 0)
    # dim0 insists on chunk1's stage1 (needs dim1 stage0 of chunk1) first;
    # dim1 insists on chunk0's stage1 (needs dim0 stage0 of chunk0) first.
    bad = [[(1, 1), (0, 0), (0, 3), (1, 2)], [(0, 1), (1, 0), (1, 3), (0, 2)]]
    with pytest.raises(RuntimeError):
        E.simulate(s, E.FIFO, enforced=bad)


def test_brute_force_dominates():
    """optimum <= min(Themis, baseline) (NOT Themis <= baseline)."""
    rng = random.Random(5)
    for _ in range(25):
        t = T.Topology.make([rng.choice([2, 4]) for _ in range(2)], [rng.randint(1, 8) for _ in range(2)])
        C = rng.randint(1, 4)
        Sz = 1 << 20
        best, _, _ = brute.exhaustive_best(t, S.AR, Sz, C, E.SCF)
        th = E.simulate(S.schedule_collective(t, S.AR, Sz, C, S.THEMIS), E.SCF).makespan
        ba = E.simulate(S.schedule_collective(t, S.AR, Sz, C, S.BASELINE), E.SCF).makespan
        assert best <= th and best <= ba
        assert best >= E.ideal_time(S.schedule_collective(t, S.AR, Sz, C, S.THEMIS))


def test_activity_rate():
    t = fig3_topo()
    s = S.schedule_collective(t, S.AR, 256 * MB, 4, S.BASELINE)
    m = E.simulate(s, E.FIFO)
    a = E.activity_rate(m, s, m.makespan)
    assert a[0] == [1] and a[1] == [m.busy[1] / m.makespan]
    a = E.activity_rate(m, s, m.makespan / 8)
    assert a[0] == [1] * 8


# ---------------------------------------------------------------- paper numbers
def test_current_platform_util():
    """97.7% utilisation of the current 16x64 (1200/100 Gbps)
    platform under the baseline; :340: 75 of dim2's 100 Gbps used."""
    g = GOLD["current_platform"]
    t = T.CURRENT_2D
    s = S.schedule_collective(t, S.AR, 1 << 30, 64, S.BASELINE)
    m = E.simulate(s, E.FIFO)
    assert abs(float(m.util) - g["util"]) < 0.02
    # :340 uses the approximate chain 1200/16 = 75 Gbps; the exact stage
    # volumes carry (P-1)/P factors (reading R20): 75 * (63/64) / (15/16).
    assert F(1200, 16) == g["dim2_used_gbps"]
    assert m.busy[1] / m.makespan * 100 == F(g["dim2_used_gbps"]) * F(63, 64) / F(15, 16)


def test_3d_homo_underutilisation():
    """balanced chain 800 = 16*50 = 128*6.25 Gbps, so the
    baseline uses 800+50+6.25 of 2400 Gbps; paper's minimum next-gen baseline
    utilisation is 35.1% (:317)."""
    g = GOLD["balance_3d_homo"]
    t = T.PRESETS["3D-SW_SW_SW_homo"]
    chain = [F(g["dim1_gbps"])]
    for k in range(1, t.D):
        chain.append(chain[-1] / t.dims[k - 1].size)
    assert chain == [F(x).limit_denominator() for x in g["balanced_gbps"]]
    assert [800 - c for c in chain] == [F(x).limit_denominator() for x in g["wasted_gbps"]]
    s = S.schedule_collective(t, S.AR, 1 << 30, 64, S.BASELINE)
    u = float(E.simulate(s, E.FIFO).util)
    assert abs(u - float(sum(chain)) / 2400) < 0.005
    assert abs(u - GOLD["next_gen_baseline_min_util"]["min"]) < 0.01


def _microbenchmark():
    g = GOLD["microbenchmark"]
    ub, uf, us, sf, ss = [], [], [], [], []
    for name, t in T.PRESETS.items():
        for sz in g["sizes_mb"]:
            b = S.schedule_collective(t, S.AR, sz * MB, g["chunks"], S.BASELINE)
            th = S.schedule_collective(t, S.AR, sz * MB, g["chunks"], S.THEMIS)
            mb, mf, ms = E.simulate(b, E.FIFO), E.simulate(th, E.FIFO), E.simulate(th, E.SCF)
            ub.append(mb.util); uf.append(mf.util); us.append(ms.util)
            sf.append(mb.makespan / mf.makespan); ss.append(mb.makespan / ms.makespan)
    avg = lambda x: float(sum(x)) / len(x)
    return dict(ub=avg(ub), uf=avg(uf), us=avg(us), sf=avg(sf), ss=avg(ss), smax=float(max(ss)))


def test_microbenchmark_averages_match_paper():
    """averages over 6 topologies x 100MB-1GB at 64 chunks.
    The zero-latency exact model is not ASTRA-SIM, so tolerances apply."""
    g = GOLD["microbenchmark"]
    r = _microbenchmark()
    assert abs(r["ub"] - g["util_baseline"]) < 0.03
    assert abs(r["sf"] - g["speedup_fifo"]) < 0.08
    assert abs(r["ss"] - g["speedup_scf"]) < 0.12
    assert abs(r["smax"] - g["speedup_scf_max"]) < 0.12
    assert abs(r["us"] - g["util_scf"]) < 0.03
    assert abs(r["uf"] - g["util_fifo"]) < 0.03
    assert r["ss"] > r["sf"] > 1


def test_fig8_chunk_sensitivity():
    """4 -> 512 chunks raises Themis utilisation (48.58 -> 91.18%
    SCF, 43.13 -> 87.81% FIFO); SCF beats FIFO."""
    g = GOLD["fig8"]
    res = {}
    for C in (4, 512):
        us, uf = [], []
        for name in g["topologies"]:
            th = S.schedule_collective(T.PRESETS[name], S.AR, g["size_mb"] * MB, C, S.THEMIS)
            us.append(float(E.simulate(th, E.SCF).util))
            uf.append(float(E.simulate(th, E.FIFO).util))
        res[C] = (sum(us) / 2, sum(uf) / 2)
    assert res[512][0] - res[4][0] >= 0.25
    assert res[512][1] - res[4][1] >= 0.25
    for C in (4, 512):
        assert res[C][0] >= res[C][1]
        assert abs(res[C][0] - g["scf"][str(C)]) < 0.1
        assert abs(res[C][1] - g["fifo"][str(C)]) < 0.1


def test_export_csv():
    t = fig3_topo()
    s = S.schedule_collective(t, S.AR, 256 * MB, 4, S.THEMIS)
    lines = S.export_csv(s).strip().split("\n")
    assert lines[0] == "chunk_id,rs_order,ag_order,bytes"
    assert lines[2].startswith("1,2 1,1 2,")


def test_choose_chunks_single_dim_closed_form():
    """D = 1: the one dim serves all 2C ops back to back, so the makespan is
    2C*A + 2S(P-1)/P * B (PAPER.md:468 with idle = 0): strictly increasing in C
    when A > 0 (choice C = 1), constant when A = 0 (tie -> smallest C = 1)."""
    from fractions import Fraction as F
    from oracle import engine as E, scheduler as S, topology as T
    S_ = 1 << 20
    for lat in (0, 1000):
        t = T.Topology.make((4,), [F(100)], [T.DIRECT], [lat])
        best = E.choose_chunks(t, S.AR, S_, S.THEMIS, E.SCF, charge_latency=True)
        assert best[0] == 1
        for C in (1, 2, 8, 64):
            m = E.simulate(S.schedule_collective(t, S.AR, S_, C, S.THEMIS), E.SCF, charge_latency=True)
            assert m.makespan == 2 * C * lat + F(2 * S_ * 3, 4) / 100
    assert E.choose_chunks(T.Topology.make((4,), [F(100)]), S.AR, 4 * 16 + 8, S.THEMIS) is None


def test_choose_chunks_pipelining_without_latency():
    """D = 2, A = 0: one chunk cannot overlap the two dims (makespan = the sum
    of its four stage times), many chunks approach the Ideal bound (R13), so
    the choice is never C = 1 and its makespan is within the pipeline fill of
    the Ideal."""
    from fractions import Fraction as F
    from oracle import engine as E, scheduler as S, topology as T
    t = T.Topology.make((2, 2), [F(100), F(100)])
    S_ = 1 << 22
    C, sched, m = E.choose_chunks(t, S.AR, S_, S.BASELINE, E.FIFO)
    one = E.simulate(S.schedule_collective(t, S.AR, S_, 1, S.BASELINE), E.FIFO)
    assert one.makespan == (F(S_, 2) + F(S_, 4) + F(S_, 4) + F(S_, 2)) / 100   # chain of 4 stages, nothing overlaps
    assert C > 1 and m.makespan < one.makespan
    assert m.makespan >= E.ideal_time(sched)


def test_release_streaming_closed_form():
    """R26: when chunks arrive slower than one chunk's whole chain takes, each
    chunk runs alone: makespan = C*r + (sum of the last chunk's stage times),
    and stage 0 of chunk c starts exactly at its arrival (c+1)*r."""
    from fractions import Fraction as F
    from oracle import engine as E, scheduler as S, topology as T
    t = T.Topology.make((2, 2, 2), [F(100), F(50), F(25)])
    S_, C = 1 << 20, 8
    sched = S.schedule_collective(t, S.AR, S_, C, S.BASELINE)
    chain = sum(op.duration for op in E.chunk_ops(sched)[C - 1])
    r = chain + 1
    m = E.simulate(sched, E.FIFO, release=r)
    assert m.makespan == C * r + chain
    for c in range(C):
        assert m.start[(c, 0)] == (c + 1) * r
    # release = 0 is the paper's model (everything ready at t = 0)
    assert E.simulate(sched, E.FIFO, release=0).makespan == E.simulate(sched, E.FIFO).makespan
