"""Hand-derived pins for the oracle (VERDICT r01 "Next
round" item 1).

Every expected value below is derived by hand in the docstring of its test —
the tracker walked chunk by chunk, the event timeline written out op by op —
from the paper's definitions (Algorithm 1; threshold,
:614; per-stage volume n_K = (P-1)/P x chunk for RS and (P-1) x bytes for AG,
:331/:487; util, :292) and typed in as literals.  None comes from running the
oracle or the CUDA path.
"""

from fractions import Fraction as F

from oracle import brute, engine as E, scheduler as S, topology as T

MiB = 2 ** 20


def test_2x2x2_111_first_eight_orders_and_tracker():
    """2x2x2, BW 1:1:1, 1 GiB, C = 64 (BASELINE configs[1] topology, SURVEY
    §8(a) a3).  Unit u = chunk x B.  An RS on a P = 2 dim sends half the
    bytes it holds, an AG sends what it holds, so order (a, b, c) charges
    a: 1/2 + 1/2 = 1, b: 1/4 + 1/4 = 1/2, c: 1/8 + 1/8 = 1/4.
    Threshold = RS of chunk/16 on the min-load dim = 1/32 u.
      c1 loads 0,0,0: gap 0 < 1/32 -> baseline (1,2,3); L = [1, 1/2, 1/4]
      c2 gap 3/4: sort by (L, k) -> (3,2,1);  L = [5/4, 1, 5/4]
      c3 -> (2,1,3);  L = [7/4, 2, 3/2]
      c4 -> (3,1,2);  L = [9/4, 9/4, 5/2]
      c5 -> (1,2,3) (tie dim1/dim2 broken by index);  L = [13/4, 11/4, 11/4]
      c6 -> (2,3,1);  L = [7/2, 15/4, 13/4]
      c7 -> (3,1,2);  L = [4, 4, 17/4]
      c8 -> (1,2,3)"""
    t = T.Topology.make((2, 2, 2), (1, 1, 1))
    S_ = 2 ** 30
    s = S.schedule_collective(t, S.AR, S_, 64, S.THEMIS)
    assert [tuple(d + 1 for d in c.rs) for c in s.chunks[:8]] == [
        (1, 2, 3), (3, 2, 1), (2, 1, 3), (3, 1, 2), (1, 2, 3), (2, 3, 1), (3, 1, 2), (1, 2, 3)]
    u = F(S_, 64)                 # B = 1 byte/ns
    want = [[1, F(1, 2), F(1, 4)], [F(5, 4), 1, F(5, 4)], [F(7, 4), 2, F(3, 2)], [F(9, 4), F(9, 4), F(5, 2)],
            [F(13, 4), F(11, 4), F(11, 4)], [F(7, 2), F(15, 4), F(13, 4)], [4, 4, F(17, 4)]]
    for n, w in enumerate(want, start=1):
        part = S.schedule_collective(t, S.AR, S_ * n // 64, n, S.THEMIS)   # same chunk size, first n chunks
        assert part.loads == [x * u for x in w], n


def test_2x2x2_111_dim_bytes_and_speedup():
    """Per-dim bytes N_K: a chunk of 16 MiB charges its
    first dim 16 MiB (RS 8 + AG 8), its second 8 MiB, its third 4 MiB; over
    the Themis orders N = [596, 596, 600] MiB ([derived]);
    the baseline puts every chunk on (1,2,3): [1024, 512, 256] MiB.  Sum =
    2 S (P-1)/P = 1792 MiB for both (F2).
    Baseline makespan = dim1's busy time 64 u (dim1 never idles: RS ops of
    later chunks are always ready); Themis+SCF makespan 75/128 S B = 37.5 u,
    speedup 128/75 = 1.7067."""
    t = T.Topology.make((2, 2, 2), (1, 1, 1))
    S_ = 2 ** 30
    th = S.schedule_collective(t, S.AR, S_, 64, S.THEMIS)
    bl = S.schedule_collective(t, S.AR, S_, 64, S.BASELINE)
    assert S.dim_volumes(th) == [596 * MiB, 596 * MiB, 600 * MiB]
    assert S.dim_volumes(bl) == [1024 * MiB, 512 * MiB, 256 * MiB]
    mt, mb = E.simulate(th, E.SCF), E.simulate(bl, E.SCF)
    assert mb.makespan == S_ and mb.busy[0] == S_
    assert mt.makespan == F(75, 128) * S_
    assert mb.makespan / mt.makespan == F(128, 75)


def test_config1_engine_values():
    """BASELINE configs[0]: 2x4, 200:50 GB/s (bytes/ns), 64 KiB, C = 4,
    chunk 16384 B, every chunk (1,2) (under-provisioned).
    Op times: RS d1 8192/200 = 40.96 ns; RS d2 (3/4)8192/50 = 122.88;
    AG d2 3 x 2048/50 = 122.88; AG d1 8192/200 = 40.96.
    dim1 busy 4 x 81.92 = 327.68 = 8192/25 ns; dim2 busy 8 x 122.88 =
    983.04 = 24576/25 ns.  dim2 starts at 40.96 and always has a ready op
    (RS c_i ready at 40.96 (i+1), AGs as RSs finish), so it ends at 1024.0;
    the last AG d1 adds 40.96: makespan 1064.96 = 26624/25 ns.
    util = (200 x 327.68 + 50 x 983.04) / (250 x 1064.96) = 114688/266240."""
    t = T.Topology.make((2, 4), (200, 50))
    s = S.schedule_collective(t, S.AR, 65536, 4, S.THEMIS)
    assert all(c.rs == (0, 1) for c in s.chunks)
    assert S.dim_volumes(s) == [65536, 49152]
    for pol in (E.SCF, E.FIFO):
        m = E.simulate(s, pol)
        assert m.makespan == F(26624, 25)
        assert m.busy == [F(8192, 25), F(24576, 25)]
        assert m.util == F(114688, 266240)
        assert round(float(m.util), 4) == 0.4308


def test_fig6_tracker_all_chunks():
    """Fig 6: 4x4, BW(dim1) = 2 BW(dim2), 256 MB AR,
    4 chunks of 64 MB; unit u = RS of 64 MB on dim1.
      c1 (1,2): RS d1 1, RS d2 1/2, AG d2 1/2, AG d1 1 -> L = [2, 1]
      c2: gap 1 >= thr (RS of 4 MB on dim2 = 1/8) -> (2,1):
          RS d2 of 64 MB = 2, RS d1 of 16 MB = 1/4, AG d1 1/4, AG d2 2 -> [5/2, 5]
      c3: min dim1, gap 5/2 -> (1,2): +[2, 1] -> [9/2, 6]
      c4: (1,2) -> [13/2, 7]"""
    t = T.Topology.make((4, 4), (2, 1))
    u = F(3, 4) * 64 * MiB / 2
    want = [[2, 1], [F(5, 2), 5], [F(9, 2), 6], [F(13, 2), 7]]
    for n, w in enumerate(want, start=1):
        s = S.schedule_collective(t, S.AR, n * 64 * MiB, n, S.THEMIS)
        assert s.loads == [x * u for x in w], n


def test_f4_regression_themis_can_lose():
    """Themis <= baseline is not an invariant.  4x2, BW 7:3
    bytes/ns, S = 256 B, C = 2 (chunk 128 B).
    Baseline, both chunks (1,2): RS d1 96/7, RS d2 16/3, AG d2 16/3,
    AG d1 96/7.  dim1: RS c0 [0, 288/21], RS c1 [288/21, 576/21], AG c0
    [576/21, 864/21], AG c1 [864/21, 1152/21] -> makespan 384/7.
    Themis: c1 (1,2); c2 -> (2,1): RS d2 64/3, RS d1 48/7, AG d1 48/7,
    AG d2 64/3.  dim2: RS c1 [0, 448/21], RS c0 [448/21, 560/21], AG c0
    [560/21, 672/21], idle, AG c1 [736/21, 1184/21]; dim1: RS c0
    [0, 288/21], RS c1 [448/21, 592/21], AG c1 [592/21, 736/21] (SCF: the
    smaller volume), AG c0 [736/21, 1024/21] -> makespan 1184/21 > 384/7.
    The brute-force optimum is <= both (SURVEY §8(c.4) Optimality)."""
    t = T.Topology.make((4, 2), (7, 3))
    bl = E.simulate(S.schedule_collective(t, S.AR, 256, 2, S.BASELINE), E.SCF)
    th = E.simulate(S.schedule_collective(t, S.AR, 256, 2, S.THEMIS), E.SCF)
    assert bl.makespan == F(384, 7)
    assert th.makespan == F(1184, 21)
    assert th.makespan > bl.makespan
    best, _, count = brute.exhaustive_best(t, S.AR, 256, 2, E.SCF)
    assert count == 4                        # (2!)^2 reversed-AG assignments
    best = getattr(best, "makespan", best)
    assert best <= bl.makespan


def test_ideal_time_values():
    """Ideal (Table 3; reading R13) = algorithmic bytes per NPU
    / sum BW: AR 2 S (P-1)/P, RS or AG S (P-1)/P.
      2x2x2, 1:1:1, S = 2^30: 2 x 2^30 x 7/8 / 3 = 7/12 x 2^30
      2x4, 200:50, S = 65536: 2 x 65536 x 7/8 / 250 = 114688/250 ns
      4x4, 2:1, RS of 256 MiB: 256 MiB x 15/16 / 3 = 80 MiB"""
    t = T.Topology.make((2, 2, 2), (1, 1, 1))
    assert E.ideal_time(S.schedule_collective(t, S.AR, 2 ** 30, 64, S.THEMIS)) == F(7, 12) * 2 ** 30
    t = T.Topology.make((2, 4), (200, 50))
    assert E.ideal_time(S.schedule_collective(t, S.AR, 65536, 4, S.THEMIS)) == F(114688, 250)
    t = T.Topology.make((4, 4), (2, 1))
    assert E.ideal_time(S.schedule_collective(t, "RS", 256 * MiB, 4, S.THEMIS)) == 80 * MiB
    assert E.ideal_time(S.schedule_collective(t, "AG", 256 * MiB, 4, S.THEMIS)) == 80 * MiB


# ---------------------------------------------------------------- R29: NVLS row
def test_nvls_fused_pair_bytes_by_message_count():
    """The fused in-switch RS+AG pair's n = (1 + 1/p) b (R29), counted message
    by message on the multimem protocol (PAPER.md:493-494 offload): every
    member m owns piece m (b/p bytes) of the b bytes it holds; for each piece j
    the switch pulls member m's copy of piece j (ld_reduce on behalf of its
    owner j) and the owner multicasts the reduced piece once (multimem.st).
    Sent by member m: its copy of every piece (p x b/p) + one multicast (b/p)."""
    from oracle import collectives as col
    for p in (2, 4, 8):
        b = F(64 * p)
        piece = b / p
        sent = [F(0)] * p
        for j in range(p):                 # piece j, reduced for its owner j
            for m in range(p):             # the switch reads member m's copy
                sent[m] += piece
            sent[j] += piece               # owner j multicasts the sum
        assert sent == [col.fused_bytes_sent(p, b)] * p


def test_nvls_single_dim_closed_form():
    """D = 1, P = 4, S = 64 B, C = 4, BW 1 B/ns.  Per chunk (16 B): NVLS = one
    fused op of 16 + 16/4 = 20 ns, its AG half 0 ns -> makespan 4 x 20 = 80 =
    (5/4) S; the direct algorithm sends 3/4 x 16 = 12 (RS) + 3 x 4 = 12 (AG)
    per chunk -> 96 = (3/2) S.  P = 2: NVLS 4 x (16 + 8) = 96 = (3/2) S vs
    direct 4 x (8 + 8) = 64 = S (offload loses at P = 2)."""
    for p, nv, di in ((4, 80, 96), (2, 96, 64)):
        for kind, want in ((T.NVLS, nv), (T.DIRECT, di)):
            t = T.Topology.make((p,), (1,), (kind,))
            m = E.simulate(S.schedule_collective(t, S.AR, 64, 4, S.THEMIS), E.SCF)
            assert m.makespan == want
            assert m.volume == [want]


def test_nvls_2x4_tracker_and_timeline():
    """2x4, dim2 NVLS, BW 1:1 (1 B/ns), S = 16 B, C = 2 (chunk 8 B).
    Tracker (R1 + R29):
      c0: loads 0,0 -> baseline (1,2).  RS d1 holds 8: 4 -> L1 = 4; the fused
          pair on d2 holds 4: 4 + 4/4 = 5 -> L2 = 5; AG d1 holds 4: 4 -> L1 = 8.
      c1: gap 3 >= thr = 3/4 x 8/16 = 3/8 on m = d2 -> sort (2,1), not fused
          (last RS dim d1 is direct): RS d2 holds 8: 6; RS d1 holds 2: 1; AG d1
          holds 1: 1; AG d2 holds 2: 3 x 2 = 6  -> L = [10, 17] = N (B = 1).
    Timeline (SCF key volume, ready, chunk):
      t=0  d1: c0s0 [0,4]   d2: c1s0 [0,6]
      t=6  d1: c1s1 [6,7]   d2: c0s1 fused [6,11]
      t=7  d1: c1s2 [7,8]   (c1s3 on d2 ready at 8)
      t=11 d2: ready c1s3 (vol 6, t 8), c0s2 (vol 0, t 11) -> c0s2 [11,11];
           then d1: c0s3 [11,15]; d2: c1s3 [11,17]      makespan 17
      busy [10, 17], util 27/34.
    FIFO (ready, chunk) at t=11 takes c1s3 [11,17], then c0s2 [17,17] and
    c0s3 [17,21]: makespan 21."""
    t = T.Topology.make((2, 4), (1, 1), (T.DIRECT, T.NVLS))
    s = S.schedule_collective(t, S.AR, 16, 2, S.THEMIS)
    assert [c.rs for c in s.chunks] == [(0, 1), (1, 0)]
    assert s.loads == [10, 17]
    assert S.dim_volumes(s) == [10, 17]
    m = E.simulate(s, E.SCF)
    assert m.makespan == 17 and m.busy == [10, 17] and m.util == F(27, 34)
    assert m.start[(0, 1)] == 6 and m.end[(0, 1)] == 11 and m.start[(0, 2)] == 11 and m.end[(0, 2)] == 11
    assert m.start[(0, 3)] == 11 and m.start[(1, 3)] == 11
    assert E.simulate(s, E.FIFO).makespan == 21


def test_nvls_data_path_is_the_all_reduce():
    """The fused pair is RS then AG on one dim: the oracle's data executor is
    unchanged by R29 and still produces the plain All-Reduce (int32 exact)."""
    from oracle import data as O
    from synth import host_inputs
    t = T.Topology.make((2, 4), (1, 1), (T.DIRECT, T.NVLS))
    xs = host_inputs(8, 8 * 4 * 16, "i32")
    s = S.schedule_collective(t, S.AR, 8 * 4 * 16 * 4, 4, S.THEMIS)
    out = O.run_schedule(xs, s, "i32")
    want = O.allreduce_definition(xs, "i32")
    assert all((o == want).all() for o in out)


def test_nvls_fixed_delay_seed_and_charge():
    """R29 A_K of the fused pair = 2 steps (reduce + multicast) x step_latency.
    D = 1, P = 4, NVLS, step latency 700 ns, S = 64 B, C = 4, BW 1 B/ns:
      tracker seed (AR) = 2 x 700 = 1400 (a plain switch dim: 2 phases x
      log2 4 steps x 700 = 2800); final tracker = 1400 + 4 x 20 = 1480;
      with per-op latency charged each fused op takes 20 + 1400 ns and its AG
      half 0 -> makespan 4 x 1420 = 5680."""
    t = T.Topology.make((4,), (1,), (T.NVLS,), (700,))
    s = S.schedule_collective(t, S.AR, 64, 4, S.THEMIS)
    assert S.tracker_reset(t, S.AR) == [1400]
    assert S.tracker_reset(T.Topology.make((4,), (1,), (T.SWITCH,), (700,)), S.AR) == [2800]
    assert s.loads == [1480]
    assert E.simulate(s, E.SCF, charge_latency=True).makespan == 5680
