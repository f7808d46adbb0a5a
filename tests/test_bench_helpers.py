"""CPU checks of bench.py's roofline / emulation arithmetic."""

from fractions import Fraction

import bench
from paper_2110_04478_b200 import themis as th


def test_hbm_bytes_closed_form_2x2x2():
    """Per rank, RS holding H on a P_k = 2 dim reads H, writes H/2; AG holding
    h reads and writes h: 2x2x2 totals 4.375 S for every order."""
    S = 1 << 30
    for pol in (th.BASELINE, th.THEMIS):
        p = th.Plan(th.Topology((2, 2, 2), (1, 1, 1)), th.ALLREDUCE, S, 64, pol)
        assert bench.hbm_bytes_per_rank(p, S) == 4.375 * S
        p.close()


def test_nvlink_bytes_equal_bus_bytes_at_one_rank_per_gpu():
    """With every dim crossing GPUs the pulled bytes are sum_K N_K = 2S(P-1)/P (F2)."""
    S = 1 << 30
    p = th.Plan(th.Topology((2, 2, 2), (4, 2, 1)), th.ALLREDUCE, S, 64)
    lay = bench.logical_layout((2, 2, 2), 8)
    assert lay["V"] == 1 and lay["cross_gpu_dims"] == [0, 1, 2]
    assert bench.nvlink_bytes_per_gpu(p, (2, 2, 2), 8) == 2 * S * 7 / 8
    assert bench.nvlink_bytes_per_gpu(p, (2, 2, 2), 1) == 0
    p.close()


def test_nvlink_bytes_straddling_dim():
    """4x2 on 4 GPUs (V = 2): dim1's group {0,1,2,3} spans GPUs {0,0,1,1}, so
    2 of each rank's 3 dim1 peers are remote; dim2's peer is always remote."""
    S = 1 << 30
    p = th.Plan(th.Topology((4, 2), (1, 1)), th.ALLREDUCE, S, 64)
    n1, n2 = [v / p.info["byte_scale"] for v in p.info["dim_volume"]]
    assert bench.nvlink_bytes_per_gpu(p, (4, 2), 4) == 2 * (n1 * 2 / 3 + n2)
    assert bench.remote_fraction((4, 2), 4, 0, 1, ring=True) == 0.0      # rank 1's left neighbour is rank 0
    assert bench.remote_fraction((4, 2), 4, 0, 2, ring=True) == 1.0      # rank 2's is rank 1 (GPU 0)
    p.close()


def test_paced_bw_exact_ratio():
    for rat in [(4, 2, 1), (1, 1, 1), (2, 2, 1), (200, 50), (1,)]:
        bw = bench.paced_bw(rat, 500.0)
        assert all(Fraction(b, bw[0]) == Fraction(r, rat[0]) for b, r in zip(bw, rat))
        assert sum(bw) <= 500_000 + 1000 * len(rat) and all(b % 1000 == 0 for b in bw)


def test_launch_config_per_gpu_count():
    """bench.py's launch configuration (shared with the full-size parity
    tests): every-SM HBM runs at N = 1, the mixed and all-NVLink budgets, the
    runtime order where <= 2 ranks share a GPU."""
    c1 = bench.launch_config((2, 2, 2), 1, 148)
    assert (c1["total_ctas"], c1["stages"], c1["stage_kb"], c1["lookahead"]) == (148, 3, 64, 1)
    c2 = bench.launch_config((2, 2, 2), 2, 148)
    assert (c2["total_ctas"], c2["stages"], c2["stage_kb"], c2["lookahead"]) == (148, 4, 48, 1)
    c4 = bench.launch_config((2, 2, 2), 4, 148)
    assert (c4["total_ctas"], c4["stages"], c4["stage_kb"], c4["lookahead"]) == (96, 4, 48, 16)
    c8 = bench.launch_config((2, 2, 2), 8, 148)
    assert (c8["total_ctas"], c8["stages"], c8["stage_kb"], c8["lookahead"]) == (128, 2, 32, 16)
    assert all(c["stages"] * c["stage_kb"] <= 192 for c in (c1, c2, c4, c8))
