"""Full-size parity (BASELINE.json configs[1]) in the launch configuration
bench.py times at N = 1: logical 2x2x2 emulated in one GPU, 1 GiB per rank,
64 chunks, emulated 4:2:1 CTA caps [85, 42, 21], 6 TMA stages.

* sampled elements: bit-exact against the oracle's per-element formulation
  (oracle.data.allreduce_element, pinned to the step-by-step simulator) with
  the oracle's own Themis schedule;
* whole buffer: every rank bitwise identical; fp32 error vs the fp64 sum
  within 1e-5 * sum|x| (north_star); int32 exact vs the wrapped int64 sum.
"""

import numpy as np
import pytest
import torch

from oracle import data as O, scheduler as S, topology as T
from paper_2110_04478_b200 import themis as th
from synth import device_input

pytestmark = pytest.mark.gpu

SIZES, RATIO, C, MIB = (2, 2, 2), (4, 2, 1), 64, 1024


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("dtype", ["f32", "i32"])
def test_config2_full_size(dtype):
    topo = th.Topology(SIZES, RATIO)
    P = topo.P
    S_ = MIB << 20
    N = S_ // 4
    import bench
    cfg = bench.launch_config(SIZES, 1, torch.cuda.get_device_properties(0).multi_processor_count)
    comm = th.Comm(topo, S_)                            # bench.py's N = 1 launch configuration
    comm.set_stages(1)
    comm.set_stage_bytes(cfg["stage_kb"] * 1024)
    comm.set_stages(cfg["stages"])
    comm.set_lookahead(cfg["lookahead"])
    comm.set_min_cta_bytes(cfg["min_cta_bytes"])
    comm.set_timeout(30.0)
    plan = th.Plan(topo, th.ALLREDUCE, S_, C, th.THEMIS).bind(comm, th.default_ctas(RATIO, cfg["total_ctas"]))
    try:
        xs = [device_input(r, N, dtype, torch.device("cuda", 0)) for r in range(P)]
        for r in range(P):
            comm.rank_view(r, N, dtype).copy_(xs[r])
        th.run(th.ALLREDUCE, comm, plan, N, dtype)
        torch.cuda.synchronize()
        comm.status()
        outs = [comm.rank_view(r, N, dtype) for r in range(P)]
        for r in range(1, P):                               # all ranks bitwise identical
            assert torch.equal(outs[r], outs[0])
        if dtype == "i32":                                  # exact vs the definition (library sum)
            s = torch.zeros(N, dtype=torch.int64, device="cuda")
            for x in xs:
                s += x.to(torch.int64)
            want = ((s + 2 ** 31) % 2 ** 32 - 2 ** 31).to(torch.int32)
            assert torch.equal(outs[0], want)
        else:                                               # |y - sum| <= 1e-5 sum|x|
            s = torch.zeros(N, dtype=torch.float64, device="cuda")
            a = torch.zeros(N, dtype=torch.float64, device="cuda")
            for x in xs:
                s += x.to(torch.float64)
                a += x.to(torch.float64).abs()
            err = (outs[0].to(torch.float64) - s).abs()
            assert bool((err <= 1e-5 * a).all())
            # sampled elements bit-exact vs the oracle, with the oracle's schedule
            o = T.Topology.make(SIZES, RATIO)
            sched = S.schedule_collective(o, S.AR, S_, C, S.THEMIS)
            rng = np.random.default_rng(5)
            idx = np.unique(np.concatenate([rng.integers(0, N, 1500), [0, N - 1, N // 2, N // P - 1]]))
            it = torch.from_numpy(idx).cuda()
            xv = torch.stack([x[it] for x in xs]).cpu().numpy()
            got = torch.stack([o_[it] for o_ in outs]).cpu().numpy()
            for n, i in enumerate(idx):
                b, c = O.element_location(o, N, C, int(i))
                v = O.allreduce_element(list(xv[:, n]), o, sched.chunks[c].rs, "f32", b)
                assert np.float32(v).tobytes() == got[0, n].tobytes(), f"element {i}"
    finally:
        plan.close()
        comm.close()


def test_max_size_bf16_over_2pow31_elements():
    """Maximum-size edge case: 2^31 + 2^25 bf16 elements (4.06 GiB) per rank,
    8 ranks in one GPU (33 GB heap): element indices exceed int32 and byte
    offsets exceed 32 bits.  Every rank bitwise identical; sampled elements
    (including both ends of every block) bit-exact vs the oracle's
    per-element formulation with the oracle's Themis schedule at 1:1:1."""
    ratio = (1, 1, 1)
    topo = th.Topology(SIZES, ratio)
    P = topo.P
    N = (1 << 31) + (1 << 25)
    S_ = N * 2
    comm = th.Comm(topo, S_)
    comm.set_timeout(60.0)
    plan = th.Plan(topo, th.ALLREDUCE, S_, C, th.THEMIS).bind(comm)
    try:
        rng = np.random.default_rng(11)
        blk = N // P
        idx = np.unique(np.concatenate([rng.integers(0, N, 800), [b * blk for b in range(P)],
                                        [b * blk + blk - 1 for b in range(P)], [(1 << 31) - 1, 1 << 31, N - 1]]))
        it = torch.from_numpy(idx).cuda()
        xv = []
        for r in range(P):
            x = device_input(r, N, "bf16", torch.device("cuda", 0))
            comm.rank_view(r, N, "bf16").copy_(x)
            xv.append(x[it].view(torch.int16).cpu().numpy().view(np.uint16))
            del x
        th.run(th.ALLREDUCE, comm, plan, N, "bf16")
        torch.cuda.synchronize()
        comm.status()
        outs = [comm.rank_view(r, N, "bf16") for r in range(P)]
        for r in range(1, P):
            assert torch.equal(outs[r].view(torch.int16), outs[0].view(torch.int16))
        got = outs[0][it].view(torch.int16).cpu().numpy().view(np.uint16)
        o = T.Topology.make(SIZES, ratio)
        sched = S.schedule_collective(o, S.AR, S_, C, S.THEMIS)
        xv = np.stack(xv)
        for n, i in enumerate(idx):
            b, c = O.element_location(o, N, C, int(i))
            v = O.allreduce_element(list(xv[:, n]), o, sched.chunks[c].rs, "bf16", b)
            assert np.asarray(v).view(np.uint16).ravel()[0] == got[n], f"element {i}"
    finally:
        plan.close()
        comm.close()
