"""Headline configuration per dtype at N = 1 (2x2x2, 1 GiB per rank, 64
chunks, 4:2:1 CTA caps over all SMs, 6 stages): bus GB/s and algorithmic HBM
GB/s for f32 / bf16 / f16 / i32 — the reduction's arithmetic should never
bind (bf16 sums 2x the elements per byte in fp32)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402
from synth import device_input  # noqa: E402
import bench  # noqa: E402

torch.cuda.set_device(0)
S = 1 << 30
topo = th.Topology((2, 2, 2), (4, 2, 1))
comm = th.Comm(topo, S)
comm.set_stages(6)
sms = torch.cuda.get_device_properties(0).multi_processor_count
plan = th.Plan(topo, th.ALLREDUCE, S, 64, th.THEMIS).bind(comm, th.default_ctas((4, 2, 1), sms))
for dt, esz in (("f32", 4), ("bf16", 2), ("f16", 2), ("i32", 4)):
    N = S // esz
    src = [device_input(r, N, dt, torch.device("cuda", 0)) for r in range(8)]
    ts = []
    for i in range(6):
        for r in range(8):
            comm.rank_view(r, N, dt).copy_(src[r])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        th.run(th.ALLREDUCE, comm, plan, N, dt)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / 1e3)
    comm.status()
    t = sum(ts) / len(ts)
    hbm = 8 * bench.hbm_bytes_per_rank(plan, S)
    print(json.dumps({"dtype": dt, "ms": round(t * 1e3, 3), "bus_gbs": round(2 * S * 7 / 8 / t / 1e9, 1),
                      "hbm_gbs": round(hbm / t / 1e9, 0)}), flush=True)
    del src
