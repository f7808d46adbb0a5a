"""K5 calibration of the CTA-cap bandwidth emulation (SURVEY.md §8(d),
north_star (d)): one dimension group alone — a P_k = 2 All-Reduce of S bytes
per rank, both ranks emulated in one GPU — on c CTAs, for a sweep of c.

Each c runs `--launches` collectives back to back (CUDA-event timed) and prints
one JSON line per c: the group's achieved per-rank bus GB/s and the algorithmic
HBM bytes per launch (RS holding S: read S + write S/2 per rank; AG: read and
write S/2 per rank -> 2.5 S per rank).  Under `ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum` the same
launches give the measured DRAM bytes and rate per c (launch order = the
printed order).

    python scripts/k5_probe.py --ctas 8,16,21,32,42,64,85,148
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402
from synth import device_input  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctas", default="8,16,21,32,42,64,85,148")
ap.add_argument("--mib", type=int, default=1024)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--chunks", type=int, default=4, help="few, large chunks: bandwidth- not latency-bound")
ap.add_argument("--stages", type=int, default=6)
a = ap.parse_args()
torch.cuda.set_device(0)
S = a.mib << 20
N = S // 4
topo = th.Topology((2,), (1,))
comm = th.Comm(topo, S)
comm.set_stages(a.stages)
src = [device_input(r, N, "f32", torch.device("cuda", 0)) for r in range(2)]
for c in [int(x) for x in a.ctas.split(",")]:
    plan = th.Plan(topo, th.ALLREDUCE, S, a.chunks, th.BASELINE).bind(comm, [c])
    ts = []
    for _ in range(a.launches):
        for r in range(2):
            comm.rank_view(r, N, "f32").copy_(src[r])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        th.run(th.ALLREDUCE, comm, plan, N, "f32")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    comm.status()
    t = min(ts)
    print(json.dumps({"ctas": c, "mib_per_rank": a.mib, "chunks": a.chunks, "launches": a.launches, "best_ms": round(t * 1e3, 4),
                      "bus_gbs_per_rank": round(2 * S * 0.5 / t / 1e9, 1),
                      "algorithmic_hbm_bytes_per_launch": int(2 * 2.5 * S),
                      "algorithmic_hbm_gbs": round(2 * 2.5 * S / t / 1e9, 1)}), flush=True)
    plan.close()
comm.close()
