"""Quick timing probe (development aid, not the bench): emulated P-rank AR on one GPU."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="2,2,2")
ap.add_argument("--bw", default="1,1,1")
ap.add_argument("--mib", type=int, default=1024)
ap.add_argument("--chunks", type=int, default=64)
ap.add_argument("--ctas", default="")
ap.add_argument("--engine", default="tma")
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
sizes = tuple(int(x) for x in a.sizes.split(","))
bw = tuple(int(x) for x in a.bw.split(","))
topo = th.Topology(sizes, bw)
N = (a.mib << 20) // 4
comm = th.Comm(topo, N * 4)
comm.set_engine(a.engine)
for r in range(topo.P):
    comm.rank_view(r, N, "f32").fill_(1.0)
for pol in (th.BASELINE, th.THEMIS):
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, a.chunks, pol)
    ctas = [int(x) for x in a.ctas.split(",")] if a.ctas else None
    plan.bind(comm, ctas)
    for _ in range(2):
        th.run(th.ALLREDUCE, comm, plan, N, "f32")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(a.iters):
        e0.record()
        th.run(th.ALLREDUCE, comm, plan, N, "f32")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    comm.status()
    t = min(ts) * 1e-3
    P = topo.P
    bus = 2 * N * 4 * (P - 1) / P / t / 1e9
    hbm = 0.0
    print(f"{'themis' if pol else 'baseline'} sizes={sizes} bw={bw} ctas={plan.bound_ctas()} engine={a.engine} "
          f"t={t*1e3:.3f} ms busBW/rank={bus:.1f} GB/s  pred_ratio_makespan={plan.makespan_ns()}")
    plan.close()
comm.close()
