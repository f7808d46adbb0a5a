"""Development probe: per-op device trace of one paced All-Reduce vs the plan's
pre-simulated times (where does the time go?).  Emulated on one GPU."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bw", default="80,80,80")       # GB/s per dim (paced)
ap.add_argument("--mib", type=int, default=1024)
ap.add_argument("--chunks", type=int, default=64)
ap.add_argument("--policy", default="themis")
ap.add_argument("--ctas", default="")
ap.add_argument("--pace", type=int, default=1)
a = ap.parse_args()
bw = tuple(int(x) * 1000 for x in a.bw.split(","))
topo = th.Topology((2, 2, 2), bw)
N = (a.mib << 20) // 4
comm = th.Comm(topo, N * 4)
comm.set_pacing(bool(a.pace))
comm.enable_trace(True)
for r in range(8):
    comm.rank_view(r, N, "f32").fill_(1.0)
plan = th.Plan(topo, th.ALLREDUCE, N * 4, a.chunks, th.THEMIS if a.policy == "themis" else th.BASELINE)
ctas = [int(x) for x in a.ctas.split(",")] if a.ctas else th.default_ctas([b for b in bw], 148)
plan.bind(comm, ctas)
for _ in range(3):
    th.run(th.ALLREDUCE, comm, plan, N, "f32")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
th.run(th.ALLREDUCE, comm, plan, N, "f32")
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e6
tr = comm.fetch_trace(plan).astype(np.int64)
t0 = tr[:, :, 0].min()
tr = tr - t0
flat = np.unique(tr.ravel())
print("globaltimer granularity (gcd of trace stamps):", int(np.gcd.reduce(flat[flat > 0])) if flat.size > 1 else -1)
st, en = plan.times()
ts = plan.info["time_scale"]
NS = plan.info["n_stages"]
ms = float(plan.makespan_ns())
print(f"kernel {t/1e3:.1f} us; trace span {tr.max()/1e3:.1f} us; model makespan {ms/1e3:.1f} us; ctas {plan.bound_ctas()}")
for k, ops in enumerate(plan.dim_ops()):
    dur = np.array([tr[c, s, 1] - tr[c, s, 0] for c, s in ops])
    mdur = np.array([(int(en[c * NS + s]) - int(st[c * NS + s])) / ts for c, s in ops])
    starts = np.array([tr[c, s, 0] for c, s in ops])
    ends = np.array([tr[c, s, 1] for c, s in ops])
    gaps = starts[1:] - ends[:-1]
    print(f"dim{k+1}: ops {len(ops)} busy {dur.sum()/1e3:.1f} us (model {mdur.sum()/1e3:.1f}); "
          f"first start {starts[0]/1e3:.1f} last end {ends[-1]/1e3:.1f}; gap mean {gaps.mean()/1e3:.2f} "
          f"max {gaps.max()/1e3:.2f} us; op dur/model mean {np.mean(dur/mdur):.3f} min {np.min(dur/mdur):.3f}")
    print("   first ops (dur us, model us):", [(round(d / 1e3, 1), round(m / 1e3, 1)) for d, m in zip(dur[:6], mdur[:6])])
lat = []
for c in range(plan.info["n_chunks"]):
    for s in range(1, NS):
        lat.append(tr[c, s, 0] - tr[c, s - 1, 1])
lat = np.array(lat)
print(f"stage transition (start(c,s) - end(c,s-1)) us: p10 {np.percentile(lat,10)/1e3:.2f} median "
      f"{np.median(lat)/1e3:.2f} p90 {np.percentile(lat,90)/1e3:.2f} min {lat.min()/1e3:.2f}")
# per-dim idle while the dim still has pending ops (model idle_K analogue)
for k, ops in enumerate(plan.dim_ops()):
    iv = sorted((tr[c, s, 0], tr[c, s, 1]) for c, s in ops)
    busy, cur_s, cur_e = 0, iv[0][0], iv[0][1]
    for a_, b_ in iv[1:]:
        if a_ > cur_e:
            busy += cur_e - cur_s
            cur_s, cur_e = a_, b_
        else:
            cur_e = max(cur_e, b_)
    busy += cur_e - cur_s
    print(f"dim{k+1}: union-busy {busy/1e3:.1f} us of span {(iv[-1][1]-iv[0][0])/1e3:.1f} us")
plan.close()
comm.close()
