"""Fig 7-style per-dimension activity on the GPU.

One paced 2x2x2 All-Reduce (1 GiB fp32 per rank, 64 chunks, emulated
BW_1:BW_2:BW_3 = 1:1:1 unless --ratio) per policy, N = 1 (8 ranks emulated in
one GPU).  The device trace gives each op's start/end; a dimension is
"active" in a window while one of its ops is in service.  The same quantity
from the planner's pre-simulated op times is printed beside it (the model the
paper plots).  Output: markdown on stdout.

    python scripts/activity.py [--ratio 1:1:1] [--windows 20]
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402
from synth import device_input  # noqa: E402
import bench  # noqa: E402


def activity(intervals, t0, t1, nwin):
    """Fraction of each of nwin equal windows of [t0, t1) covered by the union of intervals."""
    edges = np.linspace(t0, t1, nwin + 1)
    iv = sorted(intervals)
    merged = []
    for a, b in iv:
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    out = []
    for w in range(nwin):
        lo, hi = edges[w], edges[w + 1]
        cov = sum(max(0.0, min(hi, b) - max(lo, a)) for a, b in merged)
        out.append(cov / (hi - lo))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ratio", default="1:1:1")
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--chunks", type=int, default=64)
    ap.add_argument("--windows", type=int, default=10)
    ap.add_argument("--pace-gbs", type=float, default=240.0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    sizes = (2, 2, 2)
    rat = tuple(int(x) for x in a.ratio.split(":"))
    bw = bench.paced_bw(rat, a.pace_gbs)
    S = a.mib << 20
    N = S // 4
    comm = th.Comm(th.Topology(sizes, bw), S)
    comm.set_stages(6)
    comm.set_pacing(True)
    src = [device_input(r, N, "f32", torch.device("cuda", 0)) for r in range(8)]
    print(f"# Per-dimension activity (Fig 7 analogue), 2x2x2, {a.mib} MiB fp32/rank, {a.chunks} chunks, "
          f"paced BW {':'.join(str(b // 1000) for b in bw)} GB/s, N = 1\n")
    print("Activity = fraction of each window in which the dimension has an op in service; measured from the\n"
          "device trace (`%globaltimer` per op) and, in parentheses, from the planner's pre-simulated times.\n")
    for pol, name in ((th.BASELINE, "baseline"), (th.THEMIS, "Themis")):
        plan = th.Plan(th.Topology(sizes, bw), th.ALLREDUCE, S, a.chunks, pol,
                       th.SCF if pol == th.THEMIS else th.FIFO).bind(comm, th.default_ctas(rat, 148))
        comm.enable_trace(True)
        for _ in range(2):
            for r in range(8):
                comm.rank_view(r, N, "f32").copy_(src[r])
            torch.cuda.synchronize()
            th.run(th.ALLREDUCE, comm, plan, N, "f32")
            torch.cuda.synchronize()
        comm.status()
        tr = comm.fetch_trace(plan).astype(np.int64)
        comm.enable_trace(False)
        st, en = plan.times()
        ts = plan.info["time_scale"]
        NS = plan.info["n_stages"]
        t0, t1 = tr[:, :, 0].min(), tr[:, :, 1].max()
        span_model = max(int(e) for e in en) / ts
        rows = []
        for k, ops in enumerate(plan.dim_ops()):
            meas = activity([(tr[c, s, 0], tr[c, s, 1]) for c, s in ops], t0, t1, a.windows)
            model = activity([(int(st[c * NS + s]) / ts, int(en[c * NS + s]) / ts) for c, s in ops], 0.0,
                             span_model, a.windows)
            rows.append((k, meas, model))
        print(f"## {name}: measured span {(t1 - t0) / 1e3:.0f} us, model makespan {span_model / 1e3:.0f} us\n")
        print("| dim | mean activity | " + " | ".join(f"w{i}" for i in range(a.windows)) + " |")
        print("|---|---|" + "---|" * a.windows)
        for k, meas, model in rows:
            cells = " | ".join(f"{m:.2f} ({p:.2f})" for m, p in zip(meas, model))
            print(f"| dim{k + 1} | {np.mean(meas):.3f} ({np.mean(model):.3f}) | {cells} |")
        print()
        plan.close()
    comm.close()


if __name__ == "__main__":
    main()
