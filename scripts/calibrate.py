"""Latency-model calibration on B200.

The paper's latency model is Latency(dim K) = A_K + N_K * B_K + idle_K with A_K
a fixed per-op delay and B_K = 1 / BW_K.  This script measures both on the
executor from device traces and feeds them back into the planner:

1. A_K: a minimum-size All-Reduce (one 16-byte vector per piece) — the median
   traced op duration on dim K plus the median stage-to-stage hand-off.
2. BW_K: a 1 GiB All-Reduce with the dims' CTA caps (or pacing): the dim's
   volume N_K over its traced busy time (union of op intervals) minus n_ops
   times the fixed part of an op.
3. Validation: for small and medium collectives the measured time is compared
   with the makespan the pre-simulation predicts from (A_K, BW_K) with
   `charge_latency` on, and with the paper's bandwidth-only model, and the
   latency-aware Themis plan (tracker seeded with A_K, A charged per op) is
   timed against the plain Themis plan and the baseline; finally the planner
   also picks the chunk count (n_chunks = 0) from the calibrated model.

    python scripts/calibrate.py [--ratio 4:2:1] [--paced]
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/calibrate.py --gpus 4

One JSON object per line on stdout (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_04478_b200 import themis as th  # noqa: E402
from paper_2110_04478_b200.dist import barrier, init_from_env, max_over_ranks  # noqa: E402
from synth import device_input  # noqa: E402
import bench  # noqa: E402


def op_dims(plan):
    rs, ag = plan.orders()
    return np.concatenate([rs, ag], axis=1)          # [C][2D] dim of stage s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--ratio", default="4:2:1")
    ap.add_argument("--paced", action="store_true")
    ap.add_argument("--pace-gbs", type=float, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--min-cta-kb", type=int, default=0, help="op windows: min bytes per CTA (KiB), 0 = full width")
    ap.add_argument("--rotate", type=int, default=1, help="op windows: consecutive windows (1) or from CTA 0 (0)")
    ap.add_argument("--sizes-mib", default="1,4,16,64,256")
    a = ap.parse_args()
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    out_fd = os.dup(1)
    os.dup2(2, 1)
    rank, world, local, group = init_from_env("nccl" if int(os.environ.get("WORLD_SIZE", 1)) > 1 else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sizes = (2, 2, 2)
    P, D = 8, 3
    lay = bench.logical_layout(sizes, world)
    V, ncross = lay["V"], len(lay["cross_gpu_dims"])
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ctas_total = sms if ncross == 0 else (32 * D + 32 if ncross == D else (sms if V >= 4 else 96))
    rat = tuple(int(x) for x in a.ratio.split(":"))
    bw_plan = bench.paced_bw(rat, a.pace_gbs or (240.0 if V > 1 else 500.0)) if a.paced else rat
    ctas = th.default_ctas(rat, ctas_total)
    big = 1 << 30
    comm = th.Comm(th.Topology(sizes, bw_plan), big, group=group, device=local)
    comm.set_timeout(60.0)
    comm.set_stages(3 if ncross == D else 6)
    comm.set_pacing(a.paced)
    comm.set_min_cta_bytes(a.min_cta_kb * 1024)
    comm.set_window_rotation(bool(a.rotate))

    def emit(obj):
        if rank == 0:
            os.write(out_fd, (json.dumps(obj) + "\n").encode())

    def timed(plan, count, steps, trace=False):
        src = [device_input(rank * V + v, count, "f32", dev) for v in range(V)]
        ts, tr = [], None
        comm.enable_trace(1 if trace else 0)
        for i in range(2 + steps):
            for v in range(V):
                comm.rank_view(v, count, "f32").copy_(src[v])
            barrier(group, dev)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            th.run(th.ALLREDUCE, comm, plan, count, "f32")
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1) * 1e6)
        comm.status()
        if trace:
            tr = comm.fetch_trace(plan).astype(np.int64)
            comm.enable_trace(0)
        return max_over_ranks(float(np.median(ts)), group, dev), tr

    # 1. A_K from a minimum-size collective (C = 4 chunks, one vector per piece)
    C0 = 4
    cnt0 = P * C0 * 4
    p0 = th.Plan(th.Topology(sizes, bw_plan), th.ALLREDUCE, cnt0 * 4, C0, th.BASELINE, th.FIFO).bind(comm, ctas)
    t_min, tr = timed(p0, cnt0, a.steps, trace=True)
    dims = op_dims(p0)
    dur = [[] for _ in range(D)]
    hand = []
    for c in range(C0):
        for s in range(2 * D):
            dur[dims[c, s]].append(tr[c, s, 1] - tr[c, s, 0])
            if s:
                hand.append(tr[c, s, 0] - tr[c, s - 1, 1])
    handoff = float(np.median(hand))
    op_min = [max_over_ranks(float(np.median(d)), group, dev) for d in dur]   # fixed part of one op
    handoff = max_over_ranks(handoff, group, dev)
    A = [x + handoff for x in op_min]
    p0.close()

    # 2. BW_K from a 1 GiB collective (baseline order: N_K fixed by the closed form)
    cnt = big // 4
    p1 = th.Plan(th.Topology(sizes, bw_plan), th.ALLREDUCE, big, 64, th.BASELINE, th.FIFO).bind(comm, ctas)
    t_big, tr = timed(p1, cnt, 3, trace=True)
    dims = op_dims(p1)
    vol = [v / p1.info["byte_scale"] for v in p1.info["dim_volume"]]
    # busy_K = union of the dim's traced op intervals (CTAs of a group drift, so
    # consecutive ops overlap a little and durations must not be summed)
    iv = [[] for _ in range(D)]
    for c in range(64):
        for s in range(2 * D):
            iv[dims[c, s]].append((int(tr[c, s, 0]), int(tr[c, s, 1])))
    busy, nops = [0.0] * D, [len(x) for x in iv]
    for k in range(D):
        cs, ce = None, None
        for a0, b0 in sorted(iv[k]):
            if ce is None or a0 > ce:
                busy[k] += 0 if ce is None else ce - cs
                cs, ce = a0, b0
            else:
                ce = max(ce, b0)
        busy[k] += ce - cs
    # B_K: busy time net of the fixed per-op part, bytes/ns = GB/s; slowest GPU
    bw_meas = [vol[k] / max(1.0, busy[k] - nops[k] * op_min[k]) for k in range(D)]
    bw_meas = [-max_over_ranks(-x, group, dev) for x in bw_meas]
    p1.close()
    # planner units: MB/s on a 5 GB/s grid (keeps the lcm of bandwidths small), ns latencies
    bw_cal = tuple(max(1, int(round(x / 5))) * 5000 for x in bw_meas)
    lat_cal = tuple(int(round(x)) for x in A)
    emit({"calibration": True, "n_gpus": world, "ranks_per_gpu": V, "ratio": a.ratio,
          "min_cta_kb": a.min_cta_kb, "rotate": a.rotate,
          "mode": "paced" if a.paced else "caps", "ctas_per_dim": ctas, "A_ns": [round(x, 1) for x in A],
          "handoff_ns": round(handoff, 1), "min_collective_us": round(t_min / 1e3, 2),
          "bw_gbs_measured": [round(x, 1) for x in bw_meas], "big_collective_ms": round(t_big / 1e6, 3),
          "planner_topology": {"sizes": sizes, "bw_mbps": bw_cal, "step_latency_ns": lat_cal}})

    # 3. validation: model vs measured; latency-aware Themis vs plain Themis vs baseline
    cal = th.Topology(sizes, bw_cal, None, lat_cal)
    for mib in [int(x) for x in a.sizes_mib.split(",")]:
        fixed = {}
        for C in (4, 16, 64):
            nbytes = mib << 20
            cnt = nbytes // 4
            if cnt % (P * C * 4):
                continue
            row = {"mib": mib, "chunks": C, "n_gpus": world, "ratio": a.ratio, "mode": "paced" if a.paced else "caps"}
            for name, topo, pol, charge in (("baseline", cal, th.BASELINE, True), ("themis", th.Topology(sizes, bw_cal),
                                                                                   th.THEMIS, False),
                                            ("themis_latency_aware", cal, th.THEMIS, True)):
                try:
                    p = th.Plan(topo, th.ALLREDUCE, nbytes, C, pol, th.SCF if pol == th.THEMIS else th.FIFO,
                                charge_latency=charge)
                except th.ThemisError as e:
                    row[name] = {"error": str(e)}
                    continue
                # execution: CTA caps / pacing follow the emulated ratio, independent of the plan's numbers
                p.bind(comm, ctas)
                t, _ = timed(p, cnt, a.steps)
                pm = th.Plan(cal, th.ALLREDUCE, nbytes, C, pol, th.SCF if pol == th.THEMIS else th.FIFO,
                             charge_latency=True, rs_orders=p.orders()[0], ag_orders=p.orders()[1])
                pb = th.Plan(th.Topology(sizes, bw_cal), th.ALLREDUCE, nbytes, C, pol,
                             th.SCF if pol == th.THEMIS else th.FIFO, rs_orders=p.orders()[0],
                             ag_orders=p.orders()[1])
                row[name] = {"us": round(t / 1e3, 2), "model_latency_us": round(float(pm.makespan_ns()) / 1e3, 2),
                             "model_bw_only_us": round(float(pb.makespan_ns()) / 1e3, 2),
                             "greedy_chunks": p.info["n_greedy"]}
                pm.close()
                pb.close()
                p.close()
            if "us" in row.get("themis", {}) and "us" in row.get("themis_latency_aware", {}):
                row["latency_aware_vs_plain"] = round(row["themis"]["us"] / row["themis_latency_aware"]["us"], 3)
                row["latency_aware_vs_baseline"] = round(row["baseline"]["us"] / row["themis_latency_aware"]["us"], 3)
                fixed[C] = row
            emit(row)
        # n_chunks = 0: the latency-aware planner also picks the chunk count
        nbytes = mib << 20
        pa = th.Plan(cal, th.ALLREDUCE, nbytes, th.AUTO_CHUNKS, th.THEMIS, th.SCF, charge_latency=True).bind(comm, ctas)
        t, _ = timed(pa, nbytes // 4, a.steps)
        row = {"mib": mib, "chunks": "auto", "chosen_chunks": pa.n_chunks, "n_gpus": world, "ratio": a.ratio,
               "mode": "paced" if a.paced else "caps", "themis_auto": {"us": round(t / 1e3, 2),
               "model_latency_us": round(float(pa.makespan_ns()) / 1e3, 2)}}
        pa.close()
        if 64 in fixed:
            row["auto_vs_themis_c64"] = round(fixed[64]["themis"]["us"] * 1e3 / t, 3)
            row["auto_vs_baseline_c64"] = round(fixed[64]["baseline"]["us"] * 1e3 / t, 3)
        best = min((r["themis_latency_aware"]["us"], C) for C, r in fixed.items())
        row["best_fixed_latency_aware"] = {"us": best[0], "chunks": best[1]}
        emit(row)
    comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
