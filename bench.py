"""Benchmark: Themis chunked hierarchical All-Reduce on B200 (BASELINE.json).

    python bench.py [--gpus N --steps K --warmup W]            # our CUDA path
    python bench.py --impl reference [...]                      # the CPU oracle arm

Workload (BASELINE.json configs[1]): logical 2x2x2 topology (P = 8 ranks),
1 GiB fp32 per rank, 64 chunks, per-dimension bandwidth emulated 4:2:1 by
capping each dimension group's CTAs.  With N GPUs each GPU hosts V = 8 / N
logical ranks (N = 1: the whole topology inside one GPU's HBM; N = 8: one rank
per GPU, every dimension over NVLink).  A step is one All-Reduce through the
C ABI (one kernel launch).  Before every step the inputs are refreshed from a
pristine copy (untimed; writes 8 GiB > L2).  `value` = bus GB/s per logical
rank, 2 S (P-1)/P / t (NCCL-tests convention; comparable to 900 GB/s
NVLink), t = max over GPUs of the device-timed step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "All-Reduce bus GB/s vs 900 GB/s NVLink at 2/4/8 B200, Themis vs baseline order"
SIZES = (2, 2, 2)
NVLINK_PEAK = 770.0       # measured peer-copy GB/s per direction (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0    # nominal per direction per GPU (the metric's denominator)


def logical_layout(sizes, n_gpus):
    """V ranks per GPU; dims whose peers live on other GPUs (dim1 fastest)."""
    P = 1
    for s in sizes:
        P *= s
    V = P // n_gpus
    cross, stride = [], 1
    for k, s in enumerate(sizes):
        if stride * s > V or stride >= V:   # peers differ in a digit at or above V's span
            cross.append(k)
        stride *= s
    return {"P": P, "V": V, "cross_gpu_dims": cross}


def launch_config(sizes, n_gpus, sms, nvls=False):
    """bench.py's launch configuration for a logical topology on n_gpus GPUs
    (also used by the full-size parity tests, so they check exactly what is
    timed):
      CTA budget / TMA ring (K5 calibration, profiles/r01_nvlink_calibration.md,
      profiles/r02/ceilings): NVLink saturates with a bounded amount in flight
      per GPU (all-NVLink best at 128 CTAs x 2 x 32 KiB; more stages lose);
      HBM-resident dims want every SM and larger tiles (3 x 64 KiB at N = 1,
      4 x 48 KiB mixed);
      runtime intra-dim order (R28): L = 16 with <= 2 ranks per GPU (head-of-line
      blocking of the static order where NVLink dims dominate: 2x2 on 4 GPUs
      487 -> 638 GB/s), else the enforced order (neutral at N = 1, -3 % on the
      N = 2 headline)."""
    lay = logical_layout(sizes, n_gpus)
    V, ncross = lay["V"], len(lay["cross_gpu_dims"])
    if ncross == 0:
        total = sms
    elif ncross == len(sizes):
        total = min(sms, 128) if len(sizes) > 1 else (64 if nvls else 32)   # NVLS wants more threads in flight
    else:
        total = sms if V >= 4 else 96
    if ncross == len(sizes):
        stages, kb = (2 if len(sizes) > 1 else 4), 32
    elif ncross == 0:
        stages, kb = 3, 64
    else:
        stages, kb = 4, 48
    return {"total_ctas": total, "stages": stages, "stage_kb": kb, "lookahead": 16 if V <= 2 else 1,
            "min_cta_bytes": 64 * 1024}


def calibrated_bw(rates_gbs, group=None, device=None):
    """Per-dim BW (MB/s) for a calibrated Themis plan from this rank's measured
    per-dim rates (GB/s): the minimum over ranks (every rank must build the
    identical plan, R22), quantised to 1/32 of the fastest dim's rate (keeps
    lcm(BW) -- the planner's exact time scale -- small, R21)."""
    from paper_2110_04478_b200.dist import max_over_ranks
    r = [-max_over_ranks(-float(x), group, device) for x in rates_gbs]
    q = max(1.0, max(r) / 32)
    return tuple(max(1, int(round(x / q))) * int(round(q * 1000)) for x in r)


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])
        except Exception:
            pass

    def __enter__(self):
        try:   # a persistent sampler (-lms 50) started before the timed region
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except Exception:
                self.proc.kill()
            self.t.join(5)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows if len(r) > 8 for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def paced_bw(rat, total_gbs):
    """Absolute per-dim MB/s in the exact ratio `rat`, summing to ~total_gbs,
    on a whole-GB/s unit (keeps the planner's lcm of bandwidths small)."""
    unit = max(1, int(round(total_gbs / sum(rat)))) * 1000
    return tuple(int(r) * unit for r in rat)


def hbm_bytes_per_rank(plan, S):
    """Algorithmic HBM bytes one rank's ops move (reads + writes): RS stage
    holding H on dim k reads H (P_k pieces of H/P_k) and writes H/P_k; AG
    stage holding h reads and writes (P_k-1) h."""
    rs, _ = plan.orders()
    C = plan.info["n_chunks"]
    tot = 0.0
    for c in range(C):
        h = S / C
        hist = []
        for d in rs[c]:
            p = SIZES[int(d)]
            tot += h + h / p
            h /= p
            hist.append(p)
        for p in reversed(hist):
            tot += 2 * (p - 1) * h
            h *= p
    return tot


def remote_fraction(sizes, n_gpus, k, q, ring=False):
    """Share of logical rank q's dim-k pulls that cross to another GPU: the
    direct algorithm pulls equally from its P_k - 1 dim peers, the ring only
    from its left neighbour (rank r lives on GPU r // V)."""
    P = 1
    for s_ in sizes:
        P *= s_
    V = P // n_gpus
    stride = 1
    for s_ in sizes[:k]:
        stride *= s_
    pk = sizes[k]
    c = (q // stride) % pk
    peer = lambda j: q + (j - c) * stride
    if ring:
        return float(peer((c - 1) % pk) // V != q // V)
    return sum(peer(j) // V != q // V for j in range(pk) if j != c) / (pk - 1)


def nvlink_bytes_per_gpu(plan, sizes, n_gpus, ring_dims=()):
    """Bytes one GPU pulls over NVLink per collective (max over GPUs): its V
    ranks' N_K, each weighted by the share of dim-K peers on other GPUs."""
    vol = [v / plan.info["byte_scale"] for v in plan.info["dim_volume"]]
    P = plan.info["n_ranks"]
    V = P // n_gpus
    return max(sum(vol[k] * remote_fraction(sizes, n_gpus, k, q, k in ring_dims)
                   for q in range(g * V, (g + 1) * V) for k in range(len(sizes)))
               for g in range(n_gpus))


def run_themis(a):
    import torch
    from paper_2110_04478_b200 import themis as th
    from paper_2110_04478_b200.dist import barrier, check_same_plan, init_from_env, max_over_ranks
    from synth import device_input

    os.environ["NCCL_DEBUG"] = "WARN"      # keep stdout to the one JSON line (NCCL prints its version at INFO)
    rank, world, local, group = init_from_env("nccl" if int(os.environ.get("WORLD_SIZE", 1)) > 1 else "gloo")
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lay = logical_layout(SIZES, world)
    P, V = lay["P"], lay["V"]
    S = a.mib << 20
    N = S // 4
    ratio = tuple(int(x) for x in a.ratio.split(":"))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cfg = launch_config(SIZES, world, sms, nvls=a.nvls)
    total_ctas = a.ctas_total or cfg["total_ctas"]
    stages, stage_kb = a.stages or cfg["stages"], a.stage_kb or cfg["stage_kb"]
    kinds = (th.NVLS,) * len(SIZES) if a.nvls else None   # NVSwitch dims with in-switch reduction where eligible (R27, R29)
    topo = th.Topology(SIZES, ratio, kinds)
    ll_max = a.ll_max_mib << 20
    comm = th.Comm(topo, S, group=group, device=local, nvls=a.nvls and world > 1,
                   ll_bytes=4 * min(S, ll_max) if ll_max else 0)
    comm.set_timeout(30.0)
    if ll_max:
        comm.set_ll(ll_max)
    a.lookahead = a.lookahead or cfg["lookahead"]
    comm.set_lookahead(a.lookahead)
    comm.set_min_cta_bytes(a.min_cta_kb * 1024)
    comm.set_stages(1)
    comm.set_stage_bytes(stage_kb * 1024)
    comm.set_stages(stages)
    pristine = [device_input(rank * V + v, N, "f32", dev) for v in range(V)]

    def refill():
        for v in range(V):
            comm.rank_view(v, N, "f32").copy_(pristine[v])

    def make(pol, rat, total_gbs=None):
        # total_gbs: absolute per-rank bandwidth budget split in the ratio (paced
        # emulation); otherwise the ratio itself (only ratios matter to the plan).
        bw = paced_bw(rat, total_gbs) if total_gbs else rat
        t = th.Topology(SIZES, bw, kinds)
        p = th.Plan(t, th.ALLREDUCE, S, a.chunks, pol, th.SCF if pol == th.THEMIS else th.FIFO,
                    concurrency=a.concurrency)
        check_same_plan(p, group)            # fail fast before any kernel (R22)
        p.bind(comm, caps_for(rat))
        return p

    def caps_for(rat):
        if a.ctas_split and tuple(rat) == tuple(ratio):
            return [int(x) for x in a.ctas_split.split(",")]
        return th.default_ctas(rat, total_ctas)

    def timed(plan, steps, warmup):
        for _ in range(warmup):
            refill()
            th.run(th.ALLREDUCE, comm, plan, N, "f32")
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            refill()
            barrier(group, dev)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            th.run(th.ALLREDUCE, comm, plan, N, "f32")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        comm.status()
        mean = sum(ts) / len(ts)
        timed.median = max_over_ranks(sorted(ts)[len(ts) // 2], group, dev)
        return max_over_ranks(mean, group, dev), max_over_ranks(min(ts), group, dev)

    busbw = lambda t: 2 * S * (P - 1) / P / t / 1e9

    def dim_rates(plan):
        """Achieved per-dim GB/s per rank of one traced run of `plan`:
        N_K / busy_K, busy_K = union of dim K's op intervals (%globaltimer);
        the minimum over GPUs (so every rank plans identically)."""
        comm.enable_trace(True)
        refill()
        th.run(th.ALLREDUCE, comm, plan, N, "f32")
        torch.cuda.synchronize()
        comm.status()
        tr = comm.fetch_trace(plan).astype("int64")
        comm.enable_trace(False)
        out = []
        for k, ops in enumerate(plan.dim_ops()):
            iv = sorted((int(tr[c, s_, 0]), int(tr[c, s_, 1])) for c, s_ in ops)
            busy, cs, ce = 0, iv[0][0], iv[0][1]
            for s0, e0 in iv[1:]:
                if s0 > ce:
                    busy += ce - cs
                    cs, ce = s0, e0
                else:
                    ce = max(ce, e0)
            busy += ce - cs
            nk = plan.info["dim_volume"][k] / plan.info["byte_scale"]
            out.append(nk / max(busy, 1))
        return out

    main = make(th.THEMIS, ratio)
    # planner cost (SURVEY.md:557): the C++ planner (themis_plan: Algorithm 1 +
    # pre-simulation) for this exact request, median of 21 calls
    pts = []
    for _ in range(21):
        t0 = time.perf_counter()
        th.Plan(th.Topology(SIZES, ratio, kinds), th.ALLREDUCE, S, a.chunks, th.THEMIS, th.SCF).close()
        pts.append(time.perf_counter() - t0)
    planner_cpp_us = round(statistics.median(pts) * 1e6, 1)
    clocks = ClockSampler(local)
    with clocks:
        t_main, t_best = timed(main, a.steps, a.warmup)
        t_median = timed.median
    launches = a.steps * th.launches_per_call()

    # Themis vs baseline order under the emulated ratios
    compare = {}
    # Paced budget per rank that this box can carry: NVLink (~700 GB/s per GPU
    # over the cross-GPU dims' share) and HBM (~6 TB/s at ~2.5 B per bus byte).
    ncross = len(lay["cross_gpu_dims"])
    # ~80% of the physical limits, so the emulated BW (not the fabric) binds
    # even when Themis keeps every dimension busy at once.
    # NVLink: ~640 GB/s per GPU is the executor's bidirectional ceiling
    # (profiles/r02/ceilings: all GPUs pulling at once, no dependencies), so
    # ~600 per GPU over the cross-GPU dims' share keeps the emulated BW binding
    caps_ = [600.0, 0.8 * 6000.0 / (2.5 * V)]
    if ncross:
        caps_.append(600.0 * len(SIZES) / (V * ncross))
    pace_gbs = a.pace_gbs or float(int(min(caps_) // 24) * 24)
    if not a.no_compare:
        for mode in ("caps", "paced"):
            comm.set_pacing(mode == "paced")
            for rat in [ratio] + [r for r in a.compare if r != ratio]:
                row = {}
                sum_bw = sum(paced_bw(rat, pace_gbs)) / 1000
                for pol, name in ((th.BASELINE, "baseline"), (th.THEMIS, "themis")):
                    reuse = mode == "caps" and pol == th.THEMIS and rat == ratio
                    p = main if reuse else make(pol, rat, pace_gbs if mode == "paced" else None)
                    tt = t_main if reuse else timed(p, max(2, min(a.steps, 5)), 1)[0]
                    row[name] = {"bus_gbs": round(busbw(tt), 1), "ms": round(tt * 1e3, 3),
                                 "model_makespan_ns": float(p.makespan_ns()), "ctas": p.bound_ctas()}
                    if mode == "paced":   # the paper's utilisation: busBW / sum BW (F2)
                        row[name]["util"] = round(busbw(tt) / sum_bw, 4)
                    if mode == "caps" and pol == th.BASELINE and len(SIZES) > 1:
                        # calibrated BW: the per-dim rates this fabric actually
                        # delivers under these caps (one traced baseline run),
                        # as the planner's BW_K (B_K from the system)
                        cal_gbs = dim_rates(p)
                    if not reuse:
                        p.close()
                if mode == "caps" and len(SIZES) > 1:
                    # quantised to 1/32 of the fastest dim's rate (keeps lcm(BW) -- the
                    # planner's exact time scale -- small; R21)
                    def cal_plan(rates):
                        cal = calibrated_bw(rates, group, dev)
                        pc_ = th.Plan(th.Topology(SIZES, cal, kinds), th.ALLREDUCE, S, a.chunks, th.THEMIS, th.SCF)
                        check_same_plan(pc_, group)
                        return pc_.bind(comm, caps_for(rat))
                    # a dim delivers at least the best rate it showed in any run:
                    # one refinement with the calibrated plan's own rates
                    pc = cal_plan(cal_gbs)
                    cal_gbs = [max(x, y) for x, y in zip(cal_gbs, dim_rates(pc))]
                    pc.close()
                    pc = cal_plan(cal_gbs)
                    tc_ = timed(pc, max(2, min(a.steps, 5)), 1)[0]
                    row["themis_calibrated"] = {"bus_gbs": round(busbw(tc_), 1), "ms": round(tc_ * 1e3, 3),
                                                "calibrated_gbs": [round(r, 1) for r in cal_gbs],
                                                "greedy_chunks": pc.info["n_greedy"]}
                    row["calibrated_speedup"] = round(row["baseline"]["ms"] / row["themis_calibrated"]["ms"], 3)
                    pc.close()
                row["measured_speedup"] = round(row["baseline"]["ms"] / row["themis"]["ms"], 3)
                row["model_speedup"] = round(row["baseline"]["model_makespan_ns"] /
                                             row["themis"]["model_makespan_ns"], 4)
                if mode == "paced":
                    row["sum_bw_gbs"] = sum_bw
                    # the plan's makespan is in real ns here (absolute bw): model busBW / sum BW
                    row["model_util"] = {n: round(busbw(row[n]["model_makespan_ns"] * 1e-9) / sum_bw, 4)
                                         for n in ("baseline", "themis")}
                    # latency-aware Themis with a planner-chosen chunk count (R25; A_K as measured
                    # by scripts/calibrate.py) beside the fixed 64-chunk plans
                    lat = a.latency_ns or (8500 if not lay["cross_gpu_dims"] else 11000)
                    pa = th.Plan(th.Topology(SIZES, paced_bw(rat, pace_gbs), kinds, (lat,) * len(SIZES)),
                                 th.ALLREDUCE, S, th.AUTO_CHUNKS, th.THEMIS, th.SCF, charge_latency=True)
                    check_same_plan(pa, group)
                    pa.bind(comm, caps_for(rat))
                    ta = timed(pa, max(2, min(a.steps, 5)), 1)[0]
                    row["themis_auto"] = {"bus_gbs": round(busbw(ta), 1), "ms": round(ta * 1e3, 3),
                                          "chunks": pa.n_chunks, "latency_ns": lat,
                                          "util": round(busbw(ta) / sum_bw, 4)}
                    row["auto_speedup"] = round(row["baseline"]["ms"] / row["themis_auto"]["ms"], 3)
                    pa.close()
                compare[f"{mode} {':'.join(map(str, rat))}"] = row
        comm.set_pacing(False)

    # Achieved per-dimension GB/s (north_star (d)): one traced, paced Themis
    # All-Reduce; busy_K = union of dim K's op intervals (%globaltimer),
    # achieved_K = N_K / busy_K per rank, against the emulated BW_K.
    per_dim = None
    if not a.no_compare:
        rat = a.compare[0] if a.compare else ratio
        bw = paced_bw(rat, pace_gbs)
        comm.set_pacing(True)
        comm.enable_trace(True)
        p = make(th.THEMIS, rat, pace_gbs)
        refill()
        th.run(th.ALLREDUCE, comm, p, N, "f32")
        torch.cuda.synchronize()
        comm.status()
        tr = comm.fetch_trace(p).astype("int64")
        per_dim = {"ratio": ":".join(map(str, rat)), "dims": []}
        for k, ops in enumerate(p.dim_ops()):
            iv = sorted((int(tr[c, s, 0]), int(tr[c, s, 1])) for c, s in ops)
            busy, cs, ce = 0, iv[0][0], iv[0][1]
            for s0, e0 in iv[1:]:
                if s0 > ce:
                    busy += ce - cs
                    cs, ce = s0, e0
                else:
                    ce = max(ce, e0)
            busy += ce - cs
            nk = p.info["dim_volume"][k] / p.info["byte_scale"]
            per_dim["dims"].append({"dim": k + 1, "emulated_gbs": bw[k] / 1000, "bytes_per_rank": nk,
                                    "busy_us": round(busy / 1e3, 1),
                                    "achieved_gbs": round(nk / busy, 2) if busy else None})
        span = int(tr[:, :, 1].max() - tr[:, :, 0].min())
        per_dim["span_us"] = round(span / 1e3, 1)
        per_dim["note"] = ("trace-derived inside the full collective (busy = union of a dim's op intervals); "
                           "the hardware check -- each dim group alone on the real kernel, ncu "
                           "nvlrx__bytes_data_user.sum / duration = 0.94-1.01 of BW_K -- is "
                           "profiles/r02/k5_nvlink/README.md")
        p.close()
        comm.enable_trace(False)
        comm.set_pacing(False)

    # NCCL all_reduce on the same bytes (context row, N > 1 only)
    nccl = None
    if world > 1 and (not a.no_compare or a.nccl):
        import torch.distributed as dist
        x = pristine[0].clone()
        for _ in range(2):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dist.all_reduce(x)
        e1.record()
        torch.cuda.synchronize()
        tn = max_over_ranks(e0.elapsed_time(e1) / 5e3, group, dev)
        nccl = {"bus_gbs": round(2 * S * (world - 1) / world / tn / 1e9, 1), "ranks": world,
                "note": "torch.distributed.all_reduce (NCCL), flat over the N GPUs, same bytes per GPU; context"}
        del x

    # e2e through the C ABI with pinned HOST buffers (H2D + AR + D2H timed)
    e2e = None
    if not a.no_e2e:
        hin = torch.empty(V * N, dtype=torch.float32, pin_memory=True)
        for v in range(V):
            hin[v * N:(v + 1) * N].copy_(pristine[v])
        hout = torch.empty_like(hin, pin_memory=True)
        # host streaming plan (R26): chunks arrive at the measured pinned H2D
        # rate, so the pre-simulated per-dim order drains early chunks (and
        # their D2H copies start) while later ones are still in flight
        probe = min(N, 64 << 20)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        comm.rank_view(0, probe, "f32").copy_(hin[:probe], non_blocking=True)
        d1.record()
        torch.cuda.synchronize()
        # the slowest GPU's rate: every rank must build the identical plan
        h2d_gbs = -max_over_ranks(-(probe * 4 / (d0.elapsed_time(d1) / 1e3) / 1e9), group, dev)
        # PCIe bound of the e2e step: both directions at once (per-direction rate)
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        scratch = torch.empty(probe, dtype=torch.float32, device=dev)
        hout_probe = torch.empty(probe, dtype=torch.float32, pin_memory=True)
        torch.cuda.synchronize()
        d0.record()
        sa.wait_event(d0)
        sb.wait_event(d0)
        with torch.cuda.stream(sa):
            comm.rank_view(0, probe, "f32").copy_(hin[:probe], non_blocking=True)
        with torch.cuda.stream(sb):
            hout_probe.copy_(scratch, non_blocking=True)
        torch.cuda.current_stream().wait_stream(sa)
        torch.cuda.current_stream().wait_stream(sb)
        d1.record()
        torch.cuda.synchronize()
        duplex_gbs = -max_over_ranks(-(probe * 4 / (d0.elapsed_time(d1) / 1e3) / 1e9), group, dev)
        del scratch, hout_probe
        release_ns = int(V * S / a.chunks / h2d_gbs)
        bw_abs = paced_bw(ratio, max(24.0, busbw(t_main)))
        try:
            hplan = th.Plan(th.Topology(SIZES, bw_abs, kinds), th.ALLREDUCE, S, a.chunks, th.THEMIS, th.SCF,
                            concurrency=a.concurrency, chunk_release_ns=release_ns)
        except th.ThemisError:       # (planner overflow) all chunks ready at 0 instead
            release_ns = 0
            hplan = th.Plan(th.Topology(SIZES, ratio, kinds), th.ALLREDUCE, S, a.chunks, th.THEMIS, th.SCF,
                            concurrency=a.concurrency)
        check_same_plan(hplan, group)
        hplan.bind(comm, caps_for(ratio))
        th.themis_allreduce_host(hin.data_ptr(), hout.data_ptr(), comm.data_ptr, N, "f32", hplan)
        torch.cuda.synchronize()
        k = max(1, min(a.steps, 3))
        barrier(group, dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            th.themis_allreduce_host(hin.data_ptr(), hout.data_ptr(), comm.data_ptr, N, "f32", hplan)
        e1.record()
        torch.cuda.synchronize()
        te = max_over_ranks(e0.elapsed_time(e1) / 1e3 / k, group, dev)
        comm.status()
        e2e = {"value": round(busbw(te), 2), "unit": "GB/s", "h2d_bytes_per_step": V * S, "d2h_bytes_per_step": V * S,
               "ms_per_step": round(te * 1e3, 3), "h2d_gbs_measured": round(h2d_gbs, 1),
               "pcie_duplex_gbs_measured": round(duplex_gbs, 1),
               "pcie_bound_ms": round(V * S / duplex_gbs / 1e6, 3),
               "frac_of_pcie_bound": round(V * S / duplex_gbs / 1e9 / te, 3),
               "chunk_release_ns": release_ns,
               "note": "themis_allreduce_host: chunk-streamed H2D -> collective -> D2H (pinned host buffers)"}
        hplan.close()
        del hin, hout

    # roofline of the dominant (only) kernel
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_bytes = V * hbm_bytes_per_rank(main, S)
    nvl_bytes = nvlink_bytes_per_gpu(main, SIZES, world)
    hbm_ach = hbm_bytes / t_main / 1e9
    nvl_ach = nvl_bytes / t_main / 1e9
    if world == 1 or hbm_ach / hbm_peak >= nvl_ach / NVLINK_PEAK:
        roof = {"bound": "hbm", "achieved": round(hbm_ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(hbm_ach / hbm_peak, 4), "traffic": None,
                "algorithmic_bytes_per_launch": hbm_bytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650"}
    else:
        roof = {"bound": "nvlink", "achieved": round(nvl_ach, 1), "peak": NVLINK_PEAK, "unit": "GB/s",
                "frac": round(nvl_ach / NVLINK_PEAK, 4), "frac_of_900_nominal": round(nvl_ach / NVLINK_NOMINAL, 4),
                "traffic": None,
                "algorithmic_bytes_per_launch": nvl_bytes,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction (900 nominal)"}
    roof["kernel"] = "themis_exec_kernel<F32Tag,true> (TMA engine)"
    try:   # ncu-measured DRAM bytes per launch for this exact config (profiles/ncu_traffic.json)
        key = f"n{world}_{'x'.join(map(str, SIZES))}_{a.mib}MiB_c{a.chunks}_{a.ratio}"
        ent = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(key)
        if ent and roof["bound"] == "hbm":
            roof["traffic"] = ent["traffic"]
            roof["traffic_source"] = ent["source"]
    except Exception:
        pass

    cpu = None
    if world == 1 and not a.no_cpu:
        cpu = cpu_baseline(a.cpu_mib, a.chunks, ratio, reps=8)   # ~10 s of CPU work

    # Themis vs baseline under emulated heterogeneous BW (the metric's second
    # half): the paced rows carry the paper's utilisation; the headline ratio
    # 4:2:1 is the Just-Enough control (equal by construction)
    tvb = {}
    for key, row in compare.items():
        ent = {"measured_speedup": row["measured_speedup"], "model_speedup": row["model_speedup"],
               "themis_bus_gbs": row["themis"]["bus_gbs"], "baseline_bus_gbs": row["baseline"]["bus_gbs"]}
        if "themis_calibrated" in row:
            ent.update(calibrated_speedup=row["calibrated_speedup"],
                       themis_calibrated_bus_gbs=row["themis_calibrated"]["bus_gbs"],
                       calibrated_gbs=row["themis_calibrated"]["calibrated_gbs"])
        if "sum_bw_gbs" in row:
            ent.update(sum_bw_gbs=row["sum_bw_gbs"], themis_util=row["themis"]["util"],
                       baseline_util=row["baseline"]["util"],
                       frac_of_model_speedup=round(row["measured_speedup"] / row["model_speedup"], 3))
        tvb[key] = ent

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(busbw(t_main), 2), "unit": "GB/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(t_main * 1e3, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded U[-1,1) fp32 gradient buffers, torch generator seed 20211010+rank)",
            "config": {"workload": ("BASELINE.json configs[1]: 2x2x2 logical topology, 1 GiB fp32 All-Reduce per "
                                    "rank, 64 chunks, emulated per-dim BW 4:2:1")
                       if (SIZES == (2, 2, 2) and a.ratio == "4:2:1" and a.mib == 1024 and a.chunks == 64) else
                       (f"BASELINE.json configs[2] sweep point: {'x'.join(map(str, SIZES))}, {a.mib} MiB fp32 per "
                        f"rank, {a.chunks} chunks, emulated BW {a.ratio}"),
                       "topology": "x".join(map(str, SIZES)), "bytes_per_rank": S, "chunks": a.chunks,
                       "bw_ratio": a.ratio, "policy": "themis+scf", "ranks_per_gpu": V,
                       "ratio_note": ("4:2:1 on 2x2x2 is the paper's Just-Enough ratio (PAPER.md:703-705): Algorithm 1 "
                                      "keeps all 64 chunks on the baseline order, so Themis == baseline here by "
                                      "construction; the Themis effect is in themis_vs_baseline (over-provisioned "
                                      "1:1:1 / 2:2:1, paced emulation)") if a.ratio == "4:2:1" and SIZES == (2, 2, 2)
                                     else None,
                       "emulation": ("CTA caps only (value is the unthrottled kernel: with every dim's group "
                                     "sharing one HBM / NVLink fabric the caps do not bind; paced rows in "
                                     "themis_vs_baseline emulate BW_K exactly)"),
                       "ops_in_flight_per_dim": max(1, a.concurrency), "intra_dim_lookahead": a.lookahead,
                       "op_window_min_cta_kib": a.min_cta_kb, "ll": main.bound_ll(),
                       "cross_gpu_dims": [k + 1 for k in lay["cross_gpu_dims"]],
                       "ctas_per_dim": main.bound_ctas(), "engine": "tma", "tma_stages": stages, "tma_stage_kib": stage_kb,
                       "value_definition": "bus GB/s per logical rank = 2 S (P-1)/P / t, t = max over GPUs",
                       "scaling_note": ("the same 8-rank logical topology at every N: N = 1 emulates all ranks in "
                                        "one GPU's HBM, N = 8 is one rank per GPU over NVLink (V = 8 / N ranks "
                                        "per GPU); total work is fixed, hence 'strong'"),
                       "aggregate_bus_gbs": round(busbw(t_main) * P, 1),
                       "best_step_bus_gbs": round(busbw(t_best), 2),
                       "median_step_bus_gbs": round(busbw(t_median), 2),
                       "l2": "inputs refreshed from a pristine copy before every step (>= 1 GiB per GPU written, "
                             "> 126 MB L2); inputs larger than L2"},
            "clocks": clocks.summary(), "gpu_launches": launches, "roofline": roof, "e2e": e2e,
            "themis_vs_baseline": tvb, "planner": {"cpp_us": planner_cpp_us,
                                                   "oracle_ms": cpu.get("planner_oracle_ms") if cpu else None},
            "compare": compare, "per_dim_emulation": per_dim, "nccl_context": nccl, "cpu_baseline": cpu,
        }
        emit(out)
    main.close()
    comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def cpu_baseline(mib, chunks, ratio, reps=1):
    """The oracle (as it stands) on a bounded sample of the same workload."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import data as O, scheduler as S_, topology as T
    from synth import host_inputs
    t = T.Topology.make(SIZES, ratio)
    P = t.P
    N = (mib << 20) // 4
    xs = host_inputs(P, N, "f32")
    sched = S_.schedule_collective(t, S_.AR, N * 4, chunks, S_.THEMIS)
    t0 = time.perf_counter()
    for _ in range(reps):
        O.run_schedule(xs, sched, "f32")
    dt = (time.perf_counter() - t0) / reps
    # the oracle planner (Fractions: Algorithm 1 + the event pre-simulation) on
    # the full-size request, for the planner-time comparison (SURVEY.md:557)
    from oracle import engine as E_
    t1 = time.perf_counter()
    E_.simulate(S_.schedule_collective(t, S_.AR, 1 << 30, chunks, S_.THEMIS), E_.SCF)
    plan_ms = (time.perf_counter() - t1) * 1e3
    return {"value": round(2 * N * 4 * (P - 1) / P / dt / 1e9, 4), "unit": "GB/s", "cores": 1,
            "planner_oracle_ms": round(plan_ms, 2),
            "host_cores_available": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"{'x'.join(map(str, SIZES))} Themis All-Reduce, {mib} MiB fp32 per rank x {P} simulated "
                      f"ranks, {chunks} chunks, numpy single-threaded, {reps} rep(s), {dt:.2f} s per All-Reduce"}


def run_reference(a):
    """Reference arm: the CPU oracle timed on the host, same metric/config."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import data as O, scheduler as S_, topology as T
    from synth import host_inputs
    ratio = tuple(int(x) for x in a.ratio.split(":"))
    t = T.Topology.make(SIZES, ratio)
    P = t.P
    N = (a.cpu_mib << 20) // 4
    xs = host_inputs(P, N, "f32")
    sched = S_.schedule_collective(t, S_.AR, N * 4, a.chunks, S_.THEMIS)
    for _ in range(a.warmup):
        O.run_schedule(xs, sched, "f32")
    ts = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        O.run_schedule(xs, sched, "f32")
        ts.append(time.perf_counter() - t0)
    dt = sum(ts) / len(ts)
    v = round(2 * N * 4 * (P - 1) / P / dt / 1e9, 4)
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": a.gpus, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": "BASELINE.json configs[1]: 2x2x2 logical topology, 1 GiB fp32 All-Reduce per "
                                  "rank, 64 chunks, emulated per-dim BW 4:2:1",
                      "topology": "x".join(map(str, SIZES)), "bytes_per_rank": a.mib << 20, "chunks": a.chunks,
                      "bw_ratio": a.ratio, "policy": "themis+scf",
                      "sample": f"each step is a bounded sample: {a.cpu_mib} MiB fp32 per rank x {P} simulated ranks "
                                "on the host CPU (numpy, one core)", "sample_bytes_per_rank": N * 4},
           "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                            "sample": f"{a.cpu_mib} MiB fp32 per rank x {P} simulated ranks per step"},
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


_JSON_FD = None


def emit(obj) -> None:
    """Write the one JSON result line to the real stdout (fd saved at start;
    everything else, e.g. NCCL's version banner, goes to stderr)."""
    line = (json.dumps(obj) + "\n").encode()
    os.write(_JSON_FD if _JSON_FD is not None else 1, line)


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="themis", choices=["themis", "reference"])
    ap.add_argument("--mib", type=int, default=1024, help="All-Reduce bytes per logical rank (MiB)")
    ap.add_argument("--chunks", type=int, default=64)
    ap.add_argument("--ratio", default="4:2:1", help="emulated BW(dim1):BW(dim2):BW(dim3)")
    ap.add_argument("--ctas-total", type=int, default=0, help="CTAs split over the dims (default: all SMs)")
    ap.add_argument("--ctas-split", default="", help="explicit CTAs per dim for the headline ratio (experiments)")
    ap.add_argument("--nvls", action="store_true",
                    help="switch dims + multicast heap: eligible dims reduce in the NVSwitch (experimental, R27)")
    ap.add_argument("--latency-ns", type=int, default=0,
                    help="per-op A_K for the latency-aware auto-chunk compare rows (default: measured 8.5 / 11 us)")
    ap.add_argument("--cpu-mib", type=int, default=256, help="oracle sample size per rank (MiB)")
    ap.add_argument("--pace-gbs", type=float, default=0, help="per-rank sum of paced dim BWs (GB/s)")
    ap.add_argument("--ll-max-mib", type=int, default=0,
                    help="LL packets (R31) for collectives of at most this many MiB per rank (0 = off)")
    ap.add_argument("--no-compare", action="store_true")
    ap.add_argument("--nccl", action="store_true", help="NCCL context row even with --no-compare")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--stages", type=int, default=0, help="TMA ring depth (default 4 with NVLink dims, else 6)")
    ap.add_argument("--stage-kb", type=int, default=0, help="TMA ring stage size (KiB; default by topology)")
    ap.add_argument("--lookahead", type=int, default=0,
                    help="runtime intra-dim order: 1 = enforced pre-simulated order, L > 1 = first ready of the next L "
                         "(R28); 0 = auto: 16 with <= 2 ranks per GPU, else 1")
    ap.add_argument("--min-cta-kb", type=int, default=64,
                    help="op windows: an op gets one CTA per this many KiB it moves (small ops run several per dim "
                         "at once; 0 = every op on all its dim's CTAs)")
    ap.add_argument("--concurrency", type=int, default=1,
                    help="ops in flight per dimension in the plan's pre-simulation (1 = the paper's model)")
    ap.add_argument("--sizes", default="2,2,2", help="logical topology P_1,...,P_D (sweeps, config 3)")
    ap.add_argument("--compare-ratios", default="", help="extra emulated ratios, e.g. '1:1:1,2:2:1'")
    a = ap.parse_args()
    global SIZES
    SIZES = tuple(int(x) for x in a.sizes.split(","))
    if len(a.ratio.split(":")) != len(SIZES):
        a.ratio = ":".join(["1"] * len(SIZES))
    if not a.compare_ratios:
        a.compare_ratios = {3: "1:1:1,2:2:1", 2: "1:1", 1: ""}.get(len(SIZES), "")
    a.compare = [tuple(int(x) for x in r.split(":")) for r in a.compare_ratios.split(",") if r]
    if a.warmup < 3 and a.impl == "themis":
        a.warmup = 3
    if a.impl == "reference":
        run_reference(a)
    else:
        run_themis(a)


if __name__ == "__main__":
    main()
