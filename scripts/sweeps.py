"""Sweeps for BASELINE.json configs 3-5 (development / reporting tool).

    python scripts/sweeps.py --config 3|4|5 [--quick]            # N = 1 (emulated)
    torchrun --nproc-per-node N scripts/sweeps.py --config 3 ...  # N GPUs

Prints one JSON object per measured point (rank 0).  Every point is one
collective through the C ABI, timed with CUDA events (max over GPUs), inputs
refreshed before each timed call.

config 3: size x chunk-count sweep on 2x4 / 4x2 (and 2x2, flat) — Themis vs
          baseline, paced BW emulation at 1:1 and 200:50 (PAPER.md:278 notation).
config 4: DDP-style bf16 gradient-bucket All-Reduce traces on 2x2x2 (ResNet-152
          60.19 M, GNMT ~280 M parameters; 25 MiB buckets, 64 chunks each).
config 5: bf16 Reduce-Scatter + All-Gather buckets; the schedule is planned for
          the paper-scale 2x8x8x8 topology (BW of Table 2's 4D-Ring_FC_Ring_SW)
          and each chunk's 4D order is projected onto dims 1-3 (dim4 deleted)
          and executed on the 2x2x2 sub-slice (a plumbing test, not Themis-optimal).
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
from synth import WORKLOAD_PARAMS, bucket_sizes, device_input, torch_dtype  # noqa: E402
import bench  # noqa: E402

CONC = 1
LA = 0        # --lookahead: runtime intra-dim order (R28); 0 = auto (16 at <= 2 ranks per GPU, else 1)
MCB = 65536   # --min-cta-kb: op windows
LAT = 0       # --latency-ns: measured per-op A_K for the latency-aware auto-chunk column (config 3)


class Runner:
    def __init__(self, group, rank, world, local):
        self.group, self.rank, self.world, self.local = group, rank, world, local
        self.dev = torch.device("cuda", local)
        self.sms = torch.cuda.get_device_properties(self.dev).multi_processor_count

    def comm(self, sizes, max_bytes):
        topo = th.Topology(tuple(sizes), (1,) * len(sizes))
        c = th.Comm(topo, max_bytes, group=self.group, device=self.local)
        c.set_timeout(30.0)
        lay = bench.logical_layout(sizes, self.world)
        c.set_lookahead(LA or (16 if lay["V"] <= 2 else 1))       # R28, as bench.py's auto
        c.set_min_cta_bytes(MCB)                                   # op windows (small ops several per dim)
        ncross = len(lay["cross_gpu_dims"])
        c.set_stages(6 if ncross < len(sizes) else (2 if len(sizes) > 1 else 4))
        self.ctas_total = self.sms if ncross == 0 else ((min(self.sms, 128) if len(sizes) > 1 else 32) if ncross == len(sizes) else
                                                          (self.sms if lay["V"] >= 4 else 96))
        self.V = lay["V"]
        return c

    def time(self, comm, plan, coll, count, dtype, steps=3, warmup=1):
        V = self.V
        src = [device_input(self.rank * V + v, count, dtype, self.dev) for v in range(V)]
        ts = []
        for i in range(warmup + steps):
            for v in range(V):
                comm.rank_view(v, count, dtype).copy_(src[v])
            barrier(self.group, self.dev)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            th.run(coll, comm, plan, count, dtype)
            e1.record()
            torch.cuda.synchronize()
            if i >= warmup:
                ts.append(e0.elapsed_time(e1) / 1e3)
        comm.status()
        return max_over_ranks(sum(ts) / len(ts), self.group, self.dev)

    def nccl_bus_gbs(self, nbytes, dtype="f32", steps=5):
        """Context row: torch.distributed.all_reduce (NCCL) of nbytes per GPU,
        flat over the W GPUs, bus GB/s (max over GPUs of the mean time)."""
        if self.world == 1:
            return None
        import torch.distributed as dist
        x = torch.ones(nbytes // (2 if dtype == "bf16" else 4), device=self.dev,
                       dtype=torch.bfloat16 if dtype == "bf16" else torch.float32)
        for _ in range(2):
            dist.all_reduce(x, group=self.group)
        barrier(self.group, self.dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            dist.all_reduce(x, group=self.group)
        e1.record()
        torch.cuda.synchronize()
        t = max_over_ranks(e0.elapsed_time(e1) / 1e3 / steps, self.group, self.dev)
        return round(2 * nbytes * (self.world - 1) / self.world / t / 1e9, 2)

    def emit(self, row):
        if self.rank == 0:
            print(json.dumps(row), flush=True)


def pad_count(count, P, C, esz):
    g = P * C * (16 // esz)
    return (count + g - 1) // g * g


def config3(r: Runner, quick):
    W = r.world
    topos = {1: [(2, 4), (4, 2), (2, 2)], 2: [(2, 4), (4, 2), (2,)], 4: [(2, 4), (4, 2), (2, 2), (4,)],
             8: [(2, 4), (4, 2), (8,)]}[W]
    sizes_mib = [1, 16, 256, 1024] if quick else [1, 4, 16, 64, 256, 1024, 4096]
    chunks = [1, 4, 16, 64, 256] if quick else [1, 2, 4, 8, 16, 32, 64, 128, 256]
    for sizes in topos:
        P = int(np.prod(sizes))
        maxb = max(sizes_mib) << 20
        comm = r.comm(sizes, maxb)
        ratios = [(1,) * len(sizes)] + ([(200, 50)] if len(sizes) == 2 else [])
        pace_total = 240.0 if r.V > 1 else 500.0
        for S_mib in sizes_mib:
            if r.world > 1:   # NCCL context row for this size (flat, same bytes per GPU)
                r.emit({"config": 3, "n_gpus": W, "topology": "nccl-flat", "mib": S_mib,
                        "nccl_bus_gbs": r.nccl_bus_gbs(S_mib << 20)})
            for C in chunks:
                S = S_mib << 20
                if (S // 4) % (P * C * 4):
                    continue
                for rat in ratios:
                    row = {"config": 3, "n_gpus": W, "topology": "x".join(map(str, sizes)), "mib": S_mib,
                           "chunks": C, "ratio": ":".join(map(str, rat))}
                    for mode in ("caps", "paced"):
                        comm.set_pacing(mode == "paced")
                        bw = bench.paced_bw(rat, pace_total) if mode == "paced" else rat
                        for pol, name in ((th.BASELINE, "baseline"), (th.THEMIS, "themis")):
                            t = th.Topology(tuple(sizes), tuple(bw))
                            plan = th.Plan(t, th.ALLREDUCE, S, C, pol, th.SCF if pol else th.FIFO,
                                           concurrency=CONC)
                            plan.bind(comm, th.default_ctas(rat, r.ctas_total))
                            sec = r.time(comm, plan, th.ALLREDUCE, S // 4, "f32")
                            row[f"{mode}_{name}_bus_gbs"] = round(2 * S * (P - 1) / P / sec / 1e9, 2)
                            row[f"{mode}_{name}_model_ms"] = float(plan.makespan_ns()) * 1e-6 if mode == "paced" \
                                else None
                            plan.close()
                        row[f"{mode}_speedup"] = round(row[f"{mode}_themis_bus_gbs"] / row[f"{mode}_baseline_bus_gbs"],
                                                       3)
                        if LAT and mode == "paced" and C == 64:   # once per (size, ratio)
                            # latency-aware Themis with the planner-chosen chunk count (R25, NEXT-1)
                            t = th.Topology(tuple(sizes), tuple(bw), None, tuple([LAT] * len(sizes)))
                            try:
                                plan = th.Plan(t, th.ALLREDUCE, S, th.AUTO_CHUNKS, th.THEMIS, th.SCF,
                                               charge_latency=True)
                                plan.bind(comm, th.default_ctas(rat, r.ctas_total))
                                sec = r.time(comm, plan, th.ALLREDUCE, S // 4, "f32")
                                row["paced_themis_auto_bus_gbs"] = round(2 * S * (P - 1) / P / sec / 1e9, 2)
                                row["paced_themis_auto_chunks"] = plan.n_chunks
                                row["paced_auto_vs_baseline"] = round(row["paced_themis_auto_bus_gbs"] /
                                                                      row["paced_baseline_bus_gbs"], 3)
                                plan.close()
                            except th.ThemisError as e:
                                row["paced_themis_auto_error"] = str(e)
                    comm.set_pacing(False)
                    r.emit(row)
        comm.close()


def config4(r: Runner, quick):
    sizes = (2, 2, 2)
    P, C = 8, 64
    for model, nparams in WORKLOAD_PARAMS.items():
        buckets = bucket_sizes(nparams, 2)
        if quick:
            buckets = buckets[:3] + buckets[-1:]
        maxc = pad_count(max(buckets), P, th.AUTO_MAX_CHUNKS, 2)     # room for every chunk-count candidate
        comm = r.comm(sizes, maxc * 2)
        if r.world > 1:   # NCCL context: the same bf16 bucket trace through torch.distributed.all_reduce
            per = [r.nccl_bus_gbs(pad_count(n, P, C, 2) * 2, "bf16") for n in buckets]
            tot = sum(2 * pad_count(n, P, C, 2) * 2 * (r.world - 1) / r.world / (g * 1e9) for n, g in zip(buckets, per))
            r.emit({"config": 4, "n_gpus": r.world, "model": model, "mode": "nccl-flat", "bucket_bus_gbs": per,
                    "total_ms": round(tot * 1e3, 3)})
        for rat in [(1, 1, 1), (4, 2, 1)]:
            for mode in ("caps", "paced"):
                comm.set_pacing(mode == "paced")
                bw = bench.paced_bw(rat, 240.0 if r.V > 1 else 500.0) if mode == "paced" else rat
                res = {}
                for pol, name in ((th.BASELINE, "baseline"), (th.THEMIS, "themis")):
                    tot, per = 0.0, []
                    for n in buckets:
                        cnt = pad_count(n, P, C, 2)
                        plan = th.Plan(th.Topology(sizes, bw), th.ALLREDUCE, cnt * 2, C, pol,
                                       th.SCF if pol else th.FIFO, concurrency=CONC)
                        plan.bind(comm, th.default_ctas(rat, r.ctas_total))
                        sec = r.time(comm, plan, th.ALLREDUCE, cnt, "bf16", steps=2, warmup=1)
                        plan.close()
                        tot += sec
                        per.append(round(2 * cnt * 2 * (P - 1) / P / sec / 1e9, 1))
                    res[name] = {"total_ms": round(tot * 1e3, 3), "bucket_bus_gbs": per}
                if LAT and mode == "paced":   # latency-aware Themis, planner-chosen chunks (R25)
                    tot, per, chosen = 0.0, [], []
                    t = th.Topology(sizes, bw, None, (LAT,) * len(sizes))
                    for n in buckets:
                        cnt = pad_count(n, P, th.AUTO_MAX_CHUNKS, 2)
                        plan = th.Plan(t, th.ALLREDUCE, cnt * 2, th.AUTO_CHUNKS, th.THEMIS, th.SCF,
                                       charge_latency=True)
                        plan.bind(comm, th.default_ctas(rat, r.ctas_total))
                        sec = r.time(comm, plan, th.ALLREDUCE, cnt, "bf16", steps=2, warmup=1)
                        chosen.append(plan.n_chunks)
                        plan.close()
                        tot += sec
                        per.append(round(2 * cnt * 2 * (P - 1) / P / sec / 1e9, 1))
                    res["themis_auto"] = {"total_ms": round(tot * 1e3, 3), "bucket_bus_gbs": per, "chunks": chosen}
                r.emit({"config": 4, "n_gpus": r.world, "model": model, "params": nparams, "buckets": len(buckets),
                        "bucket_elems": buckets, "ratio": ":".join(map(str, rat)), "mode": mode, **res,
                        "speedup": round(res["baseline"]["total_ms"] / res["themis"]["total_ms"], 3)})
            comm.set_pacing(False)
        comm.close()


def config5(r: Runner, quick):
    big = th.Topology((2, 8, 8, 8), (3000000, 1400000, 1200000, 800000))   # MB/s (Table 2 4D-Ring_FC_Ring_SW)
    sizes, P, C = (2, 2, 2), 8, 64
    mibs = [4, 16, 64] if quick else [4, 16, 64, 256, 1024]
    comm = r.comm(sizes, max(mibs) << 20)
    for coll, name in ((th.REDUCE_SCATTER, "RS"), (th.ALL_GATHER, "AG")):
        for mib in mibs:
            S = mib << 20
            p4 = th.Plan(big, coll, S, C, th.THEMIS)
            rs4, ag4 = p4.orders()
            o4 = rs4 if coll == th.REDUCE_SCATTER else ag4
            proj = np.array([[d for d in row if d != 3] for row in o4], np.uint8)   # delete dim4
            sub = th.Topology(sizes, (3000, 1400, 1200))
            kw = {"rs_orders": proj} if coll == th.REDUCE_SCATTER else {"ag_orders": proj}
            plan = th.Plan(sub, coll, S, C, th.THEMIS, th.SCF, **kw)
            plan.bind(comm, th.default_ctas((3000, 1400, 1200), r.ctas_total))
            sec = r.time(comm, plan, coll, S // 2, "bf16")
            native = th.Plan(sub, coll, S, C, th.THEMIS).bind(comm, th.default_ctas((3000, 1400, 1200), r.ctas_total))
            sec_native = r.time(comm, native, coll, S // 2, "bf16")
            r.emit({"config": 5, "n_gpus": r.world, "coll": name, "mib": mib, "planned_on": "2x8x8x8",
                    "plan4d_hash": p4.info["hash"], "plan4d_greedy_chunks": p4.info["n_greedy"],
                    "projected_bus_gbs": round(S * (P - 1) / P / sec / 1e9, 2),
                    "native_2x2x2_themis_bus_gbs": round(S * (P - 1) / P / sec_native / 1e9, 2),
                    "projected_orders_first8": [list(map(int, row)) for row in proj[:8]]})
            p4.close()
            plan.close()
            native.close()
    comm.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=[3, 4, 5])
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--concurrency", type=int, default=1, help="ops in flight per dim (plans)")
    ap.add_argument("--lookahead", type=int, default=0, help="runtime intra-dim order window (R28); 0 = auto")
    ap.add_argument("--min-cta-kb", type=int, default=64, help="op windows: KiB per CTA (0 = full-width ops)")
    ap.add_argument("--latency-ns", type=int, default=0,
                    help="config 3: also time a latency-aware Themis plan with planner-chosen chunks (A_K ns)")
    a = ap.parse_args()
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    rank, world, local, group = init_from_env("nccl" if int(os.environ.get("WORLD_SIZE", 1)) > 1 else "gloo")
    torch.cuda.set_device(local)
    global CONC, LAT, LA, MCB
    CONC = a.concurrency
    LA = a.lookahead
    MCB = a.min_cta_kb * 1024
    LAT = a.latency_ns
    r = Runner(group, rank, world, local)
    {3: config3, 4: config4, 5: config5}[a.config](r, a.quick)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
