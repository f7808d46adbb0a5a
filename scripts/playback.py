"""Synthetic workload playback (Fig 9).

A DDP-style backward pass: for each 25 MiB bf16 gradient bucket (ResNet-152
60.19 M / GNMT ~280 M parameters) a synthetic compute kernel (one bf16 cuBLAS
GEMM sized to the bucket's backward FLOPs) runs on the compute stream; when it
finishes, the bucket's All-Reduce (one Themis kernel through the C ABI) is
enqueued on a high-priority communication stream.  Iteration time runs from
the first GEMM to the last All-Reduce; exposed communication = iteration -
compute alone (the paper's Fig 9 split of compute vs exposed comm).

    python scripts/playback.py [--model gnmt] [--ratio 1:1:1] [--paced]      # N = 1 (emulated)
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/playback.py --gpus 4

Synthetic compute recipe: backward FLOPs per logical rank and bucket =
4 x params_in_bucket x tokens (backward ~ 2 x forward, forward ~ 2 x params x
tokens); tokens per rank: ResNet-152 3056 (32 images x 95.5 FLOPs/param/2),
GNMT 6400 (128 sentences x 50 tokens).  A GPU hosting V logical ranks runs V
ranks' compute.  Not the paper's traces (OUT): a shape-alike.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_04478_b200 import themis as th  # noqa: E402
from paper_2110_04478_b200.dist import barrier, init_from_env, max_over_ranks  # noqa: E402
from synth import WORKLOAD_PARAMS, bucket_sizes  # noqa: E402
import bench  # noqa: E402

TOKENS = {"resnet152": 3056, "gnmt": 6400}
GEMM_MN = 4096


def pad_count(count, P, C, esz):
    g = P * C * (16 // esz)
    return (count + g - 1) // g * g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--model", default="all", choices=["all"] + list(WORKLOAD_PARAMS))
    ap.add_argument("--ratio", default="1:1:1")
    ap.add_argument("--paced", action="store_true", help="pace each dim at its emulated BW (else CTA caps)")
    ap.add_argument("--pace-gbs", type=float, default=0, help="per-rank sum of paced dim BWs (GB/s)")
    ap.add_argument("--chunks", type=int, default=64)
    ap.add_argument("--concurrency", type=int, default=1)
    ap.add_argument("--latency-ns", type=int, default=0,
                    help="also run latency-aware Themis plans with planner-chosen chunks (measured A_K, ns)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    out_fd = os.dup(1)            # JSON rows to the real stdout, banners to stderr
    os.dup2(2, 1)
    rank, world, local, group = init_from_env("nccl" if int(os.environ.get("WORLD_SIZE", 1)) > 1 else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sizes = (2, 2, 2)
    P = 8
    lay = bench.logical_layout(sizes, world)
    V = lay["V"]
    ncross = len(lay["cross_gpu_dims"])
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # fewer CTAs than the stand-alone bench so compute can share the GPU
    ctas_total = 64 if ncross else sms // 2
    rat = tuple(int(x) for x in a.ratio.split(":"))
    pace_total = a.pace_gbs or (240.0 if V > 1 else 500.0)
    bw = bench.paced_bw(rat, pace_total) if a.paced else rat
    models = list(WORKLOAD_PARAMS) if a.model == "all" else [a.model]
    lo, hi = torch.cuda.Stream.priority_range()
    comm_stream = torch.cuda.Stream(device=dev, priority=hi)
    comp_stream = torch.cuda.Stream(device=dev, priority=lo)

    for model in models:
        buckets = bucket_sizes(WORKLOAD_PARAMS[model], 2)
        counts = [pad_count(n, P, a.chunks, 2) for n in buckets]
        counts_auto = [pad_count(n, P, th.AUTO_MAX_CHUNKS, 2) for n in buckets]
        comm = th.Comm(th.Topology(sizes, bw), max(counts + counts_auto) * 2, group=group, device=local)
        comm.set_timeout(60.0)
        comm.set_stages(4 if ncross else 6)
        comm.set_pacing(a.paced)
        for v in range(V):
            comm.rank_view(v, max(counts + counts_auto), "bf16").normal_(0, 1e-2)
        # per-bucket GEMM: 2 * MN * MN * k = V * 4 * params * tokens
        ks = [max(64, int(V * 4 * n * TOKENS[model] / (2 * GEMM_MN * GEMM_MN)) // 64 * 64) for n in buckets]
        A = torch.randn(GEMM_MN, max(ks), device=dev, dtype=torch.bfloat16)
        B = torch.randn(max(ks), GEMM_MN, device=dev, dtype=torch.bfloat16)
        Cm = torch.empty(GEMM_MN, GEMM_MN, device=dev, dtype=torch.bfloat16)
        flops = sum(2 * GEMM_MN * GEMM_MN * k for k in ks)
        row = {"workload": "playback", "model": model, "params": WORKLOAD_PARAMS[model], "buckets": len(buckets),
               "n_gpus": world, "ranks_per_gpu": V, "ratio": a.ratio, "mode": "paced" if a.paced else "caps",
               "bw_mbps": list(bw) if a.paced else None, "ctas_total": ctas_total,
               "compute_tflop_per_gpu": round(flops / 1e12, 3), "concurrency": a.concurrency}
        variants = [(th.BASELINE, "baseline"), (th.THEMIS, "themis")]
        if a.latency_ns:
            variants.append((th.THEMIS, "themis_auto"))
        for pol, name in variants:
            plans = {}
            auto = name == "themis_auto"
            cnts = counts_auto if auto else counts
            for c in sorted(set(cnts)):
                if auto:    # latency-aware, planner-chosen chunk count (R25)
                    t = th.Topology(sizes, bw, None, (a.latency_ns,) * len(sizes))
                    p = th.Plan(t, th.ALLREDUCE, c * 2, th.AUTO_CHUNKS, th.THEMIS, th.SCF, charge_latency=True)
                else:
                    p = th.Plan(th.Topology(sizes, bw), th.ALLREDUCE, c * 2, a.chunks, pol,
                                th.SCF if pol == th.THEMIS else th.FIFO, concurrency=a.concurrency)
                plans[c] = p.bind(comm, th.default_ctas(rat, ctas_total))

            def iteration(do_comp, do_comm):
                ev = []
                for i, k in enumerate(ks):
                    if do_comp:
                        with torch.cuda.stream(comp_stream):
                            torch.mm(A[:, :k], B[:k, :], out=Cm)
                            e = torch.cuda.Event()
                            e.record(comp_stream)
                            ev.append(e)
                    if do_comm:
                        if do_comp:
                            comm_stream.wait_event(ev[-1])
                        th.run(th.ALLREDUCE, comm, plans[cnts[i]], cnts[i], "bf16", comm_stream)

            def timed(do_comp, do_comm):
                ts = []
                for it in range(a.warmup + a.steps):
                    barrier(group, dev)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(comp_stream)
                    comm_stream.wait_event(e0)
                    iteration(do_comp, do_comm)
                    comp_stream.wait_stream(comm_stream)
                    e1.record(comp_stream)
                    torch.cuda.synchronize()
                    if it >= a.warmup:
                        ts.append(e0.elapsed_time(e1))
                comm.status()
                return max_over_ranks(sorted(ts)[len(ts) // 2], group, dev)

            t_comp = timed(True, False) if name == "baseline" else row["compute_ms"]
            t_comm = timed(False, True)
            t_iter = timed(True, True)
            row["compute_ms"] = round(t_comp, 3)
            row[name] = {"comm_only_ms": round(t_comm, 3), "iteration_ms": round(t_iter, 3),
                         "exposed_comm_ms": round(t_iter - t_comp, 3),
                         "overlap_frac": round(1 - (t_iter - t_comp) / t_comm, 3) if t_comm > 0 else None}
            for p in plans.values():
                p.close()
        row["iteration_speedup"] = round(row["baseline"]["iteration_ms"] / row["themis"]["iteration_ms"], 3)
        if "themis_auto" in row:
            row["auto_iteration_speedup"] = round(row["baseline"]["iteration_ms"] / row["themis_auto"]["iteration_ms"], 3)
        row["comm_speedup"] = round(row["baseline"]["comm_only_ms"] / row["themis"]["comm_only_ms"], 3)
        if rank == 0:
            os.write(out_fd, (json.dumps(row) + "\n").encode())
        comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
