"""K5 over NVLink: one dimension group alone, on the real executor kernel, with
its CTA cap and (optionally) pacing -- the per-dimension emulation check of
SURVEY.md:549-551 measured on NVLink.

One process.  GPU 0 runs the executor for a D = 1, P = 2 logical topology
(every dim of the 2x2x2 BASELINE topology is such a pair) whose other rank
lives on GPU 1; that rank's flags are faked in GPU 0's signal pads
(themis_debug_fake_peer_gpu), so GPU 0's kernel never waits and pulls the
peer's half over NVLink: an All-Reduce of S bytes moves N = S/2 (RS) + S/2
(AG) = S over NVLink into GPU 0 (2 (P-1)/P S with P = 2).  Because no other
GPU takes part, ncu can profile (replay) it:

    python scripts/k5_nvlink.py --bw-gbs 300 --ctas 42 --paced      # plain run
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
        -k regex:themis_exec -c 3 python scripts/k5_nvlink.py ...  # hardware NVLink bytes

Prints one JSON line: in-kernel achieved GB/s (CUDA events) vs the emulated
BW_K.  The data results are meaningless (the peer never computes).

--sizes 2,2 (4 GPUs) runs a whole multi-dimensional plan this way: GPU 0's
kernel of the all-NVLink 2x2 executes alone against three faked peers, a
single-GPU launch ncu --set full can profile with real NVLink traffic.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_04478_b200 import themis as th  # noqa: E402
from paper_2110_04478_b200._lib import MAX_GPUS, check, lib  # noqa: E402


def enable_peer(dev: int, peer: int) -> None:
    from cuda.bindings import runtime as rt
    torch.cuda.set_device(dev)
    torch.cuda.synchronize()
    err, = rt.cudaDeviceEnablePeerAccess(peer, 0)
    if err not in (rt.cudaError_t.cudaSuccess, rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
        raise RuntimeError(f"cudaDeviceEnablePeerAccess({peer}): {err}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2", help="logical topology, one rank per GPU (P <= GPUs); "
                    "GPU 0 runs alone, every other GPU's ranks are faked")
    ap.add_argument("--mib", type=int, default=512, help="All-Reduce bytes per rank")
    ap.add_argument("--chunks", type=int, default=64)
    ap.add_argument("--ctas", default="32", help="CTA cap per dimension group (comma list)")
    ap.add_argument("--bw-gbs", default="300", help="emulated BW_K per dim (GB/s per rank, comma list)")
    ap.add_argument("--lookahead", type=int, default=1)
    ap.add_argument("--paced", action="store_true")
    ap.add_argument("--stages", type=int, default=2)
    ap.add_argument("--stage-kb", type=int, default=32)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    S = a.mib << 20
    N = S // 4
    sizes = tuple(int(x) for x in a.sizes.split(","))
    bw = [float(x) for x in a.bw_gbs.split(",")]
    ctas = [int(x) for x in a.ctas.split(",")]
    topo = th.Topology(sizes, tuple(int(b * 1000) for b in bw))
    P = topo.P
    sig, stride, hb = th.heap_layout(P, P, S)
    heaps = [0] * P
    for g in range(1, P):
        enable_peer(0, g)
        torch.cuda.set_device(g)
        h = C.c_void_p()
        check(lib().themis_heap_alloc(hb, C.byref(h)))
        heaps[g] = h.value
    torch.cuda.set_device(0)
    h0 = C.c_void_p()
    check(lib().themis_heap_alloc(hb, C.byref(h0)))
    heaps[0] = h0.value
    comm = C.c_void_p()
    tc = topo.to_c()
    check(lib().themis_comm_create(0, P, C.byref(tc), (C.c_void_p * MAX_GPUS)(*heaps), hb, stride, C.byref(comm)))
    check(lib().themis_comm_set_stages(comm, 1))
    check(lib().themis_comm_set_stage_bytes(comm, a.stage_kb * 1024))
    check(lib().themis_comm_set_stages(comm, a.stages))
    check(lib().themis_comm_set_pacing(comm, int(a.paced)))
    check(lib().themis_comm_set_lookahead(comm, a.lookahead))
    plan = th.Plan(topo, th.ALLREDUCE, S, a.chunks)
    arr = (C.c_int32 * MAX_GPUS)(*ctas)
    check(lib().themis_plan_bind(plan.h, comm, arr))
    for g in range(1, P):
        check(lib().themis_debug_fake_peer_gpu(plan.h, g, N, 0))
    buf = h0.value + sig
    stream = torch.cuda.current_stream()
    ts = []
    for i in range(a.iters + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(lib().themis_allreduce(buf, N, 0, plan.h, stream.cuda_stream))
        e1.record()
        torch.cuda.synchronize()
        check(lib().themis_comm_status(comm))
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / 1e3)
    t = sum(ts) / len(ts)
    # one rank per GPU: every pulled byte crosses NVLink, sum_K N_K = 2 S (P-1)/P (F2)
    vol = [v / plan.info["byte_scale"] for v in plan.info["dim_volume"]]
    nvlink_bytes = sum(vol)
    out = {"tag": a.tag, "sizes": list(sizes), "mib": a.mib, "chunks": a.chunks, "ctas": ctas, "paced": a.paced,
           "emulated_gbs": bw, "stages": a.stages, "stage_kb": a.stage_kb, "lookahead": a.lookahead,
           "ms": round(t * 1e3, 4), "nvlink_bytes": nvlink_bytes, "bus_gbs": round(nvlink_bytes / t / 1e9, 2)}
    if len(sizes) == 1:
        out["ratio_to_emulated"] = round(nvlink_bytes / t / 1e9 / bw[0], 4)
    print(json.dumps(out), flush=True)
    plan.close()
    lib().themis_comm_free(comm)
    lib().themis_heap_free(h0)
    for g in range(1, P):
        torch.cuda.set_device(g)
        lib().themis_heap_free(C.c_void_p(heaps[g]))


if __name__ == "__main__":
    main()
