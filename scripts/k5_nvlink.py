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
    ap.add_argument("--all-gpus", action="store_true",
                    help="every GPU runs its rank alone at once (all peers faked): bidirectional NVLink "
                         "traffic with no cross-GPU waits -- the executor's ceiling without dependencies")
    a = ap.parse_args()
    S = a.mib << 20
    N = S // 4
    sizes = tuple(int(x) for x in a.sizes.split(","))
    bw = [float(x) for x in a.bw_gbs.split(",")]
    ctas = [int(x) for x in a.ctas.split(",")]
    topo = th.Topology(sizes, tuple(int(b * 1000) for b in bw))
    P = topo.P
    sig, stride, hb = th.heap_layout(P, P, S)
    for g in range(P):
        for h in range(P):
            if h != g:
                enable_peer(g, h)
    runners = list(range(P)) if a.all_gpus else [0]
    # runner g's view: its own heap on GPU g, and for every other GPU h a heap
    # of its own on GPU h (pulled over NVLink; g's flag writes land there, so
    # runners never see each other's flags and none ever waits)
    allocs = []

    def alloc(dev_):
        torch.cuda.set_device(dev_)
        h_ = C.c_void_p()
        check(lib().themis_heap_alloc(hb, C.byref(h_)))
        allocs.append((dev_, h_.value))
        return h_.value

    view = {g: [alloc(h) for h in range(P)] for g in runners}
    comms, plans, streams = {}, {}, {}
    for g in runners:
        torch.cuda.set_device(g)
        comm = C.c_void_p()
        tc = topo.to_c()
        check(lib().themis_comm_create(g, P, C.byref(tc), (C.c_void_p * MAX_GPUS)(*view[g]), hb, stride,
                                       C.byref(comm)))
        check(lib().themis_comm_set_stages(comm, 1))
        check(lib().themis_comm_set_stage_bytes(comm, a.stage_kb * 1024))
        check(lib().themis_comm_set_stages(comm, a.stages))
        check(lib().themis_comm_set_pacing(comm, int(a.paced)))
        check(lib().themis_comm_set_lookahead(comm, a.lookahead))
        plan = th.Plan(topo, th.ALLREDUCE, S, a.chunks)
        arr = (C.c_int32 * MAX_GPUS)(*ctas)
        check(lib().themis_plan_bind(plan.h, comm, arr))
        for h in range(P):
            if h != g:
                check(lib().themis_debug_fake_peer_gpu(plan.h, h, N, 0))
        comms[g], plans[g], streams[g] = comm, plan, torch.cuda.current_stream(g)
    ts = []
    for i in range(a.iters + 2):
        ev = {}
        for g in runners:
            torch.cuda.set_device(g)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(streams[g])
            check(lib().themis_allreduce(view[g][g] + sig, N, 0, plans[g].h, streams[g].cuda_stream))
            e1.record(streams[g])
            ev[g] = (e0, e1)
        for g in runners:
            torch.cuda.set_device(g)
            torch.cuda.synchronize(g)
            check(lib().themis_comm_status(comms[g]))
        if i >= 2:
            ts.append(max(ev[g][0].elapsed_time(ev[g][1]) / 1e3 for g in runners))
    t = sum(ts) / len(ts)
    plan = plans[0]
    # one rank per GPU: every pulled byte crosses NVLink, sum_K N_K = 2 S (P-1)/P (F2)
    vol = [v / plan.info["byte_scale"] for v in plan.info["dim_volume"]]
    nvlink_bytes = sum(vol)
    out = {"tag": a.tag, "sizes": list(sizes), "mib": a.mib, "chunks": a.chunks, "ctas": ctas, "paced": a.paced,
           "emulated_gbs": bw, "stages": a.stages, "stage_kb": a.stage_kb, "lookahead": a.lookahead,
           "all_gpus": a.all_gpus,
           "ms": round(t * 1e3, 4), "nvlink_bytes": nvlink_bytes, "bus_gbs": round(nvlink_bytes / t / 1e9, 2)}
    if len(sizes) == 1:
        out["ratio_to_emulated"] = round(nvlink_bytes / t / 1e9 / bw[0], 4)
    print(json.dumps(out), flush=True)
    for g in runners:
        torch.cuda.set_device(g)
        plans[g].close()
        lib().themis_comm_free(comms[g])
    for dev_, h_ in allocs:
        torch.cuda.set_device(dev_)
        lib().themis_heap_free(C.c_void_p(h_))


if __name__ == "__main__":
    main()
