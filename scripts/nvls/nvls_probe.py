"""NVLS bandwidth probe (experiment for NEXT-2; not the product path).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 scripts/nvls/nvls_probe.py

Builds scripts/nvls/nvls_probe.cu with nvcc (sm_100a) into /tmp, allocates a
torch symmetric-memory buffer with a multicast address, and times the flat
NVLS All-Reduce (ld_reduce + multimem.st), the RS half (ld_reduce) and the AG
half (multimem.st) on 1 GiB fp32 per GPU.  Prints one JSON line (rank 0):
bus GB/s per the nccl-tests convention (AR 2S(W-1)/W / t; RS, AG S(W-1)/W / t).
"""
import ctypes
import json
import os
import subprocess
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    so = f"/tmp/nvls_probe_{os.getuid()}.so"
    if rank == 0:
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                               "-fPIC", "-o", so, os.path.join(HERE, "nvls_probe.cu")])
    dist.barrier()
    lib = ctypes.CDLL(so)
    lib.nvls_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    import torch.distributed._symmetric_memory as symm
    n = (1 << 30) // 4
    t = symm.empty(n, dtype=torch.float32, device=f"cuda:{local}")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    mc = getattr(h, "multicast_ptr", 0)
    if not mc:
        if rank == 0:
            print(json.dumps({"nvls_probe": "unavailable", "why": "no multicast pointer from torch symmetric memory"}))
        dist.destroy_process_group()
        return
    res = {"world": world, "bytes_per_gpu": n * 4}
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    for name, mode, busf in (("ar", 0, 2.0), ("rs", 1, 1.0), ("ag", 2, 1.0)):
        best = None
        for blocks in (sms, 2 * sms, 4 * sms):
            ts = []
            for it in range(5):
                t.fill_(1.0 + rank)
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                err = lib.nvls_launch(ctypes.c_void_p(mc), ctypes.c_void_p(t.data_ptr()), n, rank, world, mode, blocks,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                e1.record()
                torch.cuda.synchronize()
                dist.barrier()
                if err:
                    raise RuntimeError(f"launch error {err}")
                if it >= 2:
                    ts.append(e0.elapsed_time(e1) / 1e3)
            tt = torch.tensor([sum(ts) / len(ts)], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            gbs = busf * n * 4 * (world - 1) / world / tt.item() / 1e9
            if best is None or gbs > best[0]:
                best = (round(gbs, 1), blocks)
        if name == "ar":     # check: every element = sum over ranks of (1 + r)
            want = sum(1.0 + r for r in range(world))
            ok = bool(torch.all(t == want).item())
            res["ar_correct"] = ok
        res[name + "_bus_gbs"], res[name + "_blocks"] = best
    if rank == 0:
        print(json.dumps({"nvls_probe": res}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
