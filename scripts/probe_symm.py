"""Probe (development): is torch symmetric memory / NVLS multicast available here?"""
import os

import torch
import torch.distributed as dist

rank = int(os.environ.get("RANK", 0))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
try:
    from cuda.bindings import driver as drv
    drv.cuInit(0)
    err, dev = drv.cuDeviceGet(local)
    err, mc = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    print(rank, "multicast supported attr:", mc, err, flush=True)
    err, fab = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
    print(rank, "fabric handle supported:", fab, err, flush=True)
except Exception as e:
    print(rank, "cuda-python probe failed:", repr(e), flush=True)
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, dtype=torch.float32, device=f"cuda:{local}")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print(rank, "symm ok; multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", len(h.buffer_ptrs),
          flush=True)
except Exception as e:
    print(rank, "symm failed:", repr(e), flush=True)
dist.destroy_process_group()
