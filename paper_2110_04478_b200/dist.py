"""Process-group plumbing (one process per GPU, torch.distributed).

Only bootstrap and bookkeeping live here — the exchange of CUDA IPC heap
handles at comm creation and max-over-ranks timing.  No data-path collective:
the All-Reduce itself runs inside libthemis's kernel over NVLink peer memory.
"""

from __future__ import annotations

import os


def env_world() -> tuple:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init_from_env(backend: str = "nccl"):
    """Initialise the default process group from torchrun's env (127.0.0.1
    rendezvous).  Returns (rank, world, local_rank, group-or-None)."""
    import torch
    import torch.distributed as dist
    rank, world, local = env_world()
    if world <= 1:
        return 0, 1, 0, None
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return rank, world, local, dist.group.WORLD


def allgather_bytes(payload: bytes, group=None) -> list:
    """Every rank's `payload`, in rank order (used for 64-byte IPC handles)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, payload, group=group)
    return out


def max_over_ranks(x: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (device-timed step time) over the group."""
    import torch
    import torch.distributed as dist
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def barrier(group=None, device=None) -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        if device is not None and dist.get_backend(group) == "nccl":
            dist.barrier(group=group, device_ids=[device.index])
        else:
            dist.barrier(group=group)


def check_same_plan(plan, group=None) -> None:
    """Fail fast on the host if the ranks built different plans (the kernel's
    entry check would latch THEMIS_ERR_PLAN_MISMATCH, R22): all-gathers the
    plan hash (inputs, schedule, per-dim order) and raises ValueError naming
    the ranks that differ from rank 0.  No-op without a process group."""
    import torch.distributed as dist
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return
    hashes = allgather_bytes(int(plan.info["hash"]).to_bytes(8, "little"), group)
    bad = [r for r, h in enumerate(hashes) if h != hashes[0]]
    if bad:
        raise ValueError(f"ranks {bad} built a different plan than rank 0 (plan hash differs)")
