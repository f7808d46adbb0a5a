"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

Holds NONE of the method's arithmetic: it only draws per-rank input buffers.
Recipe: rank r uses seed
SEED_BASE + r; fp32 ~ U[-1, 1); bf16 / fp16 = N(0, 1) * 1e-2 cast to the
dtype; int32 ~ U[-2^20, 2^20) (plus explicit wrap tests in tests/).
Shapes: one flat gradient buffer of `count` elements per rank, the shape of a
data-parallel gradient bucket (PAPER.md:219 footnote, :689).

Gradient-bucket traces (configs 4/5) come from ``bucket_sizes``: DDP-style
25 MiB buckets over the parameter counts BASELINE.json names (ResNet-152
~60.19 M, GNMT ~280 M parameters).
"""

from __future__ import annotations

import numpy as np

SEED_BASE = 20211010
DTYPES = ("f32", "bf16", "f16", "i32")
ELEM_SIZE = {"f32": 4, "bf16": 2, "f16": 2, "i32": 4}


def host_inputs(P: int, count: int, dtype: str, seed: int = SEED_BASE, dist: str = "recipe") -> list:
    """Per-rank numpy inputs.  bf16 is returned as uint16 bit patterns.
    dist="wide": N(0,1) * 2^U{-8..8} for floats — magnitudes spread over 16
    binades so that sums are inexact and the summation order shows in the
    bits (U[-1,1) fp32 values are multiples of 2^-23: 2-3 term sums are exact)."""
    import torch
    out = []
    for r in range(P):
        g = torch.Generator(device="cpu")
        g.manual_seed(seed + r)
        x = _draw_wide(count, dtype, g) if (dist == "wide" and dtype != "i32") else _draw(count, dtype, g, "cpu")
        out.append(x.numpy().copy() if dtype != "bf16" else x.view(torch.int16).numpy().view(np.uint16).copy())
    return out


def _draw_wide(count, dtype, g):
    import torch
    x = torch.randn(count, generator=g, dtype=torch.float32)
    e = torch.randint(-8, 9, (count,), generator=g).to(torch.float32)
    return (x * torch.exp2(e)).to(torch_dtype(dtype))


def device_input(rank: int, count: int, dtype: str, device, seed: int = SEED_BASE):
    """One rank's input drawn on `device` with torch's generator (large sizes)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed + rank)
    return _draw(count, dtype, g, device)


def torch_dtype(dtype: str):
    import torch
    return {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16,
            "i32": torch.int32}[dtype]


def _draw(count, dtype, g, device):
    import torch
    if dtype == "f32":
        return torch.rand(count, generator=g, device=device, dtype=torch.float32) * 2 - 1
    if dtype in ("bf16", "f16"):
        x = torch.randn(count, generator=g, device=device, dtype=torch.float32) * 1e-2
        return x.to(torch_dtype(dtype))
    if dtype == "i32":
        return torch.randint(-(1 << 20), 1 << 20, (count,), generator=g, device=device, dtype=torch.int32)
    raise ValueError(dtype)


def bucket_sizes(n_params: int, elem_size: int = 2, bucket_bytes: int = 25 << 20) -> list:
    """Element counts of DDP-style gradient buckets (25 MiB default)."""
    per = bucket_bytes // elem_size
    full, rem = divmod(n_params, per)
    return [per] * full + ([rem] if rem else [])


WORKLOAD_PARAMS = {"resnet152": 60_190_000, "gnmt": 280_000_000}
