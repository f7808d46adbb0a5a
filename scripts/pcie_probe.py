"""PCIe reference for the e2e number: pinned host <-> device copy rates of one
GPU, H2D alone, D2H alone and both at once on two streams (CUDA events)."""
import json

import torch

n = 1 << 28                                  # 1 GiB fp32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.ones(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(h2d, d2h):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    if h2d:
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


for _ in range(2):
    timed(True, True)
out = {}
for name, h, d in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
    t = min(timed(h, d) for _ in range(3))
    out[name + "_gbs_per_direction"] = round(n * 4 / t / 1e9, 1)
print(json.dumps({"pcie_probe": out, "bytes": n * 4}))
