"""Development probe: where does a small op's time go?  Detailed per-op
device stamps (trace level 2) of one All-Reduce, emulated on one GPU or over
N GPUs (torchrun).  Prints medians relative to the op's start."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402
from paper_2110_04478_b200.dist import init_from_env  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="2,2,2")
ap.add_argument("--mib", type=int, default=16)
ap.add_argument("--kib", type=int, default=0, help="size in KiB (overrides --mib)")
ap.add_argument("--chunks", type=int, default=64)
ap.add_argument("--ctas", default="8,8,8")
ap.add_argument("--policy", default="baseline")
a = ap.parse_args()
os.environ.setdefault("NCCL_DEBUG", "WARN")
rank, world, local, group = init_from_env("nccl" if int(os.environ.get("WORLD_SIZE", 1)) > 1 else "gloo")
torch.cuda.set_device(local)
sizes = tuple(int(x) for x in a.sizes.split(","))
topo = th.Topology(sizes, (1,) * len(sizes))
N = ((a.kib << 10) if a.kib else (a.mib << 20)) // 4
comm = th.Comm(topo, N * 4, group=group, device=local)
comm.set_stages(int(os.environ.get("PROBE_STAGES", "4")))
comm.enable_trace(2)
for v in range(comm.V):
    comm.rank_view(v, N, "f32").fill_(1.0)
plan = th.Plan(topo, th.ALLREDUCE, N * 4, a.chunks, th.THEMIS if a.policy == "themis" else th.BASELINE)
plan.bind(comm, [int(x) for x in a.ctas.split(",")])
for _ in range(3):
    th.run(th.ALLREDUCE, comm, plan, N, "f32")
torch.cuda.synchronize()
if group is not None:
    torch.distributed.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
th.run(th.ALLREDUCE, comm, plan, N, "f32")
e1.record()
torch.cuda.synchronize()
tr = comm.fetch_trace(plan).astype(np.int64)
de = comm.fetch_trace_detail(plan).astype(np.int64)
if rank == 0:
    st = tr[:, :, 0]
    rel = lambda x: (x - st) / 1e3
    names = ["producer_last_tile", "consumers_done", "cta_at_counter", "last_atomic_ret", "after_sys_fence",
             "after_proxy_fence"]
    print(f"kernel {e0.elapsed_time(e1)*1e3:.1f} us  ops {st.size}")
    for j, n in enumerate(names):
        print(f"  {n:20s} median {np.median(rel(de[:, :, j])):7.2f} us  p90 {np.percentile(rel(de[:, :, j]), 90):7.2f}")
    print(f"  {'published':20s} median {np.median(rel(tr[:, :, 1])):7.2f} us")
    lat = [tr[c, s, 0] - tr[c, s - 1, 1] for c in range(tr.shape[0]) for s in range(1, tr.shape[1])]
    print(f"  stage transition median {np.median(lat)/1e3:.2f} us p10 {np.percentile(lat, 10)/1e3:.2f}")
    for c, s_ in ((1, 1), (2, 3), (3, 4)):                    # a few raw ops, relative to the op start
        print(f"  op (c{c}, s{s_}) rel us:", [round((x - st[c, s_]) / 1e3, 2) for x in de[c, s_, :6]],
              "end", round((tr[c, s_, 1] - st[c, s_]) / 1e3, 2))
    # per (dim, phase): median op duration and the per-rank bytes it moves -> GB/s
    rs, ag = plan.orders()
    D = len(sizes)
    NS = plan.info["n_stages"]
    Sb = N * 4 / a.chunks
    for k in range(D):
        for ph in ("RS", "AG"):
            durs, vols = [], []
            for c in range(a.chunks):
                order = list(rs[c]) + list(ag[c])
                h = Sb
                for s in range(NS):
                    d = int(order[s])
                    pk = sizes[d]
                    is_rs = s < D
                    v = h * (pk - 1) / pk if is_rs else h * (pk - 1)
                    if d == k and (ph == "RS") == is_rs:
                        durs.append(tr[c, s, 1] - tr[c, s, 0])
                        vols.append(v)
                    h = h / pk if is_rs else h * pk
            if durs:
                print(f"  dim{k+1} {ph}: median op {np.median(durs)/1e3:.1f} us, {np.median(vols)/1e6:.2f} MB/rank "
                      f"-> {np.median(vols)/np.median(durs):.1f} GB/s per rank")
plan.close()
comm.close()
if group is not None:
    torch.distributed.destroy_process_group()
