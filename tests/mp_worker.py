"""Multi-GPU parity worker (one process per GPU; launched by test_gpu_multi.py
with torchrun).  Every rank checks its own logical ranks against the oracle."""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import data as O, scheduler as S, topology as T  # noqa: E402
from paper_2110_04478_b200 import themis as th  # noqa: E402
from paper_2110_04478_b200.dist import init_from_env  # noqa: E402
from synth import ELEM_SIZE, host_inputs  # noqa: E402

COLL = {S.AR: th.ALLREDUCE, "RS": th.REDUCE_SCATTER, "AG": th.ALL_GATHER}


KIND_O = {th.RING: T.RING, th.DIRECT: T.DIRECT, th.SWITCH: T.SWITCH}


def case(group, W, g, sizes, bw, dtype, C, slice_elems, coll, policy, engine, kinds=None, lookahead=1, push=False,
         ll=False):
    topo = th.Topology(sizes, bw, kinds)
    P = topo.P
    V = P // W
    N = P * C * slice_elems
    esz = ELEM_SIZE[dtype]
    comm = th.Comm(topo, N * esz, group=group, ll_bytes=4 * N * esz if ll else 0)
    if ll:
        comm.set_ll(N * esz)
    comm.set_engine(engine)
    comm.set_timeout(20.0)
    comm.set_lookahead(lookahead)
    comm.set_push(push)
    plan = th.Plan(topo, COLL[coll], N * esz, C, policy).bind(comm)
    if ll and not plan.bound_ll():
        return [-1]
    xs = host_inputs(P, N, dtype, dist="wide")
    for v in range(V):
        r = g * V + v
        src = torch.from_numpy(xs[r].view(np.int16) if dtype == "bf16" else xs[r])
        view = comm.rank_view(v, N, dtype)
        view.copy_(src.view(torch.bfloat16) if dtype == "bf16" else src)
    torch.cuda.synchronize()
    th.run(COLL[coll], comm, plan, N, dtype)
    torch.cuda.synchronize()
    comm.status()
    o = T.Topology.make(sizes, bw, [KIND_O[k] for k in kinds] if kinds else None)
    sched = S.schedule_collective(o, coll, N * esz, C, S.THEMIS if policy == th.THEMIS else S.BASELINE)
    want = O.run_schedule(xs, sched, dtype)
    bad = []
    blk = N // P
    for v in range(V):
        r = g * V + v
        t = comm.rank_view(v, N, dtype).cpu()
        got = t.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else t.numpy()
        if coll == "RS":
            ok = np.array_equal(got[r * blk:(r + 1) * blk], want[r][r * blk:(r + 1) * blk])
        else:
            ok = np.array_equal(got, want[r])
        if not ok:
            bad.append(r)
    plan.close()
    comm.close()
    return bad


def fullsize_case(group, W, g):
    """configs[1] at full size (2x2x2, 1 GiB fp32 per rank, 64 chunks, 4:2:1)
    in bench.py's launch configuration for this W; sampled elements bit-exact
    against the oracle's per-element formulation with its own schedule."""
    import bench
    sizes, ratio, C = (2, 2, 2), (4, 2, 1), 64
    S_ = 1 << 30
    N = S_ // 4
    topo = th.Topology(sizes, ratio)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cfg = bench.launch_config(sizes, W, sms)               # exactly what bench.py times
    V = bench.logical_layout(sizes, W)["V"]
    comm = th.Comm(topo, S_, group=group)
    comm.set_timeout(30.0)
    comm.set_stages(1)
    comm.set_stage_bytes(cfg["stage_kb"] * 1024)
    comm.set_stages(cfg["stages"])
    comm.set_lookahead(cfg["lookahead"])
    comm.set_min_cta_bytes(cfg["min_cta_bytes"])
    plan = th.Plan(topo, th.ALLREDUCE, S_, C, th.THEMIS).bind(comm, th.default_ctas(ratio, cfg["total_ctas"]))
    from synth import device_input
    xs = [device_input(g * V + v, N, "f32", torch.device("cuda")) for v in range(V)]
    for v in range(V):
        comm.rank_view(v, N, "f32").copy_(xs[v])
    torch.cuda.synchronize()
    th.run(th.ALLREDUCE, comm, plan, N, "f32")
    torch.cuda.synchronize()
    comm.status()
    rng = np.random.default_rng(11)
    idx = np.unique(np.concatenate([rng.integers(0, N, 400), [0, N - 1]]))
    it = torch.from_numpy(idx).cuda()
    # every rank's inputs at the sampled positions (regenerated: the generator is seeded per rank)
    P = topo.P
    allx = np.stack([device_input(r, N, "f32", torch.device("cuda"))[it].cpu().numpy() for r in range(P)])
    o = T.Topology.make(sizes, ratio)
    sched = S.schedule_collective(o, S.AR, S_, C, S.THEMIS)
    bad = 0
    for v in range(V):
        got = comm.rank_view(v, N, "f32")[it].cpu().numpy()
        for n, i in enumerate(idx):
            b, c = O.element_location(o, N, C, int(i))
            want = O.allreduce_element(list(allx[:, n]), o, sched.chunks[c].rs, "f32", b)
            bad += np.float32(want).tobytes() != got[n].tobytes()
    plan.close()
    comm.close()
    return bad


def nccl_and_stress_case(group, W, g, iters=60):
    """int32 results equal torch.distributed.all_reduce (NCCL) of the per-GPU
    sums (the library routine, SURVEY §4 tier 4), and a stress loop: many
    back-to-back collectives with plans switching between policies / chunk
    counts / engines on one comm, every result checked (flag protocol under
    load: any ordering bug shows up as corruption or a watchdog timeout)."""
    import random
    import torch.distributed as dist
    sizes = (2, 2, 2)
    topo = th.Topology(sizes, (1, 1, 1))
    P, V = 8, 8 // W
    N = P * 256 * 4 * 4                     # divisible for C in {1, 4, 16, 64, 256}
    comm = th.Comm(topo, N * 4, group=group)
    comm.set_timeout(20.0)
    rng = random.Random(1234)              # same sequence on every rank
    plans = {}
    bad = 0
    for it in range(iters):
        C = rng.choice([1, 4, 16, 64, 256])
        pol = rng.choice([th.BASELINE, th.THEMIS])
        intra = rng.choice([th.SCF, th.FIFO])
        eng = rng.choice(["tma", "tma", "ldg"])
        ctas = rng.choice([None, [4, 4, 4], [12, 6, 3]])
        push = rng.random() < 0.5                        # R30, same on every rank (launch hash)
        key = (C, pol, intra, str(ctas), push)
        if key not in plans:
            comm.set_push(push)
            plans[key] = th.Plan(topo, th.ALLREDUCE, N * 4, C, pol, intra).bind(comm, ctas)
        comm.set_engine(eng)
        # R28: ranks may run a dim's ops in different orders -- give every GPU
        # its own intra-dim mode in the same collective (static / runtime L)
        comm.set_lookahead([1, 4, 16, 32][(it + g) % 4])
        xs = [torch.randint(-(1 << 20), 1 << 20, (N,), dtype=torch.int32, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(1000 * it + g * V + v))
              for v in range(V)]
        for v in range(V):
            comm.rank_view(v, N, "i32").copy_(xs[v])
        torch.cuda.synchronize()
        th.run(th.ALLREDUCE, comm, plans[key], N, "i32")
        ref = torch.stack(xs).sum(0, dtype=torch.int32) if V > 1 else xs[0].clone()
        dist.all_reduce(ref, group=group)       # NCCL over the W GPUs
        torch.cuda.synchronize()
        comm.status()
        for v in range(V):
            bad += int(not torch.equal(comm.rank_view(v, N, "i32"), ref))
    for p_ in plans.values():
        p_.close()
    comm.close()
    return bad


def api_case(group, W, g):
    """User-facing paths at W GPUs: Comm.all_reduce on ragged tensors,
    Comm.reduce_scatter / all_gather, themis_allreduce_host (chunk-streamed,
    with a chunk-arrival plan) and a CUDA-graph replay — int32 exact against
    the plain definitions.  Returns the number of mismatches on this GPU."""
    topo = th.Topology((2, 2, 2), (1, 1, 1))
    P = 8
    V = P // W
    bad = 0
    comm = th.Comm(topo, 1 << 22, group=group)
    comm.set_timeout(20.0)
    dev = torch.device("cuda", torch.cuda.current_device())
    # ragged all_reduce
    n = 12345
    xs = host_inputs(P, n, "i32", seed=7)
    ts = [torch.from_numpy(xs[g * V + v]).to(dev) for v in range(V)]
    comm.all_reduce(ts, n_chunks=4)
    want = O.allreduce_definition(xs, "i32")
    bad += sum(not np.array_equal(t.cpu().numpy(), want) for t in ts)
    # reduce_scatter -> all_gather
    n = P * 4 * 4 * 16
    xs = host_inputs(P, n, "i32", seed=8)
    outs = comm.reduce_scatter([torch.from_numpy(xs[g * V + v]).to(dev) for v in range(V)], n_chunks=4)
    want = O.allreduce_definition(xs, "i32")
    blk = n // P
    bad += sum(not np.array_equal(outs[v].cpu().numpy(), want[(g * V + v) * blk:(g * V + v + 1) * blk])
               for v in range(V))
    full = comm.all_gather(outs, n_chunks=4)
    bad += sum(not np.array_equal(f.cpu().numpy(), want) for f in full)
    # host buffers, chunk-streamed with an arrival-time plan
    n = P * 16 * 4 * 8
    xs = host_inputs(P, n, "i32", seed=9)
    plan = th.Plan(th.Topology((2, 2, 2), (4000, 2000, 1000)), th.ALLREDUCE, n * 4, 16,
                   chunk_release_ns=5000).bind(comm)
    hin = torch.from_numpy(np.concatenate([xs[g * V + v] for v in range(V)])).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    for _ in range(2):
        th.themis_allreduce_host(hin.data_ptr(), hout.data_ptr(), comm.data_ptr, n, "i32", plan)
    torch.cuda.synchronize()
    want = O.allreduce_definition(xs, "i32")
    bad += sum(not np.array_equal(hout.numpy()[v * n:(v + 1) * n], want) for v in range(V))
    # CUDA graph: two All-Reduces captured, replayed twice
    for v in range(V):
        comm.rank_view(v, n, "i32").copy_(torch.from_numpy(xs[g * V + v]))
    torch.cuda.synchronize()
    gph, st = torch.cuda.CUDAGraph(), torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(gph, stream=st):
            th.run(th.ALLREDUCE, comm, plan, n, "i32")
            th.run(th.ALLREDUCE, comm, plan, n, "i32")
    torch.cuda.synchronize()
    for _ in range(2):
        gph.replay()
    torch.cuda.synchronize()
    w = xs
    for _ in range(4):
        w = [O.allreduce_definition(w, "i32")] * P
    bad += sum(not np.array_equal(comm.rank_view(v, n, "i32").cpu().numpy(), w[0]) for v in range(V))
    comm.status()
    plan.close()
    comm.close()
    return bad


def nvls_case(group, W, g):
    """NVLS dims (R27, R29) on a multicast heap: int32 exact vs the plain
    definition; floats within the north_star tolerance of the fp64 sum (the
    switch sums in its own order) and identical on every rank.  Returns the
    number of mismatches (-1 if this box has no multicast)."""
    SW, DI = th.NVLS, th.DIRECT
    cfgs = [((W,), (SW,), "i32", 8), ((W,), (SW,), "f32", 8), ((2, W), (DI, SW), "f32", 4),
            ((2, W), (DI, SW), "bf16", 4)]
    if W == 2:
        cfgs.append(((2, 2, 2), (DI, DI, SW), "i32", 8))
    bad = 0
    for sizes, kinds, dtype, C in cfgs:
        topo = th.Topology(sizes, (1,) * len(sizes), kinds)
        P = topo.P
        V = P // W
        N = P * C * (16 // ELEM_SIZE[dtype]) * 257
        try:
            comm = th.Comm(topo, N * ELEM_SIZE[dtype], group=group, nvls=True)
        except th.ThemisError:
            return -1
        comm.set_timeout(20.0)
        plan = th.Plan(topo, th.ALLREDUCE, N * ELEM_SIZE[dtype], C).bind(comm)
        bad += int(plan.bound_nvls() == 0)       # the modelled in-switch pairs really run in the switch
        xs = host_inputs(P, N, dtype)
        for v in range(V):
            src = torch.from_numpy(xs[g * V + v].view(np.int16) if dtype == "bf16" else xs[g * V + v])
            comm.rank_view(v, N, dtype).copy_(src.view(torch.bfloat16) if dtype == "bf16" else src)
        torch.cuda.synchronize()
        for _ in range(2):                       # twice: the second call reduces the first's result
            th.run(th.ALLREDUCE, comm, plan, N, dtype)
        torch.cuda.synchronize()
        comm.status()
        outs = []
        for v in range(V):
            t = comm.rank_view(v, N, dtype).cpu()
            outs.append(t.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else t.numpy())
        once = O.allreduce_definition(xs, dtype)
        if dtype == "i32":
            want = O.allreduce_definition([once] * P, "i32")
            bad += sum(not np.array_equal(o, want) for o in outs)
        else:
            want = P * once
            scale = P * O.abs_sum(xs, dtype)
            tol = {"f32": 1e-5, "bf16": 1e-2}[dtype]   # north_star
            bad += sum(not np.all(np.abs(O.to_f64(o, dtype) - want) <= tol * scale) for o in outs)
        # every rank holds the same bits: compare a digest across GPUs
        dig = torch.tensor([float(np.frombuffer(outs[0].tobytes(), np.uint8).astype(np.int64).sum() % 1000003)],
                           device="cuda")
        mx, mn = dig.clone(), dig.clone()
        import torch.distributed as dist
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
        bad += int(mx.item() != mn.item()) + sum(not np.array_equal(o, outs[0]) for o in outs[1:])
        plan.close()
        comm.close()
    return bad


def fault_case(group, W, g):
    """Fault injection: rank 1 launches a plan
    with a different intra-dimension policy.  Every rank must report
    THEMIS_ERR_PLAN_MISMATCH (in-kernel plan-hash check) instead of hanging."""
    topo = th.Topology((W,), (1,))
    N = W * 4 * 1024
    comm = th.Comm(topo, N * 4, group=group)
    comm.set_timeout(10.0)
    plan = th.Plan(topo, th.ALLREDUCE, N * 4, 4, th.THEMIS, th.FIFO if g == 1 else th.SCF).bind(comm)
    th.run(th.ALLREDUCE, comm, plan, N, "f32")
    torch.cuda.synchronize()
    try:
        comm.status()
        status = 0
    except th.ThemisError as e:
        status = e.status
    plan.close()
    comm.close()
    return status


def main():
    rank, W, local, group = init_from_env("nccl")
    cases = []
    for engine in ("tma", "ldg"):
        cases += [((2, 2, 2), (1, 1, 1), "i32", 8, 2052, S.AR, th.THEMIS, engine),
                  ((2, 2, 2), (4, 2, 1), "f32", 8, 5124, S.AR, th.BASELINE, engine)]
    cases += [((2, 2, 2), (1, 1, 1), "bf16", 4, 8200, S.AR, th.THEMIS, "tma"),
              ((2, 2, 2), (2, 2, 1), "f16", 64, 264, S.AR, th.THEMIS, "tma"),
              ((2, 2, 2), (1, 1, 1), "i32", 4, 2048, "RS", th.THEMIS, "tma"),
              ((2, 2, 2), (1, 1, 1), "i32", 4, 2048, "AG", th.THEMIS, "tma"),
              ((W,), (1,), "f32", 4, 8196, S.AR, th.THEMIS, "tma"),
              ((2, 4), (1, 1), "f32", 16, 1028, S.AR, th.THEMIS, "tma"),
              ((4, 2), (1, 1), "i32", 16, 1028, S.AR, th.THEMIS, "tma"),
              ((W,), (1,), "f32", 4, 8196, S.AR, th.THEMIS, "tma", (th.RING,)),
              ((W,), (1,), "bf16", 4, 8200, S.AR, th.THEMIS, "tma", (th.RING,)),        # per-hop rounding (R18)
              ((4, 2), (1, 1), "f16", 8, 2056, S.AR, th.THEMIS, "tma", (th.RING, th.DIRECT)),
              ((2, 2, 2), (1, 1, 1), "f32", 4, 4100, S.AR, th.THEMIS, "tma", (th.RING,) * 3),
              ((2, 4), (1, 1), "f32", 8, 2052, S.AR, th.THEMIS, "tma", (th.DIRECT, th.RING)),
              ((4, 2), (1, 1), "f32", 8, 2052, "RS", th.THEMIS, "tma", (th.RING, th.DIRECT))]
    import random
    rng = random.Random(int(os.environ.get("THEMIS_RANDOM_SEED", 4478)) + W)   # identical on every rank
    for _ in range(int(os.environ.get("THEMIS_MP_RANDOM", 12))):               # randomised cases
        D = rng.randint(1, 3)
        sizes = tuple(rng.choice([2, 2, 4]) for _ in range(D))
        kinds = tuple(rng.choice([th.DIRECT, th.RING]) for _ in range(D))
        dtype = rng.choice(["i32", "f32", "bf16", "f16"])
        vec = 16 // ELEM_SIZE[dtype]
        cases.append((sizes, tuple(rng.choice([1, 2, 4]) for _ in range(D)), dtype, rng.choice([1, 4, 8]),
                      vec * rng.randint(1, 300), rng.choice([S.AR, S.AR, "RS", "AG"]),
                      rng.choice([th.THEMIS, th.BASELINE]), "tma", kinds,
                      rng.choice([1, 4, 16]), rng.random() < 0.5))
    for sizes, dtype in (((2, 2, 2), "i32"), ((2, 2, 2), "f32"), ((4, 2), "bf16"), ((2, 4), "i32"), ((8,), "f32")):
        for coll in (S.AR, "RS", "AG"):                                          # R31 LL small collectives
            cases.append((sizes, tuple([1] * len(sizes)), dtype, 8, (16 // ELEM_SIZE[dtype]) * 97, coll, th.THEMIS,
                          "tma", None, 1, False, True))
    fails = []
    for c in cases:
        if int(np.prod(c[0])) % W:
            continue
        bad = case(group, W, rank, *c)
        if bad:
            fails.append((c, bad))
    import torch.distributed as dist
    if 8 % W == 0:
        nb = api_case(group, W, rank)
        if nb:
            fails.append((("tensor API / host streaming / CUDA graph",), [f"{nb} mismatches"]))
    nb = nvls_case(group, W, rank)
    if nb > 0:
        fails.append((("NVLS switch dims",), [f"{nb} mismatches"]))
    elif nb < 0 and rank == 0:
        print("mp_worker: NVLS cases skipped (no multicast on this box)")
    st = fault_case(group, W, rank)
    if st != 6:
        fails.append((("fault-injection plan mismatch",), [f"status {st}"]))
    if 8 % W == 0:
        nb = nccl_and_stress_case(group, W, rank)
        if nb:
            fails.append((("NCCL comparison / stress loop",), [f"{nb} mismatching results"]))
        nb = fullsize_case(group, W, rank)
        if nb:
            fails.append((("full-size configs[1] sampled parity",), [f"{nb} mismatching samples"]))
    t = torch.tensor([len(fails)], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print(f"mp_worker W={W}: {len(cases)} cases, failing ranks total {int(t.item())}")
    for c, bad in fails:
        print(f"rank {rank} FAIL {c} logical ranks {bad}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
