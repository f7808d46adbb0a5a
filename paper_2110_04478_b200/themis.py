"""Thin Python binding of libthemis (include/themis.h).

Argument marshalling only.  The names mirror the C ABI
(``themis_plan``, ``themis_allreduce``, ``themis_reduce_scatter``,
``themis_all_gather`` ...); ``Plan`` / ``Comm`` are small RAII wrappers around
the opaque handles.  PyTorch is used for device selection, streams and — for
multi-process comms — the process group that exchanges CUDA IPC handles.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional, Sequence

import numpy as np

from ._lib import (IPC_HANDLE_BYTES, MAX_DIMS, MAX_GPUS, PlanInfo_t, PlanReq_t, ThemisError, Topology_t, check,
                   lib)

RING, DIRECT, SWITCH = 0, 1, 2                 # Table 1
NVLS = 3                                       # switch with in-switch reduction (R29)
ALLREDUCE, REDUCE_SCATTER, ALL_GATHER = 0, 1, 2
BASELINE, THEMIS = 0, 1                        # Table 3
SCF, FIFO, SCF_LITERAL = 0, 1, 2               # §4.3
DTYPES = {"f32": 0, "bf16": 1, "f16": 2, "i32": 3}
ELEM_SIZE = {"f32": 4, "bf16": 2, "f16": 2, "i32": 4}
COLL_NAMES = {"AR": ALLREDUCE, "RS": REDUCE_SCATTER, "AG": ALL_GATHER}
AUTO_CHUNKS, AUTO_MAX_CHUNKS = 0, 256           # n_chunks = 0: planner picks C (THEMIS_AUTO_MAX_CHUNKS)


@dataclass(frozen=True)
class Topology:
    """P_1 x ... x P_D; bw in MB/s per dimension."""
    sizes: tuple
    bw_mbps: tuple
    kinds: tuple = field(default=None)
    latency_ns: tuple = field(default=None)

    @property
    def D(self) -> int:
        return len(self.sizes)

    @property
    def P(self) -> int:
        return int(np.prod(self.sizes))

    def to_c(self) -> Topology_t:
        if not 1 <= self.D <= MAX_DIMS:
            raise ThemisError(1, f"ndims must be 1..{MAX_DIMS}")
        t = Topology_t()
        t.ndims = self.D
        kinds = self.kinds or (DIRECT,) * self.D
        lat = self.latency_ns or (0,) * self.D
        for k in range(self.D):
            t.size[k] = int(self.sizes[k])
            t.bw_mbps[k] = int(self.bw_mbps[k])
            t.step_latency_ns[k] = int(lat[k])
            t.kind[k] = int(kinds[k])
        return t


def _table2(sizes, gbps_per_link, links, latency_ns, kinds) -> Topology:
    """Aggregate per-NPU BW of a dim = Gb/s per link x links / 8 (GB/s) -> MB/s."""
    return Topology(tuple(sizes), tuple(b * n * 125 for b, n in zip(gbps_per_link, links)), tuple(kinds),
                    tuple(latency_ns))


# PAPER.md Table 2 (:509-519): the paper's simulated platforms (planner use;
# 1024 NPUs): sizes, BW per link (Gb/s), links per NPU, step latency (ns), Table 1 kind.
TABLE2 = {
    "2D-SW_SW": _table2((16, 64), (200, 800), (6, 1), (700, 1700), (SWITCH, SWITCH)),
    "3D-SW_SW_SW_homo": _table2((16, 8, 8), (200, 200, 800), (4, 4, 1), (700, 700, 1700), (SWITCH,) * 3),
    "3D-SW_SW_SW_hetero": _table2((16, 8, 8), (200, 200, 400), (8, 4, 1), (700, 700, 1700), (SWITCH,) * 3),
    "3D-FC_Ring_SW": _table2((8, 16, 8), (200, 200, 400), (7, 4, 1), (700, 700, 1700), (DIRECT, RING, SWITCH)),
    "4D-Ring_SW_SW_SW": _table2((4, 4, 8, 8), (1000, 200, 200, 400), (2, 8, 4, 1), (20, 700, 700, 1700),
                                (RING, SWITCH, SWITCH, SWITCH)),
    "4D-Ring_FC_Ring_SW": _table2((4, 8, 4, 8), (1500, 200, 200, 800), (2, 7, 6, 1), (20, 700, 700, 1700),
                                  (RING, DIRECT, RING, SWITCH)),
}


def themis_plan(topo: Topology, coll: int, nbytes: int, n_chunks: int, policy: int = THEMIS, intra: int = SCF,
                threshold_div: int = 16, charge_latency: bool = False, concurrency: int = 1,
                chunk_release_ns: int = 0) -> C.c_void_p:
    req = PlanReq_t(coll, policy, intra, n_chunks, int(nbytes), threshold_div, int(charge_latency), concurrency, 0,
                    int(chunk_release_ns))
    out = C.c_void_p()
    tc = topo.to_c()
    check(lib().themis_plan(C.byref(tc), C.byref(req), C.byref(out)))
    return out


class Plan:
    """A Themis (or baseline) plan: per-chunk dim orders + per-dim op order."""

    def __init__(self, topo: Topology, coll: int = ALLREDUCE, nbytes: int = 0, n_chunks: int = 64,
                 policy: int = THEMIS, intra: int = SCF, threshold_div: int = 16, charge_latency: bool = False,
                 rs_orders=None, ag_orders=None, concurrency: int = 1, chunk_release_ns: int = 0):
        """rs_orders / ag_orders (C x D, 0-based): caller-given per-chunk
        orders (themis_plan_custom) instead of Algorithm 1.  chunk_release_ns:
        chunk c arrives at (c+1) * r ns in the pre-simulation (host streaming)."""
        self.topo = topo
        self.coll = coll
        self.nbytes = int(nbytes)
        self.n_chunks = n_chunks
        self.policy = policy
        self.intra = intra
        if rs_orders is None and ag_orders is None:
            self.h = themis_plan(topo, coll, nbytes, n_chunks, policy, intra, threshold_div, charge_latency,
                                 concurrency, chunk_release_ns)
        else:
            req = PlanReq_t(coll, policy, intra, n_chunks, int(nbytes), threshold_div, int(charge_latency),
                            concurrency, 0, int(chunk_release_ns))
            rs = None if rs_orders is None else np.ascontiguousarray(np.asarray(rs_orders, np.uint8).reshape(-1))
            ag = None if ag_orders is None else np.ascontiguousarray(np.asarray(ag_orders, np.uint8).reshape(-1))
            out = C.c_void_p()
            tc = topo.to_c()
            check(lib().themis_plan_custom(C.byref(tc), C.byref(req), None if rs is None else rs.ctypes.data,
                                           None if ag is None else ag.ctypes.data, C.byref(out)))
            self.h = out
        self.comm = None
        i = PlanInfo_t()
        check(lib().themis_plan_info(self.h, C.byref(i)))
        D = i.ndims
        self.info = {
            "ndims": D, "n_chunks": i.n_chunks, "n_ranks": i.n_ranks, "n_stages": i.n_stages,
            "n_greedy": i.n_greedy, "time_scale": i.time_scale, "byte_scale": i.byte_scale,
            "makespan": i.makespan, "busy": list(i.busy[:D]), "idle": list(i.idle[:D]),
            "dim_volume": list(i.dim_volume[:D]), "final_load": list(i.final_load[:D]), "hash": i.hash,
            "util_num": i.util_num, "util_den": i.util_den, "util_exact": bool(i.util_exact),
        }
        self.n_chunks = i.n_chunks          # the planner's choice when n_chunks = 0 (auto)

    # -- queries -------------------------------------------------------------
    @property
    def D(self) -> int:
        return self.info["ndims"]

    def orders(self):
        C_, D = self.info["n_chunks"], self.D
        rs = np.zeros(C_ * D, np.uint8)
        ag = np.zeros(C_ * D, np.uint8)
        check(lib().themis_plan_orders(self.h, rs.ctypes.data, ag.ctypes.data))
        return rs.reshape(C_, D), ag.reshape(C_, D)

    def dim_ops(self) -> list:
        C_, D, NS = self.info["n_chunks"], self.D, self.info["n_stages"]
        buf = np.zeros(D * C_ * NS, np.uint32)
        n = np.zeros(D, np.int32)
        check(lib().themis_plan_dim_ops(self.h, buf.ctypes.data, n.ctypes.data))
        out = []
        for k in range(D):
            row = buf[k * C_ * NS: k * C_ * NS + n[k]]
            out.append([(int(e) >> 8, int(e) & 0xFF) for e in row])
        return out

    def servers(self) -> np.ndarray:
        """Pre-simulated server of every op, [C][n_stages]."""
        n = self.info["n_chunks"] * self.info["n_stages"]
        out = np.zeros(n, np.int32)
        check(lib().themis_plan_servers(self.h, out.ctypes.data))
        return out.reshape(self.info["n_chunks"], self.info["n_stages"])

    def times(self):
        n = self.info["n_chunks"] * self.info["n_stages"]
        s = np.zeros(n, np.uint64)
        e = np.zeros(n, np.uint64)
        check(lib().themis_plan_times(self.h, s.ctypes.data, e.ctypes.data))
        return s, e

    def to_csv(self) -> str:
        """Schedule export: `chunk_id,rs_order,ag_order,bytes`,
        1-based dims, bytes = S / C — the format the oracle writes, so a plan
        can be saved, diffed and replayed (themis_plan_custom)."""
        rs, ag = self.orders()
        cb = Fraction(self.nbytes, self.n_chunks)
        lines = ["chunk_id,rs_order,ag_order,bytes"]
        for c in range(self.n_chunks):
            r = " ".join(str(int(d) + 1) for d in rs[c] if d != 0xFF)
            a = " ".join(str(int(d) + 1) for d in ag[c] if d != 0xFF)
            lines.append(f"{c},{r},{a},{cb}")
        return "\n".join(lines) + "\n"

    def utilization(self) -> Fraction:
        """The paper's average BW utilisation of the pre-simulated run,
        sum_K BW_K busy_K / (sum BW * makespan) (R14), as the
        library computes it (themis_plan_info_t.util_num / util_den)."""
        return Fraction(self.info["util_num"], self.info["util_den"])

    def makespan_ns(self) -> Fraction:
        return Fraction(self.info["makespan"], self.info["time_scale"])

    # -- execution -------------------------------------------------------------
    def bind(self, comm: "Comm", ctas_per_dim: Optional[Sequence[int]] = None) -> "Plan":
        arr = None
        if ctas_per_dim is not None:
            arr = (C.c_int32 * MAX_DIMS)(*[int(x) for x in ctas_per_dim])
        check(lib().themis_plan_bind(self.h, comm.h, arr))
        self.comm = comm
        return self

    def bound_ll(self) -> bool:
        """True if this bound plan runs with LL packets (R31)."""
        n = C.c_int32()
        check(lib().themis_plan_bound_ll(self.h, C.byref(n)))
        return bool(n.value)

    def bound_nvls(self) -> int:
        """RS+AG pairs of this bound plan that run in the switch (R29)."""
        n = C.c_int32()
        check(lib().themis_plan_bound_nvls(self.h, C.byref(n)))
        return n.value

    def bound_ctas(self) -> list:
        arr = (C.c_int32 * MAX_DIMS)()
        check(lib().themis_plan_bound_ctas(self.h, arr))
        return list(arr[:self.D])

    def close(self):
        if self.h:
            lib().themis_plan_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def heap_layout(n_ranks: int, n_gpus: int, data_bytes: int):
    s, st, hb = C.c_uint64(), C.c_uint64(), C.c_uint64()
    check(lib().themis_heap_layout(n_ranks, n_gpus, int(data_bytes), C.byref(s), C.byref(st), C.byref(hb)))
    return s.value, st.value, hb.value


class _CAI:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


class Comm:
    """Heap + peer table for the W GPUs hosting a P-rank logical topology.

    Single process (group None): W = 1, all P ranks live in this GPU's HBM
    (V = P).  Multi-process: one process per GPU in `group`; V = P / W ranks
    per GPU; heaps are exchanged as CUDA IPC handles over the process group.
    """

    def __init__(self, topo: Topology, data_bytes: int, group=None, device=None, nvls: bool = False,
                 ll_bytes: int = 0):
        """nvls=True (W > 1): the heap is torch symmetric memory with an NVSwitch
        multicast mapping, so switch dims can reduce in the switch (R27).
        ll_bytes > 0: reserve an LL inbox of that many bytes per local rank
        after the data regions (R31; enable with set_ll)."""
        import torch
        self.topo = topo
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        torch.cuda.set_device(self.device)
        if group is not None:
            import torch.distributed as dist
            self.W = dist.get_world_size(group)
            self.gpu_rank = dist.get_rank(group)
        else:
            self.W, self.gpu_rank = 1, 0
        if self.W > MAX_GPUS or topo.P % self.W:
            raise ValueError(f"{topo.P} logical ranks cannot be spread over {self.W} GPUs")
        self.P = topo.P
        self.V = topo.P // self.W
        self.sig_bytes, self.vrank_stride, self.heap_bytes = heap_layout(self.P, self.W, data_bytes)
        self.ll_stride = (int(ll_bytes) + (1 << 16) - 1) >> 16 << 16
        self.heap_bytes += self.V * self.ll_stride
        self.imported = []
        self._symm = None
        self.mc_heap = 0
        heaps = [0] * self.W
        if nvls and self.W > 1:
            import torch.distributed._symmetric_memory as symm
            buf = symm.empty(self.heap_bytes, dtype=torch.uint8, device=self.device)
            buf.zero_()
            torch.cuda.synchronize(self.device)
            hdl = symm.rendezvous(buf, group.group_name)
            self.mc_heap = int(getattr(hdl, "multicast_ptr", 0) or 0)
            if not self.mc_heap:
                raise ThemisError(7, "NVLS requested but torch symmetric memory has no multicast mapping here")
            self._symm = (buf, hdl)
            heaps = [int(x) for x in hdl.buffer_ptrs]
            self.heap = heaps[self.gpu_rank]
        else:
            heap = C.c_void_p()
            check(lib().themis_heap_alloc(self.heap_bytes, C.byref(heap)))
            self.heap = heap.value
            heaps[self.gpu_rank] = self.heap
        if self.W > 1 and self._symm is None:
            from .dist import allgather_bytes
            h = (C.c_uint8 * IPC_HANDLE_BYTES)()
            check(lib().themis_heap_export(self.heap, h))
            allh = allgather_bytes(bytes(h), group)
            for g in range(self.W):
                if g == self.gpu_rank:
                    continue
                hh = (C.c_uint8 * IPC_HANDLE_BYTES).from_buffer_copy(allh[g])
                p = C.c_void_p()
                check(lib().themis_heap_import(hh, C.byref(p)))
                heaps[g] = p.value
                self.imported.append(p.value)
        arr = (C.c_void_p * MAX_GPUS)(*heaps)
        tc = topo.to_c()
        out = C.c_void_p()
        check(lib().themis_comm_create(self.gpu_rank, self.W, C.byref(tc), arr, self.heap_bytes, self.vrank_stride,
                                       C.byref(out)))
        self.h = out
        self.data_ptr = self.heap + self.V * self.sig_bytes    # local rank 0's data region
        if self.mc_heap:
            check(lib().themis_comm_set_multicast(self.h, self.mc_heap))

    def rank_view(self, v: int, count: int, dtype: str):
        """torch view of local rank v's first `count` elements."""
        import torch
        ptr = self.data_ptr + v * self.vrank_stride
        ts = {"f32": "<f4", "i32": "<i4", "f16": "<f2", "bf16": "<i2"}[dtype]
        t = torch.as_tensor(_CAI(ptr, count, ts), device=self.device)
        return t.view(torch.bfloat16) if dtype == "bf16" else t

    def status(self) -> None:
        check(lib().themis_comm_status(self.h))

    def set_engine(self, engine: str) -> None:
        check(lib().themis_comm_set_engine(self.h, {"ldg": 0, "tma": 1}[engine]))

    def set_pacing(self, on: bool) -> None:
        """Cap each dim at its topology bw_mbps by pacing (BW emulation)."""
        check(lib().themis_comm_set_pacing(self.h, int(on)))

    def set_stages(self, stages: int) -> None:
        """TMA ring depth per CTA (bytes in flight = stages x stage_bytes)."""
        check(lib().themis_comm_set_stages(self.h, int(stages)))

    def set_stage_bytes(self, nbytes: int) -> None:
        check(lib().themis_comm_set_stage_bytes(self.h, int(nbytes)))

    def set_min_cta_bytes(self, nbytes: int) -> None:
        """Op-window sizing: small ops run on fewer CTAs, several in flight."""
        check(lib().themis_comm_set_min_cta_bytes(self.h, int(nbytes)))

    def set_window_rotation(self, rotate: bool) -> None:
        """Op windows: consecutive windows (True) or every narrow op from CTA 0."""
        check(lib().themis_comm_set_window_rotation(self.h, int(rotate)))

    def set_ll(self, max_bytes: int, inbox_bytes: Optional[int] = None) -> None:
        """LL packets for collectives of at most max_bytes per rank (R31);
        inbox_bytes defaults to the whole inbox reserved at construction.
        Takes effect at the next Plan.bind; max_bytes = 0 turns it off."""
        inbox = self.ll_stride if inbox_bytes is None else int(inbox_bytes)
        check(lib().themis_comm_set_ll(self.h, inbox if max_bytes else 0, int(max_bytes)))

    def set_push(self, on: bool) -> None:
        """Direct AG ops by writes (TMA bulk stores into the peers, R30);
        takes effect at the next Plan.bind."""
        check(lib().themis_comm_set_push(self.h, int(on)))

    def set_lookahead(self, lookahead: int) -> None:
        """Runtime intra-dim order: 1 = the enforced pre-simulated order;
        L > 1 = first ready op among the next L of it (direct dims, R28)."""
        check(lib().themis_comm_set_lookahead(self.h, int(lookahead)))

    def set_timeout(self, seconds: float) -> None:
        check(lib().themis_comm_set_timeout(self.h, int(seconds * 1e9)))

    def enable_trace(self, on=True) -> None:
        """on: False/0 off, True/1 per-op start/end, 2 detailed stamps."""
        check(lib().themis_comm_enable_trace(self.h, int(on)))

    def fetch_trace_detail(self, plan: "Plan") -> np.ndarray:
        n = plan.info["n_chunks"] * plan.info["n_stages"] * 6
        out = np.zeros(n, np.uint64)
        check(lib().themis_trace_fetch_detail(self.h, out.ctypes.data, n))
        return out.reshape(plan.info["n_chunks"], plan.info["n_stages"], 6)

    def fetch_trace(self, plan: Plan) -> np.ndarray:
        n = plan.info["n_chunks"] * plan.info["n_stages"] * 2
        out = np.zeros(n, np.uint64)
        check(lib().themis_trace_fetch(self.h, out.ctypes.data, n))
        return out.reshape(plan.info["n_chunks"], plan.info["n_stages"], 2)

    # -- convenience: tensors in, tensors out (copies through the heap) -------
    def _tensors(self, tensors):
        import torch
        ts = [tensors] if isinstance(tensors, torch.Tensor) else list(tensors)
        if len(ts) != self.V:
            raise ValueError(f"expected {self.V} tensors (one per local logical rank), got {len(ts)}")
        dt = {torch.float32: "f32", torch.bfloat16: "bf16", torch.float16: "f16", torch.int32: "i32"}.get(ts[0].dtype)
        if dt is None:
            raise ThemisError(3, f"unsupported dtype {ts[0].dtype}")
        n = ts[0].numel()
        if any(t.numel() != n or t.dtype != ts[0].dtype or t.device != self.device for t in ts):
            raise ValueError("tensors must share numel, dtype and this comm's device")
        return ts, dt, n

    def _plan(self, coll, nbytes, n_chunks, policy, bw_mbps, ctas_per_dim) -> "Plan":
        """Plans cached per (collective, bytes, chunks, policy, bw, CTAs)."""
        if nbytes > self.vrank_stride:
            raise ValueError(f"{nbytes} B exceeds the heap's {self.vrank_stride} B per rank")
        bw = tuple(bw_mbps or self.topo.bw_mbps)
        key = (coll, nbytes, n_chunks, policy, bw, None if ctas_per_dim is None else tuple(ctas_per_dim))
        cache = self.__dict__.setdefault("_plans", {})
        plan = cache.get(key)
        if plan is None:
            topo = Topology(self.topo.sizes, bw, self.topo.kinds, self.topo.latency_ns)
            plan = Plan(topo, coll, nbytes, n_chunks, policy, SCF if policy == THEMIS else FIFO)
            plan.bind(self, ctas_per_dim)
            cache[key] = plan
        return plan

    def _granule(self, n_chunks, dt):
        return self.P * (n_chunks or AUTO_MAX_CHUNKS) * (16 // ELEM_SIZE[dt])

    def all_reduce(self, tensors, n_chunks: int = 64, policy: int = THEMIS, bw_mbps=None,
                   ctas_per_dim: Optional[Sequence[int]] = None, stream=None):
        """All-Reduce user tensors in place: one tensor (V = 1) or a list of V
        tensors, one per local logical rank, same numel / dtype.

        Any numel (R17): the copy into the heap is zero-padded up to the
        executor's granule P·C·(16 B / elem), the collective runs on the
        padded buffer (zeros add nothing) and the first numel elements are
        copied back.  The copies are extra HBM traffic: latency-critical
        callers write into `rank_view` and call `themis_allreduce` directly.
        """
        import torch
        ts, dt, n = self._tensors(tensors)
        if n == 0:                                   # nothing to reduce (every rank must agree: same numel)
            return tensors
        g = self._granule(n_chunks, dt)             # 0 = auto: every candidate fits
        count = max(g, (n + g - 1) // g * g)
        plan = self._plan(ALLREDUCE, count * ELEM_SIZE[dt], n_chunks, policy, bw_mbps, ctas_per_dim)
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        with torch.cuda.stream(s):
            for v, t in enumerate(ts):
                view = self.rank_view(v, count, dt)
                view[:n].copy_(t.reshape(-1))
                if count > n:
                    view[n:].zero_()
            themis_allreduce(self.data_ptr, count, dt, plan, s)
            for v, t in enumerate(ts):
                t.copy_(self.rank_view(v, n, dt).view(t.shape))
        return tensors

    def reduce_scatter(self, tensors, n_chunks: int = 64, policy: int = THEMIS, bw_mbps=None,
                       ctas_per_dim: Optional[Sequence[int]] = None, stream=None) -> list:
        """Reduce-Scatter: V full-size inputs (numel a multiple of P·C·16 B /
        elem); returns, per local rank q, a new tensor holding block q of the
        sum (output block r at r·numel/P, R16)."""
        import torch
        ts, dt, n = self._tensors(tensors)
        if n % self._granule(n_chunks, dt):
            raise ThemisError(2, f"numel must be a multiple of {self._granule(n_chunks, dt)}")
        plan = self._plan(REDUCE_SCATTER, n * ELEM_SIZE[dt], n_chunks, policy, bw_mbps, ctas_per_dim)
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        blk = n // self.P
        with torch.cuda.stream(s):
            for v, t in enumerate(ts):
                self.rank_view(v, n, dt).copy_(t.reshape(-1))
            themis_reduce_scatter(self.data_ptr, n, dt, plan, s)
            out = []
            for v in range(self.V):
                q = self.gpu_rank * self.V + v
                out.append(self.rank_view(v, n, dt)[q * blk:(q + 1) * blk].clone())
        return out

    def all_gather(self, blocks, n_chunks: int = 64, policy: int = THEMIS, bw_mbps=None,
                   ctas_per_dim: Optional[Sequence[int]] = None, stream=None) -> list:
        """All-Gather: V per-rank blocks (numel m, m·P a multiple of P·C·16 B /
        elem); returns, per local rank, a new tensor of all P blocks in rank
        order."""
        import torch
        ts, dt, m = self._tensors(blocks)
        n = m * self.P
        if n % self._granule(n_chunks, dt):
            raise ThemisError(2, f"numel * P must be a multiple of {self._granule(n_chunks, dt)}")
        plan = self._plan(ALL_GATHER, n * ELEM_SIZE[dt], n_chunks, policy, bw_mbps, ctas_per_dim)
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        with torch.cuda.stream(s):
            for v, t in enumerate(ts):
                q = self.gpu_rank * self.V + v
                self.rank_view(v, n, dt)[q * m:(q + 1) * m].copy_(t.reshape(-1))
            themis_all_gather(self.data_ptr, n, dt, plan, s)
            out = [self.rank_view(v, n, dt).clone() for v in range(self.V)]
        return out

    def close(self):
        for p in self.__dict__.pop("_plans", {}).values():
            p.close()
        if getattr(self, "h", None):
            lib().themis_comm_free(self.h)      # also unbinds any plan still bound to it
            self.h = None
            for p in self.imported:
                lib().themis_heap_close(p)
            self.imported = []
            if self._symm is None:
                lib().themis_heap_free(self.heap)
            self._symm = None                    # torch frees the symmetric buffer
            self.heap = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream_ptr(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def themis_allreduce(buf: int, count: int, dtype: str, plan: Plan, stream=None) -> None:
    check(lib().themis_allreduce(buf, count, DTYPES[dtype], plan.h, _stream_ptr(stream)))


def themis_reduce_scatter(buf: int, count: int, dtype: str, plan: Plan, stream=None) -> None:
    check(lib().themis_reduce_scatter(buf, count, DTYPES[dtype], plan.h, _stream_ptr(stream)))


def themis_all_gather(buf: int, count: int, dtype: str, plan: Plan, stream=None) -> None:
    check(lib().themis_all_gather(buf, count, DTYPES[dtype], plan.h, _stream_ptr(stream)))


def themis_allreduce_host(host_in: int, host_out: int, buf: int, count: int, dtype: str, plan: Plan,
                          stream=None) -> None:
    check(lib().themis_allreduce_host(host_in, host_out, buf, count, DTYPES[dtype], plan.h, _stream_ptr(stream)))


def run(coll: int, comm: Comm, plan: Plan, count: int, dtype: str, stream=None) -> None:
    """Enqueue `coll` on the comm's data region (local rank 0 at comm.data_ptr)."""
    fn = {ALLREDUCE: themis_allreduce, REDUCE_SCATTER: themis_reduce_scatter, ALL_GATHER: themis_all_gather}[coll]
    fn(comm.data_ptr, count, dtype, plan, stream)


def default_ctas(bw: Sequence[int], total: int) -> list:
    """CTA caps per dimension proportional to bandwidth — the bandwidth-
    emulation knob (north_star (d)): themis_default_ctas."""
    t = Topology(tuple([2] * len(bw)), tuple(int(b) for b in bw)).to_c()
    out = (C.c_int32 * MAX_DIMS)()
    check(lib().themis_default_ctas(C.byref(t), int(total), out))
    return list(out[:len(bw)])


def launches_per_call() -> int:
    return lib().themis_launches_per_call()


def version() -> str:
    return lib().themis_version().decode()


__all__ = ["Topology", "Plan", "Comm", "themis_plan", "themis_allreduce", "themis_reduce_scatter",
           "themis_all_gather", "themis_allreduce_host", "run", "heap_layout", "default_ctas", "ThemisError",
           "RING", "DIRECT", "SWITCH", "NVLS", "ALLREDUCE", "REDUCE_SCATTER", "ALL_GATHER", "BASELINE", "THEMIS", "SCF",
           "FIFO", "SCF_LITERAL", "DTYPES", "ELEM_SIZE"]
