"""All-Reduce / Reduce-Scatter / All-Gather over P simulated ranks in host memory
(oracle; test infrastructure).

Plain definitions the method must reach (figure
`CollectiveOperations` :212):
  AR  every rank ends with sum_r x_r (elementwise);
  RS  rank r ends with block r of sum_r x_r ("each NPU holds a portion");
  AG  every rank ends with the concatenation of all ranks' block r.
See ``allreduce_definition`` etc.  Integer sums wrap mod 2^32 (reading R19).

Step-by-step execution of a schedule (PAPER.md:258-268 hierarchical stages;
per-chunk orders from Algorithm 1), with the data layout the paper leaves open
(reading R16 / SURVEY F9):
  * block b = elements [b*N/P, (b+1)*N/P) — block index in mixed radix with
    dim1 fastest, digit_k(b) = floor(b / prod_{i<k} P_i) mod P_k;
  * chunk c = the c-th 1/C slice of every block (strided chunks);
  * a rank's held set for a chunk = blocks whose digit_d equals the rank's
    coordinate c_d on every dim d currently reduce-scattered;
  * RS(c, k): inside each dim-k group, member t keeps the held blocks with
    digit_k = t and stores sum_{j=0}^{P_k-1} x_{member j} over them, summed in
    coordinate order j (reading R18);
  * AG(c, k): member t copies, from every member j != t, j's held blocks
    (digit_k = j) into the same offsets.
After any RS order rank r holds exactly block r; AG is the exact inverse.

Float arithmetic (reading R18): 'f32' sums in float32, one add at a time in
coordinate order; 'bf16' / 'f16' accumulate in float32 and round once to
nearest-even at the end of each RS stage; 'i32' wraps; 'f64' is exact-ish
reference arithmetic.  bf16 values are carried as uint16 bit patterns.
"""

from __future__ import annotations

import numpy as np

from .collectives import AG, RS
from .scheduler import AR, Schedule

DTYPES = ("f32", "bf16", "f16", "i32", "f64")


# --- bf16 helpers (round-to-nearest-even, NaN kept quiet) --------------------
def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    nan = (b & np.uint32(0x7FFFFFFF)) > np.uint32(0x7F800000)
    lsb = (b >> np.uint32(16)) & np.uint32(1)
    r = ((b + np.uint32(0x7FFF) + lsb) >> np.uint32(16)).astype(np.uint16)
    r[nan] = ((b[nan] >> np.uint32(16)) | np.uint32(0x40)).astype(np.uint16)
    return r


def _np_dtype(dtype: str):
    return {"f32": np.float32, "bf16": np.uint16, "f16": np.float16,
            "i32": np.int32, "f64": np.float64}[dtype]


def reduce_hops(parts, dtype: str) -> np.ndarray:
    """Ring dims (R18): the executor sends ring messages in the buffer's dtype
    (a design choice of the executor — PAPER.md is silent on message
    precision; pinned against north_star's 1e-2 bound by
    test_ring_low_precision_within_north_star_bound), so the tree-exact mode
    rounds the partial after every hop:
    acc = parts[0]; acc = round(acc + parts[j]) for j = 1.. (fp32 adds)."""
    if dtype in ("f32", "i32", "f64"):
        return reduce_in_order(parts, dtype)       # storing the partial rounds nothing
    acc = parts[0]
    for p in parts[1:]:
        acc = reduce_in_order([acc, p], dtype)
    return acc


def reduce_in_order(parts, dtype: str) -> np.ndarray:
    """sum_j parts[j] in coordinate order j with the dtype's arithmetic."""
    if dtype == "f32":
        acc = parts[0].astype(np.float32, copy=True)
        for p in parts[1:]:
            acc = acc + p
        return acc
    if dtype == "bf16":
        acc = bf16_to_f32(parts[0]).copy()
        for p in parts[1:]:
            acc = acc + bf16_to_f32(p)
        return f32_to_bf16(acc)
    if dtype == "f16":
        acc = parts[0].astype(np.float32)
        for p in parts[1:]:
            acc = acc + p.astype(np.float32)
        return acc.astype(np.float16)
    if dtype == "i32":
        acc = parts[0].astype(np.int32, copy=True)
        with np.errstate(over="ignore"):
            for p in parts[1:]:
                acc = acc + p
        return acc
    if dtype == "f64":
        acc = parts[0].astype(np.float64, copy=True)
        for p in parts[1:]:
            acc = acc + p
        return acc
    raise ValueError(dtype)


# --- layout -----------------------------------------------------------------
def digit(topo, b: int, k: int) -> int:
    return (b // topo.stride(k)) % topo.dims[k].size


def held_blocks(topo, coords, reduced) -> list:
    """Blocks whose digit on every reduced dim equals the rank's coordinate."""
    return [b for b in range(topo.P) if all(digit(topo, b, d) == coords[d] for d in reduced)]


def slice_of(N: int, P: int, C: int, c: int, b: int) -> slice:
    blk = N // P
    sl = blk // C
    return slice(b * blk + c * sl, b * blk + (c + 1) * sl)


def _groups(topo, k):
    """All dim-k groups, each as the member ranks in coordinate order."""
    return [topo.dim_peers(r, k) for r in range(topo.P) if topo.coords(r)[k] == 0]


def ring_hops(topo, k) -> bool:
    """Table 1 ring dims with P_k >= 3 run the ring algorithm (P_k = 2 is direct)."""
    return topo.dims[k].kind == "ring" and topo.dims[k].size >= 3


def summation_order(topo, k, t) -> list:
    """Member order in which part t (digit_k = t) is summed on dim k.
    Direct / switch dims: coordinate order 0..P_k-1 (R18).  Ring dims
    (Table 1; figure RingAllReduce :214): the partial travels the
    ring and ends at its owner t, so it is x_{t+1} + x_{t+2} + ... + x_t."""
    pk = topo.dims[k].size
    if topo.dims[k].kind == "ring" and pk >= 3:
        return [(t + 1 + i) % pk for i in range(pk)]
    return list(range(pk))


def apply_rs(bufs, topo, C, c, k, reduced, dtype):
    N = bufs[0].shape[0]
    for members in _groups(topo, k):
        new = []
        for t, mt in enumerate(members):
            ct = topo.coords(mt)
            order = summation_order(topo, k, t)
            for b in held_blocks(topo, ct, reduced):
                if digit(topo, b, k) != t:
                    continue
                s = slice_of(N, topo.P, C, c, b)
                red = reduce_hops if ring_hops(topo, k) else reduce_in_order
                new.append((mt, s, red([bufs[members[j]][s] for j in order], dtype)))
        for mt, s, v in new:
            bufs[mt][s] = v


def apply_ag(bufs, topo, C, c, k, reduced, dtype):
    N = bufs[0].shape[0]
    rest = [d for d in reduced if d != k]
    for members in _groups(topo, k):
        for t, mt in enumerate(members):
            ct = topo.coords(mt)
            for j, mj in enumerate(members):
                if j == t:
                    continue
                for b in held_blocks(topo, ct, rest):
                    if digit(topo, b, k) != j:
                        continue
                    s = slice_of(N, topo.P, C, c, b)
                    bufs[mt][s] = bufs[mj][s]


def run_schedule(inputs, sched: Schedule, dtype: str, order=None):
    """Execute `sched` on copies of `inputs` (one array per rank, N elements).
    `order`: global op order [(chunk, stage)] (e.g. RunMetrics.global_order);
    default = chunk by chunk.  Any order consistent with each chunk's stage
    chain gives the same result (chunks touch disjoint slices)."""
    topo = sched.topo
    C = sched.n_chunks
    P = topo.P
    N = inputs[0].shape[0]
    if len(inputs) != P:
        raise ValueError("one input per rank")
    if N % (P * C):
        raise ValueError("N must be a multiple of P*C")
    bufs = [np.array(x, dtype=_np_dtype(dtype), copy=True) for x in inputs]
    if order is None:
        order = [(cs.chunk, s) for cs in sched.chunks for s in range(len(cs.stages()))]
    reduced = {cs.chunk: (set() if cs.rs else set(range(topo.D))) for cs in sched.chunks}
    nxt = {cs.chunk: 0 for cs in sched.chunks}
    for c, s in order:
        if nxt[c] != s:
            raise ValueError("order violates the chunk's stage chain")
        nxt[c] += 1
        d, ph = sched.chunks[c].stages()[s]
        if ph == RS:
            apply_rs(bufs, topo, C, c, d, reduced[c], dtype)
            reduced[c].add(d)
        else:
            apply_ag(bufs, topo, C, c, d, reduced[c], dtype)
            reduced[c].discard(d)
    return bufs


def element_location(topo, N: int, C: int, i: int) -> tuple:
    """(block b, chunk c) of element i under the layout R16."""
    blk = N // topo.P
    b = i // blk
    c = (i % blk) // (blk // C)
    return b, c


def allreduce_element(vals, topo, rs_order, dtype: str, block: int):
    """All-Reduce result of ONE element position, computed directly from the
    stage structure: arrange the P ranks' values of the element on the
    P_1 x ... x P_D grid and reduce along the chunk's RS dims in `rs_order`,
    each axis in the dim's summation order (coordinate order; ring dims end at
    the owner digit of `block`), with the dtype's rounding per stage (per hop
    on ring dims, R18).
    AG only copies, so every rank ends with this value.  `vals[r]` is rank r's
    value (bf16 as uint16 bits).  Used to check full-size runs on samples."""
    P = topo.P
    grid = {}
    for r in range(P):
        grid[topo.coords(r)] = np.array([vals[r]], dtype=_np_dtype(dtype))
    live = dict(grid)
    for k in rs_order:
        t = digit(topo, block, k)
        order = summation_order(topo, k, t)
        nxt = {}
        for coords, _ in live.items():
            if coords[k] != 0:
                continue
            members = []
            for j in order:
                cc = list(coords)
                cc[k] = j
                members.append(live[tuple(cc)])
            out = list(coords)
            out[k] = t
            nxt[tuple(out)] = (reduce_hops if ring_hops(topo, k) else reduce_in_order)(members, dtype)
        # keep only the owner digit along k (the other digits are not held)
        live = {}
        for coords, v in nxt.items():
            for j in range(topo.dims[k].size):
                cc = list(coords)
                cc[k] = j
                live[tuple(cc)] = v
    return live[topo.coords(block)][0]


# --- plain definitions ------------------------------------------------------
def allreduce_definition(inputs, dtype: str) -> np.ndarray:
    """sum_r x_r: exact int64 sum wrapped mod 2^32 for i32; fp64 otherwise."""
    if dtype == "i32":
        s = np.sum(np.stack([x.astype(np.int64) for x in inputs]), axis=0)
        return ((s + 2 ** 31) % 2 ** 32 - 2 ** 31).astype(np.int32)
    if dtype == "bf16":
        inputs = [bf16_to_f32(x) for x in inputs]
    return np.sum(np.stack([x.astype(np.float64) for x in inputs]), axis=0)


def reduce_scatter_definition(inputs, dtype: str, P: int) -> list:
    s = allreduce_definition(inputs, dtype)
    blk = s.shape[0] // P
    return [s[r * blk:(r + 1) * blk] for r in range(P)]


def all_gather_definition(inputs, P: int) -> np.ndarray:
    blk = inputs[0].shape[0] // P
    return np.concatenate([inputs[r][r * blk:(r + 1) * blk] for r in range(P)])


def abs_sum(inputs, dtype: str) -> np.ndarray:
    """sum_r |x_r| in fp64 — the scale of the float error bound (reading R18)."""
    if dtype == "bf16":
        inputs = [bf16_to_f32(x) for x in inputs]
    return np.sum(np.stack([np.abs(x.astype(np.float64)) for x in inputs]), axis=0)


def to_f64(x: np.ndarray, dtype: str) -> np.ndarray:
    return bf16_to_f32(x).astype(np.float64) if dtype == "bf16" else x.astype(np.float64)
