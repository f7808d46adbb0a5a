"""Baseline schedule and Themis Algorithm 1 (oracle; test infrastructure).

Followed step by step, in the paper's order and notation:

PAPER.md:258-268 (§2.3) — baseline: RS stages dim1 -> dimD, then AG stages
dimD -> dim1, identical for every chunk; RS-only / AG-only collectives run only
the corresponding half (:268 footnote).

PAPER.md:365-407 (Algorithm 1):
  SCHEDULE_COLLECTIVE(CT, CS, CPC):
    2  DimLoadTracker.reset(CT)                 -> loads seeded with A_K (:479)
    3  ChunkSize = CS / CPC
    5  for each chunk:
    6-9   if CT == AR: RS_Sch = SCHEDULER.SCHEDULE(RS, ChunkSize);
                       AG_Sch = reverseOrder(RS_Sch); Schedule = RS_Sch ++ AG_Sch
   10-11  else Schedule = SCHEDULER.SCHEDULE(CT, ChunkSize)
  SCHEDULER.SCHEDULE(CT, ChunkSize):
   18  loads = DimLoadTracker.getLoads()
   19  if loads.max - loads.min < Threshold: baseline order          (:392)
   21-26 else RS: dims sorted by load ascending; AG: descending      (:395-399)
   28-30 newLoad = LatencyModel.calcLoads(chunkSize, schedule, CT);
         DimLoadTracker.update(newLoad)                               (:401-403)
PAPER.md:614 — Threshold = latency-model runtime of an RS/AG of size
chunkSize/16 on the dimension with the lowest current load.
PAPER.md:489 — the Latency Model's load of chunk i on dimK is n_K^i x B_K.

Readings where the paper is silent (R1-R4, R8):
  R1  for AR the tracker is charged with the RS walk AND the AG walk;
  R2  threshold probe = volume ((P_m-1)/P_m) * chunk/div on m = argmin(L_k, k),
      compared with strict '<' (:392);
  R3  sort ties: stable by (load, dim index); AG-only "descending" = reverse of
      the ascending sort (equal loads reproduce the baseline AG order D->1);
  R4  AG-only ChunkSize is the gathered size; its first stage holds chunk/P;
  R8  the tracker is reset per collective (per plan).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .collectives import AG, RS, chunk_load, fixed_delay, fused_bytes_sent, fused_delay, is_fused, size_after
from .topology import NVLS, Topology

AR = "AR"
BASELINE, THEMIS = "baseline", "themis"


@dataclass(frozen=True)
class ChunkSchedule:
    chunk: int
    rs: tuple            # RS dim order (0-based); () for AG-only
    ag: tuple            # AG dim order (0-based); () for RS-only

    def stages(self):
        """[(dim, phase)] in execution order (RS stages then AG stages)."""
        return [(d, RS) for d in self.rs] + [(d, AG) for d in self.ag]


@dataclass
class Schedule:
    topo: Topology
    coll: str
    total_bytes: Fraction
    n_chunks: int
    chunks: list            # [ChunkSchedule]
    loads: list             # final Dim Load Tracker (ns)
    n_greedy: int           # chunks that took the sorted (non-baseline) order

    @property
    def chunk_bytes(self) -> Fraction:
        return self.total_bytes / self.n_chunks


def tracker_reset(topo: Topology, coll: str) -> list:
    """DimLoadTracker.reset(CT): each load starts at A_K of the phases the
    collective will run (reading R7)."""
    phases = {AR: (RS, AG), RS: (RS,), AG: (AG,)}[coll]
    return [fused_delay(d) if coll == AR and d.kind == NVLS else
            sum((fixed_delay(d, ph) for ph in phases), Fraction(0)) for d in topo.dims]    # R29


def baseline_order(topo: Topology, ct: str) -> tuple:
    """getBaselineScheduling(CT): RS dim1..dimD; AG dimD..dim1."""
    D = topo.D
    return tuple(range(D)) if ct == RS else tuple(reversed(range(D)))


def walk_loads(topo: Topology, ct: str, order, bytes_before) -> tuple:
    """LatencyModel.calcLoads: per-dim increments n_K^i * B_K walking the
    chunk through `order`, the chunk size changing by P_k after each stage
    (PAPER.md:221, :281).  Returns (increments, bytes after the walk)."""
    inc = [Fraction(0)] * topo.D
    b = Fraction(bytes_before)
    for d in order:
        dim = topo.dims[d]
        inc[d] += chunk_load(dim, ct, b)
        b = size_after(ct, dim.size, b)
    return inc, b


def ar_walk(topo: Topology, rs, ag, chunk) -> list:
    """An All-Reduce chunk's tracker increments: the RS walk then the AG walk
    (R1); on an NVLS dim the last RS + first AG stage is one in-switch
    All-Reduce of n = (1 + 1/p) b bytes (R29)."""
    if is_fused(topo, AR, rs, ag):
        inc_rs, b = walk_loads(topo, RS, rs[:-1], chunk)
        k = rs[-1]
        inc_rs[k] += fused_bytes_sent(topo.dims[k].size, b) / topo.dims[k].bw
        inc_ag, _ = walk_loads(topo, AG, ag[1:], b)
    else:
        inc_rs, b = walk_loads(topo, RS, rs, chunk)
        inc_ag, _ = walk_loads(topo, AG, ag, b)
    return [x + y for x, y in zip(inc_rs, inc_ag)]


def threshold(topo: Topology, loads, chunk_bytes, threshold_div) -> Fraction:
    """runtime of an RS/AG of chunkSize/16 on the min-load dim.
    An RS of X bytes and an AG gathering X bytes send the same volume
    ((P-1)/P) X, so the probe is phase independent (reading R2)."""
    m = min(range(topo.D), key=lambda k: (loads[k], k))
    return chunk_load(topo.dims[m], RS, Fraction(chunk_bytes) / threshold_div)


def scheduler_schedule(topo: Topology, ct: str, loads, chunk_bytes, threshold_div) -> tuple:
    """SCHEDULER.SCHEDULE(CT, ChunkSize) lines 18-27: pick this chunk's order
    (the tracker update is done by the caller, lines 28-30)."""
    if max(loads) - min(loads) < threshold(topo, loads, chunk_bytes, threshold_div):
        return baseline_order(topo, ct), False
    asc = tuple(sorted(range(topo.D), key=lambda k: (loads[k], k)))
    if ct == RS:
        return asc, True
    return tuple(reversed(asc)), True          # AG: descending (reading R3)


def schedule_collective(topo: Topology, coll: str, total_bytes, n_chunks: int,
                        policy: str = THEMIS, threshold_div=16) -> Schedule:
    """SCHEDULE_COLLECTIVE(CT, CS, CPC) (Algorithm 1 lines 1-14), or the
    baseline schedule when policy == 'baseline'.  The tracker is run for the
    baseline too so its final loads can be compared."""
    if n_chunks < 1:
        raise ValueError("n_chunks >= 1")
    topo.validate()
    S = Fraction(total_bytes)
    chunk = S / n_chunks                                    # line 3
    loads = tracker_reset(topo, coll)                       # line 2
    out, n_greedy = [], 0
    for i in range(n_chunks):                               # line 5
        if coll == AR:
            if policy == THEMIS:
                rs, greedy = scheduler_schedule(topo, RS, loads, chunk, threshold_div)
            else:
                rs, greedy = baseline_order(topo, RS), False
            ag = tuple(reversed(rs))                        # line 8
            inc = ar_walk(topo, rs, ag, chunk)              # reading R1 (+ R29)
            cs = ChunkSchedule(i, rs, ag)
        else:
            if policy == THEMIS:
                order, greedy = scheduler_schedule(topo, coll, loads, chunk, threshold_div)
            else:
                order, greedy = baseline_order(topo, coll), False
            first = chunk if coll == RS else chunk / topo.P  # reading R4
            inc, _ = walk_loads(topo, coll, order, first)
            cs = ChunkSchedule(i, order, ()) if coll == RS else ChunkSchedule(i, (), order)
        loads = [l + x for l, x in zip(loads, inc)]         # line 30
        n_greedy += int(greedy)
        out.append(cs)
    return Schedule(topo, coll, S, n_chunks, out, loads, n_greedy)


def dim_volumes(sched: Schedule) -> list:
    """N_K = sum_i n_K^i: bytes each NPU sends on each dim."""
    topo = sched.topo
    N = [Fraction(0)] * topo.D
    chunk = sched.chunk_bytes
    for cs in sched.chunks:
        b = chunk if cs.rs else chunk / topo.P
        fused = is_fused(topo, sched.coll, cs.rs, cs.ag)
        for i, (d, ph) in enumerate(cs.stages()):
            p = topo.dims[d].size
            if fused and i == len(cs.rs) - 1:            # the in-switch pair (R29)
                N[d] += fused_bytes_sent(p, b)
            elif fused and i == len(cs.rs):
                pass
            else:
                N[d] += Fraction(p - 1, p) * b if ph == RS else (p - 1) * b
            b = size_after(ph, p, b)
    return N


def export_csv(sched: Schedule) -> str:
    """SPEC.md:298 export: `chunk_id, rs_order, ag_order, bytes` (1-based dims)."""
    lines = ["chunk_id,rs_order,ag_order,bytes"]
    for cs in sched.chunks:
        rs = " ".join(str(d + 1) for d in cs.rs)
        ag = " ".join(str(d + 1) for d in cs.ag)
        lines.append(f"{cs.chunk},{rs},{ag},{sched.chunk_bytes}")
    return "\n".join(lines) + "\n"
