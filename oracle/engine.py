"""Deterministic pre-simulation / event engine (oracle; test infrastructure).

PAPER.md:530 — "once Inter-Dimension Schedules are determined, Themis simulates
their execution to get an estimation of when each chunk operation will be
available on each dimension ... enforces this intra-dimension ordering";
:532 — the simulation is deterministic, so all NPUs produce the same order.
PAPER.md:450-459 (§4.3) — intra-dimension policy: FIFO, or Smallest-Chunk-First.
PAPER.md:281 — chunks are fed through the 2D-stage pipeline; a chunk's next
stage starts after its previous stage.
PAPER.md:464-471 — Latency(dimK) = A_K + N_K*B_K + idle_K.
PAPER.md:292 — average BW utilisation = BW-weighted average of per-dim
utilisation.  Table 3 (:551) — Ideal.

Model (readings R9-R14):
  * one server per dimension, one op at a time (R12); every chunk's first
    stage is ready at t = 0;
  * op duration = volume * B_K (+ A_K(phase) only if charge_latency, F5);
  * at each time t all completions are processed first (the successor becomes
    ready at t), then every idle dim starts its best ready op (R11);
  * FIFO key (ready, chunk) (R10); SCF key (volume on that dim, ready, chunk)
    (R9); 'scf_literal' key (bytes_before, chunk);
  * idle_K = time dim K is idle before its last op completes, so
    finish_K = busy_K + idle_K exactly and makespan = max_K finish_K;
  * util = sum BW_K busy_K / (sum BW * makespan) (R14);
  * Ideal = algorithmic bytes / sum BW (R13): 2S(P-1)/P for AR.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

from .collectives import AG, RS, bytes_sent, fixed_delay, fused_bytes_sent, fused_delay, is_fused, size_after
from .scheduler import AR, Schedule

FIFO, SCF, SCF_LITERAL = "fifo", "scf", "scf_literal"


@dataclass(frozen=True)
class Op:
    chunk: int
    stage: int
    dim: int
    phase: str
    bytes_before: Fraction
    volume: Fraction          # n_K^i
    duration: Fraction


@dataclass
class RunMetrics:
    makespan: Fraction
    busy: list
    idle: list
    finish: list
    volume: list                                   # N_K
    dim_order: list                                # per dim [(chunk, stage)]
    start: dict = field(default_factory=dict)      # (chunk, stage) -> start
    end: dict = field(default_factory=dict)        # (chunk, stage) -> end
    util: Fraction = Fraction(0)
    global_order: list = field(default_factory=list)  # [(chunk, stage)] by (start, dim)


def chunk_ops(sched: Schedule, charge_latency: bool = False, servers: int = 1) -> list:
    """Per chunk, its ops in stage order (size before each stage).
    With `servers` parallel servers per dim each has BW_K / servers."""
    topo = sched.topo
    out = []
    for cs in sched.chunks:
        b = sched.chunk_bytes if cs.rs else sched.chunk_bytes / topo.P
        fused = is_fused(topo, sched.coll, cs.rs, cs.ag)
        ops = []
        for s, (d, ph) in enumerate(cs.stages()):
            dim = topo.dims[d]
            if fused and s == len(cs.rs) - 1:       # in-switch RS+AG pair (R29)
                v = fused_bytes_sent(dim.size, b)
                dur = v / dim.bw * servers + (fused_delay(dim) if charge_latency else 0)
            elif fused and s == len(cs.rs):         # its AG half: dependency only
                v, dur = Fraction(0), Fraction(0)
            else:
                v = bytes_sent(ph, dim.size, b)
                dur = v / dim.bw * servers + (fixed_delay(dim, ph) if charge_latency else 0)
            ops.append(Op(cs.chunk, s, d, ph, b, v, dur))
            b = size_after(ph, dim.size, b)
        out.append(ops)
    return out


def _key(policy: str, op: Op, ready):
    if policy == FIFO:
        return (ready, op.chunk)
    if policy == SCF:
        return (op.volume, ready, op.chunk)
    if policy == SCF_LITERAL:
        return (op.bytes_before, op.chunk)
    raise ValueError(policy)


def simulate(sched: Schedule, policy: str = SCF, charge_latency: bool = False,
             enforced=None, servers: int = 1, enforced_server=None, release=0) -> RunMetrics:
    """Run the chunk pipelines.  With `enforced` (per-dim [(chunk, stage)]),
    each dim must start its ops in exactly that order (the runtime contract,
    PAPER.md:530); raises RuntimeError on deadlock.

    servers > 1 generalises R12 to PAPER.md:461/:491 ("multiple chunks per
    dimension should be run in parallel"): each dim is `servers` parallel
    servers with BW_K / servers each (an op takes volume*B_K*servers); idle
    servers, in index order, each start the best ready op; m.server records
    which server ran each op.  With enforced_server ((chunk, stage) ->
    server), each server replays its own sub-list of `enforced` in order.

    release > 0 (extension, R26): chunk c's first stage becomes
    ready at (c+1)*release instead of 0 (chunks streamed in from the host);
    arrivals at t are processed after the completions at t and before the
    starts."""
    topo = sched.topo
    D = topo.D
    ops = chunk_ops(sched, charge_latency, servers)
    total = sum(len(o) for o in ops)
    queue = [dict() for _ in range(D)]          # (chunk, stage) -> ready time
    release = Fraction(release)
    arrivals = [(release * (c + 1), c) for c, o in enumerate(ops) if o]   # ready time of stage 0
    nxt_arrival = 0
    running = [[None] * servers for _ in range(D)]   # (chunk, stage, end)
    lists = None
    if enforced is not None:
        es = enforced_server or {}
        lists = [[[tuple(cs) for cs in enforced[k] if es.get(tuple(cs), 0) == sv] for sv in range(servers)]
                 for k in range(D)]
    pos = [[0] * servers for _ in range(D)]
    m = RunMetrics(Fraction(0), [Fraction(0)] * D, [Fraction(0)] * D, [Fraction(0)] * D,
                   [Fraction(0)] * D, [[] for _ in range(D)])
    m.server = {}
    t = Fraction(0)
    done = 0
    while done < total:
        while nxt_arrival < len(arrivals) and arrivals[nxt_arrival][0] <= t:   # arrivals at time t
            r, c = arrivals[nxt_arrival]
            queue[ops[c][0].dim][(c, 0)] = r
            nxt_arrival += 1
        for k in range(D):                      # starts at time t
            for sv in range(servers):
                if running[k][sv] is not None or not queue[k]:
                    continue
                if lists is not None:
                    if pos[k][sv] >= len(lists[k][sv]):
                        continue
                    nxt = lists[k][sv][pos[k][sv]]
                    if nxt not in queue[k]:
                        continue
                    pick = nxt
                    pos[k][sv] += 1
                else:
                    pick = min(queue[k], key=lambda cs: _key(policy, ops[cs[0]][cs[1]], queue[k][cs]))
                del queue[k][pick]
                op = ops[pick[0]][pick[1]]
                running[k][sv] = (pick[0], pick[1], t + op.duration)
                m.start[pick] = t
                m.server[pick] = sv
                m.dim_order[k].append(pick)
                m.global_order.append(pick)
                m.busy[k] += op.duration / servers
                m.volume[k] += op.volume
        ends = [r[2] for rk in running for r in rk if r is not None]
        if nxt_arrival < len(arrivals):
            ends.append(arrivals[nxt_arrival][0])
        if not ends:
            raise RuntimeError("deadlock: no op running and unfinished ops remain")
        t = min(ends)
        for k in range(D):                      # completions at time t
            for sv in range(servers):
                r = running[k][sv]
                if r is None or r[2] != t:
                    continue
                c, s, _ = r
                running[k][sv] = None
                m.end[(c, s)] = t
                m.finish[k] = t
                done += 1
                if s + 1 < len(ops[c]):
                    queue[ops[c][s + 1].dim][(c, s + 1)] = t
    m.makespan = max(m.finish)
    m.idle = [f - b for f, b in zip(m.finish, m.busy)]
    tb = topo.total_bw
    m.util = sum((d.bw * b for d, b in zip(topo.dims, m.busy)), Fraction(0)) / (tb * m.makespan)
    return m


def ideal_time(sched: Schedule) -> Fraction:
    """Volume-based Ideal (reading R13): algorithmic bytes per NPU / sum BW
    of the host-driven algorithms (a lower bound only without NVLS dims,
    whose in-switch pairs send less, R29)."""
    topo = sched.topo
    f = Fraction(topo.P - 1, topo.P) * sched.total_bytes
    if sched.coll == AR:
        f *= 2
    return f / topo.total_bw


def activity_rate(m: RunMetrics, sched: Schedule, window) -> list:
    """Fig 7: per dim, the fraction of each window during which
    the dim has an op in service."""
    window = Fraction(window)
    nwin = max(1, -(-m.makespan // window))
    out = []
    for k in range(sched.topo.D):
        iv = [(m.start[cs], m.end[cs]) for cs in m.dim_order[k]]
        row = []
        for w in range(int(nwin)):
            a, b = w * window, min((w + 1) * window, m.makespan)
            cov = sum((max(Fraction(0), min(b, e) - max(a, s)) for s, e in iv), Fraction(0))
            row.append(cov / (b - a))
        out.append(row)
    return out


def choose_chunks(topo, coll: str, total_bytes: int, policy: str, intra: str = SCF, charge_latency: bool = False,
                  servers: int = 1, max_chunks: int = 256, threshold_div: int = 16):
    """Chunk count chosen by the pre-simulation (extension of the CPC
    parameter; R25): among C = 1, 2, 4, ..., max_chunks
    with total_bytes % (P * C * 16) == 0, plan each (Algorithm 1 + this engine)
    and keep the smallest makespan; ties keep the smaller C.  Returns
    (C, schedule, metrics), or None when no candidate divides the buffer."""
    from .scheduler import schedule_collective
    best = None
    C = 1
    while C <= max_chunks:
        if total_bytes % (topo.P * C * 16) == 0:
            sched = schedule_collective(topo, coll, total_bytes, C, policy, threshold_div)
            m = simulate(sched, intra, charge_latency, servers=servers)
            if best is None or m.makespan < best[2].makespan:
                best = (C, sched, m)
        C *= 2
    return best
