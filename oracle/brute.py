"""Exhaustive schedule search for tiny instances (oracle; test infrastructure).

PAPER.md:420-430 (Observations 1-2): any RS order and any AG order per chunk
is valid (D! x D! per chunk), and chunks are scheduled independently, so the
space is (D! x D!)^C for AR (D!^C for RS/AG).  Themis restricts AG to
reverse(RS) (Algorithm 1 line 8), giving (D!)^C.  Every candidate is run
through the same engine and intra-dimension policy; the minimum makespan is
the optimum the greedy is compared with.
"""

from __future__ import annotations

import itertools
from fractions import Fraction

from .engine import SCF, simulate
from .scheduler import AR, ChunkSchedule, Schedule


def space_size(D: int, C: int, coll: str = AR, full: bool = False) -> int:
    f = 1
    for i in range(2, D + 1):
        f *= i
    per = f * f if (coll == AR and full) else f
    return per ** C


def candidates(topo, coll: str, C: int, full: bool = False):
    perms = list(itertools.permutations(range(topo.D)))
    if coll == AR:
        per = [(p, q) for p in perms for q in perms] if full else [(p, tuple(reversed(p))) for p in perms]
    elif coll == "RS":
        per = [(p, ()) for p in perms]
    else:
        per = [((), p) for p in perms]
    return itertools.product(per, repeat=C)


def exhaustive_best(topo, coll: str, total_bytes, C: int, policy: str = SCF,
                    full: bool = False, cap: int = 10 ** 6, charge_latency: bool = False):
    """Returns (best makespan, best assignment, number enumerated)."""
    n = space_size(topo.D, C, coll, full)
    if n > cap:
        raise ValueError(f"space {n} exceeds cap {cap}")
    best, arg, count = None, None, 0
    for assign in candidates(topo, coll, C, full):
        chunks = [ChunkSchedule(i, rs, ag) for i, (rs, ag) in enumerate(assign)]
        sched = Schedule(topo, coll, Fraction(total_bytes), C, chunks, [], 0)
        m = simulate(sched, policy, charge_latency)
        count += 1
        if best is None or m.makespan < best:
            best, arg = m.makespan, assign
    return best, arg, count
