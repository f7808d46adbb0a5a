"""Greedy gap of Algorithm 1.

Calls only `oracle/` (test infrastructure): for small chunk counts, enumerate
every reversed-AG assignment ((D!)^C; and the full (D! x D!)^C space where it
is small), run each through the same pre-simulation and intra-dimension
policy, and compare the optimum with Themis's greedy schedule and the
baseline.  Writes a markdown table to stdout.

    python scripts/greedy_gap.py > profiles/r01_greedy_gap.md
"""

import os
import sys
import time
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import brute as B, engine as E, scheduler as S, topology as T  # noqa: E402

CASES = [  # (name, sizes, bw GB/s, bytes, C, full-space?)
    ("2x2x2 1:1:1", (2, 2, 2), (100, 100, 100), 1 << 30, 4, False),
    ("2x2x2 1:1:1", (2, 2, 2), (100, 100, 100), 1 << 30, 5, False),
    ("2x2x2 2:2:1", (2, 2, 2), (200, 200, 100), 1 << 30, 5, False),
    ("2x2x2 4:2:1", (2, 2, 2), (400, 200, 100), 1 << 30, 5, False),
    ("4x2 1:1", (4, 2), (100, 100), 1 << 30, 8, False),
    ("2x4 1:1", (2, 4), (100, 100), 1 << 30, 8, False),
    ("4x2 200:50", (4, 2), (200, 50), 1 << 30, 8, False),
    ("4x2 7:3", (4, 2), (7, 3), 1 << 30, 2, True),
    ("4x2 1:1", (4, 2), (100, 100), 1 << 30, 5, True),
    ("4x4 2:1 (Fig 3)", (4, 4), (2, 1), 256 << 20, 4, True),
]


def main():
    print("# Greedy gap of Algorithm 1 (round 1)\n")
    print("`scripts/greedy_gap.py` (oracle only): every assignment of the given space through the same")
    print("pre-simulation (SCF; FIFO for the baseline), optimum vs Themis's greedy and the fixed baseline.\n")
    print("| topology, BW | C | space | assignments | optimum | Themis | baseline | Themis / opt | baseline / opt |")
    print("|---|---|---|---|---|---|---|---|---|")
    for name, sizes, bw, nbytes, C, full in CASES:
        t = T.Topology.make(sizes, [Fraction(b) for b in bw])
        t0 = time.time()
        opt, _, n = B.exhaustive_best(t, S.AR, nbytes, C, E.SCF, full=full, cap=2 * 10 ** 6)
        th = E.simulate(S.schedule_collective(t, S.AR, nbytes, C, S.THEMIS), E.SCF).makespan
        bl = E.simulate(S.schedule_collective(t, S.AR, nbytes, C, S.BASELINE), E.FIFO).makespan
        space = "(D! x D!)^C" if full else "(D!)^C reversed AG"
        print(f"| {name} | {C} | {space} | {n} | {float(opt):.4g} | {float(th):.4g} | {float(bl):.4g} | "
              f"{float(th / opt):.4f} | {float(bl / opt):.4f} |", flush=True)
        print(f"<!-- {time.time() - t0:.1f} s -->", file=sys.stderr)
    print("\nTimes in the oracle's units (bytes / (GB/s) = ns).  Themis / opt = 1 means the greedy found an")
    print("optimal schedule; > 1 is the greedy gap the paper accepts for O(C*D log D) planning (PAPER.md:430).")


if __name__ == "__main__":
    main()
