"""Greedy gap of Algorithm 1.

For small chunk counts, enumerate every reversed-AG assignment ((D!)^C; and
the full (D! x D!)^C space where it is small) through the C++ planner's
pre-simulation (`themis_plan_custom`, bit-exact against the oracle's engine,
`tests/test_planner_parity.py::test_custom_orders_full_space`) and compare
the optimum with Themis's greedy schedule and the fixed baseline.  Writes a
markdown table to stdout.  (Round 1 ran the same enumeration on the oracle;
analysis tools now use the product planner -- the oracle is test
infrastructure only.)

    python scripts/greedy_gap.py > profiles/r02_greedy_gap.md
"""

import itertools
import os
import sys
import time
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402

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


def makespan(plan) -> Fraction:
    try:
        return plan.makespan_ns()
    finally:
        plan.close()


def main():
    print("# Greedy gap of Algorithm 1\n")
    print("`scripts/greedy_gap.py`: every assignment of the given space through the C++ planner's")
    print("pre-simulation (SCF; FIFO for the baseline), optimum vs Themis's greedy and the fixed baseline.\n")
    print("| topology, BW | C | space | assignments | optimum | Themis | baseline | Themis / opt | baseline / opt |")
    print("|---|---|---|---|---|---|---|---|---|")
    for name, sizes, bw, nbytes, C, full in CASES:
        topo = th.Topology(sizes, tuple(b * 1000 for b in bw))
        D = len(sizes)
        t0 = time.time()
        perms = list(itertools.permutations(range(D)))
        chunk_choices = [(r, a) for r in perms for a in perms] if full else [(r, tuple(reversed(r))) for r in perms]
        opt, n = None, 0
        for assign in itertools.product(chunk_choices, repeat=C):
            rs = [r for r, _ in assign]
            ag = [a for _, a in assign]
            m = makespan(th.Plan(topo, th.ALLREDUCE, nbytes, C, th.THEMIS, th.SCF, rs_orders=rs, ag_orders=ag))
            opt = m if opt is None or m < opt else opt
            n += 1
        tm = makespan(th.Plan(topo, th.ALLREDUCE, nbytes, C, th.THEMIS, th.SCF))
        bl = makespan(th.Plan(topo, th.ALLREDUCE, nbytes, C, th.BASELINE, th.FIFO))
        space = "(D! x D!)^C" if full else "(D!)^C reversed AG"
        print(f"| {name} | {C} | {space} | {n} | {float(opt):.4g} | {float(tm):.4g} | {float(bl):.4g} | "
              f"{float(tm / opt):.4f} | {float(bl / opt):.4f} |", flush=True)
        print(f"<!-- {time.time() - t0:.1f} s -->", file=sys.stderr)
    print("\nTimes in ns (bytes / (GB/s)).  Themis / opt = 1 means the greedy found an optimal schedule; > 1 is")
    print("the greedy gap the paper accepts for O(C*D log D) planning (PAPER.md:430).")


if __name__ == "__main__":
    main()
