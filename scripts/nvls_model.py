"""In-network offload in the latency model (DESIGN R29):
planner-only comparison on the paper's 1024-NPU Table-2 topologies.

For every preset, every Switch dimension is modelled either as a plain switch
(halving-doubling, R7/R23) or as an NVLS-style reducing switch (the chunk's
last-RS / first-AG pair fused into one op of (1 + 1/P_k) x bytes, R29).
Baseline and Themis orders, SCF intra-dim order, 64 chunks, 100 MB and 1 GB
All-Reduces, the paper's model (Table-2 step latencies seed the Dim Load
Tracker, no per-op charge: F5, the setting that reproduces the paper's
microbenchmark averages).  Reports the pre-simulated makespans and Themis's
speedup -- the paper's claim that Themis still balances the dimensions when a
dimension offloads its collective.

    python scripts/nvls_model.py > profiles/r02_nvls_model.md
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_04478_b200 import themis as th  # noqa: E402


def plan_ms(topo, nbytes, policy):
    p = th.Plan(topo, th.ALLREDUCE, nbytes, 64, policy, th.SCF)   # A_K seeds the tracker only (F5)
    try:
        return float(p.makespan_ns()) * 1e-6, p.info["n_greedy"]
    finally:
        p.close()


def main():
    print("# In-network offload (NVLS-style switch dims) in the Themis latency model\n")
    print("Planner only (`scripts/nvls_model.py`, the C++ planner; R29 bit-exact against the oracle in "
          "`tests/test_planner_parity.py::test_nvls_algorithm_row`).  PAPER.md Table 2 topologies, 1024 NPUs, "
          "64 chunks, SCF, the paper's model (Table-2 step latencies seed the tracker; no per-op charge, F5).  "
          "`switch`: every Switch dim runs "
          "halving-doubling RS / AG; `nvls`: every Switch dim fuses each chunk's last-RS / first-AG pair "
          "into one in-switch op ((1 + 1/P_k) x bytes, 2 latency steps).  Speedup = baseline / Themis makespan.\n")
    print("| topology | size | switch dims as | baseline ms | Themis ms | Themis speedup | greedy chunks |")
    print("|---|---|---|---|---|---|---|")
    for name, t in th.TABLE2.items():
        for mb in (100, 1000):
            nbytes = mb * 10 ** 6 // (t.P * 64 * 16) * (t.P * 64 * 16) or t.P * 64 * 16
            for mode in ("switch", "nvls"):
                kinds = tuple(th.NVLS if (mode == "nvls" and k == th.SWITCH) else k for k in t.kinds)
                if mode == "nvls" and kinds == t.kinds:
                    continue                          # no switch dim to offload
                topo = th.Topology(t.sizes, t.bw_mbps, kinds, t.latency_ns)
                b, _ = plan_ms(topo, nbytes, th.BASELINE)
                m, g = plan_ms(topo, nbytes, th.THEMIS)
                print(f"| {name} | {mb} MB | {mode} | {b:.3f} | {m:.3f} | {b / m:.3f} | {g}/64 |")
    print("\nWith the fused in-switch pairs Themis keeps its gain (1.53-2.79x here) and mostly grows it "
          "(2D-SW_SW 1 GB 1.53 -> 1.59x, 4D-Ring_SW_SW_SW 1 GB 1.66 -> 1.76x): the offload makes the switch "
          "dims cheaper per byte, the baseline order cannot use that (its bottleneck stays dim1), Algorithm 1 "
          "shifts load onto them -- PAPER.md:493-494's point that offload and Themis compose.  Where the "
          "offload dim already carries little (3D-FC_Ring_SW, 4D-Ring_FC_Ring_SW at 1 GB) the greedy "
          "choices shift slightly and the gain moves by ~1-2 % either way.")


if __name__ == "__main__":
    main()
