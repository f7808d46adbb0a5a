"""Themis CPU oracle — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

A plain, slow, obviously-correct CPU implementation of what the Themis hot
path computes (arXiv 2110.04478, ``/root/reference/PAPER.md``):

* ``topology``    — P_1 x ... x P_D topologies (Table 2 :509-519)
* ``collectives`` — per-dimension step counts / volumes / size change
                    (PAPER.md:221, Table 1 :226-238, :475-487)
* ``scheduler``   — baseline order and Themis
                    Algorithm 1 with Dim Load Tracker, Latency Model and
                    Threshold
* ``engine``      — the deterministic pre-simulation that yields the
                    intra-dimension op order
                    plus the paper's utilisation metric
* ``brute``       — exhaustive search of the schedule space
                    
* ``data``        — an All-Reduce / Reduce-Scatter / All-Gather over P
                    simulated ranks in host memory

All time/byte arithmetic uses ``fractions.Fraction`` (exact); data
arithmetic uses numpy in the dtype the method computes in.

Rules: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
anything under ``oracle/``.  The oracle shares no code with the CUDA / C++
path (``paper_2110_04478_b200``) and imports nothing from it.

Parity status: every public function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``; see DESIGN.md "Oracle pins".  The one item left
"parity unpinned" is the absolute makespan of the paper's Fig 3b (the
figure is not in PAPER.md); the oracle's value 7 is pinned only by brute
force (it equals the optimum over all 16 schedules).
"""

from . import topology, collectives, scheduler, engine, brute, data  # noqa: F401
