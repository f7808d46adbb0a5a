"""Per-dimension basic collective algorithms (oracle; test infrastructure).

PAPER.md:221 — "when performing RS/AG on P participating NPUs, the data size
residing on each NPU shrinks/multiplies by P x".
PAPER.md:281 — the size of a chunk in a stage is the size residing on each NPU
*before* the stage.
PAPER.md:487 footnote — n_K^i = (P_K - 1)/P_K x 4MB for a 4MB chunk on dimK
(RS).  PAPER.md:331 — "the 64MB RS (or 16MB AG) takes 1 unit", so an AG of
b bytes-before sends (P-1) x b (reading R5).
PAPER.md:475-477 — A_K = number_of_steps x step_latency; ring All-Reduce takes
2P-2 steps (so P-1 per phase).  Table 1 (:226-238): Ring -> ring,
FullyConnected -> direct (1 step), Switch -> halving-doubling (log2 P steps,
DESIGN.md reading R7).
"""

from __future__ import annotations

from fractions import Fraction

from .topology import DIRECT, NVLS, RING, SWITCH, Dim

RS, AG = "RS", "AG"


def num_steps(phase: str, kind: str, p: int) -> int:
    if p < 2:
        raise ValueError("p >= 2")
    if kind == RING:
        return p - 1
    if kind == DIRECT:
        return 1
    if kind in (SWITCH, NVLS):
        if p & (p - 1):
            raise ValueError("halving-doubling needs a power of two")
        return p.bit_length() - 1
    raise ValueError(kind)


def bytes_sent(phase: str, p: int, bytes_before) -> Fraction:
    """Bytes each NPU sends on the dimension for one stage (n_K^i)."""
    b = Fraction(bytes_before)
    if phase == RS:
        return Fraction(p - 1, p) * b
    if phase == AG:
        return (p - 1) * b
    raise ValueError(phase)


def size_after(phase: str, p: int, bytes_before) -> Fraction:
    b = Fraction(bytes_before)
    return b / p if phase == RS else b * p


def fixed_delay(dim: Dim, phase: str) -> Fraction:
    """A_K = number_of_steps x step_latency."""
    return num_steps(phase, dim.kind, dim.size) * dim.step_latency


def chunk_load(dim: Dim, phase: str, bytes_before) -> Fraction:
    """Latency-model increment n_K^i x B_K with B_K = 1/BW_K."""
    return bytes_sent(phase, dim.size, bytes_before) / dim.bw


# ---- in-network offload ("Switch collective offload reduces
# the collective's network traffic (n_K^i) and fixed delay (A_K)"; the
# hierarchical structure and Themis's balancing stay).  Reading R29: on an NVLS
# dim an All-Reduce chunk's last RS stage and its first AG stage (the same dim,
# Algorithm 1 line 8) run as ONE in-switch All-Reduce of the stage's data.  Per
# NPU, holding b bytes before the pair, each member sends its copy of every
# member's piece into the switch (b) and the reduced piece back for the
# multicast (b/p): n = (1 + 1/p) * b, in 2 switch traversals (reduce, then
# multicast store).  The AG half is then a zero-volume op that only orders the
# chunk's pipeline.

FUSED_STEPS = 2


def fused_bytes_sent(p: int, bytes_before) -> Fraction:
    """n_K^i of the fused in-switch RS+AG pair on a dim of size p."""
    b = Fraction(bytes_before)
    return b + b / p


def fused_delay(dim: Dim) -> Fraction:
    return FUSED_STEPS * dim.step_latency


def is_fused(topo, coll: str, rs, ag) -> bool:
    """AR chunk whose last RS dim is its first AG dim and an NVLS dim (R29)."""
    return coll == "AR" and bool(rs) and bool(ag) and rs[-1] == ag[0] and topo.dims[rs[-1]].kind == NVLS
