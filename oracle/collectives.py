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

from .topology import DIRECT, RING, SWITCH, Dim

RS, AG = "RS", "AG"


def num_steps(phase: str, kind: str, p: int) -> int:
    if p < 2:
        raise ValueError("p >= 2")
    if kind == RING:
        return p - 1
    if kind == DIRECT:
        return 1
    if kind == SWITCH:
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
