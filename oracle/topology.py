"""Multi-dimensional topology P_1 x ... x P_D (oracle; test infrastructure).

PAPER.md:278 — "we use the notation P_1 x P_2 x ... x P_D to refer to the size
of a multi-dimensional network where P_i is ... the size of peer NPUs
participating in the communication on the i'th dimension".
PAPER.md:505 / Table 2 (:509-519) — per-dimension aggregate BW/NPU = BW/link x
#links/NPU; network latency = step_latency (:525).
PAPER.md:136 footnote — all bandwidths are uni-directional.

Units (reading R21): bandwidth in bytes/ns (numerically GB/s),
time in ns, sizes in bytes.  Table 2 is in Gb/s; ``gbps()`` divides by 8.

Rank <-> coordinates (reading R15, paper silent): dim 1 varies
fastest, c_k = floor(r / prod_{i<k} P_i) mod P_k.  Dimensions are 0-based in
code (dim1 of the paper == index 0).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Sequence

RING, DIRECT, SWITCH = "ring", "direct", "switch"   # Table 1
# A Switch dimension whose switch can reduce (in-network collective offload,
# PAPER.md:493-494; on B200: NVSwitch NVLS multimem).  DESIGN.md reading R29.
NVLS = "nvls"
KINDS = (RING, DIRECT, SWITCH, NVLS)


def gbps(x) -> Fraction:
    """Gb/s (decimal, Table 2) -> bytes/ns."""
    return Fraction(x) / 8


@dataclass(frozen=True)
class Dim:
    size: int                       # P_k
    bw: Fraction                    # aggregate uni-directional BW per NPU, bytes/ns
    kind: str = DIRECT              # topology of the dimension (Table 1)
    step_latency: Fraction = Fraction(0)  # ns, "step_latency"


@dataclass(frozen=True)
class Topology:
    dims: tuple

    @staticmethod
    def make(sizes: Sequence[int], bws: Sequence, kinds=None, latencies=None) -> "Topology":
        kinds = kinds or [DIRECT] * len(sizes)
        latencies = latencies or [0] * len(sizes)
        t = Topology(tuple(Dim(int(p), Fraction(b), k, Fraction(l))
                           for p, b, k, l in zip(sizes, bws, kinds, latencies)))
        t.validate()
        return t

    # --- basic quantities -------------------------------------------------
    @property
    def D(self) -> int:
        return len(self.dims)

    @property
    def P(self) -> int:
        n = 1
        for d in self.dims:
            n *= d.size
        return n

    @property
    def sizes(self) -> tuple:
        return tuple(d.size for d in self.dims)

    @property
    def total_bw(self) -> Fraction:
        return sum((d.bw for d in self.dims), Fraction(0))

    def validate(self) -> None:
        """SPEC.md:39,43 rules: D >= 1; P_k >= 2; BW > 0; latency >= 0;
        Switch => P_k a power of two (halving-doubling)."""
        if self.D < 1:
            raise ValueError("topology needs at least one dimension")
        for i, d in enumerate(self.dims):
            if d.size < 2:
                raise ValueError(f"dim{i+1}: size {d.size} < 2")
            if d.bw <= 0:
                raise ValueError(f"dim{i+1}: bandwidth must be > 0")
            if d.step_latency < 0:
                raise ValueError(f"dim{i+1}: negative latency")
            if d.kind not in KINDS:
                raise ValueError(f"dim{i+1}: unknown kind {d.kind!r}")
            if d.kind in (SWITCH, NVLS) and (d.size & (d.size - 1)):
                raise ValueError(f"dim{i+1}: switch size {d.size} not a power of two")

    # --- rank coordinates (dim1 fastest) ---------------------------------
    def stride(self, k: int) -> int:
        s = 1
        for i in range(k):
            s *= self.dims[i].size
        return s

    def coords(self, r: int) -> tuple:
        out = []
        for d in self.dims:
            out.append(r % d.size)
            r //= d.size
        return tuple(out)

    def rank_of(self, coords: Sequence[int]) -> int:
        r = 0
        for k in reversed(range(self.D)):
            r = r * self.dims[k].size + coords[k]
        return r

    def dim_peers(self, r: int, k: int) -> list:
        """Ranks sharing every coordinate of r except dim k, in coordinate
        order j = 0..P_k-1 (rank r itself at j = c_k)."""
        c = list(self.coords(r))
        out = []
        for j in range(self.dims[k].size):
            c[k] = j
            out.append(self.rank_of(c))
        return out


def _table2(sizes, bw_link, links, lat, kinds):
    return Topology.make(sizes, [gbps(b * l) for b, l in zip(bw_link, links)], kinds, lat)


S_, R_, F_ = SWITCH, RING, DIRECT
# PAPER.md Table 2 (:509-519): name -> (sizes, BW/link Gb/s, links/NPU, latency ns)
PRESETS = {
    "2D-SW_SW": _table2((16, 64), (200, 800), (6, 1), (700, 1700), (S_, S_)),
    "3D-SW_SW_SW_homo": _table2((16, 8, 8), (200, 200, 800), (4, 4, 1), (700, 700, 1700), (S_, S_, S_)),
    "3D-SW_SW_SW_hetero": _table2((16, 8, 8), (200, 200, 400), (8, 4, 1), (700, 700, 1700), (S_, S_, S_)),
    "3D-FC_Ring_SW": _table2((8, 16, 8), (200, 200, 400), (7, 4, 1), (700, 700, 1700), (F_, R_, S_)),
    "4D-Ring_SW_SW_SW": _table2((4, 4, 8, 8), (1000, 200, 200, 400), (2, 8, 4, 1), (20, 700, 700, 1700),
                                (R_, S_, S_, S_)),
    "4D-Ring_FC_Ring_SW": _table2((4, 8, 4, 8), (1500, 200, 200, 800), (2, 7, 6, 1), (20, 700, 700, 1700),
                                  (R_, F_, R_, S_)),
}
# "current" 2D platform of Fig 2: 16 x 64, 1200 / 100 Gb/s.
# Its latencies are not given in the paper; zero.
CURRENT_2D = Topology.make((16, 64), (gbps(1200), gbps(100)), (SWITCH, SWITCH))
