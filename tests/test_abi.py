"""The C-ABI library loads on a CPU-only host and exports every symbol
include/themis.h declares; the Python binding uses the same names."""

import pytest

import os
import re

from paper_2110_04478_b200 import _lib, themis as th

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "themis.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(themis_[a-z_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = declared()
    assert "themis_allreduce" in names and "themis_plan" in names and "themis_reduce_scatter" in names
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n), n
        assert n in _lib.SIGNATURES, f"binding lacks {n}"


def test_binding_names_match_abi():
    for n in ("themis_plan", "themis_allreduce", "themis_reduce_scatter", "themis_all_gather",
              "themis_allreduce_host"):
        assert hasattr(th, n)


def test_version_and_launch_count():
    assert "sm_100a" in th.version()
    assert th.launches_per_call() == 1


def test_heap_layout():
    sig, stride, heap = th.heap_layout(8, 1, 1 << 30)
    assert stride == 1 << 30 and heap == 8 * (sig + stride)
    sig2, stride2, heap2 = th.heap_layout(8, 8, 1000)
    assert stride2 % 65536 == 0 and heap2 == sig2 + stride2


def test_default_ctas_is_the_a9_formula():
    """themis_default_ctas == SURVEY a9's c_k = max(1, round(c_tot BW_k / sum BW))
    whenever those roundings already sum to c_tot; always sums to c_tot, >= 1."""
    import random
    from fractions import Fraction
    rng = random.Random(7)
    agree = 0
    for _ in range(2000):
        D = rng.randint(1, 8)
        bw = [rng.choice([1, 2, 3, 4, 7, 50, 200, 1000, rng.randint(1, 10**6)]) for _ in range(D)]
        total = rng.randint(D, 400)
        got = th.default_ctas(bw, total)
        assert sum(got) == total and min(got) >= 1, (bw, total, got)
        want = [max(1, round(Fraction(total * b, sum(bw)))) for b in bw]   # half-to-even ties are remainder ties
        if sum(want) == total and all(Fraction(total * b, sum(bw)) % 1 != Fraction(1, 2) for b in bw):
            assert got == want, (bw, total, got, want)
            agree += 1
    assert agree > 500


def test_default_ctas():
    assert th.default_ctas((4, 2, 1), 28) == [16, 8, 4]
    assert th.default_ctas((1000, 1, 1), 3) == [1, 1, 1]           # the one-CTA floor binds
    with pytest.raises(th.ThemisError):
        th.default_ctas((1, 1, 1), 2)                              # budget < ndims
    assert th.default_ctas((1, 1, 1), 148) == [50, 49, 49]
    assert sum(th.default_ctas((200, 50), 7)) == 7
