"""The C-ABI library loads on a CPU-only host and exports every symbol
include/themis.h declares; the Python binding uses the same names."""

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


def test_default_ctas():
    assert th.default_ctas((4, 2, 1), 28) == [16, 8, 4]
    assert th.default_ctas((1, 1, 1), 148) == [50, 49, 49]
    assert sum(th.default_ctas((200, 50), 7)) == 7
