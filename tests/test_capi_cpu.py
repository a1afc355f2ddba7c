"""CPU-only checks of the C-ABI boundary: the library loads, exports every
symbol include/gpujoin.h declares, and its pure-host entry points behave
(no GPU compute is issued here)."""
import ctypes
import os
import re

import pytest

import paper_1809_09930_b200 as pkg
from paper_1809_09930_b200 import gpujoin

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpujoin.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"GJ_API\s+[\w\s\*]+?\b(gj_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build()
    return gpujoin.lib()


def test_every_declared_symbol_is_exported(L):
    decl = declared_symbols()
    assert len(decl) >= 15
    assert sorted(gpujoin.EXPORTS) == decl
    for name in decl:
        assert hasattr(L, name), name
    out = os.popen(f"nm -D --defined-only {gpujoin.LIB_PATH}").read()
    exported = set(re.findall(r" T (gj_\w+)", out))
    assert set(decl) <= exported
    assert not [s for s in re.findall(r" T (\w+)", out) if not s.startswith("gj_") and not s.startswith("_")]


def test_library_is_built_for_sm100a(L):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {gpujoin.LIB_PATH}").read()
    assert "sm_100a" in out


def test_host_only_entry_points(L):
    assert pkg.abi_version() == 3
    o = gpujoin.default_options()
    assert (o.reorder, o.sortidu, o.shortc, o.symmetric, o.filter) == (1, 1, 1, 1, 2) and o.sample_frac == 0.01
    # computeNumBatches (§3.2.2 l.199-200)
    assert pkg.num_batches(3 * 10 ** 8, 10 ** 8) == 3
    assert pkg.num_batches(10 ** 5, 10 ** 8) == 3
    assert pkg.num_batches(10 ** 9, 10 ** 8) == 10
    assert pkg.num_batches(10 ** 9, 0) == 10          # auto b_s: no device here -> the paper's 1e8


def test_invalid_arguments_fail_without_touching_the_gpu(L):
    h = ctypes.c_void_p()
    rc = L.gj_build_index(None, 10, 4, 0.1, 2, None, ctypes.byref(h))
    assert rc == gpujoin.GJ_ERR_INVALID and b"null" in L.gj_last_error()
    buf = (ctypes.c_double * 8)()
    for n, dim, eps, k in [(0, 4, 0.1, 2), (2, 0, 0.1, 1), (2, 4, 0.0, 2), (2, 4, 0.1, 5), (2, 4, 0.1, 0),
                           (2, 200, 0.1, 2)]:
        rc = L.gj_build_index(buf, n, dim, eps, k, None, ctypes.byref(h))
        assert rc == gpujoin.GJ_ERR_INVALID, (n, dim, eps, k)
    assert L.gj_index_info(None, None) == gpujoin.GJ_ERR_INVALID
    L.gj_free_index(None)
