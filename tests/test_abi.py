"""C-ABI library checks that need no GPU: the in-tree libcg.so builds for
sm_100a, loads, exports every symbol include/cg.h declares, and rejects bad
arguments before touching the device."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1503_06029_b200 import build_lib

    build_lib.build()
    from paper_1503_06029_b200 import cg

    return cg.lib()


def _declared():
    txt = open(os.path.join(ROOT, "include", "cg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cg_[a-z_]+)\s*\(", txt)))


def test_header_symbols_exported(L):
    from paper_1503_06029_b200 import cg

    names = _declared()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", cg.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (cg_[a-z_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    for n in names:
        getattr(L, n)  # resolvable through the loader
    assert set(cg.EXPORTED) <= exported


def test_sm100a_cubin_embedded():
    from paper_1503_06029_b200 import cg

    out = subprocess.run(["cuobjdump", "--list-elf", cg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_without_device(L):
    from paper_1503_06029_b200.cg import (CG_EINVAL, CG_ETOOBIG, cg_cells, cg_edges, cg_opts)

    c, e = cg_cells(), cg_edges()
    fake = ctypes.c_void_p(0x1000)
    assert L.cg_build(None, 10, 8, ctypes.byref(c), ctypes.byref(e)) == CG_EINVAL
    assert L.cg_build(fake, 0, 8, ctypes.byref(c), ctypes.byref(e)) == CG_EINVAL
    assert L.cg_build(fake, -3, 8, ctypes.byref(c), ctypes.byref(e)) == CG_EINVAL
    assert L.cg_build(fake, 10, 0, ctypes.byref(c), ctypes.byref(e)) == CG_EINVAL
    assert L.cg_build(fake, 10, 4097, ctypes.byref(c), ctypes.byref(e)) == CG_EINVAL
    assert L.cg_build(fake, 1 << 32, 8, ctypes.byref(c), ctypes.byref(e)) == CG_ETOOBIG
    assert c.words is None and c.n_cells == 0 and e.ij is None and e.n_edges == 0
    assert b"2^32" in L.cg_last_error()
    L.cg_build(fake, 10, 4097, ctypes.byref(c), ctypes.byref(e))
    assert b"ell" in L.cg_last_error()
    o = cg_opts()
    L.cg_opts_init(ctypes.byref(o))
    assert o.dict_kind == 4 and o.lcp_prune == 1 and o.bucket_log2 == -1  # CG_DICT_AUTO
    assert L.cg_query(None, None, 1, None, None, None) == CG_EINVAL
    assert L.cg_strerror(-2) == b"input byte not in {0,1} / pad bit set"
    assert L.cg_version() >= 1


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle or numpy-based compute."""
    pkg = os.path.join(ROOT, "paper_1503_06029_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn


def test_kernel_launch_counter_and_new_entries_reject_bad_arguments(L):
    """cg_kernel_launches is monotone; the f1-f4 entries reject NULL / bad
    sizes before touching the device."""
    from paper_1503_06029_b200.cg import CG_EINVAL, cg_cells, cg_edges

    a = L.cg_kernel_launches()
    assert a >= 0 and L.cg_kernel_launches() == a
    i64 = ctypes.c_int64
    assert L.cg_signatures(None, 4, 3, None, 8, None, None) == CG_EINVAL
    fake = ctypes.c_void_p(0x1000)
    assert L.cg_signatures(fake, 4, 0, fake, 8, fake, None) == CG_EINVAL   # dim 0
    assert L.cg_signatures(fake, 4, 17, fake, 8, fake, None) == CG_EINVAL  # dim 17
    assert L.cg_signatures(fake, 0, 3, fake, 8, fake, None) == CG_EINVAL   # n 0
    c, e = cg_cells(), cg_edges()
    assert L.cg_insert(None, 1, None, 0, 8, fake, 1, None, ctypes.byref(c), ctypes.byref(e)) == CG_EINVAL
    assert L.cg_insert(fake, 0, None, 0, 8, fake, 1, None, ctypes.byref(c), ctypes.byref(e)) == CG_EINVAL
    assert L.cg_allpairs(None, 4, 64, 0, ctypes.byref(e), None, None) == CG_EINVAL
    assert L.cg_allpairs(fake, 4, 64, 9, ctypes.byref(e), None, None) == CG_EINVAL  # anchors > 8
    assert L.cg_csr(fake, 1, 0, fake, fake, None) == CG_EINVAL   # n_cells 0
    ecc = ctypes.c_int32()
    assert L.cg_bfs(fake, fake, 4, 4, fake, None, ctypes.byref(ecc), None) == CG_EINVAL  # source
    assert L.cg_bfs(None, fake, 4, 0, fake, None, ctypes.byref(ecc), None) == CG_EINVAL
    assert c.words is None and e.ij is None
