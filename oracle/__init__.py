"""CPU oracle for the cell-graph path of arXiv 1503.06029 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_1503_06029_b200``) never imports it and shares no code with it.

The arithmetic lives in ``cg_oracle.cpp`` (see its header for the paper
citations); this module only builds the shared library with g++ and marshals
numpy arrays through ctypes.

Functions
---------
build(bytes_u8[n, ell])          ORACLE-A: std::set + single-bit-flip lookup
build_packed(words_u64[n, W], ell)
brute(bytes_u8[n, ell])          ORACLE-B: sort/unique + all-pairs distance
query(cells_u64[nc, W], ell, q_u64[nq, W])  self / neighbour indices
signatures(points_f64[n, dim], planes_f64[ell, dim+1])  f1: bytes u8[n, ell]
csr(edges_u32[m, 2], nv) / bfs(row_ptr, col, src)      f4: adjacency, distances, parents
All return ``(rc, cells u64[nc, W], edges u32[m, 2])`` (query: ``(rc, self, nbr)``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cg_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, EINVAL, EINPUT, ENOMEM, ETOOBIG, ESELF = 0, -1, -2, -3, -5, -9


def build_lib(force: bool = False) -> str:
    """Compile cg_oracle.cpp with g++ (no optimisation tricks beyond -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(
            ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC]
        )
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        pp = ctypes.POINTER(ctypes.c_void_p)
        pi64 = ctypes.POINTER(ctypes.c_int64)
        pd = ctypes.POINTER(ctypes.c_double)
        lib.oracle_build.argtypes = [P, i64, i32, i32, i32, pp, pi64, pp, pi64, pd]
        lib.oracle_build_packed.argtypes = [P, i64, i32, i32, pp, pi64, pp, pi64, pd]
        lib.oracle_brute.argtypes = [P, i64, i32, i32, pp, pi64, pp, pi64]
        lib.oracle_query.argtypes = [P, i64, i32, P, i64, P, P]
        lib.oracle_signatures.argtypes = [P, i64, i32, P, i32, P]
        lib.oracle_csr.argtypes = [P, i64, i64, P, P]
        lib.oracle_csr.restype = ctypes.c_int
        lib.oracle_bfs.argtypes = [P, P, i64, i64, P, P]
        lib.oracle_bfs.restype = ctypes.c_int
        lib.oracle_signatures.restype = ctypes.c_int
        lib.oracle_free.argtypes = [P]
        for f in (lib.oracle_build, lib.oracle_build_packed, lib.oracle_brute, lib.oracle_query):
            f.restype = ctypes.c_int
        lib.oracle_free.restype = None
        _lib = lib
    return _lib


def _threads(nthreads):
    if nthreads is None or nthreads <= 0:
        return os.cpu_count() or 1
    return nthreads


def _collect(lib, rc, cp, nc, ep, ne, W):
    try:
        if rc != OK:
            return rc, None, None
        cells = np.ctypeslib.as_array(
            ctypes.cast(cp.value, ctypes.POINTER(ctypes.c_uint64)), shape=(nc.value * W,)
        ).copy().reshape(nc.value, W) if nc.value else np.zeros((0, W), np.uint64)
        edges = np.ctypeslib.as_array(
            ctypes.cast(ep.value, ctypes.POINTER(ctypes.c_uint32)), shape=(ne.value * 2,)
        ).copy().reshape(ne.value, 2) if ne.value else np.zeros((0, 2), np.uint32)
        return rc, cells, edges
    finally:
        if cp.value:
            lib.oracle_free(cp)
        if ep.value:
            lib.oracle_free(ep)


def _as_bytes(x):
    x = np.ascontiguousarray(x)
    if x.dtype != np.uint8:
        raise TypeError("oracle expects uint8 bytes")
    return x


def build(x: np.ndarray, nthreads: int | None = None, self_check: bool = False,
          timings: dict | None = None):
    """ORACLE-A on uint8[n, ell] (``x.shape == (n, ell)``)."""
    lib = _load()
    x = _as_bytes(x)
    n, ell = (x.shape[0], x.shape[1]) if x.ndim == 2 else (0, 0)
    W = (ell + 63) // 64 if ell > 0 else 1
    cp, ep = ctypes.c_void_p(), ctypes.c_void_p()
    nc, ne = ctypes.c_int64(), ctypes.c_int64()
    t = (ctypes.c_double * 4)()
    rc = lib.oracle_build(x.ctypes.data if x.size else None, n, ell, _threads(nthreads),
                          int(self_check), ctypes.byref(cp), ctypes.byref(nc),
                          ctypes.byref(ep), ctypes.byref(ne), t)
    if timings is not None:
        timings.update(pack=t[0], set=t[1], lookup=t[2], sort=t[3],
                       threads=_threads(nthreads))
    return _collect(lib, rc, cp, nc, ep, ne, W)


def build_packed(words: np.ndarray, ell: int, nthreads: int | None = None,
                 timings: dict | None = None):
    """ORACLE-A on packed MSB-first words u64[n, ceil(ell/64)]."""
    lib = _load()
    words = np.ascontiguousarray(words, dtype=np.uint64)
    W = (ell + 63) // 64
    n = words.shape[0] if words.ndim == 2 else 0
    if n and words.shape[1] != W:
        raise ValueError("words must have ceil(ell/64) columns")
    cp, ep = ctypes.c_void_p(), ctypes.c_void_p()
    nc, ne = ctypes.c_int64(), ctypes.c_int64()
    t = (ctypes.c_double * 4)()
    rc = lib.oracle_build_packed(words.ctypes.data if n else None, n, ell, _threads(nthreads),
                                 ctypes.byref(cp), ctypes.byref(nc), ctypes.byref(ep),
                                 ctypes.byref(ne), t)
    if timings is not None:
        timings.update(unpack=t[0], set=t[1], lookup=t[2], sort=t[3],
                       threads=_threads(nthreads))
    return _collect(lib, rc, cp, nc, ep, ne, W)


def brute(x: np.ndarray, nthreads: int | None = None):
    """ORACLE-B on uint8[n, ell]."""
    lib = _load()
    x = _as_bytes(x)
    n, ell = (x.shape[0], x.shape[1]) if x.ndim == 2 else (0, 0)
    W = (ell + 63) // 64 if ell > 0 else 1
    cp, ep = ctypes.c_void_p(), ctypes.c_void_p()
    nc, ne = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.oracle_brute(x.ctypes.data if x.size else None, n, ell, _threads(nthreads),
                          ctypes.byref(cp), ctypes.byref(nc), ctypes.byref(ep),
                          ctypes.byref(ne))
    return _collect(lib, rc, cp, nc, ep, ne, W)


def query(cells: np.ndarray, ell: int, q: np.ndarray):
    """Self / single-flip neighbour indices of packed queries against a table."""
    lib = _load()
    cells = np.ascontiguousarray(cells, dtype=np.uint64)
    q = np.ascontiguousarray(q, dtype=np.uint64)
    nq = q.shape[0]
    self_idx = np.empty(nq, np.int32)
    nbr = np.empty((nq, ell), np.int32)
    rc = lib.oracle_query(cells.ctypes.data, cells.shape[0], ell,
                          q.ctypes.data if nq else None, nq, self_idx.ctypes.data,
                          nbr.ctypes.data)
    return rc, self_idx, nbr


def timed_build(x: np.ndarray, nthreads: int | None = None):
    """ORACLE-A with wall time; returns (cells, edges, seconds, timings)."""
    tm: dict = {}
    t0 = time.perf_counter()
    rc, cells, edges = build(x, nthreads=nthreads, timings=tm)
    dt = time.perf_counter() - t0
    if rc != OK:
        raise RuntimeError(f"oracle_build failed rc={rc}")
    return cells, edges, dt, tm


def signatures(points: np.ndarray, planes: np.ndarray):
    """f1 cell signatures: ``(rc, bytes u8[n, ell])``; bit k of point r
    is [fma-chain value of a_k . p_r + b_k >= 0] (DESIGN G12, G21)."""
    lib = _load()
    P = np.ascontiguousarray(points, dtype=np.float64)
    A = np.ascontiguousarray(planes, dtype=np.float64)
    n, dim = P.shape
    ell = A.shape[0]
    assert A.shape[1] == dim + 1
    out = np.zeros((n, ell), dtype=np.uint8)
    rc = lib.oracle_signatures(P.ctypes.data, n, dim, A.ctypes.data, ell, out.ctypes.data)
    return rc, out


def csr(edges: np.ndarray, nv: int):
    """f4 adjacency of G_X: ``(rc, row_ptr u64[nv+1], col u32[2m])``."""
    lib = _load()
    E = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
    m = E.shape[0]
    row_ptr = np.zeros(nv + 1, dtype=np.uint64)
    col = np.zeros(max(1, 2 * m), dtype=np.uint32)
    rc = lib.oracle_csr(E.ctypes.data, m, nv, row_ptr.ctypes.data, col.ctypes.data)
    return rc, row_ptr, col[: 2 * m]


def bfs(row_ptr: np.ndarray, col: np.ndarray, src: int):
    """f4 BFS: ``(rc, dist i32[nv], parent i32[nv])``."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    cl = np.ascontiguousarray(col, dtype=np.uint32)
    if cl.size == 0:
        cl = np.zeros(1, dtype=np.uint32)
    nv = rp.shape[0] - 1
    dist = np.zeros(nv, dtype=np.int32)
    parent = np.zeros(nv, dtype=np.int32)
    rc = lib.oracle_bfs(rp.ctypes.data, cl.ctypes.data, nv, int(src), dist.ctypes.data,
                        parent.ctypes.data)
    return rc, dist, parent
