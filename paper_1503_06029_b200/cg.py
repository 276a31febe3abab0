"""Thin Python binding of the C ABI in include/cg.h (ctypes; marshalling only).

Every step of the path runs in the CUDA kernels of ``lib/libcg.so``; this
module only passes device pointers, sizes and the stream handle, and wraps
the returned device buffers as torch tensors without copying (through
``__cuda_array_interface__``; the tensor owns the buffer and frees it with
``cg_cells_free`` / ``cg_edges_free`` when collected).  There is no CPU
fallback: if the library is missing or the device is not a B200 the calls
raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libcg.so")

CG_OK, CG_EINVAL, CG_EINPUT, CG_ENOMEM, CG_ECUDA, CG_ETOOBIG, CG_EARCH, CG_ENOTIMPL = (
    0, -1, -2, -3, -4, -5, -6, -7)
CG_DICT_SORTED, CG_DICT_BSEARCH, CG_DICT_GLOBAL, CG_DICT_HASH, CG_DICT_AUTO = 0, 1, 2, 3, 4
DICT_KINDS = {"sorted": CG_DICT_SORTED, "bsearch": CG_DICT_BSEARCH, "global": CG_DICT_GLOBAL,
              "hash": CG_DICT_HASH, "auto": CG_DICT_AUTO}


class CgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"cg error {code}: {msg}")
        self.code = code


class cg_cells(ctypes.Structure):
    _fields_ = [("words", ctypes.c_void_p), ("n_cells", ctypes.c_int64),
                ("ell", ctypes.c_int32), ("words_per_cell", ctypes.c_int32)]


class cg_edges(ctypes.Structure):
    _fields_ = [("ij", ctypes.c_void_p), ("n_edges", ctypes.c_int64)]


class cg_stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in
                ("us_total", "us_pack", "us_sort", "us_dedupe", "us_layers", "us_dict",
                 "us_probe", "us_edges")] + \
               [(k, ctypes.c_int64) for k in
                ("n_in", "n_cells", "n_edges", "logical_probes", "issued_probes")] + \
               [("sort_passes", ctypes.c_int32), ("probe_reruns", ctypes.c_int32),
                ("kernel_launches", ctypes.c_int64), ("us_host_alloc", ctypes.c_double),
                ("n_allocs", ctypes.c_int64), ("us_host_total", ctypes.c_double),
                ("us_host_setup", ctypes.c_double), ("dict_bytes", ctypes.c_int64),
                ("dict_cells", ctypes.c_int64)]


class cg_opts(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_void_p), ("dict_kind", ctypes.c_int32),
                ("lcp_prune", ctypes.c_int32), ("bucket_log2", ctypes.c_int32),
                ("sort_kind", ctypes.c_int32), ("index_out", ctypes.c_void_p),
                ("stats", ctypes.POINTER(cg_stats)), ("filter_extra", ctypes.c_int32),
                ("reserved0", ctypes.c_int32), ("edge_cap", ctypes.c_int64)]


_lib = None


def lib():
    """Load libcg.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CgError(CG_ENOTIMPL, f"{LIB_PATH} not built (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    L.cg_opts_init.argtypes = [ctypes.POINTER(cg_opts)]
    L.cg_opts_init.restype = None
    for name in ("cg_build_ex",):
        f = getattr(L, name)
        f.argtypes = [P, i64, i32, ctypes.POINTER(cg_opts), ctypes.POINTER(cg_cells),
                      ctypes.POINTER(cg_edges)]
        f.restype = ctypes.c_int
    L.cg_build.argtypes = [P, i64, i32, ctypes.POINTER(cg_cells), ctypes.POINTER(cg_edges)]
    L.cg_build.restype = ctypes.c_int
    L.cg_build_packed_ex.argtypes = [P, i64, i32, ctypes.POINTER(cg_opts),
                                     ctypes.POINTER(cg_cells), ctypes.POINTER(cg_edges)]
    L.cg_build_packed_ex.restype = ctypes.c_int
    L.cg_build_host.argtypes = [P, i64, i32, ctypes.POINTER(cg_opts),
                                ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(i64),
                                ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(i64)]
    L.cg_build_host.restype = ctypes.c_int
    L.cg_host_free.argtypes = [P]
    L.cg_host_free.restype = None
    L.cg_query.argtypes = [P, P, i64, P, P, P]
    L.cg_query.restype = ctypes.c_int
    L.cg_index_info.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.cg_index_info.restype = ctypes.c_int
    L.cg_cells_free.argtypes = [ctypes.POINTER(cg_cells)]
    L.cg_cells_free.restype = None
    L.cg_edges_free.argtypes = [ctypes.POINTER(cg_edges)]
    L.cg_edges_free.restype = None
    L.cg_index_free.argtypes = [P]
    L.cg_index_free.restype = None
    L.cg_strerror.argtypes = [ctypes.c_int]
    L.cg_strerror.restype = ctypes.c_char_p
    L.cg_last_error.argtypes = []
    L.cg_last_error.restype = ctypes.c_char_p
    L.cg_version.argtypes = []
    L.cg_version.restype = ctypes.c_int
    L.cg_kernel_launches.argtypes = []
    L.cg_kernel_launches.restype = ctypes.c_int64
    L.cg_insert.argtypes = [P, i64, P, i64, i32, P, i64, ctypes.POINTER(cg_opts),
                            ctypes.POINTER(cg_cells), ctypes.POINTER(cg_edges)]
    L.cg_insert.restype = ctypes.c_int
    L.cg_allpairs.argtypes = [P, i64, i32, i32, ctypes.POINTER(cg_edges), ctypes.POINTER(i64), P]
    L.cg_allpairs.restype = ctypes.c_int
    L.cg_csr.argtypes = [P, i64, i64, P, P, P]
    L.cg_csr.restype = ctypes.c_int
    L.cg_bfs.argtypes = [P, P, i64, i64, P, P, ctypes.POINTER(i32), P]
    L.cg_bfs.restype = ctypes.c_int
    L.cg_signatures.argtypes = [P, i64, i32, P, i32, P, P]
    L.cg_signatures.restype = ctypes.c_int
    L.cg_build_points.argtypes = [P, i64, i32, P, i32, ctypes.POINTER(cg_opts),
                                  ctypes.POINTER(cg_cells), ctypes.POINTER(cg_edges)]
    L.cg_build_points.restype = ctypes.c_int
    L.cg_dist_local.argtypes = [P, i64, i32, ctypes.POINTER(cg_opts), i32,
                                ctypes.POINTER(cg_cells), ctypes.POINTER(i64)]
    L.cg_dist_local.restype = ctypes.c_int
    L.cg_dist_merge_chunk.argtypes = [P, ctypes.POINTER(i64), i32, i64, i32, i32,
                                      ctypes.POINTER(cg_opts), P, i64, ctypes.POINTER(i64)]
    L.cg_dist_merge_chunk.restype = ctypes.c_int
    L.cg_dist_probe.argtypes = [P, i64, i32, i32, i32, ctypes.POINTER(cg_opts),
                                ctypes.POINTER(cg_edges)]
    L.cg_dist_probe.restype = ctypes.c_int
    L.cg_dist_finalize.argtypes = [P, ctypes.POINTER(i64), i32, i64, ctypes.POINTER(cg_opts),
                                   ctypes.POINTER(cg_edges)]
    L.cg_dist_finalize.restype = ctypes.c_int
    _install_torch_allocator(L)
    _lib = L
    return L


# Device memory for the library's outputs and scratch arena comes from
# PyTorch's caching allocator (the cg_set_allocator hook): freed output
# blocks are reused by the next build on the same stream without a driver
# call, so steady-state builds never map memory.
_ALLOC_T = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_T = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


def _torch_alloc(size, stream, ctx):
    try:
        return torch._C._cuda_cudaCachingAllocator_raw_alloc(int(size), int(stream or 0))
    except Exception:  # out of memory -> NULL -> CG_ENOMEM
        return None


def _torch_free(ptr, stream, ctx):
    if ptr:
        try:
            torch._C._cuda_cudaCachingAllocator_raw_delete(int(ptr))
        except Exception:  # interpreter shutdown: torch is already torn down
            pass


_ALLOC_CB = _ALLOC_T(_torch_alloc)
_FREE_CB = _FREE_T(_torch_free)


def _install_torch_allocator(L):
    if os.environ.get("CG_NO_TORCH_ALLOC"):
        return
    L.cg_set_allocator.argtypes = [_ALLOC_T, _FREE_T, ctypes.c_void_p]
    L.cg_set_allocator.restype = ctypes.c_int
    rc = L.cg_set_allocator(_ALLOC_CB, _FREE_CB, None)
    if rc != CG_OK:
        raise CgError(rc, "cg_set_allocator failed")


EXPORTED = ("cg_opts_init", "cg_build", "cg_build_ex", "cg_build_packed_ex", "cg_build_host",
            "cg_host_free", "cg_query", "cg_index_info", "cg_set_allocator", "cg_cells_free",
            "cg_edges_free", "cg_index_free", "cg_strerror", "cg_last_error", "cg_version",
            "cg_kernel_launches", "cg_signatures", "cg_build_points", "cg_csr", "cg_bfs",
            "cg_allpairs", "cg_insert",
            "cg_dist_local", "cg_dist_merge_chunk", "cg_dist_probe", "cg_dist_finalize")


def _check(rc: int):
    if rc != CG_OK:
        L = lib()
        raise CgError(rc, f"{L.cg_strerror(rc).decode()}: {L.cg_last_error().decode()}")


class _DevBlock:
    """Owner of one device buffer returned by the library; exposes it through
    __cuda_array_interface__ so torch.as_tensor wraps it without a copy."""

    def __init__(self, kind: str, struct, ptr: int, shape, typestr: str):
        self._kind, self._struct = kind, struct
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
            "version": 3, "strides": None, "stream": None}

    def __del__(self):
        try:
            L = lib()
            if self._kind == "cells":
                L.cg_cells_free(ctypes.byref(self._struct))
            else:
                L.cg_edges_free(ctypes.byref(self._struct))
        except Exception:
            pass


def _wrap_cells(c: cg_cells, device) -> torch.Tensor:
    W = max(1, c.words_per_cell)
    if c.n_cells == 0:
        return torch.zeros((0, W), dtype=torch.int64, device=device)
    blk = _DevBlock("cells", c, c.words, (c.n_cells, W), "<i8")
    return torch.as_tensor(blk, device=device)


def _wrap_edges(e: cg_edges, device) -> torch.Tensor:
    if e.n_edges == 0:
        L = lib()
        L.cg_edges_free(ctypes.byref(e))
        return torch.zeros((0, 2), dtype=torch.int32, device=device)
    blk = _DevBlock("edges", e, e.ij, (e.n_edges, 2), "<i4")
    return torch.as_tensor(blk, device=device)


class Index:
    """Dictionary over a cell table (cg_index); immutable, for cg_query."""

    def __init__(self, handle: int, device):
        self.handle = handle
        self.device = device
        n = ctypes.c_int64()
        ell = ctypes.c_int32()
        _check(lib().cg_index_info(ctypes.c_void_p(handle), ctypes.byref(n), ctypes.byref(ell)))
        self.n_cells, self.ell = n.value, ell.value
        self.words = (self.ell + 63) // 64

    def query(self, q: torch.Tensor, stream: torch.cuda.Stream | None = None):
        """q: int64 [nq, W] packed cells (device).  Returns (self_idx int32 [nq],
        nbr_idx int32 [nq, ell]); asynchronous on the stream."""
        if q.dim() != 2 or q.shape[1] != self.words or q.dtype != torch.int64 or not q.is_cuda:
            raise CgError(CG_EINVAL, "q must be a CUDA int64 tensor [nq, ceil(ell/64)]")
        q = q.contiguous()
        nq = q.shape[0]
        self_idx = torch.empty(nq, dtype=torch.int32, device=q.device)
        nbr = torch.empty((nq, self.ell), dtype=torch.int32, device=q.device)
        st = stream or torch.cuda.current_stream(q.device)
        _check(lib().cg_query(ctypes.c_void_p(self.handle), ctypes.c_void_p(q.data_ptr()), nq,
                              ctypes.c_void_p(self_idx.data_ptr()),
                              ctypes.c_void_p(nbr.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
        return self_idx, nbr

    def __del__(self):
        try:
            if self.handle:
                lib().cg_index_free(ctypes.c_void_p(self.handle))
                self.handle = 0
        except Exception:
            pass


@dataclass
class BuildResult:
    cells: torch.Tensor          # int64 [n_cells, W] (u64 bit patterns, canonical order)
    edges: torch.Tensor          # int32 [n_edges, 2] (u32 values, i < j, ascending)
    stats: dict = field(default_factory=dict)
    index: Index | None = None


SORT_KINDS = {"auto": 0, "lsd": 1, "nosmall": 2, "nosweep": 3, "sweep": 4}


def _opts(stream, dict_kind, lcp_prune, bucket_log2, want_index, want_stats, sort_kind="auto",
          filter_extra=-1, edge_cap=0):
    L = lib()
    o = cg_opts()
    L.cg_opts_init(ctypes.byref(o))
    o.filter_extra = int(filter_extra)
    o.edge_cap = int(edge_cap)
    o.stream = ctypes.c_void_p(stream.cuda_stream)
    o.dict_kind = DICT_KINDS[dict_kind] if isinstance(dict_kind, str) else int(dict_kind)
    o.lcp_prune = int(bool(lcp_prune))
    o.bucket_log2 = int(bucket_log2)
    o.sort_kind = SORT_KINDS[sort_kind] if isinstance(sort_kind, str) else int(sort_kind)
    ih = ctypes.c_void_p()
    st = cg_stats()
    if want_index:
        o.index_out = ctypes.cast(ctypes.byref(ih), ctypes.c_void_p)
    if want_stats:
        o.stats = ctypes.pointer(st)
    return o, ih, st


def _stats_dict(st: cg_stats) -> dict:
    return {k: getattr(st, k) for k, _ in cg_stats._fields_}


def build(vecs: torch.Tensor, *, stream: torch.cuda.Stream | None = None,
          dict_kind="auto", lcp_prune: bool = True, bucket_log2: int = -1,
          want_index: bool = False, want_stats: bool = False,
          sort_kind="auto", filter_extra: int = -1, edge_cap: int = 0) -> BuildResult:
    """cg_build_ex on a CUDA uint8 tensor [n, ell] of 0/1 bytes."""
    if not isinstance(vecs, torch.Tensor) or vecs.dim() != 2:
        raise CgError(CG_EINVAL, "vecs must be a 2-D tensor [n, ell]")
    if vecs.dtype != torch.uint8:
        raise CgError(CG_EINVAL, "vecs must be uint8")
    if not vecs.is_cuda:
        raise CgError(CG_EINVAL, "vecs must be a CUDA tensor (no CPU fallback)")
    vecs = vecs.contiguous()
    n, ell = vecs.shape
    stream = stream or torch.cuda.current_stream(vecs.device)
    o, ih, st = _opts(stream, dict_kind, lcp_prune, bucket_log2, want_index, want_stats,
                      sort_kind, filter_extra, edge_cap)
    c, e = cg_cells(), cg_edges()
    with torch.cuda.device(vecs.device):
        _check(lib().cg_build_ex(ctypes.c_void_p(vecs.data_ptr()), n, ell, ctypes.byref(o),
                                 ctypes.byref(c), ctypes.byref(e)))
    c.ell, c.words_per_cell = ell, (ell + 63) // 64
    res = BuildResult(_wrap_cells(c, vecs.device), _wrap_edges(e, vecs.device))
    if want_stats:
        res.stats = _stats_dict(st)
    if want_index and ih.value:
        res.index = Index(ih.value, vecs.device)
    return res


def build_packed(words: torch.Tensor, ell: int, *, stream=None, dict_kind="auto",
                 lcp_prune=True, bucket_log2=-1, want_index=False, want_stats=False,
                 sort_kind="auto", filter_extra=-1, edge_cap=0):
    """cg_build_packed_ex on CUDA int64 [n, ceil(ell/64)] MSB-first words."""
    if words.dim() != 2 or words.dtype != torch.int64 or not words.is_cuda:
        raise CgError(CG_EINVAL, "words must be a CUDA int64 tensor [n, W]")
    words = words.contiguous()
    n = words.shape[0]
    stream = stream or torch.cuda.current_stream(words.device)
    o, ih, st = _opts(stream, dict_kind, lcp_prune, bucket_log2, want_index, want_stats,
                      sort_kind, filter_extra, edge_cap)
    c, e = cg_cells(), cg_edges()
    with torch.cuda.device(words.device):
        _check(lib().cg_build_packed_ex(ctypes.c_void_p(words.data_ptr()), n, ell,
                                        ctypes.byref(o), ctypes.byref(c), ctypes.byref(e)))
    c.ell, c.words_per_cell = ell, (ell + 63) // 64
    res = BuildResult(_wrap_cells(c, words.device), _wrap_edges(e, words.device))
    if want_stats:
        res.stats = _stats_dict(st)
    if want_index and ih.value:
        res.index = Index(ih.value, words.device)
    return res


def _check_points(points: torch.Tensor, planes: torch.Tensor):
    if (not isinstance(points, torch.Tensor) or points.dim() != 2 or points.dtype != torch.float64
            or not points.is_cuda):
        raise CgError(CG_EINVAL, "points must be a CUDA float64 tensor [n, dim]")
    if (not isinstance(planes, torch.Tensor) or planes.dim() != 2 or planes.dtype != torch.float64
            or not planes.is_cuda or planes.shape[1] != points.shape[1] + 1):
        raise CgError(CG_EINVAL, "planes must be a CUDA float64 tensor [ell, dim + 1]")
    return points.contiguous(), planes.contiguous()


def signatures(points: torch.Tensor, planes: torch.Tensor, *, stream=None) -> torch.Tensor:
    """cg_signatures (f1): packed cell signatures int64 [n, ceil(ell/64)] of
    points f64 [n, dim] against half-spaces planes f64 [ell, dim + 1]."""
    points, planes = _check_points(points, planes)
    n, dim = points.shape
    ell = planes.shape[0]
    words = torch.empty((n, (ell + 63) // 64), dtype=torch.int64, device=points.device)
    stream = stream or torch.cuda.current_stream(points.device)
    with torch.cuda.device(points.device):
        _check(lib().cg_signatures(ctypes.c_void_p(points.data_ptr()), n, dim,
                                   ctypes.c_void_p(planes.data_ptr()), ell,
                                   ctypes.c_void_p(words.data_ptr()),
                                   ctypes.c_void_p(stream.cuda_stream)))
    return words


def build_points(points: torch.Tensor, planes: torch.Tensor, *, stream=None, dict_kind="auto",
                 lcp_prune=True, bucket_log2=-1, want_index=False, want_stats=False,
                 sort_kind="auto") -> BuildResult:
    """cg_build_points (f1): the cell graph of the sampled points' signatures,
    computed and packed on the device (no n x ell byte matrix)."""
    points, planes = _check_points(points, planes)
    n, dim = points.shape
    ell = planes.shape[0]
    stream = stream or torch.cuda.current_stream(points.device)
    o, ih, st = _opts(stream, dict_kind, lcp_prune, bucket_log2, want_index, want_stats,
                      sort_kind)
    c, e = cg_cells(), cg_edges()
    with torch.cuda.device(points.device):
        _check(lib().cg_build_points(ctypes.c_void_p(points.data_ptr()), n, dim,
                                     ctypes.c_void_p(planes.data_ptr()), ell, ctypes.byref(o),
                                     ctypes.byref(c), ctypes.byref(e)))
    c.ell, c.words_per_cell = ell, (ell + 63) // 64
    res = BuildResult(_wrap_cells(c, points.device), _wrap_edges(e, points.device))
    if want_stats:
        res.stats = _stats_dict(st)
    if want_index and ih.value:
        res.index = Index(ih.value, points.device)
    return res


def build_host(vecs_host: torch.Tensor, *, device=None, stream=None, dict_kind="auto",
               lcp_prune=True, bucket_log2=-1, want_stats=False):
    """cg_build_host: uint8 [n, ell] HOST tensor (pinned for full speed) in,
    numpy-compatible host results out: (cells int64 [nc, W], edges int32 [m, 2],
    stats).  Host<->device copies happen inside the library call."""
    import numpy as np

    if vecs_host.is_cuda or vecs_host.dtype != torch.uint8 or vecs_host.dim() != 2:
        raise CgError(CG_EINVAL, "vecs_host must be a CPU uint8 tensor [n, ell]")
    vecs_host = vecs_host.contiguous()
    n, ell = vecs_host.shape
    device = torch.device(device or "cuda")
    with torch.cuda.device(device):
        stream = stream or torch.cuda.current_stream(device)
        o, ih, st = _opts(stream, dict_kind, lcp_prune, bucket_log2, False, want_stats)
        hc, he = ctypes.c_void_p(), ctypes.c_void_p()
        nc, ne = ctypes.c_int64(), ctypes.c_int64()
        L = lib()
        _check(L.cg_build_host(ctypes.c_void_p(vecs_host.data_ptr()), n, ell, ctypes.byref(o),
                               ctypes.byref(hc), ctypes.byref(nc), ctypes.byref(he),
                               ctypes.byref(ne)))
    W = (ell + 63) // 64
    try:
        cells = np.ctypeslib.as_array(ctypes.cast(hc.value, ctypes.POINTER(ctypes.c_int64)),
                                      shape=(nc.value * W,)).reshape(nc.value, W).copy()
        edges = (np.ctypeslib.as_array(ctypes.cast(he.value, ctypes.POINTER(ctypes.c_int32)),
                                       shape=(ne.value * 2,)).reshape(ne.value, 2).copy()
                 if ne.value else np.zeros((0, 2), np.int32))
    finally:
        L.cg_host_free(hc)
        L.cg_host_free(he)
    return cells, edges, (_stats_dict(st) if want_stats else {})


def build_host_raw(vecs_host: torch.Tensor, *, stream=None, want_stats=False):
    """As build_host but returns the library's pinned host pointers and counts
    without copying (caller must release with release_host); used by the e2e
    bench leg so the timed region holds exactly the library call."""
    n, ell = vecs_host.shape
    device = torch.device("cuda")
    stream = stream or torch.cuda.current_stream(device)
    o, ih, st = _opts(stream, "global", True, -1, False, want_stats)
    hc, he = ctypes.c_void_p(), ctypes.c_void_p()
    nc, ne = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().cg_build_host(ctypes.c_void_p(vecs_host.data_ptr()), n, ell, ctypes.byref(o),
                               ctypes.byref(hc), ctypes.byref(nc), ctypes.byref(he),
                               ctypes.byref(ne)))
    return hc.value, nc.value, he.value, ne.value, (_stats_dict(st) if want_stats else {})


def release_host(*ptrs):
    L = lib()
    for p in ptrs:
        if p:
            L.cg_host_free(ctypes.c_void_p(p))


def version() -> int:
    return lib().cg_version()


# ---------------------------------------------------------------- distributed phases
def dist_local(vecs: torch.Tensor, *, chunk_bits: int = 0, stream=None):
    """cg_dist_local: pack + sort + dedupe this rank's rows -> (sorted unique
    run int64 [c, W] (device), chunk_off list of 2^chunk_bits + 1 row offsets
    of its prefix chunks)."""
    if vecs.dtype != torch.uint8 or vecs.dim() != 2 or not vecs.is_cuda:
        raise CgError(CG_EINVAL, "vecs must be a CUDA uint8 tensor [n, ell]")
    vecs = vecs.contiguous()
    n, ell = vecs.shape
    stream = stream or torch.cuda.current_stream(vecs.device)
    o, _, _ = _opts(stream, "global", True, -1, False, False)
    c = cg_cells()
    off = (ctypes.c_int64 * ((1 << chunk_bits) + 1))()
    with torch.cuda.device(vecs.device):
        _check(lib().cg_dist_local(ctypes.c_void_p(vecs.data_ptr()), n, ell, ctypes.byref(o),
                                   int(chunk_bits), ctypes.byref(c), off))
    c.ell, c.words_per_cell = ell, (ell + 63) // 64
    return _wrap_cells(c, vecs.device), [int(x) for x in off]


def dist_merge_chunk(pieces: torch.Tensor, counts, ell: int, chunk_bits: int,
                     table: torch.Tensor, n_table: int, *, stream=None) -> int:
    """cg_dist_merge_chunk: append the sorted unique union of one prefix chunk
    of every rank's run (pieces int64 [G, stride, W], counts[g] valid rows
    each) to table (int64 [cap, W], device) after its n_table rows.  Returns
    the new row count."""
    if pieces.dtype != torch.int64 or pieces.dim() != 3 or not pieces.is_cuda:
        raise CgError(CG_EINVAL, "pieces must be a CUDA int64 tensor [G, stride, W]")
    if table.dtype != torch.int64 or table.dim() != 2 or not table.is_contiguous():
        raise CgError(CG_EINVAL, "table must be a contiguous int64 tensor [cap, W]")
    pieces = pieces.contiguous()
    G, stride, W = pieces.shape
    cnt = (ctypes.c_int64 * G)(*[int(c) for c in counts])
    nt = ctypes.c_int64(int(n_table))
    stream = stream or torch.cuda.current_stream(pieces.device)
    o, _, _ = _opts(stream, "global", True, -1, False, False)
    with torch.cuda.device(pieces.device):
        _check(lib().cg_dist_merge_chunk(ctypes.c_void_p(pieces.data_ptr()), cnt, G, stride, ell,
                                         int(chunk_bits), ctypes.byref(o),
                                         ctypes.c_void_p(table.data_ptr()), table.shape[0],
                                         ctypes.byref(nt)))
    return nt.value


def dist_probe(table: torch.Tensor, ell: int, G: int, rank: int, *, stream=None,
               want_stats=False, lcp_prune=True):
    """cg_dist_probe: this rank's share of the flip queries (popcount-layer
    split) over the canonical table int64 [n_cells, W] (device).  Returns
    (edges int32 [m_r, 2] canonical, stats)."""
    if table.dtype != torch.int64 or table.dim() != 2 or not table.is_cuda:
        raise CgError(CG_EINVAL, "table must be a CUDA int64 tensor [n_cells, W]")
    table = table.contiguous()
    stream = stream or torch.cuda.current_stream(table.device)
    o, _, st = _opts(stream, "global", lcp_prune, -1, False, want_stats)
    e = cg_edges()
    with torch.cuda.device(table.device):
        _check(lib().cg_dist_probe(ctypes.c_void_p(table.data_ptr()), table.shape[0], ell, G, rank,
                                   ctypes.byref(o), ctypes.byref(e)))
    return _wrap_edges(e, table.device), (_stats_dict(st) if want_stats else {})


def dist_finalize(gathered: torch.Tensor, counts, *, stream=None) -> torch.Tensor:
    """cg_dist_finalize: gathered = int32 [G, stride, 2] per-rank canonical,
    disjoint edge lists (counts[g] valid pairs each) -> their G-way merge,
    the canonical edge list int32 [m, 2]."""
    if gathered.dtype != torch.int32 or gathered.dim() != 3 or not gathered.is_cuda:
        raise CgError(CG_EINVAL, "gathered must be a CUDA int32 tensor [G, stride, 2]")
    gathered = gathered.contiguous()
    G, stride, _ = gathered.shape
    cnt = (ctypes.c_int64 * G)(*[int(c) for c in counts])
    stream = stream or torch.cuda.current_stream(gathered.device)
    o, _, _ = _opts(stream, "global", True, -1, False, False)
    e = cg_edges()
    with torch.cuda.device(gathered.device):
        _check(lib().cg_dist_finalize(ctypes.c_void_p(gathered.data_ptr()), cnt, G, stride,
                                      ctypes.byref(o), ctypes.byref(e)))
    return _wrap_edges(e, gathered.device)


def kernel_launches() -> int:
    """Kernels the library has launched in this process (cg_kernel_launches)."""
    return int(lib().cg_kernel_launches())


def csr(edges: torch.Tensor, n_cells: int, *, stream=None):
    """cg_csr (f4): canonical edge list int32 [m, 2] (device) -> (row_ptr int64
    [n_cells + 1], col int32 [2m]) with sorted adjacency lists."""
    if edges.dim() != 2 or edges.shape[1] != 2 or edges.dtype != torch.int32 or not edges.is_cuda:
        raise CgError(CG_EINVAL, "edges must be a CUDA int32 tensor [m, 2]")
    edges = edges.contiguous()
    m = edges.shape[0]
    dev = edges.device
    row_ptr = torch.empty(n_cells + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(1, 2 * m), dtype=torch.int32, device=dev)
    stream = stream or torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        _check(lib().cg_csr(ctypes.c_void_p(edges.data_ptr()), m, n_cells,
                            ctypes.c_void_p(row_ptr.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                            ctypes.c_void_p(stream.cuda_stream)))
    return row_ptr, col[: 2 * m]


def bfs(row_ptr: torch.Tensor, col: torch.Tensor, source: int, *, want_parent=True,
        stream=None):
    """cg_bfs (f4): (dist int32 [n], parent int32 [n] or None, eccentricity)."""
    n = row_ptr.shape[0] - 1
    dev = row_ptr.device
    dist = torch.empty(n, dtype=torch.int32, device=dev)
    parent = torch.empty(n, dtype=torch.int32, device=dev) if want_parent else None
    ecc = ctypes.c_int32()
    stream = stream or torch.cuda.current_stream(dev)
    col = col if col.numel() else torch.zeros(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _check(lib().cg_bfs(ctypes.c_void_p(row_ptr.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                            n, int(source), ctypes.c_void_p(dist.data_ptr()),
                            ctypes.c_void_p(parent.data_ptr() if parent is not None else 0),
                            ctypes.byref(ecc), ctypes.c_void_p(stream.cuda_stream)))
    return dist, parent, ecc.value


def allpairs(cells: torch.Tensor, ell: int, anchors: int = 0, *, stream=None):
    """cg_allpairs (f3): distance-1 pairs of a cell table int64 [n, W] (device)
    by pair comparison (naive, or Alg. 1-2 with `anchors` anchors).  Returns
    (edges int32 [m, 2] canonical, pairs_compared)."""
    if cells.dim() != 2 or cells.dtype != torch.int64 or not cells.is_cuda:
        raise CgError(CG_EINVAL, "cells must be a CUDA int64 tensor [n, W]")
    cells = cells.contiguous()
    n = cells.shape[0]
    e = cg_edges()
    cmp = ctypes.c_int64()
    stream = stream or torch.cuda.current_stream(cells.device)
    with torch.cuda.device(cells.device):
        _check(lib().cg_allpairs(ctypes.c_void_p(cells.data_ptr()), n, ell, anchors,
                                 ctypes.byref(e), ctypes.byref(cmp),
                                 ctypes.c_void_p(stream.cuda_stream)))
    return _wrap_edges(e, cells.device), cmp.value


def insert(cells: torch.Tensor, edges: torch.Tensor, vecs: torch.Tensor, *, stream=None):
    """cg_insert (f2): the cell graph of (accumulated input) + (new samples
    vecs uint8 [n_new, ell]), from an existing canonical table int64 [n, W]
    and edge list int32 [m, 2] (device).  Returns (cells, edges)."""
    if cells.dim() != 2 or cells.dtype != torch.int64 or not cells.is_cuda:
        raise CgError(CG_EINVAL, "cells must be a CUDA int64 tensor [n, W]")
    if vecs.dim() != 2 or vecs.dtype != torch.uint8 or not vecs.is_cuda:
        raise CgError(CG_EINVAL, "vecs must be a CUDA uint8 tensor [n_new, ell]")
    if (not isinstance(edges, torch.Tensor) or edges.dim() != 2 or edges.shape[1] != 2
            or edges.dtype != torch.int32 or not edges.is_cuda):
        raise CgError(CG_EINVAL, "edges must be a CUDA int32 tensor [m, 2]")
    if cells.device != vecs.device or edges.device != cells.device:
        raise CgError(CG_EINVAL, "cells, edges and vecs must be on the same device")
    n_new, ell = vecs.shape
    if cells.shape[1] != (ell + 63) // 64:
        raise CgError(CG_EINVAL, "cells must have ceil(ell/64) words per row")
    # keep the contiguous copies alive until the call returns (the library
    # allocates from the same caching allocator on the same stream)
    cells, vecs, edges = cells.contiguous(), vecs.contiguous(), edges.contiguous()
    m = edges.shape[0]
    eptr = edges.data_ptr() if m else 0
    stream = stream or torch.cuda.current_stream(cells.device)
    o, _, _ = _opts(stream, "global", True, -1, False, False)
    c, e = cg_cells(), cg_edges()
    with torch.cuda.device(cells.device):
        _check(lib().cg_insert(ctypes.c_void_p(cells.data_ptr()), cells.shape[0],
                               ctypes.c_void_p(eptr), m, ell,
                               ctypes.c_void_p(vecs.data_ptr()), n_new, ctypes.byref(o),
                               ctypes.byref(c), ctypes.byref(e)))
    c.ell, c.words_per_cell = ell, (ell + 63) // 64
    return _wrap_cells(c, cells.device), _wrap_edges(e, cells.device)
