"""B200-native cell-graph construction (arXiv 1503.06029): the data-parallel
hot path -- pack, radix sort, dedupe, popcount layering, prefix-indexed
sorted dictionary, single-bit-flip probes, canonical edge sort -- as
hand-written sm_100a CUDA behind the C ABI of include/cg.h.

    from paper_1503_06029_b200 import build
    res = build(vecs_uint8_cuda)      # res.cells int64 [nc, W], res.edges int32 [m, 2]
    res = build_points(points_f64_cuda, planes_f64_cuda)   # signatures on the device (f1)
"""
from .cg import (BuildResult, CgError, Index, allpairs, bfs, build, build_host,  # noqa: F401
                 build_packed, build_points, csr, insert, lib, signatures, version)

__all__ = ["build", "build_packed", "build_host", "build_points", "signatures", "csr", "bfs",
           "allpairs", "insert",
           "BuildResult",
           "Index", "CgError", "lib", "version"]
