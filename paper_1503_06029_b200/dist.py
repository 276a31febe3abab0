"""Multi-GPU cell-graph build (row e): one process per GPU, torch.distributed
for the two exchanges the north star allows (NCCL over NVLink on B200).

  phase 1  cg_dist_local        pack + sort + dedupe this rank's rows; split
                                the sorted run into 2^chunk_bits prefix chunks
  exch. 1  all-gather           per chunk, in prefix order: every rank's piece
  phase 2  cg_dist_merge_chunk  append the chunk's merge to the replicated
                                canonical table -- while the all-gather of the
                                next chunk is in flight (async NCCL op)
  phase 3  cg_dist_probe        probe this rank's share of the popcount layers
                                (a 0->1 flip goes one layer up)
                                with a dictionary over its layers only
  exch. 2  all-gather           edge counts, then the edge lists (padded)
  phase 4  cg_dist_finalize     G-way merge -> the canonical edge list

At G = 1 both exchanges and the merge vanish (the run is the table).  The
compute phases are pluggable (``ops``) so the exchange logic runs with the
gloo backend on CPU (tests/test_dist_gloo.py); the product ops (``CudaOps``)
call the C ABI.  DESIGN.md section 8.
"""
from __future__ import annotations

import time

import torch
import torch.distributed as dist


class CudaOps:
    """The C-ABI phases (device tensors)."""

    def __init__(self, stream=None, want_stats=False):
        self.stream = stream
        self.want_stats = want_stats
        self.last_stats = {}

    def local(self, vecs, chunk_bits):
        from . import cg

        if vecs.shape[0] == 0:  # an empty shard (uneven split, n < G): an empty run
            W = (vecs.shape[1] + 63) // 64
            return (torch.zeros((0, W), dtype=torch.int64, device=vecs.device),
                    [0] * ((1 << chunk_bits) + 1))
        return cg.dist_local(vecs, chunk_bits=chunk_bits, stream=self.stream)

    def new_table(self, cap, W, device):
        return torch.empty((max(1, cap), W), dtype=torch.int64, device=device)

    def merge_chunk(self, pieces, counts, ell, chunk_bits, table, n_table):
        from . import cg

        return cg.dist_merge_chunk(pieces, counts, ell, chunk_bits, table, n_table,
                                   stream=self.stream)

    def probe(self, table, ell, G, rank):
        from . import cg

        edges, st = cg.dist_probe(table, ell, G, rank, stream=self.stream,
                                  want_stats=self.want_stats)
        self.last_stats = st
        return edges

    def finalize(self, gathered, counts):
        from . import cg

        return cg.dist_finalize(gathered, counts, stream=self.stream)


def _gather_vector(v: list[int], device, group) -> list[list[int]]:
    """All-gather one int64 vector per rank -> [G][len(v)]."""
    G = dist.get_world_size(group)
    t = torch.tensor(v, dtype=torch.int64, device=device)
    outs = [torch.zeros_like(t) for _ in range(G)]
    dist.all_gather(outs, t, group=group)
    return [[int(x) for x in o.tolist()] for o in outs]


def _start_gather_padded(x: torch.Tensor, stride: int, group):
    """Asynchronous all-gather of per-rank tensors [c_r, ...] padded to
    `stride` rows -> (work, result [G, stride, ...] once work is done)."""
    G = dist.get_world_size(group)
    stride = max(1, stride)
    pad = torch.zeros((stride,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    if x.shape[0]:
        pad[: x.shape[0]] = x
    if dist.get_backend(group) == "nccl":
        out = torch.empty((G * stride,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        work = dist.all_gather_into_tensor(out, pad, group=group, async_op=True)
        return work, lambda: out.view((G, stride) + tuple(x.shape[1:]))
    outs = [torch.empty_like(pad) for _ in range(G)]
    work = dist.all_gather(outs, pad, group=group, async_op=True)
    return work, lambda: torch.cat(outs).view((G, stride) + tuple(x.shape[1:]))


def build_distributed(vecs_local: torch.Tensor, ell: int | None = None, group=None, ops=None,
                      chunk_bits: int = 1, timings: dict | None = None):
    """Build the cell graph of the union of every rank's rows.  Returns
    (table [n_c, W] int64, edges [m, 2] int32), identical on every rank.

    chunk_bits: the run exchange goes in 2^chunk_bits prefix chunks, chunk
    c+1 on NVLink while chunk c is merged.  Each chunk's merge has a fixed
    cost (C5 at G = 8, one B200: 1 chunk 2.17 ms, 2 chunks 2.59, 8 chunks
    3.46 ms of merging), against ~1.2 ms of NVLink transfer to hide: two
    chunks (the default) is the estimated optimum."""
    ops = ops or CudaOps()
    ell = ell or vecs_local.shape[1]
    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = {}
    t0 = time.perf_counter()
    if G == 1:
        chunk_bits = 0
    run, chunk_off = ops.local(vecs_local, chunk_bits)
    t["local"] = time.perf_counter() - t0
    if G == 1:
        table = run
    else:
        C = 1 << chunk_bits
        mine = [chunk_off[c + 1] - chunk_off[c] for c in range(C)]
        counts = _gather_vector(mine, run.device, group)  # [G][C]
        W = run.shape[1]
        table = ops.new_table(sum(map(sum, counts)), W, run.device)
        n_table = 0

        def start(c):
            stride = max(counts[g][c] for g in range(G))
            return _start_gather_padded(run[chunk_off[c]: chunk_off[c + 1]], stride, group)

        pending = start(0)
        for c in range(C):
            nxt = start(c + 1) if c + 1 < C else None  # in flight during this merge
            work, result = pending
            work.wait()
            n_table = ops.merge_chunk(result(), [counts[g][c] for g in range(G)], ell,
                                      chunk_bits, table, n_table)
            pending = nxt
        table = table[:n_table]
    t["table"] = time.perf_counter() - t0 - t["local"]
    local_edges = ops.probe(table, ell, G, rank)
    t["probe"] = time.perf_counter() - t0 - t["local"] - t["table"]
    if G == 1:
        edges = local_edges
    else:
        ecounts = [c[0] for c in _gather_vector([local_edges.shape[0]], local_edges.device, group)]
        work, result = _start_gather_padded(local_edges, max(ecounts), group)
        work.wait()
        edges = ops.finalize(result(), ecounts)
    t["total"] = time.perf_counter() - t0
    if timings is not None:
        timings.update(t)
    return table, edges
