"""Multi-GPU cell-graph build: one process per GPU, torch.distributed for the
two exchanges the north star allows (NCCL over NVLink on B200):

  phase 1  cg_dist_local        pack + sort + dedupe this rank's rows
  exch. 1  all-gather           run lengths, then the runs (padded)
  phase 2  cg_dist_merge_probe  global table (replicated), probe this rank's
                                share of the (popcount, index) order
  exch. 2  all-gather           edge counts, then the edge lists (padded)
  phase 3  cg_dist_finalize     canonical edge list

The compute phases are pluggable (``ops``) so the exchange logic can be
exercised with the gloo backend on CPU (tests/test_dist_gloo.py); the
product ops (``CudaOps``) call the C ABI.  DESIGN.md section 8.
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

    def local(self, vecs):
        from . import cg

        if vecs.shape[0] == 0:  # an empty shard (uneven split, n < G): an empty run
            return torch.zeros((0, (vecs.shape[1] + 63) // 64), dtype=torch.int64,
                               device=vecs.device)
        return cg.dist_local(vecs, stream=self.stream)

    def merge_probe(self, runs, counts, rank, ell):
        from . import cg

        table, edges, st = cg.dist_merge_probe(runs, counts, rank, ell, stream=self.stream,
                                               want_stats=self.want_stats)
        self.last_stats = st
        return table, edges

    def finalize(self, gathered, counts):
        from . import cg

        return cg.dist_finalize(gathered, counts, stream=self.stream)


def _gather_counts(n: int, device, group) -> list[int]:
    G = dist.get_world_size(group)
    t = torch.tensor([n], dtype=torch.int64, device=device)
    outs = [torch.zeros_like(t) for _ in range(G)]
    dist.all_gather(outs, t, group=group)
    return [int(o.item()) for o in outs]


def _gather_padded(x: torch.Tensor, counts: list[int], group) -> torch.Tensor:
    """All-gather per-rank tensors [c_r, ...] padded to max c -> [G, stride, ...]."""
    G = len(counts)
    stride = max(1, max(counts))
    pad = torch.zeros((stride,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    if x.shape[0]:
        pad[: x.shape[0]] = x
    if dist.get_backend(group) == "nccl":
        out = torch.empty((G * stride,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, pad, group=group)
    else:
        outs = [torch.empty_like(pad) for _ in range(G)]
        dist.all_gather(outs, pad, group=group)
        out = torch.cat(outs)
    return out.view((G, stride) + tuple(x.shape[1:]))


def build_distributed(vecs_local: torch.Tensor, ell: int | None = None, group=None, ops=None,
                      timings: dict | None = None):
    """Build the cell graph of the union of every rank's rows.  Returns
    (table [n_c, W] int64, edges [m, 2] int32), identical on every rank."""
    ops = ops or CudaOps()
    ell = ell or vecs_local.shape[1]
    rank = dist.get_rank(group)
    t = {}
    t0 = time.perf_counter()
    run = ops.local(vecs_local)
    counts = _gather_counts(run.shape[0], run.device, group)
    runs = _gather_padded(run, counts, group)
    t["local+exchange1"] = time.perf_counter() - t0
    table, local_edges = ops.merge_probe(runs, counts, rank, ell)
    t["merge_probe"] = time.perf_counter() - t0 - t["local+exchange1"]
    ecounts = _gather_counts(local_edges.shape[0], local_edges.device, group)
    gathered = _gather_padded(local_edges, ecounts, group)
    edges = ops.finalize(gathered, ecounts)
    t["total"] = time.perf_counter() - t0
    if timings is not None:
        timings.update(t)
    return table, edges
