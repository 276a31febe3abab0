"""The N > 1 exchange logic of paper_1503_06029_b200.dist on CPU: world size 2
and 3 with the gloo backend.  The compute phases are stood in by the CPU
oracle (tests may use it), so this checks the run/edge all-gathers, padding
and counts, and that every rank ends with the single-process result."""
from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


class OracleOps:
    """CPU stand-in for the C-ABI phases (same contracts as dist.CudaOps)."""

    def local(self, vecs, chunk_bits):
        W = (vecs.shape[1] + 63) // 64
        if vecs.shape[0] == 0:
            return torch.zeros((0, W), dtype=torch.int64), [0] * ((1 << chunk_bits) + 1)
        rc, cells, _ = oracle.build(vecs.numpy())
        assert rc == 0
        top = cells[:, 0] >> np.uint64(64 - chunk_bits) if chunk_bits else np.zeros(len(cells), np.uint64)
        off = np.searchsorted(top, np.arange((1 << chunk_bits) + 1, dtype=np.uint64), side="left")
        return torch.from_numpy(cells.view(np.int64)), [int(x) for x in off]

    def new_table(self, cap, W, device):
        return torch.zeros((max(1, cap), W), dtype=torch.int64)

    def merge_chunk(self, pieces, counts, ell, chunk_bits, table, n_table):
        G = pieces.shape[0]
        rows = np.concatenate([pieces[g, : counts[g]].numpy() for g in range(G)]).view(np.uint64)
        if rows.shape[0] == 0:
            return n_table
        rc, merged, _ = oracle.build_packed(rows, ell)
        assert rc == 0
        if n_table:  # chunks arrive in prefix order, above every row merged before
            prev = table[n_table - 1].numpy().view(np.uint64)
            assert tuple(prev) < tuple(merged[0])
        table[n_table: n_table + merged.shape[0]] = torch.from_numpy(merged.view(np.int64))
        return n_table + merged.shape[0]

    def probe(self, table, ell, G, rank):
        rc, t2, edges = oracle.build_packed(table.numpy().view(np.uint64), ell)
        assert rc == 0
        mine = edges[edges[:, 0] % G == rank]  # any disjoint split exercises the exchange
        return torch.from_numpy(np.ascontiguousarray(mine).view(np.int32))

    def finalize(self, gathered, counts):
        G = gathered.shape[0]
        e = np.concatenate([gathered[g, : counts[g]].numpy() for g in range(G)]).view(np.uint32)
        e = e[np.lexsort((e[:, 1], e[:, 0]))]
        return torch.from_numpy(np.ascontiguousarray(e).view(np.int32))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, x, ell, outdir, empty_rank, chunk_bits):
    from paper_1503_06029_b200 import dist as cgdist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    n = x.shape[0]
    lo, hi = n * rank // world, n * (rank + 1) // world
    if rank == empty_rank:
        hi = lo  # an empty shard: its rows go to nobody -- the others cover the input below
    if empty_rank >= 0 and rank == (empty_rank + 1) % world:
        lo, hi = min(lo, n * empty_rank // world), max(hi, n * (empty_rank + 1) // world)
    table, edges = cgdist.build_distributed(torch.from_numpy(x[lo:hi]), ell, ops=OracleOps(),
                                            chunk_bits=chunk_bits)
    np.save(os.path.join(outdir, f"t{rank}.npy"), table.numpy())
    np.save(os.path.join(outdir, f"e{rank}.npy"), edges.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,empty_rank,chunk_bits", [(2, -1, 3), (3, -1, 2), (3, 1, 3), (2, -1, 0)])
def test_gloo_exchange_matches_single_process(world, empty_rank, chunk_bits):
    """Chunked run exchange (prefix chunks merged in order), the edge
    exchange and an empty shard (uneven split) reproduce the single-process
    result on every rank."""
    x = synth.clustered_bytes(77, 3001, 70, n_centers=5, max_flips=3)
    x = np.concatenate([x, x[:500]])  # duplicates across ranks
    rc, want_c, want_e = oracle.build(x)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), x, 70, d, empty_rank, chunk_bits),
                 nprocs=world, join=True)
        for r in range(world):
            t = np.load(os.path.join(d, f"t{r}.npy")).view(np.uint64)
            e = np.load(os.path.join(d, f"e{r}.npy")).view(np.uint32)
            np.testing.assert_array_equal(t, want_c)
            np.testing.assert_array_equal(e, want_e)
