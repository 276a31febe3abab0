"""Distributed phases on one GPU with logical ranks (row e): cg_dist_local
per row shard, the chunked exchange (prefix chunks merged in order by
cg_dist_merge_chunk), cg_dist_probe for every rank (popcount-layer split) and
cg_dist_finalize must give the oracle's cell table and edge list for any
number of ranks G (P14: G-invariance), with each rank's dictionary holding
about 1/G of the cells plus one popcount layer."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from helpers import popcount_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1503_06029_b200 import build_lib

    build_lib.build()
    import paper_1503_06029_b200.cg as cg

    return cg


def _pad_stack(ts, dtype, tail):
    stride = max(1, max(t.shape[0] for t in ts))
    out = torch.zeros((len(ts), stride) + tail, dtype=dtype, device="cuda")
    for g, t in enumerate(ts):
        out[g, : t.shape[0]] = t
    return out


def logical_ranks(cg, x: np.ndarray, G: int, chunk_bits: int = 3):
    n, ell = x.shape
    W = (ell + 63) // 64
    xt = torch.from_numpy(x).cuda()
    C = 1 << chunk_bits
    runs, offs = [], []
    for g in range(G):
        part = xt[n * g // G: n * (g + 1) // G]
        if part.shape[0] == 0:
            runs.append(torch.zeros((0, W), dtype=torch.int64, device="cuda"))
            offs.append([0] * (C + 1))
            continue
        r, off = cg.dist_local(part, chunk_bits=chunk_bits)
        assert off[0] == 0 and off[-1] == r.shape[0] and all(a <= b for a, b in zip(off, off[1:]))
        runs.append(r)
        offs.append(off)
    table = torch.empty((sum(r.shape[0] for r in runs), W), dtype=torch.int64, device="cuda")
    nt = 0
    for c in range(C):
        pieces = [runs[g][offs[g][c]: offs[g][c + 1]] for g in range(G)]
        nt = cg.dist_merge_chunk(_pad_stack(pieces, torch.int64, (W,)), [p.shape[0] for p in pieces],
                                 ell, chunk_bits, table, nt)
    table = table[:nt]
    edges, stats = [], []
    for r in range(G):
        e, st = cg.dist_probe(table, ell, G, r, want_stats=True)
        edges.append(e)
        stats.append(st)
    ecounts = [e.shape[0] for e in edges]
    final = cg.dist_finalize(_pad_stack(edges, torch.int32, (2,)), ecounts)
    torch.cuda.synchronize()
    return (table.cpu().numpy().view(np.uint64), final.cpu().numpy().view(np.uint32), ecounts,
            stats)


@pytest.mark.parametrize("chunk_bits", [0, 3])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_logical_ranks_vs_oracle(cg, G, chunk_bits):
    x = synth.clustered_bytes(G, 60000, 100, n_centers=6, max_flips=3)
    x = np.concatenate([x, x[:9999]])  # duplicates across ranks
    c, e, ecounts, _ = logical_ranks(cg, x, G, chunk_bits)
    rc, oc, oe = oracle.build(x)
    assert rc == 0
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(e, oe)
    if G > 1:
        assert sum(1 for k in ecounts if k > 0) >= 2  # the work is really split


@pytest.mark.parametrize("ell", [64, 128, 300])
def test_logical_ranks_words(cg, ell):
    """W = 1, 2 (MSD merge of the chunk pieces) and W = 5 (full sort)."""
    d, _ = synth.planted_bytes(ell, 20000, ell)
    c, e, _, _ = logical_ranks(cg, d, 4, 2)
    rc, oc, oe = oracle.build(d)
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(e, oe)


@pytest.mark.parametrize("ell,G,chunk_bits", [(64, 4, 0), (128, 4, 2), (128, 8, 3), (100, 3, 1)])
def test_merge_with_cross_rank_duplicates(cg, ell, G, chunk_bits):
    """Random rows (the bucket merge path: every bucket fits the shared-memory
    capacity) with 20 % of the rows repeated on other ranks: the direct
    G-way merge must drop the copies and close the gaps."""
    d, _ = synth.planted_bytes(ell + G, 30000, ell)
    rng = np.random.default_rng(ell + G)
    x = np.concatenate([d, d[rng.integers(0, d.shape[0], d.shape[0] // 5)]])
    x = x[rng.permutation(x.shape[0])]
    c, e, _, _ = logical_ranks(cg, x, G, chunk_bits)
    rc, oc, oe = oracle.build(x)
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(e, oe)


def test_logical_ranks_c5_recipe_vs_oracle(cg):
    d = synth.config("C5", scale_log2=18)
    x = synth.unpack_words_np(d["words"], 128)
    c, e, ecounts, _ = logical_ranks(cg, x, 4)
    rc, oc, oe = oracle.build(x)
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(e, oe)
    # equal-weight cuts: no rank gets more than ~1.5x its share of the edges
    assert max(ecounts) < 1.5 * (sum(ecounts) / 4) + 64


def test_rank_dictionary_is_its_layers(cg):
    """G = 8 on the C5 recipe (2^20 cells): every rank's dictionary holds its
    sources plus the popcount layers one above them -- about 1/G of the
    table plus one layer -- and its index bytes shrink accordingly; the
    result is the oracle's."""
    G = 8
    d = synth.config("C5", scale_log2=20)
    x = synth.unpack_words_np(d["words"], 128)
    c, e, _, stats = logical_ranks(cg, x, G)
    rc, oc, oe = oracle.build(x)
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(e, oe)
    nc = oc.shape[0]
    layer = np.bincount(popcount_rows(oc), minlength=129)
    _, st1 = cg.dist_probe(torch.from_numpy(oc.view(np.int64)).cuda(), 128, 1, 0, want_stats=True)
    assert st1["dict_cells"] == nc
    for st in stats:
        assert st["dict_cells"] <= nc / G + 1.3 * layer.max() + (1 << 16)
        # the prefix index is sized in powers of two: at most 2x the cell share
        assert st["dict_bytes"] <= st1["dict_bytes"] * 2 * st["dict_cells"] / nc + 4096
    assert sum(st["logical_probes"] for st in stats) == nc * 128  # every cell probed once


def test_dist_errors(cg):
    pieces = torch.zeros((2, 4, 2), dtype=torch.int64, device="cuda")
    table = torch.zeros((16, 2), dtype=torch.int64, device="cuda")
    with pytest.raises(cg.CgError):
        cg.dist_merge_chunk(pieces, [5, 1], 128, 0, table, 0)  # count > stride
    with pytest.raises(cg.CgError):
        cg.dist_merge_chunk(pieces, [4, 4], 128, 0, table, 10)  # capacity
    with pytest.raises(cg.CgError):
        cg.dist_probe(table, 128, 2, 2)  # rank >= G
    with pytest.raises(cg.CgError):
        cg.dist_local(torch.zeros((4, 8), dtype=torch.uint8, device="cuda"), chunk_bits=9)
