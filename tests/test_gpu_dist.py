"""Distributed phases on one GPU with logical ranks: cg_dist_local per row
shard, the gathered runs, cg_dist_merge_probe for every rank, the gathered
edge lists and cg_dist_finalize must reproduce cg_build byte for byte for any
number of ranks G (P14: G-invariance)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

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


def logical_ranks(cg, x: np.ndarray, G: int, dict_kind="global"):
    n, ell = x.shape
    W = (ell + 63) // 64
    xt = torch.from_numpy(x).cuda()
    runs = [cg.dist_local(xt[n * g // G: n * (g + 1) // G]) for g in range(G)]
    counts = [r.shape[0] for r in runs]
    stacked = _pad_stack(runs, torch.int64, (W,))
    tables, edges = [], []
    for r in range(G):
        t, e, _ = cg.dist_merge_probe(stacked, counts, r, ell, dict_kind=dict_kind)
        tables.append(t)
        edges.append(e)
    for t in tables[1:]:
        assert torch.equal(t, tables[0])
    ecounts = [e.shape[0] for e in edges]
    final = cg.dist_finalize(_pad_stack(edges, torch.int32, (2,)), ecounts, dict_kind=dict_kind)
    torch.cuda.synchronize()
    return (tables[0].cpu().numpy().view(np.uint64), final.cpu().numpy().view(np.uint32),
            ecounts)


@pytest.mark.parametrize("dict_kind", ["global", "sorted"])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_logical_ranks_match_single_build(cg, G, dict_kind):
    x = synth.clustered_bytes(G, 60000, 100, n_centers=6, max_flips=3)
    x = np.concatenate([x, x[:9999]])
    res = cg.build(torch.from_numpy(x).cuda())
    want_c = res.cells.cpu().numpy().view(np.uint64)
    want_e = res.edges.cpu().numpy().view(np.uint32)
    c, e, ecounts = logical_ranks(cg, x, G, dict_kind)
    # the oracle decides (P14 G-invariance on top: equal to the 1-GPU build)
    rc, oc, oe = oracle.build(x)
    assert rc == 0
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(e, oe)
    np.testing.assert_array_equal(c, want_c)
    np.testing.assert_array_equal(e, want_e)
    if G > 1:
        assert sum(1 for k in ecounts if k > 0) >= 2  # the work is really split


def test_logical_ranks_c5_recipe_vs_oracle(cg):
    d = synth.config("C5", scale_log2=18)
    x = synth.unpack_words_np(d["words"], 128)
    c, e, ecounts = logical_ranks(cg, x, 4)
    rc, oc, oe = oracle.build(x)
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(e, oe)
    # equal-weight cuts: no rank gets more than ~2x its share of the edges
    assert max(ecounts) < 2 * (sum(ecounts) / 4) + 64


def test_dist_errors(cg):
    runs = torch.zeros((2, 4, 2), dtype=torch.int64, device="cuda")
    with pytest.raises(cg.CgError):
        cg.dist_merge_probe(runs, [5, 1], 0, 128)  # count > stride
    with pytest.raises(cg.CgError):
        cg.dist_merge_probe(runs, [1, 1], 2, 128)  # rank >= G
