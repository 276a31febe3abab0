"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element, on seeded inputs of the paper's workload shapes (BASELINE configs),
plus the paper fixtures, sweeps over ell (ragged tails, multi-word keys),
duplicates, options, cg_query, cg_build_host and error paths.

The bar is bit-exact (DESIGN "Parity"): same cell table bytes, same edge list."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from helpers import check_invariants, load_golden, words_from_strings

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1503_06029_b200 import build_lib

    build_lib.build()
    import paper_1503_06029_b200 as cg

    cg.lib()
    return cg


def gpu_build(cg, x: np.ndarray, **kw):
    res = cg.build(torch.from_numpy(np.ascontiguousarray(x)).cuda(), **kw)
    torch.cuda.synchronize()
    cells = res.cells.cpu().numpy().view(np.uint64)
    edges = res.edges.cpu().numpy().view(np.uint32)
    return cells, edges, res


def assert_parity(cg, x, ell=None, **kw):
    cells, edges, res = gpu_build(cg, x, **kw)
    rc, oc, oe = oracle.build(x)
    assert rc == 0
    assert cells.shape == oc.shape, (cells.shape, oc.shape)
    np.testing.assert_array_equal(cells, oc)
    assert edges.shape == oe.shape, (edges.shape, oe.shape)
    np.testing.assert_array_equal(edges, oe)
    return cells, edges, res


# ---------------------------------------------------------------- paper fixtures
@pytest.mark.parametrize("name", ["fig1.txt", "fig1_full.txt", "fig2.txt"])
def test_paper_figures(cg, name):
    x, cells, edges = load_golden(name)
    c, e, _ = assert_parity(cg, x)
    np.testing.assert_array_equal(c, words_from_strings(cells))
    np.testing.assert_array_equal(e, edges)


# ---------------------------------------------------------------- BASELINE configs
def test_c1_planted(cg):
    d = synth.config("C1")
    c, e, _ = assert_parity(cg, d["bytes"])
    assert e.shape[0] == 500 and c.shape[0] == 1000


def test_c2_arrangement_closed_form(cg):
    d = synth.config("C2")
    c, e, _ = assert_parity(cg, d["bytes"])
    assert c.shape[0] == 20101 and e.shape[0] == 40000


def test_c3_uniform_arrangement(cg):
    d = synth.config("C3")
    c, e, res = assert_parity(cg, d["bytes"], want_stats=True)
    check_invariants(c, e, 64)


def test_c3_full_closed_form(cg):
    d = synth.config("C3F")
    c, e, _ = assert_parity(cg, d["bytes"])
    assert c.shape[0] == 43745 and e.shape[0] == 129088


@pytest.mark.parametrize("name,lg", [("C4", 14), ("C5", 20)])
def test_planted_reduced_vs_oracle(cg, name, lg):
    d = synth.config(name, scale_log2=lg)
    x = synth.unpack_words_np(d["words"], d["ell"])
    c, e, _ = assert_parity(cg, x)
    assert c.shape[0] == 1 << lg and e.shape[0] == 1 << (lg - 1)


def _expected_planted(words, pair_of):
    """Canonical table and planted edges from the generator (P7): canonical
    index by numpy lexsort of the word columns (word 0 most significant)."""
    W = words.shape[1]
    order = np.lexsort(tuple(words[:, w] for w in range(W - 1, -1, -1)))
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    o2 = np.argsort(pair_of, kind="stable")
    a, b = rank[o2[0::2]], rank[o2[1::2]]
    e = np.stack([np.minimum(a, b), np.maximum(a, b)], 1).astype(np.uint32)
    e = e[np.argsort(e[:, 0], kind="stable")]
    return words[order], e


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_planted_full_size(cg, name):
    """Full BASELINE size (C4: 2^20 x 1024; C5: 2^26 x 128), bytes made on the
    device from the generator's words; checked against the generator's planted
    pairs (every row is a cell, the edges are exactly the planted pairs)."""
    d = synth.config(name)
    words = d["words"]
    wt = torch.from_numpy(words.view(np.int64)).cuda()
    x = synth.unpack_words_torch(wt, d["ell"])
    del wt
    res = cg.build(x, want_stats=True)
    torch.cuda.synchronize()
    del x
    cells = res.cells.cpu().numpy().view(np.uint64)
    edges = res.edges.cpu().numpy().view(np.uint32)
    want_c, want_e = _expected_planted(words, d["pair_of"])
    assert cells.shape == want_c.shape
    np.testing.assert_array_equal(cells, want_c)
    assert edges.shape == want_e.shape
    np.testing.assert_array_equal(edges, want_e)
    st = res.stats
    assert st["n_cells"] == d["n"] and st["n_edges"] == d["n"] // 2
    assert st["logical_probes"] == d["n"] * d["ell"]


# ---------------------------------------------------------------- sweeps
ELLS = [1, 2, 3, 7, 31, 32, 33, 63, 64, 65, 127, 128, 129, 200, 255, 256, 257, 511, 512, 513,
        1024, 2049, 4096]


@pytest.mark.parametrize("ell", ELLS)
def test_ell_sweep_clustered_with_duplicates(cg, ell):
    x = synth.clustered_bytes(ell + 7, 5000 + ell, ell, n_centers=5, max_flips=3)
    x = np.concatenate([x, x[:777]])
    c, e, _ = assert_parity(cg, x)
    check_invariants(c, e, ell)


@pytest.mark.parametrize("n", [1, 2, 31, 33, 3071, 3073, 4095, 4097, 12289])
@pytest.mark.parametrize("sort_kind", ["auto", "nosmall"])
def test_ragged_sizes(cg, n, sort_kind):
    x = synth.clustered_bytes(n, n, 40, n_centers=3, max_flips=4)
    assert_parity(cg, x, sort_kind=sort_kind)


# ---------------------------------------------------------------- one-CTA small path
@pytest.mark.parametrize("n,ell", [(1, 1), (2, 3), (1000, 32), (2047, 64), (2048, 64),
                                   (2048, 256), (2049, 256), (1500, 255), (1500, 257),
                                   (700, 129), (1024, 192)])
@pytest.mark.parametrize("kind", ["planted", "clustered"])
def test_small_path_edges(cg, n, ell, kind):
    """n <= 2048, ell <= 256 run in one CTA (bitonic sort, block-scan dedupe,
    binary-search probes); just past either limit the general path runs.
    Both against the oracle, with duplicates and dense Hamming-1 clusters."""
    if kind == "planted":
        x, _ = synth.planted_bytes(n + ell, max(1, n // 2), ell)
        x = x[:n] if x.shape[0] >= n else np.concatenate([x, x[: n - x.shape[0]]])
    else:
        x = synth.clustered_bytes(n + 3 * ell, n, ell, n_centers=3, max_flips=3)
    c, e, _ = assert_parity(cg, x)
    c2, e2, _ = gpu_build(cg, x, sort_kind="nosmall")
    np.testing.assert_array_equal(c, c2)
    np.testing.assert_array_equal(e, e2)


def test_small_path_errors_and_options(cg):
    x = synth.clustered_bytes(9, 500, 40, n_centers=3, max_flips=3)
    assert_parity(cg, x, lcp_prune=False)
    assert_parity(cg, x, dict_kind="hash")
    bad = x.copy()
    bad[17, 5] = 2
    with pytest.raises(cg.CgError) as ei:
        cg.build(torch.from_numpy(bad).cuda())
    assert ei.value.code == -2  # CG_EINPUT


def test_random_uniform_many_layers(cg):
    x = synth.random_bytes(3, 200000, 20, dup_frac=0.3)
    assert_parity(cg, x)


def test_hypercube_closed_form(cg):
    for ell in (12, 20):
        x = synth.hypercube(ell)
        x = x[np.random.default_rng(ell).permutation(x.shape[0])]
        c, e, res = gpu_build(cg, x, want_stats=True)
        n = 1 << ell
        np.testing.assert_array_equal(c[:, 0] >> np.uint64(64 - ell), np.arange(n, dtype=np.uint64))
        v = np.arange(n, dtype=np.int64)
        pairs = [np.stack([v[(v >> b) & 1 == 0], v[(v >> b) & 1 == 0] + (1 << b)], 1)
                 for b in range(ell)]
        want = np.concatenate(pairs)
        want = want[np.lexsort((want[:, 1], want[:, 0]))].astype(np.uint32)
        np.testing.assert_array_equal(e, want)  # m = ell * 2^(ell-1), every degree = ell


@pytest.mark.parametrize("dict_kind", ["global", "sorted", "hash"])
def test_dense_ball_tile_overflow(cg, dict_kind):
    """All vectors of weight <= 2 (ell = 100): weight-1 cells have 99
    out-edges each, so a 256-cell tile of the canonical-order probe overflows
    its shared edge buffer and takes the spill path."""
    ell = 100
    rows = [np.zeros(ell, np.uint8)]
    for a in range(ell):
        r = np.zeros(ell, np.uint8)
        r[a] = 1
        rows.append(r)
        for b2 in range(a + 1, ell):
            r2 = r.copy()
            r2[b2] = 1
            rows.append(r2)
    x = np.stack(rows)[np.random.default_rng(0).permutation(len(rows))]
    c, e, res = assert_parity(cg, x, dict_kind=dict_kind, want_stats=True)
    assert e.shape[0] == ell + ell * (ell - 1)


def test_all_identical_and_single(cg):
    c, e, _ = assert_parity(cg, np.ones((1000, 70), np.uint8))
    assert c.shape[0] == 1 and e.shape[0] == 0
    c, e, _ = assert_parity(cg, np.zeros((1, 5), np.uint8))
    assert c.shape[0] == 1 and e.shape[0] == 0


def test_multiset_x3_and_permutation(cg):
    x = synth.clustered_bytes(5, 20000, 96, n_centers=6, max_flips=3)
    c0, e0, _ = gpu_build(cg, x)
    rng = np.random.default_rng(1)
    x3 = np.concatenate([x, x, x])[rng.permutation(3 * x.shape[0])]
    c1, e1, _ = gpu_build(cg, x3)
    np.testing.assert_array_equal(c0, c1)
    np.testing.assert_array_equal(e0, e1)


@pytest.mark.parametrize("kw", [dict(), dict(lcp_prune=False), dict(dict_kind="bsearch"),
                                dict(dict_kind="sorted"), dict(dict_kind="sorted", lcp_prune=False),
                                dict(dict_kind="bsearch", lcp_prune=False), dict(bucket_log2=0),
                                dict(bucket_log2=6), dict(dict_kind="sorted", bucket_log2=0),
                                dict(edge_cap=1), dict(dict_kind="sorted", edge_cap=1),
                                dict(dict_kind="hash"), dict(dict_kind="hash", lcp_prune=False),
                                dict(dict_kind="hash", edge_cap=1)],
                         ids=lambda kw: ",".join(f"{k}={v}" for k, v in kw.items()) or "default")
def test_options_vs_oracle(cg, kw):
    """Every dictionary / pruning / bucket / capacity option gives the oracle's
    bytes on an arrangement-like clustered input (ell = 150, W = 3) and on a
    C5-recipe planted input (W = 2)."""
    x = synth.clustered_bytes(8, 30000, 150, n_centers=8, max_flips=3)
    assert_parity(cg, x, **kw)
    d = synth.config("C5", scale_log2=15)
    assert_parity(cg, synth.unpack_words_np(d["words"], 128), **kw)


def test_lcp_prune_issues_fewer_probes(cg):
    x = synth.clustered_bytes(8, 30000, 150, n_centers=8, max_flips=3)
    _, _, r0 = gpu_build(cg, x, want_stats=True)
    _, _, rn = gpu_build(cg, x, want_stats=True, lcp_prune=False)
    assert r0.stats["issued_probes"] <= rn.stats["issued_probes"]


@pytest.mark.parametrize("case", ["C3", "C5small", "W1uniform", "W2dups"])
def test_sort_paths_agree(cg, case):
    """MSD fast path (prefix buckets + shared-memory bitonic sort, with the
    overflow fallback) and the full LSD path give identical bytes."""
    if case == "C3":  # heavy duplicates: buckets overflow -> fallback path
        x = synth.config("C3")["bytes"]
    elif case == "C5small":
        d = synth.config("C5", scale_log2=18)
        x = synth.unpack_words_np(d["words"], 128)
    elif case == "W1uniform":
        x = synth.random_bytes(4, 300000, 64)
    else:
        x = synth.random_bytes(6, 200000, 100, dup_frac=0.5)
    c0, e0, _ = gpu_build(cg, x, sort_kind="auto")
    c1, e1, _ = gpu_build(cg, x, sort_kind="lsd")
    np.testing.assert_array_equal(c0, c1)
    np.testing.assert_array_equal(e0, e1)
    rc, oc, oe = oracle.build(x)
    np.testing.assert_array_equal(c0, oc)
    np.testing.assert_array_equal(e0, oe)


def test_determinism(cg):
    d = synth.config("C3")
    c0, e0, _ = gpu_build(cg, d["bytes"])
    for _ in range(3):
        c1, e1, _ = gpu_build(cg, d["bytes"])
        assert np.array_equal(c0, c1) and np.array_equal(e0, e1)


# ---------------------------------------------------------------- packed + host entry points
def test_packed_entry(cg):
    d = synth.config("C5", scale_log2=14)
    wt = torch.from_numpy(d["words"].view(np.int64)).cuda()
    res = cg.build_packed(wt, 128)
    torch.cuda.synchronize()
    rc, oc, oe = oracle.build_packed(d["words"], 128)
    np.testing.assert_array_equal(res.cells.cpu().numpy().view(np.uint64), oc)
    np.testing.assert_array_equal(res.edges.cpu().numpy().view(np.uint32), oe)


def test_host_entry(cg):
    d = synth.config("C2")
    xh = torch.from_numpy(d["bytes"]).pin_memory()
    cells, edges, _ = cg.build_host(xh)
    rc, oc, oe = oracle.build(d["bytes"])
    np.testing.assert_array_equal(cells.view(np.uint64), oc)
    np.testing.assert_array_equal(edges.view(np.uint32), oe)


# ---------------------------------------------------------------- cg_query
@pytest.mark.parametrize("dict_kind", ["global", "sorted"])
def test_query_against_oracle(cg, dict_kind):
    x = synth.clustered_bytes(21, 8000, 77, n_centers=4, max_flips=3)
    cells, edges, res = gpu_build(cg, x, want_index=True, dict_kind=dict_kind)
    idx = res.index
    assert idx is not None and idx.n_cells == cells.shape[0]
    rng = np.random.default_rng(2)
    extra = synth.clustered_bytes(22, 500, 77, n_centers=4, max_flips=5)
    from helpers import words_from_rows

    q = np.concatenate([cells, words_from_rows(extra)])
    q_dirty = q.copy()
    q_dirty[:, -1] |= np.uint64((1 << (64 - 77 % 64)) - 1)  # pad bits must be ignored
    qt = torch.from_numpy(q_dirty.view(np.int64)).cuda()
    s, nb = idx.query(qt)
    torch.cuda.synchronize()
    rc, os_, onb = oracle.query(cells, 77, q)
    assert rc == 0
    np.testing.assert_array_equal(s.cpu().numpy(), os_)
    np.testing.assert_array_equal(nb.cpu().numpy(), onb)
    # consistency with the edge list: row i of the adjacency
    s_cells = s.cpu().numpy()[: cells.shape[0]]
    assert np.array_equal(s_cells, np.arange(cells.shape[0]))
    assert int((nb.cpu().numpy()[: cells.shape[0]] >= 0).sum()) == 2 * edges.shape[0]


# ---------------------------------------------------------------- errors
def test_input_validation(cg):
    x = np.zeros((100, 16), np.uint8)
    x[57, 3] = 2
    with pytest.raises(cg.CgError) as ei:
        cg.build(torch.from_numpy(x).cuda())
    assert ei.value.code == -2
    # the stream and library stay usable after an error
    assert_parity(cg, synth.clustered_bytes(1, 100, 16))


def test_host_pointer_rejected(cg):
    import ctypes

    from paper_1503_06029_b200 import cg as cgm

    xh = torch.zeros((10, 8), dtype=torch.uint8)
    c, e = cgm.cg_cells(), cgm.cg_edges()
    rc = cgm.lib().cg_build(ctypes.c_void_p(xh.data_ptr()), 10, 8, ctypes.byref(c), ctypes.byref(e))
    assert rc == cgm.CG_EINVAL


def test_loaded_library_is_in_tree(cg):
    import os

    from paper_1503_06029_b200 import cg as cgm

    maps = open("/proc/self/maps").read()
    assert os.path.realpath(cgm.LIB_PATH) in maps or cgm.LIB_PATH in maps


@pytest.mark.parametrize("ell,n", [(64, 1 << 19), (128, 1 << 19), (200, 300000), (1024, 1 << 18)])
def test_heavy_duplication_hash_path(cg, ell, n):
    """Skewed inputs (few distinct cells) at n >= 2^18 overflow the MSD
    buckets and go through the hash dedupe + full sort of the distinct rows."""
    rng = np.random.default_rng(ell + n)
    base = synth.clustered_bytes(ell, 4000, ell, 6, 2)
    x = np.ascontiguousarray(base[rng.integers(0, base.shape[0], size=n)])
    cells, edges, _ = gpu_build(cg, x)
    rc, oc, oe = oracle.build(x)
    assert rc == 0
    assert np.array_equal(cells, oc) and np.array_equal(edges, oe)


@pytest.mark.parametrize("fextra", [0, 2, 4, 5, 8])
@pytest.mark.parametrize("dict_kind", ["global", "sorted"])
def test_filter_resolution(cg, fextra, dict_kind):
    """The prefix filter's extra bits (cg_opts.filter_extra) change only which
    far flips reach a bucket search, never the result; fextra >= 5 takes the
    probe's word-only filter test, smaller values the general one."""
    d = synth.config("C5", scale_log2=16)
    x = synth.unpack_words_np(d["words"], d["ell"])
    assert_parity(cg, x, filter_extra=fextra, dict_kind=dict_kind)
    assert_parity(cg, synth.clustered_bytes(7, 3000, 96, 5, 2), filter_extra=fextra,
                  dict_kind=dict_kind)


def test_bad_options_rejected(cg):
    x = torch.zeros((10, 8), dtype=torch.uint8, device="cuda")
    for kw in (dict(filter_extra=9), dict(filter_extra=-2), dict(edge_cap=-1), dict(sort_kind=5)):
        with pytest.raises(cg.CgError) as ei:
            cg.build(x, **kw)
        assert ei.value.code == -1


# ---------------------------------------------------------------- long rows (W > 2)
@pytest.mark.parametrize("ell,dup,dict_kind", [(300, 0.0, "global"), (300, 0.1, "global"),
                                               (1024, 0.2, "global"), (300, 0.0, "sorted"),
                                               (520, 0.1, "sorted"), (2048, 0.05, "global"),
                                               (1024, 0.1, "hash"), (64, 0.1, "hash"),
                                               (128, 0.0, "hash")])
def test_long_rows_prefix_sort_paths(cg, ell, dup, dict_kind):
    """Random long rows with planted partners: the (32-bit prefix, index) sort
    succeeds (short tie runs); without duplicates the rows go straight to the
    cell table (no dedupe pass), with duplicates the warp-cooperative
    gather + dedupe runs; the layered dictionary needs popcount/lcp."""
    x, _ = synth.planted_bytes(ell, 6000, ell)
    rng = np.random.default_rng(ell)
    if dup:
        x = np.concatenate([x, x[rng.integers(0, x.shape[0], int(dup * x.shape[0]))]])
    x = x[rng.permutation(x.shape[0])]
    assert_parity(cg, x, dict_kind=dict_kind)


# ---------------------------------------------------------------- hash dictionary
@pytest.mark.parametrize("ell", [1, 7, 64, 65, 128, 200, 1024, 4096])
def test_hash_dictionary_sweep(cg, ell):
    """CG_DICT_HASH (open-addressed, h ^ Z[k] per flip) gives the oracle's
    graph on clustered inputs dense in Hamming-1 pairs and duplicates (hash
    collisions of distinct cells only cost verification)."""
    x = synth.clustered_bytes(ell + 11, 4000 + ell, ell, n_centers=4, max_flips=3)
    x = np.concatenate([x, x[:333]])
    assert_parity(cg, x, dict_kind="hash")


def test_hash_dictionary_arrangement_and_hypercube(cg):
    d = synth.config("C2")
    assert_parity(cg, d["bytes"], dict_kind="hash")
    x = synth.hypercube(14)
    assert_parity(cg, x[np.random.default_rng(3).permutation(x.shape[0])], dict_kind="hash")


def test_hash_dictionary_keeps_no_index(cg):
    x = torch.from_numpy(synth.random_bytes(1, 100, 16)).cuda()
    with pytest.raises(cg.CgError):
        cg.build(x, dict_kind="hash", want_index=True)


@pytest.mark.parametrize("ell", [200, 700])
def test_long_rows_long_ties_hash_then_sort(cg, ell):
    """n >= 2^15 rows of W > 2 words with long runs of equal 32-bit prefixes
    (clustered rows, heavy duplication): the prefix sort gives up, the copies
    are dropped by hashing and the distinct rows are sorted word by word."""
    x = synth.clustered_bytes(ell, 40000, ell, n_centers=5, max_flips=3)
    assert_parity(cg, x)


def test_auto_dictionary_choice(cg):
    """CG_DICT_AUTO (the default) takes the hash dictionary for long,
    heavily duplicated rows (C2: the arrangement with 10x duplication) and the
    prefix index otherwise; both give the oracle's graph (checked on C2 and
    C4-like rows) and an index request keeps the prefix index."""
    d = synth.config("C2")
    _, _, r = assert_parity(cg, d["bytes"], want_stats=True)
    assert r.stats["dict_bytes"] != 0
    x, _ = synth.planted_bytes(4, 3000, 300)
    assert_parity(cg, x)
    rr = cg.build(torch.from_numpy(d["bytes"]).cuda(), want_index=True)
    assert rr.index is not None
