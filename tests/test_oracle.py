"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY 8.c.5 P1-P13).  No GPU.  Each pin is chosen so a plausible oracle bug
(wrong bit order, dropped dedupe, reversed edge orientation, missing flip,
off-by-one on the last word) fails at least one of them."""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from helpers import (check_invariants, definition, load_golden, words_from_rows,
                     words_from_strings)


def _both(x, **kw):
    ra, ca, ea = oracle.build(x, self_check=True, **kw)
    rb, cb, eb = oracle.brute(x, **kw)
    assert ra == 0 and rb == 0
    return ca, ea, cb, eb


# ---------------------------------------------------------------- P1-P3 paper fixtures
@pytest.mark.parametrize("name", ["fig1.txt", "fig1_full.txt", "fig2.txt"])
def test_paper_figures(name):
    x, cells, edges = load_golden(name)
    ca, ea, cb, eb = _both(x)
    want = words_from_strings(cells)
    np.testing.assert_array_equal(ca, want)
    np.testing.assert_array_equal(ea, edges)
    np.testing.assert_array_equal(cb, want)
    np.testing.assert_array_equal(eb, edges)


def test_fig1_any_order_and_multiplicity():
    x, cells, edges = load_golden("fig1.txt")
    rng = np.random.default_rng(0)
    for _ in range(10):
        y = x[rng.integers(0, 4, size=12)]
        y = np.concatenate([x, y])[rng.permutation(16)]
        _, ea, _, eb = _both(y)
        np.testing.assert_array_equal(ea, edges)
        np.testing.assert_array_equal(eb, edges)


def test_fig2_msb_first_word_values():
    """P3: MSB-first word values of Fig. 2 rows increase in the printed order
    (0, 9, 27, 52, 54, 55 as 6-bit numbers); LSB-first values would not."""
    x, cells, _ = load_golden("fig2.txt")
    rc, ca, _ = oracle.build(x)
    vals = (ca[:, 0] >> np.uint64(58)).tolist()
    assert vals == [0, 9, 27, 52, 54, 55]
    lsb = [int(s[::-1], 2) for s in cells]
    assert lsb == [0, 36, 54, 11, 27, 59] and lsb != sorted(lsb)


# ---------------------------------------------------------------- P4/P5 closed forms
@pytest.mark.parametrize("k", [3, 5, 10, 25])
def test_arrangement2d_closed_form(k):
    x = synth.arrangement2d(100 + k, k, n_uniform=500)
    ca, ea, cb, eb = _both(x)
    assert ca.shape[0] == 1 + k + k * (k - 1) // 2
    assert ea.shape[0] == k * k
    np.testing.assert_array_equal(ca, cb)
    np.testing.assert_array_equal(ea, eb)
    check_invariants(ca, ea, k)


def test_c2_full_size_closed_form():
    d = synth.config("C2")
    rc, c, e = oracle.build(d["bytes"])
    assert rc == 0
    assert c.shape[0] == d["expect_cells"] == 20101
    assert e.shape[0] == d["expect_edges"] == 40000
    check_invariants(c, e, 200)


@pytest.mark.parametrize("k", [4, 6, 10, 14])
def test_arrangement3d_closed_form(k):
    x = synth.arrangement3d_full(200 + k, k)
    ca, ea, cb, eb = _both(x)
    assert ca.shape[0] == sum(math.comb(k, i) for i in range(4))
    assert ea.shape[0] == k * sum(math.comb(k - 1, i) for i in range(3))
    np.testing.assert_array_equal(ca, cb)
    np.testing.assert_array_equal(ea, eb)


def test_c3_full_size_closed_form():
    d = synth.config("C3F")
    rc, c, e = oracle.build(d["bytes"])
    assert rc == 0
    assert c.shape[0] == d["expect_cells"] == 43745
    assert e.shape[0] == d["expect_edges"] == 129088
    check_invariants(c, e, 64)


# ---------------------------------------------------------------- P6 hypercube
@pytest.mark.parametrize("ell", [1, 2, 3, 5, 8, 10])
def test_hypercube(ell):
    x = synth.hypercube(ell)
    x = x[np.random.default_rng(ell).permutation(x.shape[0])]
    ca, ea, cb, eb = _both(x)
    n = 1 << ell
    # V_i = i (as an ell-bit number, bit 0 most significant)
    np.testing.assert_array_equal(ca[:, 0] >> np.uint64(64 - ell), np.arange(n, dtype=np.uint64))
    want = sorted((v, v + (1 << b)) for v in range(n) for b in range(ell) if not (v >> b) & 1)
    assert ea.shape[0] == ell * (1 << (ell - 1))
    np.testing.assert_array_equal(ea, np.array(want, np.uint32))
    np.testing.assert_array_equal(eb, ea)
    deg = np.bincount(ea.ravel(), minlength=n)
    assert np.all(deg == ell)  # the P:106 degree bound met exactly


# ---------------------------------------------------------------- P7 planted pairs
def _planted_expected(x, pair_of):
    """Expected edges from the generator's own knowledge, via numpy's row
    sort (independent of the oracle): canonical index of each row by
    np.unique(axis=0) (lexicographic order of the byte rows)."""
    u, inv = np.unique(x, axis=0, return_inverse=True)
    inv = inv.ravel()
    order = np.argsort(pair_of, kind="stable")
    a, b = inv[order[0::2]], inv[order[1::2]]
    e = np.stack([np.minimum(a, b), np.maximum(a, b)], 1)
    e = e[np.lexsort((e[:, 1], e[:, 0]))]
    return words_from_rows(u), e.astype(np.uint32)


def test_c1_planted_exact():
    d = synth.config("C1")
    cells_w, e_w = _planted_expected(d["bytes"], d["pair_of"])
    ca, ea, cb, eb = _both(d["bytes"])
    assert ea.shape[0] == 500
    np.testing.assert_array_equal(ca, cells_w)
    np.testing.assert_array_equal(ea, e_w)
    np.testing.assert_array_equal(eb, e_w)


@pytest.mark.parametrize("name,lg", [("C4", 10), ("C5", 12)])
def test_planted_recipe_small(name, lg):
    d = synth.config(name, scale_log2=lg)
    x = synth.unpack_words_np(d["words"], d["ell"])
    cells_w, e_w = _planted_expected(x, d["pair_of"])
    rc, ca, ea = oracle.build(x)
    assert rc == 0
    np.testing.assert_array_equal(ca, cells_w)
    np.testing.assert_array_equal(ea, e_w)
    # the packed entry point agrees with the byte entry point
    rc2, cp, ep = oracle.build_packed(d["words"], d["ell"])
    assert rc2 == 0
    np.testing.assert_array_equal(cp, ca)
    np.testing.assert_array_equal(ep, ea)


# ---------------------------------------------------------------- P8 A == B sweeps
ELLS = [1, 2, 3, 7, 31, 32, 33, 63, 64, 65, 127, 128, 129, 200, 255, 256, 257, 511, 512, 513, 1024]


@pytest.mark.parametrize("ell", ELLS)
def test_a_equals_b_sweep(ell):
    for seed, dup in ((ell, 0.0), (ell + 1000, 0.5)):
        x = synth.clustered_bytes(seed, 400, ell, n_centers=4, max_flips=2)
        if dup:
            x = np.concatenate([x, x[: int(dup * len(x))]])
        ca, ea, cb, eb = _both(x)
        np.testing.assert_array_equal(ca, cb)
        np.testing.assert_array_equal(ea, eb)
        check_invariants(ca, ea, ell)
        if ell <= 64:
            x2 = synth.random_bytes(seed, 300, ell, dup_frac=dup)
            ca, ea, cb, eb = _both(x2)
            np.testing.assert_array_equal(ca, cb)
            np.testing.assert_array_equal(ea, eb)


def test_a_equals_definition_tiny():
    rng = np.random.default_rng(5)
    for _ in range(200):
        ell = int(rng.integers(1, 9))
        n = int(rng.integers(1, 40))
        x = rng.integers(0, 2, size=(n, ell), dtype=np.uint8)
        cw, ew = definition(x)
        ca, ea, cb, eb = _both(x)
        np.testing.assert_array_equal(ca, cw)
        np.testing.assert_array_equal(ea, ew)
        np.testing.assert_array_equal(cb, cw)
        np.testing.assert_array_equal(eb, ew)


# ---------------------------------------------------------------- P9/P10 invariance
def test_multiset_and_permutation_invariance():
    x = synth.clustered_bytes(9, 500, 70, n_centers=3, max_flips=3)
    rc, c0, e0 = oracle.build(x)
    rng = np.random.default_rng(9)
    x3 = np.concatenate([x, x, x])[rng.permutation(3 * len(x))]
    rc, c1, e1 = oracle.build(x3)
    np.testing.assert_array_equal(c0, c1)
    np.testing.assert_array_equal(e0, e1)
    rc, c2, e2 = oracle.build(x[rng.permutation(len(x))], nthreads=3)
    np.testing.assert_array_equal(c0, c2)
    np.testing.assert_array_equal(e0, e2)


# ---------------------------------------------------------------- P12 exhaustive
@pytest.mark.parametrize("ell", [1, 2, 3, 4])
def test_exhaustive_subsets(ell):
    allv = synth.hypercube(ell)
    N = 1 << ell
    masks = range(1, 1 << N)
    if ell == 4:  # 65535 subsets: every 7th one plus all small/large ones
        masks = [m for m in masks if m % 7 == 0 or bin(m).count("1") <= 2
                 or bin(m).count("1") >= N - 2]
    for m in masks:
        x = allv[[i for i in range(N) if (m >> i) & 1]]
        cw, ew = definition(x)
        rc, ca, ea = oracle.build(x, nthreads=1)
        assert rc == 0
        np.testing.assert_array_equal(ca, cw)
        np.testing.assert_array_equal(ea, ew)


def test_exhaustive_ell4_a_equals_b():
    """All 2^16 - 1 nonempty subsets of {0,1}^4: ORACLE-A == ORACLE-B."""
    allv = synth.hypercube(4)
    for m in range(1, 1 << 16):
        x = allv[[i for i in range(16) if (m >> i) & 1]]
        ra, ca, ea = oracle.build(x, nthreads=1)
        rb, cb, eb = oracle.brute(x, nthreads=1)
        assert ea.shape == eb.shape and np.array_equal(ea, eb) and np.array_equal(ca, cb)


# ---------------------------------------------------------------- P13 SPEC examples + query
def test_spec_examples_pack_flip_distance():
    # pack [1,1,1] -> "111";  get_bit("110", 2) = 0
    rc, c, _ = oracle.build(np.array([[1, 1, 1]], np.uint8))
    assert int(c[0, 0]) == 0b111 << 61
    rc, c, _ = oracle.build(np.array([[1, 1, 0]], np.uint8))
    assert (int(c[0, 0]) >> 61) & 1 == 0
    # flip_bit("111", 2) = "110" and dist = 1: an edge
    rc, c, e = oracle.build(np.array([[1, 1, 1], [1, 1, 0]], np.uint8))
    assert e.tolist() == [[0, 1]]
    # dist("110","101") = 2: no edge
    rc, c, e = oracle.build(np.array([[1, 1, 0], [1, 0, 1]], np.uint8))
    assert e.shape[0] == 0


def test_query_fig2_lookup_examples():
    """Fig. 2 table, 001001 -> index 1; 000001 (digits 001) absent."""
    x, cells, _ = load_golden("fig2.txt")
    rc, c, e = oracle.build(x)
    q = words_from_strings(["001001", "000001", "110110"])
    rc, s, nbr = oracle.query(c, 6, q)
    assert rc == 0
    assert s.tolist() == [1, -1, 4]
    # 110110: flipping bit 4 -> 110100 (index 3), bit 5 -> 110111 (index 5)
    assert nbr[2].tolist() == [-1, -1, -1, -1, 3, 5]
    # 000001 flipped at bit 5 -> 000000 (index 0)
    assert nbr[1, 5] == 0


def test_query_consistent_with_edges():
    x = synth.clustered_bytes(11, 300, 45, n_centers=3, max_flips=2)
    rc, c, e = oracle.build(x)
    rc, s, nbr = oracle.query(c, 45, c)
    assert np.array_equal(s, np.arange(c.shape[0]))
    adj = set(map(tuple, e.tolist()))
    for i in range(c.shape[0]):
        for k in range(45):
            j = nbr[i, k]
            if j >= 0:
                assert (min(i, j), max(i, j)) in adj
    assert (nbr >= 0).sum() == 2 * e.shape[0]


# ---------------------------------------------------------------- errors (G5, G10)
def test_error_codes():
    assert oracle.build(np.zeros((0, 8), np.uint8))[0] == oracle.EINVAL
    assert oracle.build(np.zeros((3, 0), np.uint8))[0] == oracle.EINVAL
    assert oracle.build(np.zeros((1, 4097), np.uint8))[0] == oracle.EINVAL
    assert oracle.build(np.zeros((1, 4096), np.uint8))[0] == 0
    bad = np.zeros((4, 9), np.uint8)
    bad[2, 3] = 2
    assert oracle.build(bad)[0] == oracle.EINPUT
    assert oracle.brute(bad)[0] == oracle.EINPUT
    w = np.array([[1]], np.uint64)  # pad bit set for ell = 3
    assert oracle.build_packed(w, 3)[0] == oracle.EINPUT


def test_degenerate_sizes():
    rc, c, e = oracle.build(np.ones((5, 17), np.uint8))
    assert c.shape == (1, 1) and e.shape[0] == 0
    rc, c, e = oracle.build(np.array([[0], [1], [1], [0]], np.uint8))
    assert c[:, 0].tolist() == [0, 1 << 63] and e.tolist() == [[0, 1]]


# ---------------------------------------------------------------- grid graphs (m >= 2^32 recipe)
def grid_closed_form(side: int, dims: int):
    """Cell graph of the thermometer-coded grid [side]^dims (synth.grid_words_np):
    Hamming distance 1 between two codes <=> grid neighbours (one axis moves by
    one step), and the canonical order is the mixed-radix order with axis 0
    most significant (00..0 < 10..0 < 110..0 < ... per axis).  So V_i = grid
    point i, and E = {(i, i + side^p) : digit p of i < side - 1}, ascending;
    n_c = side^dims, m = dims (side - 1) side^(dims - 1)."""
    n = side ** dims
    i = np.arange(n, dtype=np.int64)
    rows = []
    for p in range(dims):  # ascending p = ascending j for a fixed i
        d = (i // side ** p) % side
        j = np.where(d < side - 1, i + side ** p, -1)
        rows.append(j)
    J = np.stack(rows, axis=1)
    I = np.repeat(i, dims).reshape(n, dims)
    keep = J >= 0
    return n, np.stack([I[keep], J[keep]], axis=1).astype(np.uint32)


@pytest.mark.parametrize("side,dims,mult", [(3, 6, 7), (4, 4, 5), (5, 3, 2), (2, 9, 5), (3, 18, 1000003)])
def test_grid_closed_form(side, dims, mult):
    """Pins the generator of the full-size m >= 2^32 GPU test (3^18 cells,
    4,649,045,868 edges) on small grids: the oracle's graph of the
    thermometer-coded grid equals the grid graph in closed form (for 3^18
    only the counts, from the formula)."""
    if side ** dims > 10 ** 6:
        n, m = side ** dims, dims * (side - 1) * side ** (dims - 1)
        assert (n, m) == (387420489, 4649045868) and m >= 1 << 32
        return
    w, ell = synth.grid_words_np(side, dims, mult)
    rc, c, e = oracle.build_packed(w, ell)
    assert rc == 0
    n, want = grid_closed_form(side, dims)
    assert c.shape[0] == n
    assert e.shape[0] == dims * (side - 1) * side ** (dims - 1)
    np.testing.assert_array_equal(e, want)
    check_invariants(c, e, ell)
