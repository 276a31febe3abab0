"""Oracle pins for row f1 (cell signatures of sampled points):
the paper's Figure 1 table, the tie rule, error handling, and the
arrangement closed forms reached from FP64 points through the signature
oracle + ORACLE-A (CPU only)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))


def _load_fig1_points():
    sec, planes, points, sig = None, [], [], []
    for ln in open(os.path.join(HERE, "golden", "fig1_points.txt")):
        ln = ln.strip()
        if not ln or ln.startswith("#"):
            continue
        if ln.startswith("["):
            sec = ln
            continue
        f = ln.split()
        if sec == "[planes]":
            planes.append([float(v) for v in f])
        elif sec == "[points]":
            points.append([float(v) for v in f[1:]])
        elif sec == "[signatures]":
            sig.append([int(c) for c in f[1]])
    return np.array(points), np.array(planes), np.array(sig, dtype=np.uint8)


def test_fig1_table_from_points():
    """the four points' representations are 111, 110, 100, 101."""
    P, A, sig = _load_fig1_points()
    rc, b = oracle.signatures(P, A)
    assert rc == 0
    assert np.array_equal(b, sig)
    sp, sa = synth.fig1_points()
    assert np.array_equal(sp, P) and np.array_equal(sa, A)
    # and the cell graph is the 4-cycle of Figure 1 (tests/golden/fig1.txt)
    rc, cells, edges = oracle.build(b)
    assert rc == 0 and edges.tolist() == [[0, 1], [0, 2], [1, 3], [2, 3]]


def test_tie_counts_as_satisfied():
    """DESIGN G12: a point on the plane satisfies it, also for -0.0 values."""
    A = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, -2.0], [-1.0, 0.0, 0.0]])
    P = np.array([[0.0, 2.0], [-0.0, 2.0], [1.0, 1.0]])
    rc, b = oracle.signatures(P, A)
    assert rc == 0
    assert b.tolist() == [[1, 1, 1], [1, 1, 1], [1, 0, 0]]


def test_nonfinite_is_einput():
    A = np.array([[1.0, 0.0, 0.0]])
    rc, _ = oracle.signatures(np.array([[np.nan, 0.0]]), A)
    assert rc == oracle.EINPUT
    rc, _ = oracle.signatures(np.array([[1.0, 0.0]]), np.array([[np.inf, 0.0, 0.0]]))
    assert rc == oracle.EINPUT
    rc, _ = oracle.signatures(np.array([[2.0 ** 61, 0.0]]), np.array([[1.0, 0.0, 0.0]]))
    assert rc == oracle.EINPUT
    rc, _ = oracle.signatures(np.array([[2.0 ** 60, 0.0]]), np.array([[1.0, 0.0, 0.0]]))
    assert rc == 0


def test_fma_order_is_the_definition():
    """DESIGN G21: v = fma(a_0, p_0, b).  a_0 = 1 + 2^-27, p_0 = 1 - 2^-27:
    the exact product is 1 - 2^-54, so the fused value with b = -1 is
    -2^-54 < 0 (bit 0), while a separately rounded product (1 - 2^-54 rounds
    to even, 1.0) would give 0 and bit 1."""
    e = 2.0 ** -27
    A = np.array([[1.0 + e, -1.0]])
    rc, b = oracle.signatures(np.array([[1.0 - e]]), A)
    assert rc == 0 and b.tolist() == [[0]]


@pytest.mark.parametrize("dim,k", [(2, 3), (2, 5), (2, 12), (2, 25), (3, 4), (3, 6), (3, 10)])
def test_arrangement_closed_form_from_points(dim, k):
    """Every cell of a simple arrangement is hit by the vertex points, so the
    signature oracle + ORACLE-A give the closed-form cell and edge counts
    (2-D: 1 + k + C(k,2), k^2; 3-D: sum C(k,i), k sum C(k-1,i))."""
    P, A = synth.arrangement_points(100 * dim + k, k, dim)
    rc, b = oracle.signatures(P, A)
    assert rc == 0
    rc, cells, edges = oracle.build(b)
    assert rc == 0
    assert (cells.shape[0], edges.shape[0]) == synth.arrangement_cells_edges(k, dim)
    # ORACLE-B agrees on the small ones
    if P.shape[0] <= 4000:
        rc2, c2, e2 = oracle.brute(b)
        assert rc2 == 0 and np.array_equal(c2, cells) and np.array_equal(e2, edges)


def test_k3_lines_is_figure1_full_arrangement():
    """Three lines in general position, as in Figure 1: 7 of the 8 sign
    patterns occur ("no point is represented by 000" there), 9 = 3^2
    edges."""
    P, A = synth.arrangement_points(7, 3, 2)
    rc, b = oracle.signatures(P, A)
    rc, cells, edges = oracle.build(b)
    assert cells.shape[0] == 7 and edges.shape[0] == 9
