"""Oracle pins for row f4 (CSR + BFS path queries on G_X, P:20, P:57,
P:423-424): closed forms that do not come from the oracle's own code.

* Hypercube H_l (all 2^l cells, cell v = the integer v): the BFS distance
  between s and v is popc(s ^ v) (a shortest path flips each differing bit
  once), every degree is l (the P:106 bound met), and the neighbours one
  step closer to s are v ^ 2^b for the differing bits b.
* Simple hyperplane arrangements: the cell graph is isometric to its
  embedding in the hypercube -- the distance between two cells equals the
  number of hyperplanes separating them, i.e. the Hamming distance of their
  signatures -- so BFS distances from any cell equal Hamming distances.
* Figure 1: from A, B and D are at distance 1, C at distance 2."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth


def _hamming_rows(cells: np.ndarray, s: int) -> np.ndarray:
    x = np.bitwise_xor(cells, cells[s][None, :])
    return np.array([sum(bin(int(w)).count("1") for w in row) for row in x])


@pytest.mark.parametrize("ell", [1, 2, 5, 8, 10])
def test_hypercube_distances_are_popcounts(ell):
    rc, cells, edges = oracle.build(synth.hypercube(ell))
    n = cells.shape[0]
    rc, rp, col = oracle.csr(edges, n)
    assert rc == 0
    assert np.all(np.diff(rp.astype(np.int64)) == ell)  # every degree = ell
    for s in {0, n - 1, n // 3}:
        rc, dist, parent = oracle.bfs(rp, col, s)
        assert rc == 0
        assert np.array_equal(dist, [bin(v ^ s).count("1") for v in range(n)])
        for v in range(n):
            if v == s:
                assert parent[v] == -1
            else:
                # a neighbour one step closer: v with one of its differing
                # bits moved back to s's value; the smallest such
                cands = [v ^ (1 << b) for b in range(ell) if ((v ^ s) >> b) & 1]
                assert parent[v] == min(cands)


@pytest.mark.parametrize("dim,k", [(2, 6), (2, 15), (3, 6), (3, 9)])
def test_arrangement_bfs_distance_is_hamming(dim, k):
    P, A = synth.arrangement_points(500 + 10 * dim + k, k, dim)
    rc, b = oracle.signatures(P, A)
    rc, cells, edges = oracle.build(b)
    n = cells.shape[0]
    rc, rp, col = oracle.csr(edges, n)
    for s in (0, n // 2, n - 1):
        rc, dist, parent = oracle.bfs(rp, col, s)
        assert np.all(dist >= 0)  # the cell graph of an arrangement is connected
        assert np.array_equal(dist, _hamming_rows(cells, s))


def test_fig1_distances():
    x = np.array([[1, 1, 1], [1, 1, 0], [1, 0, 0], [1, 0, 1]], dtype=np.uint8)  # A B C D
    rc, cells, edges = oracle.build(x)   # canonical: C=100, D=101, B=110, A=111
    rc, rp, col = oracle.csr(edges, 4)
    rc, dist, parent = oracle.bfs(rp, col, 3)  # from A
    assert dist.tolist() == [2, 1, 1, 0]      # C, D, B, A
    assert parent.tolist() == [1, 3, 3, -1]   # C via D (smaller than B), D and B via A


def test_unreachable_and_isolated():
    """Planted pairs: components of size 1-2; the rest is unreachable."""
    rc, cells, edges = oracle.build(synth.config("C1")["bytes"])
    n = cells.shape[0]
    rc, rp, col = oracle.csr(edges, n)
    s = int(edges[0, 0])
    rc, dist, parent = oracle.bfs(rp, col, s)
    assert sorted(dist.tolist()).count(0) == 1 and sorted(dist.tolist()).count(1) == 1
    assert (dist == -1).sum() == n - 2
    rc, rp0, col0 = oracle.csr(np.zeros((0, 2), np.uint32), 3)
    assert rp0.tolist() == [0, 0, 0, 0]
    rc, dist, parent = oracle.bfs(rp0, col0, 1)
    assert dist.tolist() == [-1, 0, -1] and parent.tolist() == [-1, -1, -1]
