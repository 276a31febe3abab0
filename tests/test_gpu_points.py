"""GPU parity for row f1: cg_signatures / cg_build_points (signatures computed
and packed on the device) vs the CPU oracle's signatures (same fma order,
DESIGN G21) + ORACLE-A, bit-exact."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from helpers import check_invariants

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


def _pack_bytes(b: np.ndarray) -> np.ndarray:
    """Reference packing of oracle bytes into the ABI word format (test helper)."""
    n, ell = b.shape
    W = (ell + 63) // 64
    pad = np.zeros((n, W * 64), dtype=np.uint8)
    pad[:, :ell] = b
    return np.packbits(pad, axis=1, bitorder="big").view(">u8").astype(np.uint64).reshape(n, W)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("dim,ell,n", [(1, 1, 1), (2, 3, 100), (3, 63, 1000), (3, 64, 777),
                                       (3, 65, 513), (4, 128, 4096), (3, 200, 300),
                                       (7, 257, 200), (16, 1024, 64)])
def test_signatures_match_oracle(cg, dim, ell, n):
    rng = np.random.default_rng(1000 + 7 * dim + ell)
    P = rng.standard_normal((n, dim))
    A = rng.standard_normal((ell, dim + 1))
    # ties: integer-valued points on integer planes give exact zeros
    if n > 8 and dim >= 2:
        P[:8] = rng.integers(-3, 4, size=(8, dim))
        A[:min(4, ell), :] = rng.integers(-2, 3, size=(min(4, ell), dim + 1))
        A[0, :dim] = 1.0
        A[0, dim] = -P[0].sum()  # point 0 exactly on plane 0
    w = cg.signatures(_dev(P), _dev(A)).cpu().numpy().view(np.uint64)
    rc, b = oracle.signatures(P, A)
    assert rc == 0
    assert np.array_equal(w, _pack_bytes(b))


def test_signatures_fma_rounding_case(cg):
    """The G21 pin on the device: fma(1 + 2^-27, 1 - 2^-27, -1) < 0."""
    e = 2.0 ** -27
    w = cg.signatures(_dev([[1.0 - e]]), _dev([[1.0 + e, -1.0]])).cpu().numpy().view(np.uint64)
    assert int(w[0, 0]) == 0


def test_fig1_points_on_device(cg):
    P, A = synth.fig1_points()
    res = cg.build_points(_dev(P), _dev(A))
    cells = res.cells.cpu().numpy().view(np.uint64)
    edges = res.edges.cpu().numpy().view(np.uint32)
    rc, b = oracle.signatures(P, A)
    rc, oc, oe = oracle.build(b)
    assert np.array_equal(cells, oc) and np.array_equal(edges, oe)
    assert edges.tolist() == [[0, 1], [0, 2], [1, 3], [2, 3]]


@pytest.mark.parametrize("dim,k", [(2, 25), (2, 100), (3, 10), (3, 40)])
def test_build_points_arrangement_closed_form(cg, dim, k):
    P, A = synth.arrangement_points(100 * dim + k, k, dim)
    res = cg.build_points(_dev(P), _dev(A))
    cells = res.cells.cpu().numpy().view(np.uint64)
    edges = res.edges.cpu().numpy().view(np.uint32)
    assert (cells.shape[0], edges.shape[0]) == synth.arrangement_cells_edges(k, dim)
    rc, b = oracle.signatures(P, A)
    rc, oc, oe = oracle.build(b)
    assert np.array_equal(cells, oc) and np.array_equal(edges, oe)
    check_invariants(cells, edges, k)


@pytest.mark.parametrize("k,n", [(64, 1 << 20), (128, 1 << 18)])
def test_build_points_uniform_vs_oracle(cg, k, n):
    """C3-shaped FP64 samples (heavy duplication), and the same input as bytes
    through cg_build: identical results."""
    P, A = synth.points_uniform(3 + k, k, n)
    res = cg.build_points(_dev(P), _dev(A))
    cells = res.cells.cpu().numpy().view(np.uint64)
    edges = res.edges.cpu().numpy().view(np.uint32)
    rc, b = oracle.signatures(P, A)
    assert rc == 0
    rc, oc, oe = oracle.build(b)
    assert np.array_equal(cells, oc) and np.array_equal(edges, oe)
    r2 = cg.build(torch.from_numpy(b).cuda())
    assert np.array_equal(r2.cells.cpu().numpy().view(np.uint64), cells)
    assert np.array_equal(r2.edges.cpu().numpy().view(np.uint32), edges)


def test_points_errors(cg):
    from paper_1503_06029_b200.cg import CG_EINPUT, CG_EINVAL, CgError

    P = np.zeros((4, 3))
    A = np.ones((5, 4))
    with pytest.raises(CgError) as ei:
        cg.signatures(_dev(np.full((4, 3), np.nan)), _dev(A))
    assert ei.value.code == CG_EINPUT
    with pytest.raises(CgError) as ei:
        cg.build_points(_dev(P), _dev(np.full((5, 4), np.inf)))
    assert ei.value.code == CG_EINPUT
    with pytest.raises(CgError) as ei:
        cg.signatures(_dev(np.full((4, 3), 2.0 ** 61)), _dev(A))
    assert ei.value.code == CG_EINPUT
    with pytest.raises(CgError) as ei:
        cg.build_points(_dev(np.zeros((4, 17))), _dev(np.ones((5, 18))))
    assert ei.value.code == CG_EINVAL
    with pytest.raises(CgError):
        cg.signatures(_dev(P), _dev(np.ones((5, 3))))  # planes must be [ell, dim + 1]
