"""GPU parity for row f4: cg_csr / cg_bfs (CUDA) vs the CPU oracle's
adjacency lists and BFS (distances and canonical parents), bit-exact, on
graphs built by cg_build, plus the closed forms (hypercube popcounts,
arrangement Hamming distances)."""
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
    import paper_1503_06029_b200 as cg

    cg.lib()
    return cg


def _graph(cg, x):
    res = cg.build(torch.from_numpy(np.ascontiguousarray(x)).cuda())
    return res


def _check(cg, res, sources):
    n = res.cells.shape[0]
    e = res.edges.cpu().numpy().view(np.uint32)
    rp, col = cg.csr(res.edges, n)
    rc, orp, ocol = oracle.csr(e, n)
    assert rc == 0
    assert np.array_equal(rp.cpu().numpy().view(np.uint64), orp)
    assert np.array_equal(col.cpu().numpy().view(np.uint32), ocol)
    out = []
    for s in sources:
        dist, parent, ecc = cg.bfs(rp, col, s)
        rc, od, op = oracle.bfs(orp, ocol, s)
        d = dist.cpu().numpy()
        assert np.array_equal(d, od)
        assert np.array_equal(parent.cpu().numpy(), op)
        assert ecc == int(d.max())
        out.append(d)
    return out


@pytest.mark.parametrize("ell", [1, 4, 10, 16])
def test_hypercube(cg, ell):
    res = _graph(cg, synth.hypercube(ell))
    n = res.cells.shape[0]
    for s, d in zip((0, n - 1, n // 3), _check(cg, res, (0, n - 1, n // 3))):
        assert np.array_equal(d, [bin(v ^ s).count("1") for v in range(n)])


@pytest.mark.parametrize("dim,k", [(2, 40), (3, 12)])
def test_arrangement_distances(cg, dim, k):
    P, A = synth.arrangement_points(900 + dim + k, k, dim)
    res = cg.build_points(torch.from_numpy(P).cuda(), torch.from_numpy(A).cuda())
    cells = res.cells.cpu().numpy().view(np.uint64)
    for s, d in zip((0, 7), _check(cg, res, (0, 7))):
        x = np.bitwise_xor(cells, cells[s][None, :])
        ham = np.array([sum(bin(int(w)).count("1") for w in row) for row in x])
        assert np.array_equal(d, ham)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_configs(cg, name):
    res = _graph(cg, synth.config(name)["bytes"])
    n = res.cells.shape[0]
    _check(cg, res, (0, n // 2, n - 1))


def test_no_edges_and_errors(cg):
    from paper_1503_06029_b200.cg import CG_EINVAL, CgError

    e = torch.zeros((0, 2), dtype=torch.int32, device="cuda")
    rp, col = cg.csr(e, 5)
    assert rp.cpu().tolist() == [0] * 6
    dist, parent, ecc = cg.bfs(rp, col, 2)
    assert dist.cpu().tolist() == [-1, -1, 0, -1, -1] and ecc == 0
    with pytest.raises(CgError) as ei:
        cg.bfs(rp, col, 5)
    assert ei.value.code == CG_EINVAL
