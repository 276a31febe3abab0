"""GPU parity for row f3: cg_allpairs (naive all-pairs, and the
anchor method of Alg. 1-2) on cg_build's cell table must return
exactly cg_build's edge list and the oracle's -- an in-GPU cross-check of
the flip-probe path by an independent method."""
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


CASES = [("C1", None), ("C2", None), ("C3", None), ("hyper10", synth.hypercube(10)),
         ("rand200", synth.random_bytes(11, 3000, 200, dup_frac=0.3)),
         ("rand1024", synth.random_bytes(12, 700, 1024)),
         ("planted65", synth.planted_bytes(13, 1500, 65)[0]),
         ("planted4096", synth.planted_bytes(14, 100, 4096)[0])]


@pytest.mark.parametrize("name,x", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("anchors", [0, 3, 8])
def test_allpairs_equals_build(cg, name, x, anchors):
    if x is None:
        x = synth.config(name)["bytes"]
    ell = x.shape[1]
    res = cg.build(torch.from_numpy(np.ascontiguousarray(x)).cuda())
    if res.cells.shape[0] < anchors:
        pytest.skip("fewer cells than anchors")
    e, compared = cg.allpairs(res.cells, ell, anchors)
    got = e.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, res.edges.cpu().numpy().view(np.uint32))
    rc, oc, oe = oracle.build(x)
    assert np.array_equal(got, oe)
    n = res.cells.shape[0]
    assert compared <= n * (n - 1) // 2
    if anchors == 0:
        assert compared == n * (n - 1) // 2  # the naive method compares every pair


def test_anchor_pruning_is_effective(cg):
    """On random 200-bit vectors the anchors skip most pairs (the point of
    Alg. 2) while the result is unchanged."""
    x = synth.random_bytes(21, 4000, 200)
    res = cg.build(torch.from_numpy(x).cuda())
    e0, c0 = cg.allpairs(res.cells, 200, 0)
    e8, c8 = cg.allpairs(res.cells, 200, 8)
    assert torch.equal(e0, e8)
    assert c8 < c0 // 10


def test_allpairs_errors(cg):
    from paper_1503_06029_b200.cg import CG_EINVAL, CgError

    c = torch.zeros((4, 1), dtype=torch.int64, device="cuda")
    with pytest.raises(CgError) as ei:
        cg.allpairs(c, 64, 9)
    assert ei.value.code == CG_EINVAL
    with pytest.raises(CgError):
        cg.allpairs(c, 0, 0)
