"""GPU parity for row f2: cg_insert (accumulating a new batch of samples
into an existing cell graph) must equal the oracle's cell graph of
the union of all samples (P:102-109, P:108 multiset) and cg_build on the
concatenated input, bit for bit."""
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


def _split_cases():
    rng = np.random.default_rng(77)
    c1 = synth.config("C1")["bytes"]
    hyp = synth.hypercube(9)
    P, A = synth.arrangement_points(31, 12, 2)
    rc, arr = oracle.signatures(P, A)
    planted, _ = synth.planted_bytes(41, 2000, 200)
    c3 = synth.config("C3")["bytes"][:50000]
    return [
        ("C1 halves", c1[:500], c1[500:]),
        ("C1 + duplicates", c1, np.concatenate([c1[:50], c1[900:]])),
        ("hypercube interleaved", hyp[::2], hyp[1::2]),
        ("hypercube batch inside", hyp, hyp[rng.permutation(len(hyp))[:100]]),
        ("arrangement", arr[: len(arr) // 3], arr[len(arr) // 3:]),
        ("planted pairs split", planted[:2500], planted[2500:]),
        ("C3 rows", c3[:30000], c3[30000:]),
        ("one new cell", c1, (1 - c1[:1]).astype(np.uint8)),
    ]


@pytest.mark.parametrize("name,x1,x2", _split_cases(), ids=[c[0] for c in _split_cases()])
def test_insert_equals_union(cg, name, x1, x2):
    d1 = torch.from_numpy(np.ascontiguousarray(x1)).cuda()
    d2 = torch.from_numpy(np.ascontiguousarray(x2)).cuda()
    r1 = cg.build(d1)
    cells, edges = cg.insert(r1.cells, r1.edges, d2)
    got_c = cells.cpu().numpy().view(np.uint64)
    got_e = edges.cpu().numpy().view(np.uint32)
    union = np.concatenate([x1, x2])
    rc, oc, oe = oracle.build(union)
    assert rc == 0
    assert np.array_equal(got_c, oc)
    assert np.array_equal(got_e, oe)
    r = cg.build(torch.from_numpy(union).cuda())
    assert torch.equal(r.cells, cells) and torch.equal(r.edges, edges)


def test_insert_repeated_batches(cg):
    """Accumulating in 5 batches gives the graph of all samples."""
    x = synth.config("C2")["bytes"]
    parts = np.array_split(x, 5)
    r = cg.build(torch.from_numpy(parts[0]).cuda())
    cells, edges = r.cells, r.edges
    for p in parts[1:]:
        cells, edges = cg.insert(cells, edges, torch.from_numpy(np.ascontiguousarray(p)).cuda())
    assert cells.shape[0] == 20101 and edges.shape[0] == 40000  # the C2 closed form
    rc, oc, oe = oracle.build(x)
    assert np.array_equal(cells.cpu().numpy().view(np.uint64), oc)
    assert np.array_equal(edges.cpu().numpy().view(np.uint32), oe)


def test_insert_errors(cg):
    from paper_1503_06029_b200.cg import CG_EINPUT, CgError

    r = cg.build(torch.from_numpy(synth.config("C1")["bytes"]).cuda())
    bad = torch.full((3, 32), 2, dtype=torch.uint8, device="cuda")
    with pytest.raises(CgError) as ei:
        cg.insert(r.cells, r.edges, bad)
    assert ei.value.code == CG_EINPUT
