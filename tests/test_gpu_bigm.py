"""Edge lists with m >= 2^32 (the bound m <= n_c*ell/2 of P:106 allows it at
the paper's sizes: 2^26 cells x 128 bits -> 2^32).  Tile block positions and
canonical offsets are 64-bit; this builds the thermometer-coded grid [3]^18
(387,420,489 cells, 4,649,045,868 edges, ell = 36) on the B200 and checks
every edge against the grid graph's closed form, pinned on small grids by the
oracle (tests/test_oracle.py::test_grid_closed_form)."""
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


def _closed_form_chunk(i: torch.Tensor, side: int, dims: int) -> torch.Tensor:
    cols = []
    for p in range(dims):  # ascending p = ascending j for a fixed i
        step = side ** p
        cols.append(torch.where((i // step) % side < side - 1, i + step, -1))
    J = torch.stack(cols, 1)
    keep = J >= 0
    I = i[:, None].expand_as(J)
    return torch.stack([I[keep], J[keep]], 1).to(torch.int32)


@pytest.mark.parametrize("side,dims", [(3, 10), (4, 7)])
def test_grid_vs_oracle(cg, side, dims):
    """The grid recipe through the default path, vs the oracle (small)."""
    w, ell = synth.grid_words_np(side, dims, 7 if side != 7 else 3)
    res = cg.build_packed(torch.from_numpy(w.view(np.int64)).cuda(), ell)
    torch.cuda.synchronize()
    rc, oc, oe = oracle.build_packed(w, ell)
    np.testing.assert_array_equal(res.cells.cpu().numpy().view(np.uint64), oc)
    np.testing.assert_array_equal(res.edges.cpu().numpy().view(np.uint32), oe)


def test_edges_beyond_2_32(cg):
    side, dims = 3, 18
    n = side ** dims
    m = dims * (side - 1) * side ** (dims - 1)
    assert m >= 1 << 32
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 110 * 2**30:
        pytest.skip(f"needs ~110 GiB of free device memory, {free / 2**30:.0f} GiB free")
    w, ell = synth.grid_words_torch(side, dims, "cuda", perm_mult=1000003)
    res = cg.build_packed(w, ell, sort_kind="lsd", want_stats=True)
    del w
    torch.cuda.synchronize()
    assert res.cells.shape[0] == n
    assert res.edges.shape[0] == m
    # cells: V_i = grid point i (canonical = mixed-radix order)
    want_cells, _ = synth.grid_words_torch(side, dims, "cuda", perm_mult=1)
    assert torch.equal(res.cells, want_cells)
    del want_cells
    # every edge, chunk by chunk of source cells, at its 64-bit offset
    E = res.edges
    off = 0
    C = 1 << 22
    for c0 in range(0, n, C):
        i = torch.arange(c0, min(n, c0 + C), device="cuda", dtype=torch.int64)
        want = _closed_form_chunk(i, side, dims)
        got = E[off: off + want.shape[0]]
        assert torch.equal(got, want), f"edges of cells [{c0}, {c0 + C}) differ"
        off += want.shape[0]
    assert off == m
    del res, E
    torch.cuda.empty_cache()
