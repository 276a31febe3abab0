"""Seeded synthetic inputs for the cell-graph path (arXiv 1503.06029).

This module is DATA, shared by the CUDA path's tests/bench and by the oracle:
it produces input vectors (``uint8[n, ell]``, one byte per bit, byte k of a row
= 1 iff constraint c_k holds) and facts the generator itself knows by
construction (planted pairs).  It holds none of the method's arithmetic: no
dedupe, no sorting of cells, no Hamming-1 search.

Workloads (BASELINE.json ``configs``; recipes in DESIGN.md "Input recipe"):
  C1  planted pairs, n=1000, ell=32, bases pairwise Hamming >= 4   (seed 1)
  C2  2-D arrangement of k=200 integer lines, exact quadrant
      signatures at all C(k,2) vertices + 2^17 uniform integer points (seed 2)
  C3  ell=64 random planes in R^3, 2^20 uniform FP64 points        (seed 3)
  C3F 3-D arrangement of k=64 integer planes, exact octant
      signatures at all C(k,3) vertices ("C3-full")                 (seed 33)
  C4  planted pairs, n=2^20, ell=1024                                (seed 4)
  C5  planted pairs, n=2^26, ell=128                                 (seed 5)

Large planted inputs are generated as packed words (``planted_words``) whose
bit layout is defined here (byte k of a row = bit 63-(k%64) of word k//64);
``unpack_words_np`` / ``unpack_words_torch`` expand them to the byte input.
Both are representation changes of *generated* data, nothing more.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

CONFIG_NAMES = ("C1", "C2", "C3", "C3F", "C4", "C5")


# --------------------------------------------------------------------------
# bit-row <-> words representation of generated data
# --------------------------------------------------------------------------
def unpack_words_np(words: np.ndarray, ell: int) -> np.ndarray:
    """u64[n, W] -> uint8[n, ell] with byte k = bit 63-(k%64) of word k//64."""
    words = np.ascontiguousarray(words, dtype=np.uint64)
    n, W = words.shape
    be = words.astype(">u8").view(np.uint8).reshape(n, W * 8)
    bits = np.unpackbits(be, axis=1, bitorder="big")
    return np.ascontiguousarray(bits[:, :ell])


def unpack_words_torch(words, ell: int):
    """Device-side twin of ``unpack_words_np`` (torch plumbing for big inputs).

    ``words``: int64 tensor [n, W] (u64 bit patterns).  Returns uint8 [n, ell].
    Done in column chunks to bound temporaries.
    """
    import torch

    n, W = words.shape
    out = torch.empty((n, ell), dtype=torch.uint8, device=words.device)
    shifts = torch.arange(63, -1, -1, device=words.device, dtype=torch.int64)
    rows_per = max(1, (1 << 27) // max(1, 64 * W))
    for r0 in range(0, n, rows_per):
        r1 = min(n, r0 + rows_per)
        blk = words[r0:r1]
        for w in range(W):
            k0, k1 = 64 * w, min(ell, 64 * w + 64)
            b = ((blk[:, w : w + 1] >> shifts[: k1 - k0]) & 1).to(torch.uint8)
            out[r0:r1, k0:k1] = b
    return out


def _random_words(rng: np.random.Generator, n: int, ell: int) -> np.ndarray:
    W = (ell + 63) // 64
    w = rng.integers(0, 2**64, size=(n, W), dtype=np.uint64, endpoint=False)
    if ell % 64:
        w[:, W - 1] &= np.uint64(((1 << (ell % 64)) - 1) << (64 - ell % 64))
    return w


def _bit_word(ell: int, k: np.ndarray):
    """(word index, u64 mask) of bit k in the representation above."""
    k = np.asarray(k, dtype=np.int64)
    return k // 64, (np.uint64(1) << (np.uint64(63) - (k % 64).astype(np.uint64)))


# --------------------------------------------------------------------------
# planted Hamming-1 pairs (C1, C4, C5)
# --------------------------------------------------------------------------
def planted_words(seed: int, n_pairs: int, ell: int, min_base_dist: int = 0):
    """Random bases with one planted partner each (partner = base with one bit
    negated), shuffled.  Returns (words u64[2*n_pairs, W], pair_of u64[2n])
    where rows r and s form a planted pair iff pair_of[r] == pair_of[s].

    ``min_base_dist`` > 0 enforces pairwise Hamming distance >= that among
    bases by rejection (used by C1 so the planted pairs are exactly all the
    distance-1 pairs); otherwise uniqueness holds with high probability.
    """
    rng = np.random.default_rng(seed)
    W = (ell + 63) // 64
    if min_base_dist > 0:
        bases = np.zeros((0, W), np.uint64)
        while bases.shape[0] < n_pairs:
            cand = _random_words(rng, 1, ell)
            if bases.shape[0]:
                x = bases ^ cand
                d = np.zeros(bases.shape[0], np.int64)
                for w in range(W):
                    d += np.bitwise_count(x[:, w]).astype(np.int64)
                if d.min() < min_base_dist:
                    continue
            bases = np.vstack([bases, cand])
    else:
        bases = _random_words(rng, n_pairs, ell)
    k = rng.integers(0, ell, size=n_pairs)
    partners = bases.copy()
    wi, m = _bit_word(ell, k)
    partners[np.arange(n_pairs), wi] ^= m
    words = np.concatenate([bases, partners], axis=0)
    pair_of = np.concatenate([np.arange(n_pairs), np.arange(n_pairs)]).astype(np.uint64)
    perm = rng.permutation(2 * n_pairs)
    return np.ascontiguousarray(words[perm]), pair_of[perm]


def planted_bytes(seed: int, n_pairs: int, ell: int, min_base_dist: int = 0):
    words, pair_of = planted_words(seed, n_pairs, ell, min_base_dist)
    return unpack_words_np(words, ell), pair_of


# --------------------------------------------------------------------------
# exact hyperplane arrangements (C2, C3F)
# --------------------------------------------------------------------------
def _lines_general_position(rng, k, amax, cmax):
    while True:
        a = rng.integers(-amax, amax + 1, size=k, dtype=np.int64)
        b = rng.integers(-amax, amax + 1, size=k, dtype=np.int64)
        c = rng.integers(-cmax, cmax + 1, size=k, dtype=np.int64)
        if np.any((a == 0) & (b == 0)):
            continue
        I, J = np.triu_indices(k, 1)
        D = a[I] * b[J] - a[J] * b[I]
        if np.any(D == 0):
            continue
        X = b[I] * c[J] - b[J] * c[I]
        Y = c[I] * a[J] - c[J] * a[I]
        # value of every line at every vertex, times D: exact in int64
        # (|a X|, |b Y|, |c D| <= 2^61 each, DESIGN input recipe)
        val = a[None, :] * X[:, None] + b[None, :] * Y[:, None] + c[None, :] * D[:, None]
        on = val == 0
        on[np.arange(len(I)), I] = False
        on[np.arange(len(I)), J] = False
        if np.any(on):
            continue  # three concurrent lines: redraw
        return a, b, c, I, J, D, X, Y, val


def arrangement2d(seed: int, k: int, n_uniform: int = 0, amax: int = 2**15,
                  cmax: int = 2**30):
    """Signatures of a 2-D arrangement of k integer lines a x + b y + c = 0 in
    general position.  Every cell touches a vertex, and the four cells around a
    vertex carry all four sign combinations of its two lines while every other
    line keeps its (exactly computed) sign at the vertex -- so the 4*C(k,2)
    quadrant signatures hit every cell.  ``n_uniform`` integer points in the
    vertex bounding box (+10 %) are appended; bit = [a x + b y + c >= 0]
    (tie counts as satisfied, DESIGN G12).  Rows are shuffled."""
    rng = np.random.default_rng(seed)
    a, b, c, I, J, D, X, Y, val = _lines_general_position(rng, k, amax, cmax)
    sgn = (val > 0) == (D > 0)[:, None]  # sign of (value / D) > 0
    nv = len(I)
    rows = np.repeat(sgn.astype(np.uint8), 4, axis=0)
    q = np.tile(np.array([[0, 0], [0, 1], [1, 0], [1, 1]], np.uint8), (nv, 1))
    vi = np.repeat(np.arange(nv), 4)
    rows[np.arange(4 * nv), I[vi]] = q[:, 0]
    rows[np.arange(4 * nv), J[vi]] = q[:, 1]
    parts = [rows]
    if n_uniform:
        xs = X / D
        ys = Y / D
        lo = np.array([xs.min(), ys.min()])
        hi = np.array([xs.max(), ys.max()])
        pad = 0.1 * (hi - lo)
        lo = np.maximum(lo - pad, -(2.0**31))
        hi = np.minimum(hi + pad, 2.0**31)
        px = rng.integers(int(math.floor(lo[0])), int(math.ceil(hi[0])) + 1, size=n_uniform)
        py = rng.integers(int(math.floor(lo[1])), int(math.ceil(hi[1])) + 1, size=n_uniform)
        v = a[None, :] * px[:, None] + b[None, :] * py[:, None] + c[None, :]
        parts.append((v >= 0).astype(np.uint8))
    out = np.concatenate(parts, axis=0)
    return np.ascontiguousarray(out[rng.permutation(out.shape[0])])


def _det3(m00, m01, m02, m10, m11, m12, m20, m21, m22):
    return (m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20)
            + m02 * (m10 * m21 - m11 * m20))


def arrangement3d_full(seed: int, k: int, amax: int = 2**12, bmax: int = 2**20):
    """Signatures of a 3-D arrangement of k integer planes a.p + b = 0 in general
    position: the eight octant signatures at each of the C(k,3) vertices (the
    three planes through a vertex take all 8 sign combinations around it; every
    other plane keeps its exact sign there), hitting every cell.  Shuffled."""
    rng = np.random.default_rng(seed)
    T = np.array(list(itertools.combinations(range(k), 3)), dtype=np.int64)
    while True:
        A = rng.integers(-amax, amax + 1, size=(k, 3), dtype=np.int64)
        B = rng.integers(-bmax, bmax + 1, size=k, dtype=np.int64)
        i, j, l = T[:, 0], T[:, 1], T[:, 2]
        ai, aj, al = A[i], A[j], A[l]
        D = _det3(ai[:, 0], ai[:, 1], ai[:, 2], aj[:, 0], aj[:, 1], aj[:, 2],
                  al[:, 0], al[:, 1], al[:, 2])
        if np.any(D == 0):
            continue
        nb = -B
        Nx = _det3(nb[i], ai[:, 1], ai[:, 2], nb[j], aj[:, 1], aj[:, 2], nb[l], al[:, 1], al[:, 2])
        Ny = _det3(ai[:, 0], nb[i], ai[:, 2], aj[:, 0], nb[j], aj[:, 2], al[:, 0], nb[l], al[:, 2])
        Nz = _det3(ai[:, 0], ai[:, 1], nb[i], aj[:, 0], aj[:, 1], nb[j], al[:, 0], al[:, 1], nb[l])
        # plane m at vertex (Nx,Ny,Nz)/D, times D (|.| < 2^62, exact in int64)
        val = (A[None, :, 0] * Nx[:, None] + A[None, :, 1] * Ny[:, None]
               + A[None, :, 2] * Nz[:, None] + B[None, :] * D[:, None])
        on = val == 0
        r = np.arange(len(T))
        on[r, i] = on[r, j] = on[r, l] = False
        if np.any(on):
            continue
        break
    sgn = ((val > 0) == (D > 0)[:, None]).astype(np.uint8)
    nv = len(T)
    rows = np.repeat(sgn, 8, axis=0)
    octs = np.array(list(itertools.product((0, 1), repeat=3)), np.uint8)
    q = np.tile(octs, (nv, 1))
    vi = np.repeat(np.arange(nv), 8)
    rr = np.arange(8 * nv)
    rows[rr, T[vi, 0]] = q[:, 0]
    rows[rr, T[vi, 1]] = q[:, 1]
    rows[rr, T[vi, 2]] = q[:, 2]
    return np.ascontiguousarray(rows[rng.permutation(rows.shape[0])])


def arrangement3d_uniform(seed: int, k: int = 64, n: int = 1 << 20):
    """k planes with N(0,I) unit normals and U(-0.5,0.5) offsets; n points
    uniform in [-1,1]^3 (FP64); bit = [a.p + b >= 0] (C3)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((k, 3))
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    B = rng.uniform(-0.5, 0.5, size=k)
    P = rng.uniform(-1.0, 1.0, size=(n, 3))
    return np.ascontiguousarray(((P @ A.T + B[None, :]) >= 0).astype(np.uint8))


# --------------------------------------------------------------------------
# f1 inputs: FP64 points + half-space planes (the signatures are computed by
# the code under test, not here)
# --------------------------------------------------------------------------
def fig1_points():
    """Three lines and the four points A, B, C, D of the paper's Figure 1
    (P:60-90): planes f64[3, 3] rows (a_x, a_y, b) for a.p + b >= 0, points
    f64[4, 2]; their signatures are the printed table A=111, B=110, C=100,
    D=101.  The coordinates are a construction with that table (the
    figure's geometry is not in the text)."""
    planes = np.array([[1.0, 0.0, 0.0],     # c_0: x >= 0
                       [0.0, 1.0, 0.0],     # c_1: y >= 0
                       [-1.0, -1.0, 2.0]])  # c_2: x + y <= 2
    points = np.array([[0.5, 0.5], [2.0, 1.0], [3.0, -0.5], [0.5, -0.5]])
    return points, planes


def arrangement_points(seed: int, k: int, dim: int, margin: float = 1e-9):
    """k random hyperplanes in general position in R^dim (dim 2 or 3), unit
    normals, offsets U(-0.5, 0.5), and 2^dim FP64 points around every vertex
    (intersection of dim planes): vertex + delta * M^-1 s for every sign
    pattern s, M the vertex's plane normals, so the points take all 2^dim
    sign combinations of those planes while every other plane keeps its
    sign at the vertex; every cell touches a vertex, so every cell is hit.
    delta is a quarter of the distance to the nearest other plane, and the
    arrangement is redrawn until every |a.p + b| >= margin (far above FP64
    rounding), so any evaluation order yields the same signs.  Returns
    (points f64[2^dim * C(k, dim), dim], planes f64[k, dim + 1]), shuffled."""
    rng = np.random.default_rng(seed)
    combos = np.array(list(itertools.combinations(range(k), dim)), dtype=np.int64)
    signs = np.array(list(itertools.product((-1.0, 1.0), repeat=dim)))
    for _ in range(200):
        A = rng.standard_normal((k, dim))
        A /= np.linalg.norm(A, axis=1, keepdims=True)
        b = rng.uniform(-0.5, 0.5, size=k)
        M = A[combos]                                   # [V, dim, dim]
        if np.min(np.abs(np.linalg.det(M))) < 1e-6:
            continue
        V = np.linalg.solve(M, -b[combos][..., None])[..., 0]  # vertices [V, dim]
        Dir = np.linalg.solve(M[:, None], signs[None, :, :, None])[..., 0]  # [V, 2^dim, dim]
        val = V @ A.T + b[None, :]                       # [V, k]
        own = np.zeros_like(val, dtype=bool)
        own[np.arange(len(combos))[:, None], combos] = True
        other = np.where(own, np.inf, np.abs(val))
        slope = np.abs(np.einsum("vsd,kd->vsk", Dir, A)).max(axis=1)  # [V, k]
        slope = np.where(own, 0.0, slope)
        delta = 0.25 * np.min(other / np.maximum(slope, 1e-300), axis=1)  # [V]
        pts = (V[:, None, :] + delta[:, None, None] * Dir).reshape(-1, dim)
        vals = pts @ A.T + b[None, :]
        if np.min(np.abs(vals)) < margin:
            continue
        planes = np.concatenate([A, b[:, None]], axis=1)
        return np.ascontiguousarray(pts[rng.permutation(len(pts))]), planes
    raise RuntimeError(f"no arrangement of {k} planes in R^{dim} with margin {margin}")


def arrangement_cells_edges(k: int, dim: int):
    """Closed forms for a simple arrangement of k hyperplanes in R^dim
    (dim 2: 1 + k + C(k,2) cells, k^2 edges; dim 3: sum_{i<=3} C(k,i) cells,
    k * sum_{i<=2} C(k-1,i) edges -- every facet on a plane is a cell of the
    induced (dim-1)-arrangement)."""
    cells = sum(math.comb(k, i) for i in range(dim + 1))
    edges = k * sum(math.comb(k - 1, i) for i in range(dim))
    return cells, edges


def points_uniform(seed: int, k: int, n: int, dim: int = 3):
    """C3-style FP64 input for f1 at any size: k planes (N(0,I) unit normals,
    U(-1/2,1/2) offsets) and n points uniform in [-1,1]^dim."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((k, dim))
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    b = rng.uniform(-0.5, 0.5, size=k)
    return rng.uniform(-1.0, 1.0, size=(n, dim)), np.concatenate([A, b[:, None]], axis=1)


# --------------------------------------------------------------------------
# small structured / random inputs for tests
# --------------------------------------------------------------------------
def hypercube(ell: int) -> np.ndarray:
    """All 2^ell vectors; row v = binary expansion of v, byte 0 most significant."""
    v = np.arange(1 << ell, dtype=np.int64)
    sh = np.arange(ell - 1, -1, -1, dtype=np.int64)
    return ((v[:, None] >> sh[None, :]) & 1).astype(np.uint8)


def grid_words_np(side: int, dims: int, perm_mult: int = 1) -> tuple[np.ndarray, int]:
    """All cells of a `dims`-dimensional grid with `side` vertices per axis,
    each axis a path embedded by the thermometer code 1^t 0^(side-1-t)
    (t = 0..side-1), concatenated axis 0 first: ell = dims*(side-1) <= 64,
    one packed word per cell (bit k = word bit 63-k).  Row r holds the grid
    point whose mixed-radix number (axis 0 most significant) is
    (r * perm_mult) mod side^dims (perm_mult coprime to side: a permutation).
    Generated data only; what the cell graph of it is, is the tests' business."""
    ell = dims * (side - 1)
    assert ell <= 64
    n = side ** dims
    r = (np.arange(n, dtype=np.uint64) * np.uint64(perm_mult)) % np.uint64(n)
    w = np.zeros(n, np.uint64)
    for c in range(dims - 1, -1, -1):
        t = r % np.uint64(side)
        r //= np.uint64(side)
        # thermometer code of t on bits c*(side-1) .. c*(side-1)+side-2
        code = ((np.uint64(1) << t) - np.uint64(1)) << (np.uint64(side - 1) - t)
        w |= code << np.uint64(64 - (c + 1) * (side - 1))
    return w.reshape(n, 1), ell


def grid_words_torch(side: int, dims: int, device, perm_mult: int = 1):
    """grid_words_np on the device (torch int64 [n, 1] holding the u64 bit
    patterns); for the full-size m >= 2^32 test."""
    import torch

    ell = dims * (side - 1)
    assert ell <= 64
    n = side ** dims
    r = (torch.arange(n, dtype=torch.int64, device=device) * perm_mult) % n
    w = torch.zeros(n, dtype=torch.int64, device=device)
    one = torch.ones((), dtype=torch.int64, device=device)
    for c in range(dims - 1, -1, -1):
        t = r % side
        r = r // side
        code = ((one << t) - 1) << (side - 1 - t)
        w |= code << (64 - (c + 1) * (side - 1))
    del r
    return w.view(n, 1), ell


def random_bytes(seed: int, n: int, ell: int, dup_frac: float = 0.0, p_one: float = 0.5):
    rng = np.random.default_rng(seed)
    nu = max(1, int(round(n * (1.0 - dup_frac))))
    base = (rng.random((nu, ell)) < p_one).astype(np.uint8)
    if n > nu:
        extra = base[rng.integers(0, nu, size=n - nu)]
        base = np.concatenate([base, extra], axis=0)
    return np.ascontiguousarray(base[rng.permutation(base.shape[0])])


def clustered_bytes(seed: int, n: int, ell: int, n_centers: int = 8, max_flips: int = 3):
    """Rows = a random center with up to ``max_flips`` random bits negated:
    dense in Hamming-1 pairs and duplicates (stress input)."""
    rng = np.random.default_rng(seed)
    centers = rng.integers(0, 2, size=(n_centers, ell), dtype=np.uint8)
    rows = centers[rng.integers(0, n_centers, size=n)].copy()
    nf = rng.integers(0, max_flips + 1, size=n)
    for f in range(max_flips):
        sel = np.nonzero(nf > f)[0]
        kk = rng.integers(0, ell, size=sel.size)
        rows[sel, kk] ^= 1
    return rows


# --------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------
def config(name: str, scale_log2: int | None = None):
    """Return a dict with ``bytes`` (uint8[n, ell]) or ``words`` (for C4/C5 when
    ``scale_log2`` is None use words to avoid a host-side byte blow-up), ``ell``,
    ``n``, and what the generator guarantees (``expect_cells``, ``expect_edges``
    where known by construction; None otherwise).

    ``scale_log2`` overrides n = 2^scale_log2 for the planted configs (same
    recipe, smaller n: parity-test and CPU-baseline samples)."""
    if name == "C1":
        x, pair_of = planted_bytes(1, 500, 32, min_base_dist=4)
        return dict(name=name, bytes=x, ell=32, n=1000, pair_of=pair_of,
                    expect_cells=1000, expect_edges=500)
    if name == "C2":
        x = arrangement2d(2, 200, n_uniform=1 << 17)
        k = 200
        return dict(name=name, bytes=x, ell=200, n=x.shape[0],
                    expect_cells=1 + k + k * (k - 1) // 2, expect_edges=k * k)
    if name == "C3":
        x = arrangement3d_uniform(3, 64, 1 << 20)
        return dict(name=name, bytes=x, ell=64, n=x.shape[0], expect_cells=None,
                    expect_edges=None)
    if name == "C3F":
        k = 64
        x = arrangement3d_full(33, k)
        nc = sum(math.comb(k, i) for i in range(4))
        m = k * sum(math.comb(k - 1, i) for i in range(3))
        return dict(name=name, bytes=x, ell=64, n=x.shape[0], expect_cells=nc,
                    expect_edges=m)
    if name in ("C4", "C5"):
        ell, seed, lg = (1024, 4, 20) if name == "C4" else (128, 5, 26)
        if scale_log2 is not None:
            lg = scale_log2
        n = 1 << lg
        words, pair_of = planted_words(seed, n // 2, ell)
        return dict(name=name, words=words, ell=ell, n=n, pair_of=pair_of,
                    expect_cells=n, expect_edges=n // 2)
    raise KeyError(name)
