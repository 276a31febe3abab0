"""Test-side helpers: golden fixtures, a tiny pure-Python restatement of the
definition (for brute force on tiny inputs), and structural invariants."""
from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name: str):
    sec, out = None, {"input": [], "cells": [], "edges": []}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("["):
                sec = line.strip("[]")
                continue
            out[sec].append(line)
    x = np.array([[int(ch) for ch in s] for s in out["input"]], np.uint8)
    cells = [s for s in out["cells"]]
    edges = np.array([[int(t) for t in s.split()] for s in out["edges"]], np.uint32).reshape(-1, 2)
    return x, cells, edges


def words_from_strings(strs, ell=None):
    """'0'/'1' strings (bit 0 first) -> u64[n, W], bit k at word k//64, bit 63-k%64."""
    ell = ell or len(strs[0])
    W = (ell + 63) // 64
    out = np.zeros((len(strs), W), np.uint64)
    for i, s in enumerate(strs):
        for k, ch in enumerate(s):
            if ch == "1":
                out[i, k // 64] |= np.uint64(1 << (63 - k % 64))
    return out


def words_from_rows(x: np.ndarray):
    return words_from_strings(["".join(str(int(b)) for b in r) for r in x], x.shape[1])


def definition(x: np.ndarray):
    """The result by definition (DESIGN G1-G4), pure Python,
    for tiny inputs: V = sorted distinct rows (tuple order = bit 0 first,
    0 < 1); E = all i < j with exactly one differing position."""
    V = sorted(set(tuple(int(b) for b in r) for r in x))
    E = [(i, j) for i in range(len(V)) for j in range(i + 1, len(V))
         if sum(a != b for a, b in zip(V[i], V[j])) == 1]
    ell = x.shape[1]
    cells = words_from_strings(["".join(map(str, v)) for v in V], ell) if V else np.zeros((0, (ell + 63) // 64), np.uint64)
    return cells, np.array(E, np.uint32).reshape(-1, 2)


def popcount_rows(cells: np.ndarray) -> np.ndarray:
    return np.bitwise_count(cells).sum(axis=1).astype(np.int64)


def check_invariants(cells: np.ndarray, edges: np.ndarray, ell: int):
    """P11: structural invariants every output must satisfy."""
    nc, W = cells.shape
    assert W == (ell + 63) // 64
    if ell % 64:
        pad = np.uint64((1 << (64 - ell % 64)) - 1)
        assert not np.any(cells[:, -1] & pad), "pad bits must be zero"
    if nc > 1:
        # strictly increasing in canonical (word-lexicographic) order
        a, b = cells[:-1], cells[1:]
        lt = np.zeros(nc - 1, bool)
        eq = np.ones(nc - 1, bool)
        for w in range(W):
            lt |= eq & (a[:, w] < b[:, w])
            eq &= a[:, w] == b[:, w]
        assert lt.all(), "cells must be strictly increasing"
    m = edges.shape[0]
    if m:
        i = edges[:, 0].astype(np.int64)
        j = edges[:, 1].astype(np.int64)
        assert np.all(i < j) and np.all(j < nc)
        key = (i << 32) | j
        assert np.all(np.diff(key) > 0), "edges ascending and unique"
        d = np.bitwise_count(cells[i] ^ cells[j]).sum(axis=1)
        assert np.all(d == 1), "every edge at Hamming distance 1"
        pc = popcount_rows(cells)
        assert np.all(pc[j] == pc[i] + 1), "i < j edge goes one popcount layer up"
        deg = np.bincount(np.concatenate([i, j]), minlength=nc)
        assert deg.max() <= ell, "degree <= ell (P:106)"
    assert 2 * m <= nc * ell, "m <= n*ell/2 (P:106)"
