"""Verify a built cell graph against the CPU oracle and say what differs.

SPEC-style verify: the result of a build -- the cell
table (u64[n_c][W], canonical order) and the edge list (u32 (i, j)) -- is
compared with ORACLE-A on the same input:
  * cells: content and canonical (strictly increasing) order,
  * edges: missing pairs, extra pairs, pairs out of order or with i >= j.
Its own self-test is fault injection (tests/test_verify.py, -m "not gpu"):
drop one edge -> 1 missing; add a distance-2 pair -> 1 extra; swap two
cells -> order failure.  Test infrastructure: it calls oracle/ (never the
product path's code).

    python tools/verify.py C1 [--inject drop|extra|swap]   (GPU build + verify)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _rows_less(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Row-wise lexicographic a < b over u64 words (MSB-first words)."""
    lt = np.zeros(a.shape[0], bool)
    eq = np.ones(a.shape[0], bool)
    for w in range(a.shape[1]):
        lt |= eq & (a[:, w] < b[:, w])
        eq &= a[:, w] == b[:, w]
    return lt


def compare(cells: np.ndarray, edges: np.ndarray, oc: np.ndarray, oe: np.ndarray,
            show: int = 5) -> dict:
    cells = np.asarray(cells, np.uint64).reshape(cells.shape[0], -1)
    oc = np.asarray(oc, np.uint64).reshape(oc.shape[0], -1)
    edges = np.asarray(edges, np.uint32).reshape(-1, 2)
    oe = np.asarray(oe, np.uint32).reshape(-1, 2)
    rep = {"n_cells": int(cells.shape[0]), "n_cells_oracle": int(oc.shape[0]),
           "n_edges": int(edges.shape[0]), "n_edges_oracle": int(oe.shape[0])}
    order_ok = bool(cells.shape[0] < 2 or _rows_less(cells[:-1], cells[1:]).all())
    rep["cells_order_ok"] = order_ok
    rep["cells_ok"] = bool(cells.shape == oc.shape and np.array_equal(cells, oc))
    key = lambda e: (e[:, 0].astype(np.uint64) << np.uint64(32)) | e[:, 1].astype(np.uint64)
    k, ko = key(edges), key(oe)
    missing = np.setdiff1d(ko, k)
    extra = np.setdiff1d(k, ko)
    rep["n_missing"] = int(missing.size)
    rep["n_extra"] = int(extra.size)
    rep["missing"] = [[int(x >> np.uint64(32)), int(x & np.uint64(0xffffffff))] for x in missing[:show]]
    rep["extra"] = [[int(x >> np.uint64(32)), int(x & np.uint64(0xffffffff))] for x in extra[:show]]
    rep["edges_order_ok"] = bool(k.size < 2 or (k[1:] > k[:-1]).all())
    rep["edges_i_lt_j"] = bool((edges[:, 0] < edges[:, 1]).all()) if edges.size else True
    rep["ok"] = bool(rep["cells_ok"] and order_ok and not missing.size and not extra.size
                     and rep["edges_order_ok"] and rep["edges_i_lt_j"])
    return rep


def verify(x: np.ndarray, cells: np.ndarray, edges: np.ndarray) -> dict:
    import oracle

    rc, oc, oe = oracle.build(np.ascontiguousarray(x, np.uint8))
    if rc != 0:
        return {"ok": False, "oracle_rc": int(rc)}
    return compare(cells, edges, oc, oe)


def inject(cells: np.ndarray, edges: np.ndarray, kind: str, seed: int = 0):
    """Fault injection for the verify self-test."""
    rng = np.random.default_rng(seed)
    cells, edges = cells.copy(), edges.copy()
    if kind == "drop" and edges.shape[0]:
        edges = np.delete(edges, int(rng.integers(edges.shape[0])), axis=0)
    elif kind == "extra":
        # a distance-2 pair (i, j): not an edge of any cell graph
        W = cells.shape[1]
        nc = cells.shape[0]
        d2 = None
        for i in range(nc):
            for j in range(i + 1, min(nc, i + 64)):
                if sum(bin(int(a) ^ int(b)).count("1") for a, b in zip(cells[i], cells[j])) == 2:
                    d2 = (i, j)
                    break
            if d2:
                break
        assert d2 is not None and W >= 1, "no distance-2 pair to inject"
        ins = np.array([d2], np.uint32)
        edges = np.concatenate([edges, ins])
        k = (edges[:, 0].astype(np.uint64) << np.uint64(32)) | edges[:, 1].astype(np.uint64)
        edges = edges[np.argsort(k, kind="stable")]
    elif kind == "swap" and cells.shape[0] >= 2:
        i = int(rng.integers(cells.shape[0] - 1))
        cells[[i, i + 1]] = cells[[i + 1, i]]
    return cells, edges


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C1")
    ap.add_argument("--inject", choices=["drop", "extra", "swap"])
    args = ap.parse_args()
    import torch

    import synth
    from paper_1503_06029_b200 import cg

    d = synth.config(args.config)
    x = d["bytes"] if d.get("bytes") is not None else synth.unpack_words_np(d["words"], d["ell"])
    r = cg.build(torch.from_numpy(np.ascontiguousarray(x)).cuda())
    cells = r.cells.cpu().numpy().view(np.uint64)
    edges = r.edges.cpu().numpy().view(np.uint32)
    if args.inject:
        cells, edges = inject(cells, edges, args.inject)
    rep = verify(x, cells, edges)
    print(json.dumps(rep))
    sys.exit(0 if rep["ok"] else 1)


if __name__ == "__main__":
    main()
