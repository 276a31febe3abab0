"""Device time of every phase of the distributed build on ONE GPU with
logical ranks (C5 recipe): per G, the slowest rank's local build, the
(replicated) chunk merges, the slowest rank's probe, the finalize merge, and
the data each exchange moves.  Feeds the Amdahl table of DESIGN.md section 8
(the exchanges themselves need NVLink; they are reported as bytes)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
Gs = [int(g) for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
chunk_bits = int(os.environ.get("CHUNK_BITS", "3"))
dev = torch.device("cuda:0")
x, d = bench.make_c5_device(torch, lg, dev)
n, ell = x.shape
W = 2


def timed(f, reps=3):
    best, out = None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = f()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best, out


ref_ms, _ = timed(lambda: cg.build(x))
print(json.dumps({"cg_build_ms": round(ref_ms, 3)}), flush=True)
for G in Gs:
    cbits = chunk_bits if G > 1 else 0
    C = 1 << cbits
    loc = []
    runs = []
    for g in range(G):
        part = x[n * g // G: n * (g + 1) // G]
        t, r = timed(lambda: cg.dist_local(part, chunk_bits=cbits))
        loc.append(t)
        runs.append(r)
    if G == 1:
        table, merge_ms = runs[0][0], 0.0
    else:
        cap = sum(r[0].shape[0] for r in runs)
        table = torch.empty((cap, W), dtype=torch.int64, device=dev)

        staged = []  # the all-gathered pieces of every chunk (the exchange's output)
        for c in range(C):
            pieces = [r[0][r[1][c]: r[1][c + 1]] for r in runs]
            stride = max(1, max(p.shape[0] for p in pieces))
            st = torch.zeros((G, stride, W), dtype=torch.int64, device=dev)
            for g, p in enumerate(pieces):
                st[g, : p.shape[0]] = p
            staged.append((st, [p.shape[0] for p in pieces]))

        def merge_all():
            nt = 0
            for st, cnt in staged:
                nt = cg.dist_merge_chunk(st, cnt, ell, cbits, table, nt)
            return nt

        merge_ms, nt = timed(merge_all, reps=2)
        table = table[:nt]
    prb, edges, sts = [], [], []
    for r in range(G):
        t, (e, st) = timed(lambda: cg.dist_probe(table, ell, G, r, want_stats=True))
        prb.append(t)
        edges.append(e)
        sts.append(st)
    if G > 1:
        stride = max(e.shape[0] for e in edges)
        ga = torch.zeros((G, stride, 2), dtype=torch.int32, device=dev)
        for g, e in enumerate(edges):
            ga[g, : e.shape[0]] = e
        fin_ms, fin = timed(lambda: cg.dist_finalize(ga, [e.shape[0] for e in edges]))
    else:
        fin_ms = 0.0
    nc = table.shape[0]
    out = {"G": G, "local_ms_max": round(max(loc), 3), "merge_ms": round(merge_ms, 3),
           "probe_ms_max": round(max(prb), 3), "probe_ms_min": round(min(prb), 3),
           "finalize_ms": round(fin_ms, 3),
           "runs_allgather_bytes": int(sum(r[0].shape[0] for r in runs) * W * 8),
           "edges_allgather_bytes": int(sum(e.shape[0] for e in edges) * 8),
           "dict_cells_max": max(st["dict_cells"] for st in sts), "n_cells": nc,
           "dict_bytes_max": max(st["dict_bytes"] for st in sts),
           "rank_stage_us": {k[3:]: round(v, 1) for k, v in sts[0].items()
                             if k.startswith("us_") and not k.startswith("us_host")}}
    out["device_ms_sum"] = round(out["local_ms_max"] + merge_ms + out["probe_ms_max"] + fin_ms, 3)
    print(json.dumps(out), flush=True)
    del runs, edges, table
    staged = None
    torch.cuda.empty_cache()
