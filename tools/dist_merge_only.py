"""One chunked merge of G logical ranks' runs (C5 recipe) inside an NVTX
range "merge" (for `ncu --nvtx --nvtx-include merge/`), diagnostics."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

lg, G, cbits = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda:0")
x, d = bench.make_c5_device(torch, lg, dev)
n, ell = x.shape
runs = [cg.dist_local(x[n * g // G: n * (g + 1) // G], chunk_bits=cbits) for g in range(G)]
C = 1 << cbits
staged = []
for c in range(C):
    pieces = [r[0][r[1][c]: r[1][c + 1]] for r in runs]
    stride = max(1, max(p.shape[0] for p in pieces))
    st = torch.zeros((G, stride, 2), dtype=torch.int64, device=dev)
    for g, p in enumerate(pieces):
        st[g, : p.shape[0]] = p
    staged.append((st, [p.shape[0] for p in pieces]))
table = torch.empty((sum(r[0].shape[0] for r in runs), 2), dtype=torch.int64, device=dev)
for rep in range(2):
    torch.cuda.synchronize()
    if rep == 1:
        torch.cuda.nvtx.range_push("merge")
    nt = 0
    for st, cnt in staged:
        nt = cg.dist_merge_chunk(st, cnt, ell, cbits, table, nt)
    torch.cuda.synchronize()
    if rep == 1:
        torch.cuda.nvtx.range_pop()
print("rows", nt)
