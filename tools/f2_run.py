"""cg_insert of the last 2^20 C5 rows into the graph of the others (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

x, d = bench.make_c5_device(torch, 26, torch.device("cuda:0"))
n = x.shape[0]
nb = 1 << 20
old = cg.build(x[: n - nb])
new = x[n - nb:].contiguous()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    c, e = cg.insert(old.cells, old.edges, new)
    torch.cuda.synchronize()
    del c, e
