"""Stage times of cg_build_points (f1) on n = 2^k uniform points in R^3 and
ell = 128 C3-style planes (diagnostics)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ell = int(sys.argv[3]) if len(sys.argv) > 3 else 128
P, A = synth.points_uniform(5, ell, 1 << 20)
dev = torch.device("cuda:0")
pts = torch.empty((1 << lg, 3), dtype=torch.float64, device=dev)
g = torch.Generator(device=dev).manual_seed(5)
pts.uniform_(-1.0, 1.0, generator=g)
planes = torch.from_numpy(A).to(dev)
for i in range(reps):
    r = cg.build_points(pts, planes, want_stats=True)
    torch.cuda.synchronize()
    st = {k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.stats.items()}
    print(json.dumps({"rep": i, **{k: st[k] for k in ("us_total", "us_pack", "us_sort", "us_dedupe", "us_dict", "us_probe", "us_edges", "n_cells", "n_edges")}}))
    del r
w = cg.signatures(pts, planes)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    w = cg.signatures(pts, planes)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"signatures_ms": round(e0.elapsed_time(e1) / 5, 3), "n": 1 << lg, "ell": ell}))
