"""Per-step stage breakdown of cg_build on the C5 workload (diagnostics)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dev = torch.device("cuda:0")
x, d = bench.make_c5_device(torch, lg, dev)
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = cg.build(x, want_stats=True, bucket_log2=int(os.environ.get('CG_BUCKET_LOG2', '-1')))
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    st = {k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.stats.items()}
    print(json.dumps({"rep": i, "wall_ms": round(wall, 2), **st}))
    del r

# python-side overhead breakdown of one call
import cProfile, pstats  # noqa: E402
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
r = cg.build(x, want_stats=True, bucket_log2=int(os.environ.get('CG_BUCKET_LOG2', '-1')))
torch.cuda.synchronize()
pr.disable()
print(json.dumps({k: round(v, 1) for k, v in r.stats.items() if k.startswith("us_host")}))
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
