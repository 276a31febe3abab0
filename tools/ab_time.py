"""A/B timing of libcg.so variants on one workload (device-resident input):
    python tools/ab_time.py CONFIG REPS LIB1 LIB2 ...
CONFIG: C5 (2^26 x 128), C5:LG (2^LG rows), C1..C4, C3F.  Variants run
interleaved (round robin, REPS rounds after a warm-up) so clock drift hits
all of them alike; prints the median per-stage microseconds of each."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

cfg, reps, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
dev = torch.device("cuda:0")
if cfg.startswith("C5"):
    import bench
    lg = int(cfg.split(":")[1]) if ":" in cfg else 26
    x, _ = bench.make_c5_device(torch, lg, dev)
else:
    d = synth.config(cfg)
    x = (torch.from_numpy(d["bytes"]).to(dev) if d.get("bytes") is not None else
         synth.unpack_words_torch(torch.from_numpy(d["words"].view(np.int64)).to(dev), d["ell"]))
handles = []
for p in libs:
    cg._lib = None
    cg.LIB_PATH = p
    handles.append(cg.lib())
res = {p: [] for p in libs}
ref = None
for r in range(reps + 1):
    for p, L in zip(libs, handles):
        cg._lib = L
        out = cg.build(x, want_stats=True)
        torch.cuda.synchronize()
        if ref is None:
            ref = (out.cells.cpu(), out.edges.cpu())
        elif r == 0 and not os.environ.get("AB_NOCHECK"):
            assert torch.equal(out.cells.cpu(), ref[0]) and torch.equal(out.edges.cpu(), ref[1]), p
        if r > 0:
            res[p].append(out.stats)
        del out
for p in libs:
    keys = [k for k in res[p][0] if k.startswith("us_") and not k.startswith("us_host")]
    med = {k[3:]: round(float(np.median([s[k] for s in res[p]])), 1) for k in keys}
    print(json.dumps({"lib": os.path.basename(p), **med}))
