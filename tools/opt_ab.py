"""Interleaved A/B of runtime cg_build options on C5 (median stage us).
    python tools/opt_ab.py REPS 'bucket_log2=1' 'filter_extra=4' ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

reps = int(sys.argv[1])
variants = [dict()] + [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in a.split(",")) for a in sys.argv[2:]]
x, _ = bench.make_c5_device(torch, 26, torch.device("cuda:0"))
res = [[] for _ in variants]
for r in range(reps + 1):
    for vi, kw in enumerate(variants):
        out = cg.build(x, want_stats=True, **kw)
        torch.cuda.synchronize()
        if r:
            res[vi].append(out.stats)
        del out
for kw, sts in zip(variants, res):
    keys = [k for k in sts[0] if k.startswith("us_") and not k.startswith("us_host")]
    print(json.dumps({"opts": kw, **{k[3:]: round(float(np.median([s[k] for s in sts])), 1) for k in keys},
                      "issued": sts[0]["issued_probes"]}))
