"""A/B timing of cg.build options on the C5 workload (device-resident input):
    python tools/kind_ab.py REPS KW1 KW2 ...   (KW = sort_kind=nosweep etc., "-" = defaults)
Variants run interleaved; prints the median per-stage microseconds of each."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

reps, variants = int(sys.argv[1]), sys.argv[2:]
lg = int(os.environ.get("LG", "26"))
x, _ = bench.make_c5_device(torch, lg, torch.device("cuda:0"))
kws = []
for v in variants:
    kw = {}
    if v != "-":
        for item in v.split(","):
            k, _, val = item.partition("=")
            kw[k] = int(val) if val.lstrip("-").isdigit() else val
    kws.append(kw)
res = {v: [] for v in variants}
ref = None
for r in range(reps + 1):
    for v, kw in zip(variants, kws):
        out = cg.build(x, want_stats=True, **kw)
        torch.cuda.synchronize()
        key = (out.cells.shape[0], out.edges.shape[0])
        if ref is None:
            ref = (key, out.cells[:4096].cpu(), out.edges[-4096:].cpu())
        else:
            assert key == ref[0] and torch.equal(out.cells[:4096].cpu(), ref[1]) and \
                torch.equal(out.edges[-4096:].cpu(), ref[2]), v
        if r:
            res[v].append(out.stats)
        del out
for v in variants:
    st = res[v]
    keys = ["us_total", "us_pack", "us_sort", "us_dedupe", "us_layers", "us_dict", "us_probe", "us_edges"]
    print(json.dumps({"variant": v, **{k[3:]: round(float(np.median([s[k] for s in st])), 1) for k in keys},
                      "sort_passes": st[-1]["sort_passes"]}))
