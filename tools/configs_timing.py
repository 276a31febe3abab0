"""Build time of every BASELINE config on one GPU (device-resident input;
median of 5 after 2 warm-ups; diagnostics for DESIGN.md)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

dev = torch.device("cuda:0")
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C3F", "C4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
for name in names:
    d = synth.config(name)
    if "bytes" in d and d["bytes"] is not None:
        x = torch.from_numpy(d["bytes"]).to(dev)
    else:
        x = synth.unpack_words_torch(torch.from_numpy(d["words"].view(np.int64)).to(dev), d["ell"])
    ts, st = [], None
    for i in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = cg.build(x, want_stats=True)
        e1.record()
        torch.cuda.synchronize()
        if i >= min(2, reps - 1):
            ts.append(e0.elapsed_time(e1))
        st = r.stats
    print(json.dumps({"config": name, "n": int(x.shape[0]), "ell": int(x.shape[1]),
                      "n_cells": st["n_cells"], "n_edges": st["n_edges"],
                      "ms": round(float(np.median(ts)), 3),
                      "stages_us": {k[3:]: round(v, 1) for k, v in st.items()
                                    if k.startswith("us_") and not k.startswith("us_host")}}))
