"""A/B of the dictionaries (prefix index vs open-addressed hash
vs layered) on every BASELINE config: median per-stage microseconds of
cg_build (device-resident input), all kinds checked equal to the default.

    python tools/dict_ab.py [C1,C2,C3,C4,C5] [reps] [kinds]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C4", "C5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kinds = sys.argv[3].split(",") if len(sys.argv) > 3 else ["global", "hash", "sorted"]
dev = torch.device("cuda:0")
for name in names:
    if name == "C5":
        import bench
        x, _ = bench.make_c5_device(torch, 26, dev)
    else:
        d = synth.config(name)
        x = (torch.from_numpy(d["bytes"]).to(dev) if d.get("bytes") is not None else
             synth.unpack_words_torch(torch.from_numpy(d["words"].view(np.int64)).to(dev), d["ell"]))
    ref = None
    for kind in kinds:
        sts = []
        for r in range(reps + 1):
            out = cg.build(x, want_stats=True, dict_kind=kind)
            torch.cuda.synchronize()
            if r == 0:
                e = out.edges.cpu()
                if ref is None:
                    ref = e
                assert torch.equal(e, ref), (name, kind)
            else:
                sts.append(out.stats)
            del out
        keys = [k for k in sts[0] if k.startswith("us_") and not k.startswith("us_host")]
        med = {k[3:]: round(float(np.median([s[k] for s in sts])), 1) for k in keys}
        print(json.dumps({"config": name, "dict": kind, "issued": sts[0]["issued_probes"],
                          "dict_bytes": sts[0]["dict_bytes"], **med}), flush=True)
    del x
    torch.cuda.empty_cache()
