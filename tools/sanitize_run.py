"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every default-path kernel plus the layered path, the spill path
and cg_query on tiny inputs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1503_06029_b200 import cg  # noqa: E402

lp, _ = synth.planted_bytes(7, 3000, 700)  # W = 11: prefix sort + staged probe
cases = [synth.config("C1")["bytes"], synth.clustered_bytes(3, 3000, 100, 4, 3),
         synth.hypercube(10), synth.random_bytes(1, 5000, 200, dup_frac=0.5),
         np.concatenate([lp, lp[:500]])]
for x in cases:
    xt = torch.from_numpy(x).cuda()
    for kw in (dict(), dict(dict_kind="sorted", want_index=True), dict(sort_kind="lsd"),
               dict(sort_kind="nosmall"), dict(dict_kind="hash")):
        r = cg.build(xt, **kw)
        if r.index is not None:
            q = r.cells[:64].contiguous()
            r.index.query(q)
        torch.cuda.synchronize()
        del r
# the sweep path (pack partition, region sweep, slot-reading bucket pass with
# the fused prefix index), forced at a size the sanitizers finish
xs, _ = synth.planted_bytes(5, (1 << 17) + 500, 128)
xs = np.concatenate([xs, xs[:3000]])
r = cg.build(torch.from_numpy(xs).cuda(), sort_kind="sweep", want_stats=True)
torch.cuda.synchronize()
assert r.stats["sort_passes"] == 1, r.stats["sort_passes"]
del r
print("sanitize build paths ok")

# rows f1-f4 on small inputs
P, A = synth.arrangement_points(3, 8, 2)
res = cg.build_points(torch.from_numpy(P).cuda(), torch.from_numpy(A).cuda())
w = cg.signatures(torch.from_numpy(P).cuda(), torch.from_numpy(A).cuda())
rp, col = cg.csr(res.edges, res.cells.shape[0])
cg.bfs(rp, col, 0)
c1 = synth.config("C1")["bytes"]
r1 = cg.build(torch.from_numpy(c1[:600]).cuda())
cg.insert(r1.cells, r1.edges, torch.from_numpy(c1[600:]).cuda())
cg.allpairs(r1.cells, 32, 3)
torch.cuda.synchronize()
print("sanitize f-rows ok")
