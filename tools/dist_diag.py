"""Host-side phase timings of the distributed build at world size 1 (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_1503_06029_b200 import dist as cgdist  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev, rank=0, world_size=1)
x, d = bench.make_c5_device(torch, 26, dev)
ops = cgdist.CudaOps(torch.cuda.current_stream(dev), want_stats=True)
for i in range(4):
    t = {}
    torch.cuda.synchronize()
    table, edges = cgdist.build_distributed(x, 128, ops=ops, timings=t)
    torch.cuda.synchronize()
    print({k: round(v * 1e3, 2) for k, v in t.items()}, {k: round(v, 1) for k, v in ops.last_stats.items() if k.startswith("us_")})
dist.destroy_process_group()
