#!/usr/bin/env python
"""Benchmark of the cell-graph construction hot path (arXiv 1503.06029).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full ``cg_build`` (pack, sort, dedupe, popcount layers,
dictionary, flip probes, canonical edge sort) over the whole workload with
the input resident in HBM.  At N = 1 the workload is BASELINE.json's CFG5
(n = 2^26 planted cells, ell = 128; the input is 8.6 GB, larger than L2, so
no L2 flush is needed between steps).  N > 1 (torchrun): the same CFG5 job
sharded over N ranks (rows split, NCCL all-gather of the sorted runs,
queries sharded by popcount layer, edge gather) -- strong scaling.

Prints ONE JSON line on rank 0 (contract in DESIGN.md "Measurement").
``--impl reference`` times the CPU oracle (the reference arm of this tier)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("cells/s and flip-probes/s building the cell graph at 1/2/4/8 B200; "
          "% HBM roofline")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 50):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self.proc = None

    def start(self):
        if self.period_ms <= 0:
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append((time.perf_counter(), parts))

    def mark(self):
        """Start of the timed region.  The sampler is started before the
        warm-up: nvidia-smi's first query initialises NVML and can hold the
        driver for ~0.2 s, which must not land inside the timed steps."""
        self.t0 = time.perf_counter()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.perf_counter()
        time.sleep(2.5 * self.period_ms / 1e3)  # one more sample after the region
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        t0 = getattr(self, "t0", 0.0)
        inside = [r for t, r in self.rows if t0 <= t <= t1 + 1.5 * self.period_ms / 1e3]
        # the region can be shorter than the sampling period: then the samples
        # closest to it stand in
        self.rows = inside or [r for _, r in sorted(self.rows, key=lambda tr: abs(tr[0] - t0))[:2]]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": float(np.median(load)) if load else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------- workload
def make_c5_device(torch, lg: int, device):
    import synth

    d = synth.config("C5", scale_log2=lg)
    wt = torch.from_numpy(d["words"].view(np.int64)).to(device)
    x = synth.unpack_words_torch(wt, d["ell"])
    del wt
    torch.cuda.synchronize(device)
    return x, d


def alg_bytes(st: dict, n: int, ell: int) -> dict:
    """Algorithmic (compulsory) HBM bytes per stage, DESIGN.md section 6:
    every byte the stage must read or write at least once with the data
    layout and number of passes of its algorithm; re-reads that caches could
    avoid are NOT counted, so achieved/peak is an honest roofline fraction."""
    W = (ell + 63) // 64
    K = 8 * W
    nc, m = st["n_cells"], st["n_edges"]
    dict_b = st.get("dict_bytes", 0)
    # MSD path (W <= 2): the top-digit passes (sort_passes: 2 one-sweep
    # passes, or 1 region sweep on the sweep path, whose first partition ran
    # inside the pack) + the bucket pass, each reads and writes every key;
    # W > 2: word-0 gather, 8 passes over (u64 word 0, u32 index) pairs, one
    # row gather (tie fixes not counted)
    passes = int(st.get("sort_passes", 2)) if W <= 2 else 0
    sort_key_bytes = (passes + 1) * 2 * K if W <= 2 else 8 + 8 * 2 * 12 + (K + 4) + K
    # the probe kernel's work unit is a tile of 32 cells (probe_global.cu
    # kTileCells); per tile it writes a u32 count and a u64 block position
    tiles = (nc + 31) // 32
    # sweep path: the bucket pass writes T and F itself (the dict stage has
    # no kernel of its own, only the index writes move into the sort)
    fused_dict = W <= 2 and passes == 1 and dict_b > 0 and st.get("us_dict", 1e9) < 50.0
    return {
        "pack": n * (ell + K),
        "sort": n * sort_key_bytes + (dict_b if fused_dict else 0),
        "dedupe": 0,
        "layers": 0,
        "dict": 0 if fused_dict else nc * K + dict_b,
        "probe": nc * K + dict_b + m * 8 + tiles * 12,
        "edges": m * 16,
    }


def survey_bytes(st: dict, n: int, ell: int) -> dict:
    """SURVEY.md section 8.d.3's per-unit byte model (a hash dictionary read
    once per issued probe): 32 B per issued probe + K per cell (own key) +
    (K + 8) B per edge for the probe; 8 passes x 2 x (8 + 4) B per key plus a
    gather of 32 + K B for the W >= 2 sort (8 x 16 B for W = 1).  The builder
    does not run that design (DESIGN.md section 6 says why), so a fraction
    above 1 under this model means the kernel answers probes without a
    dictionary sector each (prefix filter, near-bucket scan), not that it
    beats the HBM peak."""
    W = (ell + 63) // 64
    K = 8 * W
    nc, m = st["n_cells"], st["n_edges"]
    sort_b = (192 + 32 + K) if W >= 2 else 128
    return {"probe": 32 * st["issued_probes"] + nc * K + m * (K + 8),
            "sort": n * sort_b}


def _ncu_kernel(stage: str):
    """(DRAM bytes per launch, ncu duration in s, profile file) of the
    stage's main kernel from the newest committed ncu --set full summary
    (profiles/*_kernels.json), or (None, None, None)."""
    import glob

    name = STAGE_KERNEL.get(stage)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_kernels.json")))
    if not name or not files:
        return None, None, None
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}

    def val(v):
        parts = v.split()
        return float(parts[0]) * unit.get(parts[1] if len(parts) > 1 else "byte", 1)

    with open(files[-1]) as f:
        ks = json.load(f)
    for k in ks:
        if name in k["kernel"]:
            mt = k["metrics"]
            if "dram__bytes_read.sum" not in mt or "dram__bytes_write.sum" not in mt:
                return None, None, None
            tot = val(mt["dram__bytes_read.sum"]) + val(mt["dram__bytes_write.sum"])
            dur = val(mt["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in mt else None
            return int(tot), dur, os.path.basename(files[-1])
    return None, None, None


STAGE_KERNEL = {"pack": "k_pack", "sort": "k_bucket_rank", "dedupe": "k_dedupe",
                "dict": "k_global_index", "probe": "k_probe_global", "edges": "k_tile_copy",
                "layers": "k_gather_rows"}


def run_ours(args):
    import torch

    from paper_1503_06029_b200 import cg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 or world > 1 or args.dist:
        return run_dist(args)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    lg = args.scale_log2
    x, d = make_c5_device(torch, lg, dev)
    n, ell = x.shape
    stream = torch.cuda.current_stream(dev)
    sampler = ClockSampler(dev.index or 0, period_ms=int(os.environ.get("CG_CLOCK_MS", "50")))
    sampler.start()
    time.sleep(0.5)  # let nvidia-smi initialise NVML before any timing
    # warm-up (also JIT-free: the kernels are precompiled sm_100a cubins)
    # (same stream as the timed steps: the caching allocator keeps freed
    # output blocks per stream, so a different warm-up stream would make the
    # first timed step allocate)
    for _ in range(args.warmup):
        r = cg.build(x, stream=stream, want_stats=True)
        del r
    torch.cuda.synchronize(dev)
    sampler.mark()
    stats = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    l0 = cg.kernel_launches()
    ev0.record(stream)
    for _ in range(args.steps):
        r = cg.build(x, stream=stream, want_stats=True)
        stats.append(r.stats)
        del r
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    launches = cg.kernel_launches() - l0
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = stats[-1]
    nc, m = st["n_cells"], st["n_edges"]
    cells_per_s = nc / (ms * 1e-3)
    probes_per_s = st["logical_probes"] / (ms * 1e-3)
    # per-stage average over the timed steps (CUDA events inside the library,
    # recorded on the build stream)
    keys = ["us_pack", "us_sort", "us_dedupe", "us_layers", "us_dict", "us_probe", "us_edges"]
    stage_us = {k[3:]: float(np.mean([s[k] for s in stats])) for k in keys}
    stage_us_max = {k[3:]: float(np.max([s[k] for s in stats])) for k in keys}
    host_us = [round(s["us_host_total"], 1) for s in stats]
    alloc_us = [round(s["us_host_alloc"], 1) for s in stats]
    ab = alg_bytes(st, n, ell)
    peak, peak_src = _peaks()
    stages = {}
    for k, us in stage_us.items():
        if ab.get(k) and us > 0:
            gbs = ab[k] / (us * 1e-6) / 1e9
            stages[k] = {"us": round(us, 1), "alg_bytes": int(ab[k]), "GBps": round(gbs, 1),
                         "frac": round(gbs / peak, 4)}
    # dominant KERNEL: the probe stage is one kernel (k_probe_global); the sort
    # stage is several (2 one-sweep passes, bounds, bucket pass), each shorter
    dom = max(("pack", "probe", "dict"), key=lambda k: stage_us[k])
    achieved = ab[dom] / (stage_us[dom] * 1e-6) / 1e9
    traffic, ncu_s, tsrc = _ncu_kernel(dom)
    sb = survey_bytes(st, n, ell)
    t_dom = stage_us[dom] * 1e-6
    fracs = {
        # compulsory bytes / live CUDA-event time: the headline
        "compulsory": round(achieved / peak, 4),
        # DRAM bytes ncu measured for one launch / live time (wasted re-reads count)
        "ncu_dram": round(traffic / t_dom / 1e9 / peak, 4) if traffic else None,
        # the same bytes over ncu's own (cold-cache, serialised) duration
        "ncu_dram_ncu_time": round(traffic / ncu_s / 1e9 / peak, 4) if traffic and ncu_s else None,
        # SURVEY 8.d.3's per-unit model (32 B per issued probe ...) / live time
        "survey_8d": round(sb[dom] / t_dom / 1e9 / peak, 4) if dom in sb else None,
    }
    roof = {"bound": "hbm", "kernel_stage": dom, "kernel": STAGE_KERNEL.get(dom),
            "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_src,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_source": tsrc, "alg_bytes_per_launch": int(ab[dom]),
            "alg_bytes_def": "compulsory bytes, DESIGN.md section 6 (bench.alg_bytes)",
            "fractions": fracs,
            "survey_8d_bytes_per_launch": int(sb[dom]) if dom in sb else None}
    # the sort stage under the survey model too (several kernels, one stage)
    sort_fracs = {"compulsory": stages.get("sort", {}).get("frac"),
                  "survey_8d": round(sb["sort"] / (stage_us["sort"] * 1e-6) / 1e9 / peak, 4)
                  if stage_us.get("sort") else None}
    total_alg = sum(ab.values())
    whole = total_alg / (ms * 1e-3) / 1e9
    # ---- rows f1 / f4, measured alone (not part of the step)
    f1 = run_f1(torch, cg, dev, lg) if args.f1 else None
    f4 = run_f4(torch, cg, dev) if args.f1 else None
    f3 = run_f3(torch, cg, dev) if args.f1 else None
    f2 = run_f2(torch, cg, x, dev) if args.f1 else None
    qb = run_query(torch, cg, x, dev) if args.f1 else None
    cfgs = run_configs(torch, cg, dev) if args.configs else None
    # ---- e2e through the host-buffer C-ABI entry
    e2e = run_e2e(torch, cg, x, args, dev)
    # ---- CPU oracle baseline on a bounded sample
    cpu = cpu_baseline(args) if args.cpu_baseline else None
    out = {
        "metric": METRIC, "value": round(cells_per_s, 1), "unit": "cells/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "C5" if lg == 26 else f"C5@2^{lg}", "n": n, "ell": ell,
                   "n_cells": nc, "n_edges": m, "l2": "inputs larger than L2 (8.6 GB), no flush",
                   "input": "uint8[n][ell] resident in HBM", "parallelism": "single GPU"},
        "flip_probes_per_s": round(probes_per_s, 1),
        "issued_probes_per_s": round(st["issued_probes"] / (ms * 1e-3), 1),
        "issued_probes": st["issued_probes"],
        "stage_us": {k: round(v, 1) for k, v in stage_us.items()},
        "stage_roofline": stages,
        "stage_us_max": {k: round(v, 1) for k, v in stage_us_max.items()},
        "host_us_per_step": host_us,
        "host_alloc_us_per_step": alloc_us,
        "whole_path_alg_GBps": round(whole, 1),
        "whole_path_roofline_frac": round(whole / peak, 4),
        "roofline": roof,
        "sort_roofline": sort_fracs,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "f1_signatures": f1,
        "f4_csr_bfs": f4,
        "f3_allpairs": f3,
        "f2_insert": f2,
        "b_query": qb,
        "configs_latency": cfgs,
    }
    print(json.dumps(out))


def run_dist(args):
    """N ranks under torchrun (one GPU each): CFG5 split n/N rows per rank,
    the distributed phases of DESIGN.md section 8 (chunked NCCL all-gather of
    the sorted runs, popcount-layer probe shards, edge all-gather).  Strong
    scaling; device time per step = max over ranks of CUDA-event time."""
    import torch
    import torch.distributed as tdist

    import synth
    from paper_1503_06029_b200 import cg
    from paper_1503_06029_b200 import dist as cgdist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if not tdist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        tdist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    lg = args.scale_log2
    d = synth.config("C5", scale_log2=lg)
    n, ell = d["n"], d["ell"]
    lo, hi = n * rank // world, n * (rank + 1) // world
    wt = torch.from_numpy(np.ascontiguousarray(d["words"][lo:hi]).view(np.int64)).to(dev)
    x = synth.unpack_words_torch(wt, ell)
    del wt, d
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    ops = cgdist.CudaOps(stream, want_stats=True)
    sampler = ClockSampler(dev.index or 0) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.5)
    for _ in range(args.warmup):
        cgdist.build_distributed(x, ell, ops=ops)
    torch.cuda.synchronize(dev)
    tdist.barrier()
    if sampler:
        sampler.mark()
    l0 = cg.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        table, edges = cgdist.build_distributed(x, ell, ops=ops)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    tdist.barrier()
    launches = cg.kernel_launches() - l0
    clocks = sampler.stop() if sampler else None
    ms = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device=dev)
    tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
    ms = float(ms.item())
    lt = torch.tensor([launches], device=dev, dtype=torch.int64)
    tdist.all_reduce(lt)
    nc, m = int(table.shape[0]), int(edges.shape[0])
    st = dict(ops.last_stats)
    # the rank's probe stage (its contiguous canonical range) as the dominant kernel
    peak, peak_src = _peaks()
    roof = None
    if st.get("us_probe"):
        nr = (nc + world - 1) // world  # the rank's probed cells (equal-weight share)
        ab = alg_bytes(dict(st, n_cells=nr), n, ell)
        a = ab["probe"] / (st["us_probe"] * 1e-6) / 1e9
        roof = {"bound": "hbm", "kernel_stage": "probe", "kernel": "k_probe_global",
                "achieved": round(a, 1), "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": round(a / peak, 4), "traffic": None,
                "alg_bytes_per_launch": int(ab["probe"]),
                "alg_bytes_def": "compulsory bytes of rank 0's probe share (bench.alg_bytes)"}
    e2e = run_dist_e2e(torch, tdist, cgdist, x, ell, ops, stream, dev, args, rank, world, nc)
    if rank == 0:
        out = {"metric": METRIC, "value": round(nc / (ms * 1e-3), 1), "unit": "cells/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "u64", "data": "synthetic",
               "config": {"workload": "C5" if lg == 26 else f"C5@2^{lg}", "n": n, "ell": ell,
                          "n_cells": nc, "n_edges": m,
                          "l2": "inputs larger than L2 (8.6 GB / N per rank), no flush",
                          "parallelism": f"rows/{world} + chunked NCCL all-gather of sorted runs "
                          "(overlapped with the merge) + popcount-layer probe shards + NCCL "
                          "edge all-gather + G-way merge"},
               "flip_probes_per_s": round(nc * ell / (ms * 1e-3), 1),
               "rank0_stage_us": {k[3:]: round(v, 1) for k, v in st.items()
                                  if k.startswith("us_") and not k.startswith("us_host")},
               "roofline": roof, "gpu_launches": int(lt.item()), "clocks": clocks,
               "e2e": e2e, "cpu_baseline": None}
        print(json.dumps(out))
    tdist.barrier()
    tdist.destroy_process_group()


def run_dist_e2e(torch, tdist, cgdist, x, ell, ops, stream, dev, args, rank, world, nc):
    """e2e at N > 1: every step copies each rank's shard from pinned host
    memory to its GPU, runs the distributed build and copies the result (cell
    table + edge list) back to rank 0's host; max over ranks."""
    if args.e2e_steps <= 0:
        return None
    xh = torch.empty(x.shape, dtype=torch.uint8, pin_memory=True)
    xh.copy_(x)
    torch.cuda.synchronize(dev)
    tdist.barrier()
    # pinned result buffers sized by one untimed build (allocation is not
    # part of the measured work)
    table, edges = cgdist.build_distributed(xh.to(dev), ell, ops=ops)
    th = torch.empty(table.shape, dtype=table.dtype, pin_memory=True) if rank == 0 else None
    eh = torch.empty(edges.shape, dtype=edges.dtype, pin_memory=True) if rank == 0 else None
    del table, edges
    torch.cuda.synchronize(dev)
    tdist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d2h = 0
    ev0.record(stream)
    for _ in range(args.e2e_steps):
        xd = xh.to(dev, non_blocking=True)
        table, edges = cgdist.build_distributed(xd, ell, ops=ops)
        if rank == 0:
            th.copy_(table, non_blocking=True)
            eh.copy_(edges, non_blocking=True)
            d2h = th.numel() * th.element_size() + eh.numel() * eh.element_size()
        del xd
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    ms = torch.tensor([ev0.elapsed_time(ev1) / args.e2e_steps], device=dev)
    tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
    ms = float(ms.item())
    h2d = torch.tensor([x.numel()], device=dev, dtype=torch.int64)
    tdist.all_reduce(h2d)
    return {"value": round(nc / (ms * 1e-3), 1), "unit": "cells/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": int(d2h),
            "steps": args.e2e_steps, "api": "dist.build_distributed (pinned host shards)"}


def run_f1(torch, cg, dev, lg):
    """Row f1 measured alone: cg_signatures on n = 2^lg uniform FP64 points in
    R^3 against ell = 128 C3-style planes (device-resident inputs).  The
    kernel is FP64-FMA bound: peak = 148 SMs x 64 FP64 FMA/clk x 2 flop x
    the SM clock."""
    import synth

    n, ell, dim = 1 << lg, 128, 3
    _, A = synth.points_uniform(5, ell, 1, dim)
    pts = torch.empty((n, dim), dtype=torch.float64, device=dev)
    pts.uniform_(-1.0, 1.0, generator=torch.Generator(device=dev).manual_seed(5))
    planes = torch.from_numpy(A).to(dev)
    w = cg.signatures(pts, planes)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        w = cg.signatures(pts, planes)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / reps
    del w, pts
    flops = 2.0 * n * ell * dim
    peak = 148 * 64 * 2 * 1.965e9 / 1e12
    tf = flops / (ms * 1e-3) / 1e12
    hbm = n * dim * 8 + n * 16
    hpeak, hsrc = _peaks()
    hbm_gbs = hbm / (ms * 1e-3) / 1e9
    # neither roof binds alone: the kernel also compares, packs and
    # histograms (integer work); both fractions are reported, the FP64 peak
    # is derived from unit counts (no measured FP64 figure exists)
    return {"n": n, "ell": ell, "dim": dim, "ms": round(ms, 3),
            "points_per_s": round(n / (ms * 1e-3), 1),
            "roofline": {"bound": "alu", "unit": "TFLOP/s (fp64 fma)", "achieved": round(tf, 2),
                         "peak": round(peak, 2), "frac": round(tf / peak, 4),
                         "peak_source": "DERIVED, not measured: 148 SM x 64 fp64 FMA/clk x 2 x "
                                        "1.965 GHz (unit counts); the kernel also does integer "
                                        "compare/pack/histogram work, so this is not evidence "
                                        "of an FP64 bound"},
            "hbm_roofline": {"achieved": round(hbm_gbs, 1), "peak": hpeak, "unit": "GB/s",
                             "frac": round(hbm_gbs / hpeak, 4), "peak_source": hsrc},
            "hbm_bytes": hbm}


def run_f4(torch, cg, dev, ell=22):
    """Row f4 measured alone: CSR construction and a BFS over the cell graph of
    the hypercube H_ell (all 2^ell cells: 4.2M cells, 46M edges at ell = 22),
    built by cg_build (not timed); TEPS = 2m / BFS time."""
    import synth

    x = torch.from_numpy(synth.hypercube(ell)).to(dev)
    res = cg.build(x)
    n, m = res.cells.shape[0], res.edges.shape[0]
    del x
    rp, col = cg.csr(res.edges, n)
    dist, parent, ecc = cg.bfs(rp, col, 0)
    torch.cuda.synchronize(dev)
    reps = 3
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(reps):
        rp, col = cg.csr(res.edges, n)
    e1.record()
    for _ in range(reps):
        dist, parent, ecc = cg.bfs(rp, col, 0)
    e2.record()
    torch.cuda.synchronize(dev)
    csr_ms, bfs_ms = e0.elapsed_time(e1) / reps, e1.elapsed_time(e2) / reps
    return {"graph": f"hypercube H_{ell}", "n_cells": n, "n_edges": m, "csr_ms": round(csr_ms, 3),
            "bfs_ms": round(bfs_ms, 3), "bfs_levels": ecc + 1,
            "teps": round(2 * m / (bfs_ms * 1e-3), 1),
            "note": "BFS includes the canonical-parent pass and one host sync per level"}


def run_query(torch, cg, x, dev, nq_log2=20):
    """Row b measured alone: cg_query (self + ell single-bit-flip lookups per
    query) of 2^20 random cells of the C5 table against its index
    (asynchronous, device-resident queries)."""
    res = cg.build(x, want_index=True)
    n = res.cells.shape[0]
    g = torch.Generator(device=dev).manual_seed(9)
    q = res.cells[torch.randint(0, n, (1 << nq_log2,), device=dev, generator=g)].contiguous()
    self_idx, nbr = res.index.query(q)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        self_idx, nbr = res.index.query(q)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / reps
    nq = q.shape[0]
    ell = res.index.ell
    return {"table_cells": n, "queries": nq, "ms": round(ms, 3),
            "queries_per_s": round(nq / (ms * 1e-3), 1),
            "lookups_per_s": round(nq * (ell + 1) / (ms * 1e-3), 1),
            "found_self": int((self_idx >= 0).sum().item()),
            "found_neighbours": int((nbr >= 0).sum().item())}


def run_f2(torch, cg, x, dev, batch_log2=20):
    """Row f2 measured alone: the C5 graph of the first n - 2^20 rows (built,
    not timed) extended by the last 2^20 rows with cg_insert; compared with
    the full rebuild of the step."""
    n = x.shape[0]
    nb = 1 << batch_log2
    old = cg.build(x[: n - nb])
    new = x[n - nb:].contiguous()
    cells, edges = cg.insert(old.cells, old.edges, new)
    torch.cuda.synchronize(dev)
    del cells, edges
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        cells, edges = cg.insert(old.cells, old.edges, new)
        del cells, edges
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / reps
    return {"table_cells": int(old.cells.shape[0]), "batch_rows": nb, "ms": round(ms, 3),
            "batch_rows_per_s": round(nb / (ms * 1e-3), 1)}


def run_f3(torch, cg, dev):
    """Row f3 measured alone: cg_allpairs on the C5 recipe's first 2^17 cells
    (ell = 128): the naive method (every pair) and Alg. 1-2 with h = 5 anchors
    (the paper's best h on its GPU); pair-checks/s."""
    import synth

    d = synth.config("C5", scale_log2=17)
    x = synth.unpack_words_torch(torch.from_numpy(d["words"].view(np.int64)).to(dev), d["ell"])
    res = cg.build(x)
    n = res.cells.shape[0]
    out = {"workload": "C5 recipe at n = 2^17 (ell = 128)", "n_cells": n,
           "pairs": n * (n - 1) // 2}
    for h in (0, 5):
        e, cmp = cg.allpairs(res.cells, d["ell"], h)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e, cmp = cg.allpairs(res.cells, d["ell"], h)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        out[f"h{h}"] = {"ms": round(ms, 2), "pairs_compared": cmp,
                        "pairs_per_s": round(out["pairs"] / (ms * 1e-3), 1),
                        "edges_match_build": bool(torch.equal(e, res.edges))}
    return out


def run_configs(torch, cg, dev, names=("C1", "C2", "C3", "C4")):
    """The other BASELINE configs on one GPU (latency-bound at these sizes,
    SURVEY 8.d.2): device-resident input, 3 warm-ups, then per build the
    wall time of cg.build + a stream synchronize (what a caller waits for:
    host round trips and allocations included) and, separately, CUDA-event
    time on the stream; medians over 20 builds, no stats collection."""
    import time

    import synth

    out = {}
    for name in names:
        d = synth.config(name)
        if d.get("bytes") is not None:
            x = torch.from_numpy(d["bytes"]).to(dev)
        else:
            x = synth.unpack_words_torch(torch.from_numpy(d["words"].view(np.int64)).to(dev), d["ell"])
        stream = torch.cuda.current_stream(dev)
        for _ in range(3):
            r = cg.build(x, stream=stream)
            del r
        torch.cuda.synchronize(dev)
        walls, evs = [], []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            r = cg.build(x, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            walls.append((time.perf_counter() - t0) * 1e3)
            evs.append(e0.elapsed_time(e1))
            nc, m = int(r.cells.shape[0]), int(r.edges.shape[0])
            del r
        w = float(np.median(walls))
        out[name] = {"n": int(x.shape[0]), "ell": int(x.shape[1]), "n_cells": nc, "n_edges": m,
                     "wall_ms": round(w, 4), "event_ms": round(float(np.median(evs)), 4),
                     "cells_per_s": round(nc / (w * 1e-3), 1)}
        del x
    torch.cuda.empty_cache()
    return out


def run_e2e(torch, cg, x, args, dev):
    """Same metric through cg_build_host: pinned host input, H2D + build +
    D2H of the cell table and edge list inside the timed region."""
    if args.e2e_steps <= 0:
        return None
    n, ell = x.shape
    xh = torch.empty((n, ell), dtype=torch.uint8, pin_memory=True)
    xh.copy_(x)
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    hc, nc, he, ne, _ = cg.build_host_raw(xh, stream=stream)  # warm-up
    cg.release_host(hc, he)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(args.e2e_steps):
        hc, nc, he, ne, _ = cg.build_host_raw(xh, stream=stream)
        cg.release_host(hc, he)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    wall = (time.perf_counter() - t0) / args.e2e_steps
    ms = ev0.elapsed_time(ev1) / args.e2e_steps
    W = (ell + 63) // 64
    del xh
    return {"value": round(nc / (ms * 1e-3), 1), "unit": "cells/s",
            "ms_per_step": round(ms, 3), "wall_ms_per_step": round(wall * 1e3, 3),
            "h2d_bytes_per_step": int(n * ell), "d2h_bytes_per_step": int(nc * 8 * W + ne * 8),
            "steps": args.e2e_steps, "api": "cg_build_host (pinned host buffers)"}


def cpu_baseline(args, lg=None):
    import oracle
    import synth

    lg = lg if lg is not None else args.cpu_sample_log2
    d = synth.config("C5", scale_log2=lg)
    x = synth.unpack_words_np(d["words"], d["ell"])
    threads = os.cpu_count() or 1
    cells, edges, dt, tm = oracle.timed_build(x, nthreads=threads)
    nc = cells.shape[0]
    # the single-thread run SURVEY 8.d.5 asks for, on a 16x smaller sample
    d1 = synth.config("C5", scale_log2=max(10, lg - 4))
    x1 = synth.unpack_words_np(d1["words"], d1["ell"])
    c1, _, dt1, _ = oracle.timed_build(x1, nthreads=1)
    return {"value": round(nc / dt, 1), "unit": "cells/s", "cores": threads, "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": f"C5 recipe (seed 5) at n=2^{lg}, ell=128: {nc} cells, "
                      f"{edges.shape[0]} edges; ORACLE-A std::set + flip lookup, "
                      f"lookups on {threads} threads",
            "seconds": round(dt, 3),
            "flip_probes_per_s": round(nc * 128 / dt, 1),
            "phases_s": {k: round(v, 3) for k, v in tm.items() if k != "threads"},
            "single_thread": {"value": round(c1.shape[0] / dt1, 1), "unit": "cells/s",
                              "sample": f"C5 recipe at n=2^{max(10, lg - 4)}, 1 thread",
                              "seconds": round(dt1, 3)}}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth

    lg = args.ref_sample_log2
    d = synth.config("C5", scale_log2=lg)
    x = synth.unpack_words_np(d["words"], d["ell"])
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.timed_build(x, nthreads=threads)
    t0 = time.perf_counter()
    nc = 0
    for _ in range(args.steps):
        cells, edges, dt, tm = oracle.timed_build(x, nthreads=threads)
        nc = cells.shape[0]
    el = (time.perf_counter() - t0) / args.steps
    v = nc / el
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "cells/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(el * 1e3, 3), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "u64", "data": "synthetic",
           "config": {"workload": "C5", "sample": f"C5 recipe at n=2^{lg} per step",
                      "n": int(x.shape[0]), "ell": 128},
           "cpu_baseline": {"value": round(v, 1), "unit": "cells/s", "cores": threads,
                            "kind": "oracle",
                            "sample": f"C5 recipe (seed 5) at n=2^{lg}, ell=128 per step"},
           "e2e": {"value": round(v, 1), "unit": "cells/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--dist", action="store_true",
                    help="use the distributed (NCCL) path even at N = 1")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale-log2", type=int, default=26, help="C5 n = 2^k (26 = BASELINE CFG5)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-f1", dest="f1", action="store_false",
                    help="skip the row-f1 signature measurement")
    ap.add_argument("--no-configs", dest="configs", action="store_false",
                    help="skip the per-config (C1-C4) latency lines")
    ap.add_argument("--cpu-sample-log2", type=int, default=22)
    ap.add_argument("--ref-sample-log2", type=int, default=20)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours" and not os.environ.get("CG_BENCH_ALLOW_SHORT"):
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
