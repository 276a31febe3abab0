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

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
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
    """Algorithmic bytes per stage: what the method
    must move, independent of how the kernels move it."""
    W = (ell + 63) // 64
    K = 8 * W
    nc, m, issued = st["n_cells"], st["n_edges"], st["issued_probes"]
    # MSD path (W <= 2): 2 top-digit passes + the bucket pass, each 2K per key;
    # multi-word LSD (W > 2): per word 8 passes x 2 x 12 B + gathers
    sort_key_bytes = 6 * K if W <= 2 else W * (192 + 16) + 2 * K
    return {
        "pack": n * (ell + K),
        "sort": n * sort_key_bytes,
        "dedupe": n * K + nc * (K + 6),
        "layers": nc * (K + 8) + nc * 8,
        "dict": nc * 8,
        "probe": nc * (K + 10) + issued * 32 + m * 8,
        "edges": m * 8 * 2 * 8 + m * 16,
    }


STAGE_KERNEL = {"pack": "k_pack", "sort": "k_bucket_sort", "dedupe": "k_dedupe",
                "dict": "k_global_index", "probe": "k_probe_global", "edges": "k_tile_copy",
                "layers": "k_gather_rows"}


def _ncu_traffic(stage: str):
    """DRAM bytes (read + write) per launch of the stage's main kernel from the
    committed ncu --set full summary (profiles/*_kernels.json), or None."""
    import glob

    name = STAGE_KERNEL.get(stage)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_kernels.json")))
    if not name or not files:
        return None, None
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    with open(files[-1]) as f:
        ks = json.load(f)
    for k in ks:
        if name in k["kernel"]:
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v = k["metrics"].get(m)
                if v is None:
                    return None, None
                num, u = v.split()[0], v.split()[1] if len(v.split()) > 1 else "byte"
                tot += float(num) * unit.get(u, 1)
            return int(tot), os.path.basename(files[-1])
    return None, None


def run_ours(args):
    import torch

    from paper_1503_06029_b200 import cg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 or world > 1 or args.dist:
        from paper_1503_06029_b200 import dist as cgdist

        return cgdist.bench_main(args, METRIC)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    lg = args.scale_log2
    x, d = make_c5_device(torch, lg, dev)
    n, ell = x.shape
    stream = torch.cuda.current_stream(dev)
    # warm-up (also JIT-free: the kernels are precompiled sm_100a cubins)
    for _ in range(args.warmup):
        r = cg.build(x, want_stats=True)
        del r
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(dev.index or 0)
    sampler.start()
    stats = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    ev0.record(stream)
    for _ in range(args.steps):
        r = cg.build(x, stream=stream, want_stats=True)
        stats.append(r.stats)
        del r
    ev1.record(stream)
    torch.cuda.synchronize(dev)
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
    ab = alg_bytes(st, n, ell)
    peak, peak_src = _peaks()
    dom = max(stage_us, key=lambda k: stage_us[k])
    achieved = ab[dom] / (stage_us[dom] * 1e-6) / 1e9
    traffic, tsrc = _ncu_traffic(dom)
    roof = {"bound": "hbm", "kernel_stage": dom, "kernel": STAGE_KERNEL.get(dom),
            "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_src,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_source": tsrc, "alg_bytes_per_launch": int(ab[dom]),
            "alg_bytes_def": "SURVEY 8.d.3 per-unit figures (DESIGN.md section 6)"}
    total_alg = sum(ab.values())
    whole = total_alg / (ms * 1e-3) / 1e9
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
        "whole_path_alg_GBps": round(whole, 1),
        "whole_path_roofline_frac": round(whole / peak, 4),
        "roofline": roof,
        "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))


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
    return {"value": round(nc / dt, 1), "unit": "cells/s", "cores": threads, "kind": "oracle",
            "sample": f"C5 recipe (seed 5) at n=2^{lg}, ell=128: {nc} cells, "
                      f"{edges.shape[0]} edges; ORACLE-A std::set + flip lookup, "
                      f"lookups on {threads} threads",
            "seconds": round(dt, 3),
            "flip_probes_per_s": round(nc * 128 / dt, 1),
            "phases_s": {k: round(v, 3) for k, v in tm.items() if k != "threads"}}


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
