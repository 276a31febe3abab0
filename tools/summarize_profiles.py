"""Write profiles/<tag>_launches.csv (launch list of bench.py under ncu),
profiles/<tag>_kernels.json and profiles/<tag>_summary.md (key ncu --set full
metrics per profiled kernel) from the gpurun_out/ captures.

usage: python tools/summarize_profiles.py r1 gpurun_out/launches.csv gpurun_out/prof_*.ncu-rep
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")

METRICS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
           "Achieved Occupancy", "Registers Per Thread", "Executed Ipc Active", "No Eligible",
           "Compute (SM) Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_bytes.sum", "smsp__inst_executed.sum"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    ki, ni, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    ks = {}
    for row in r[1:]:
        k = ks.setdefault(row[ii], {"kernel": row[ki].split("(")[0].replace("void ", ""), "metrics": {}})
        if row[ni] in METRICS and row[ni] not in k["metrics"]:
            k["metrics"][row[ni]] = f"{row[vi]} {row[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh = rr[0]
    for n, row in enumerate(rr[2:]):
        kid = row[hh.index("ID")] if "ID" in hh else str(n)
        if kid in ks:
            for m in RAW:
                if m in hh:
                    ks[kid]["metrics"][m] = f"{row[hh.index(m)]} {rr[1][hh.index(m)]}".strip()
    return list(ks.values())


def main():
    tag, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    os.makedirs(OUT, exist_ok=True)
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(OUT, f"{tag}_launches.csv"))
    allk = []
    for rep in reps:
        for k in details(rep):
            k["report"] = os.path.basename(rep)
            allk.append(k)
    with open(os.path.join(OUT, f"{tag}_kernels.json"), "w") as f:
        json.dump(allk, f, indent=1)
    lines = [f"# ncu summaries ({tag})", "",
             "One `ncu --set full --clock-control none` capture per kernel on the C5 workload",
             "(2^26 cells, ell = 128) via `tools/diag_stages.py 26 1`; cold-cache, serialised.", ""]
    for k in allk:
        lines.append(f"## {k['kernel']}  ({k['report']})")
        for m, v in k["metrics"].items():
            lines.append(f"- {m}: {v}")
        lines.append("")
    if os.path.exists(launches):
        lines.append("## launch list of the last build (bench.py --steps 2 --warmup 1 --no-f1 under ncu)")
        lines.append("")
        p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), launches,
                            os.environ.get("LAUNCHES_PER_STEP", "20")],
                           capture_output=True, text=True).stdout
        lines += ["```", p.rstrip(), "```"]
    with open(os.path.join(OUT, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print(os.path.join(OUT, f"{tag}_summary.md"))


if __name__ == "__main__":
    main()
