"""Aggregate an ncu source page (SASS) by CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [TOP]

Maps SASS offsets to source lines with nvdisasm -g on the cubins embedded in
the in-tree libcg.so (built with -lineinfo), then sums instructions executed
and warp-stall samples per (file, line)."""
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lib = os.path.join(ROOT, "paper_1503_06029_b200", "lib", "libcg.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
# offset -> (file, line) for the function whose name contains kname
lines = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    cur_fn, cur_loc = None, None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_loc = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and kname in cur_fn:
            lines.setdefault(cur_fn, {})[int(m.group(1), 16)] = cur_loc
fns = list(lines)
if not fns:
    sys.exit(f"no function matching {kname}")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-c", "1"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = []
for x in r[2:]:
    if x and x[0] == "Kernel Name":
        break  # the next profiled launch: keep the first one
    rows.append(x)
# the profiled instance: its mangled name from the report, else by SASS length
mg = subprocess.run(["ncu", "-i", rep, "--print-kernel-base", "mangled", "--page", "details", "--csv"],
                    capture_output=True, text=True).stdout.splitlines()
mname = next((c.strip('"') for ln in mg[1:2] for c in ln.split('","') if c.strip('"').startswith("_Z")), None)
fn = mname if mname in lines else min(fns, key=lambda f: abs(len(lines[f]) - len(rows)))
ai, si, ii, ti = (h.index("Address"), h.index("Warp Stall Sampling (All Samples)"),
                  h.index("Instructions Executed"), h.index("Source"))
base = int(rows[0][ai], 16)
agg = {}
for x in rows:
    off = int(x[ai], 16) - base
    loc = lines[fn].get(off, ("?", 0))
    a = agg.setdefault(loc, [0, 0])
    a[0] += int(x[ii] or 0)
    a[1] += int(x[si] or 0)
ti_ = sum(v[0] for v in agg.values()) or 1
ts_ = sum(v[1] for v in agg.values()) or 1
print(f"{fn}: {ti_:.3e} warp-instructions, {ts_} stall samples")
for loc, (ni, ns) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{loc[0]:>20s}:{loc[1]:<5d} inst {100*ni/ti_:5.1f}%  stall {100*ns/ts_:5.1f}%")
