"""Shared-memory wavefronts per CUDA source line from an ncu source page.

    python tools/ncu_smem.py REPORT.ncu-rep KERNEL_SUBSTRING [TOP]"""
import csv, glob, os, re, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines())); h = r[1]; rows = r[2:]
wi, ii, ai = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("Address")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1503_06029_b200/lib/libcg.so")],
               cwd=tmp, capture_output=True)
lines = {}
for cub in glob.glob(tmp + "/*.cubin"):
    o = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    fn = loc = None
    for ln in o.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1); continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = (os.path.basename(m.group(1)), int(m.group(2))); continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and fn and kname in fn:
            lines.setdefault(fn, {})[int(m.group(1), 16)] = loc
# the profiled instance: its mangled name from the report, else by SASS length
mg = subprocess.run(["ncu", "-i", rep, "--print-kernel-base", "mangled", "--page", "details", "--csv"],
                    capture_output=True, text=True).stdout.splitlines()
mname = next((c.strip('"') for ln in mg[1:2] for c in ln.split('","') if c.strip('"').startswith("_Z")), None)
fn = mname if mname in lines else min(lines, key=lambda f: abs(len(lines[f]) - len(rows)))
base = int(rows[0][ai], 16)
agg = {}
for x in rows:
    l = lines[fn].get(int(x[ai], 16) - base, ("?", 0))
    a = agg.setdefault(l, [0, 0]); a[0] += int(x[wi] or 0); a[1] += int(x[ii] or 0)
tot = sum(v[0] for v in agg.values()) or 1
print(f"{fn[:60]}: {tot} shared wavefronts, ideal {sum(v[1] for v in agg.values())}")
srcs = {}
for (f, l), (w, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    p = glob.glob(os.path.join(ROOT, "paper_1503_06029_b200/csrc", f))
    txt = open(p[0]).read().splitlines()[l - 1].strip()[:64] if p and l else ""
    print(f"{f}:{l:<5d} {w:10d} ideal {i:10d} {100*w/tot:5.1f}%  {txt}")
