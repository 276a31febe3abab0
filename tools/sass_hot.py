"""Top SASS lines by stall samples and instruction counts from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]; rows = r[2:]
si, ii, ti, ai = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed'), h.index('Avg. Threads Executed')
tot_s = sum(int(x[ii] or 0) for x in rows); tot_i = sum(int(x[ti] or 0) for x in rows)
print(f"samples {tot_s}  warp-instructions {tot_i:.3e}  lines {len(rows)}")
for k, x in enumerate(rows):
    x.append(k)
for x in sorted(rows, key=lambda x: -int(x[ii] or 0))[:top]:
    print(f"{x[-1]:5d} {int(x[ii] or 0)/tot_s*100:5.1f}% inst {int(x[ti] or 0)/tot_i*100:5.1f}% thr {x[ai]:>5s}  {x[si].strip()[:90]}")
