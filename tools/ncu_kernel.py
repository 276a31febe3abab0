"""Hot SASS lines for the k-th kernel (0-based) in a multi-kernel ncu report."""
import csv, subprocess, sys
rep, k, top = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-id", f"::regex:.*:{k+1}"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
if len(r) < 3:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
print(r[0][:2])
h = r[1]; rows = r[2:]
si, ii, ti = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
tot_s = sum(int(x[ii] or 0) for x in rows) or 1; tot_i = sum(int(x[ti] or 0) for x in rows) or 1
print(f"samples {tot_s} inst {tot_i:.3e}")
for n, x in sorted(enumerate(rows), key=lambda kv: -int(kv[1][ii] or 0))[:top]:
    print(f"{n:5d} {100*int(x[ii] or 0)/tot_s:5.1f}% inst {100*int(x[ti] or 0)/tot_i:5.1f}%  {x[si].strip()[:80]}")
