"""SASS instruction-count profile by region (ncu source page): top lines + cumulative by line blocks."""
import csv, subprocess, sys
rep = sys.argv[1]; blk = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]; rows = r[2:]
si, ti, ii = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
tot = sum(int(x[ti] or 0) for x in rows); ts = sum(int(x[ii] or 0) for x in rows)
for b0 in range(0, len(rows), blk):
    seg = rows[b0:b0 + blk]
    n = sum(int(x[ti] or 0) for x in seg); s = sum(int(x[ii] or 0) for x in seg)
    if n / tot > 0.01 or s / ts > 0.02:
        ops = {}
        for x in seg:
            op = x[si].strip().split()[0] if x[si].strip() else ''
            if op.startswith('@'): op = x[si].strip().split()[1]
            ops[op.split('.')[0]] = ops.get(op.split('.')[0], 0) + int(x[ti] or 0)
        top = sorted(ops.items(), key=lambda kv: -kv[1])[:5]
        print(f"lines {b0:5d}-{b0+blk-1:5d}: inst {100*n/tot:5.1f}%  stall {100*s/ts:5.1f}%  " + " ".join(f"{k}:{100*v/tot:.1f}" for k, v in top))
