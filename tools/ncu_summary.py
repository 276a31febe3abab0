"""Key metrics of an ncu --set full report (one kernel)."""
import csv, subprocess, sys
want = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L2 Cache Throughput', 'L1/TEX Cache Throughput',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'Compute (SM) Throughput', 'Executed Ipc Active', 'Issue Slots Busy',
        'No Eligible', 'Active Warps Per Scheduler', 'Eligible Warps Per Scheduler',
        'Warp Cycles Per Issued Instruction', 'Block Limit Shared Mem', 'Block Limit Registers',
        'Dynamic Shared Memory Per Block', 'Grid Size', 'Block Size', 'Avg. Active Threads Per Warp',
        'Branch Efficiency', 'Mem Busy', 'Max Bandwidth', 'Mem Pipes Busy']
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]; ni, vi, ui = h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    ki = h.index('Kernel Name')
    print(f"== {rep}: {r[1][ki][:80]}")
    seen = set()
    for row in r[1:]:
        if row[ni] in want and row[ni] not in seen:
            seen.add(row[ni]); print(f"  {row[ni]:38s} {row[vi]:>14s} {row[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        hh = rr[0]
        for m in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'gpu__time_duration.sum'):
            if m in hh:
                i = hh.index(m); print(f"  {m:38s} {rr[2][i]:>14s} {rr[1][i]}")
