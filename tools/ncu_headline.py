"""Print headline metrics per kernel of an ncu --set full report (details page)."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L2 Hit Rate', 'L1/TEX Hit Rate', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'Issue Slots Busy',
        'Compute (SM) Throughput', 'Warp Cycles Per Issued Instruction', 'No Eligible', 'Block Limit Registers',
        'Block Limit Shared Mem', 'Mem Busy', 'Max Bandwidth', 'Mem Pipes Busy']
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
for r in rows[1:]:
    if r[mi] in WANT:
        print(r[ki][:40], '|', r[mi], '=', r[vi], r[ui])
