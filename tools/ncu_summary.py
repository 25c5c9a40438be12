"""Key metrics of every kernel in an .ncu-rep (ncu --set full): duration, DRAM/SM throughput,
issue activity, occupancy, stall reasons.  usage: python tools/ncu_summary.py file.ncu-rep"""
import csv
import io
import subprocess
import sys
KEYS = ('Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Registers Per Thread', 'Issue Slots Busy', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'Executed Ipc Active', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Block Size', 'Grid Size', 'Executed Instructions',
        'Dynamic Shared Memory Per Block', 'Waves Per SM')
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for x in rows[1:]:
    d = dict(zip(h, x))
    if d.get('Metric Name') in KEYS:
        print(d['Kernel Name'][:40], '|', d['Metric Name'], d['Metric Unit'], d['Metric Value'])
raw = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
if len(r) > 2:
    hh, vals = r[0], r[2]
    want = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum']
    for k in want:
        if k in hh:
            print(k, r[1][hh.index(k)], vals[hh.index(k)])
    st = [(float(vals[i].replace(',', '') or 0), hh[i]) for i in range(len(hh))
          if hh[i].startswith('smsp__average_warp_latency_issue_stalled_') and hh[i].endswith('.ratio')
          or hh[i].startswith('smsp__average_warps_issue_stalled_') and hh[i].endswith('_per_issue_active.ratio')]
    for v, k in sorted(st, reverse=True)[:8]:
        print('stall', k, v)
