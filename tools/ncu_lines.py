"""Summarise an ncu --csv launch list: one line per launch with its metrics."""
import csv
import collections
import sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        d.setdefault((r[ii], r[ki][:48]), {})[r[mi]] = r[vi]
short = {'gpu__time_duration.sum': 'ns', 'dram__bytes_read.sum': 'rd', 'dram__bytes_write.sum': 'wr',
         'dram__throughput.avg.pct_of_peak_sustained_elapsed': 'dram%'}
for (i, k), v in d.items():
    print(i, k, ' '.join(f'{short.get(m, m)}={x}' for m, x in v.items()))
