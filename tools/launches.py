"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: mean us per kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')))
hdr = None
acc = collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] == 'gpu__time_duration.sum':
            name = d['Kernel Name'].split('(')[0].replace('void ', '')
            v = float(d['Metric Value'].replace(',', ''))
            acc[name].append(v / 1000 if d.get('Metric Unit', 'ns') in ('ns', 'nsecond') else v)
for k, v in acc.items():
    print(f"{k[:60]:60s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us")
