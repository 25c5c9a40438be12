"""Aggregate ncu warp-stall samples per CUDA source line (report from --import-source on):
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys, collections, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname, hdr = None, None
agg = collections.Counter()
stalls = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or r[0] in ('', '-'):
        continue
    key = (fname, int(r[0]))
    src[key] = r[1].strip()[:90]
    try:
        agg[key] += float(r[4])
    except ValueError:
        pass
    for i, c in enumerate(hdr):
        if c.startswith('stall_') and 'Not Issued' not in c:
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v:
                stalls[key][c[6:]] += v
tot = sum(agg.values())
print(f'total samples {tot:.0f}')
for key, v in agg.most_common(top):
    st = ', '.join(f'{k} {int(n)}' for k, n in stalls[key].most_common(3))
    print(f'{v:6.0f} {100 * v / tot:5.1f}%  {key[0]}:{key[1]:<5d} {src[key]:90s} | {st}')
