"""Hot source lines of one kernel from `ncu -i X --page source --csv --print-source cuda,sass`:
CUDA lines ranked by warp-stall samples, with instructions executed.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kre}',
                      '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, lines, hdr = None, [], None
for r in rows:
    if r and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
    elif r and r[0] == 'Line No':
        hdr = r
    elif hdr and r and r[0] and r[0].isdigit():
        d = dict(zip(hdr[:3], r[:3]))
        try:
            samp = int(r[4]); inst = int(r[7])
        except (ValueError, IndexError):
            continue
        lines.append((samp, inst, fname, int(r[0]), r[1].strip()[:110]))
tot = sum(x[0] for x in lines) or 1
toti = sum(x[1] for x in lines) or 1
print(f'total stall samples {tot}, instructions {toti}')
for s, i, f, ln, src in sorted(lines, reverse=True)[:n]:
    print(f'{100 * s / tot:5.1f}% smp {100 * i / toti:5.1f}% ins  {f}:{ln}  {src}')
