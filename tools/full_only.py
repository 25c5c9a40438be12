"""Time the full-cache baseline (a5) variants at C4 (1 x 1M, 32q/8kv, bf16):
support-V / dense-V, tensor-core (R26) or canonical (R1) score pass."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload
dev = torch.device('cuda')
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 20)
Hq, Hkv = 32, 8
alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 1.5
wl = make_workload(1, n, Hq, Hkv, seed=1, device=dev)
c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens)
ekv.rebuild_page_stats(c)
ws = ekv.alloc_workspace(c, Hq, None)
kb = n * Hkv * 128 * 2
ref = None
for name, kw in [('support-V tc', {}), ('dense-V tc', {'dense_v': True}), ('support-V canonical', {'canonical': True}),
                 ('dense-V canonical', {'dense_v': True, 'canonical': True})]:
    ap = ekv.attn_params(alpha, **kw)
    for i in range(3):
        o, t, s = ekv.full_attend(c, wl.q, ap, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        ekv.full_attend(c, wl.q, ap, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 10
    fl = (kb * (2 if 'dense' in name else 1)) / 6550e9 * 1e6
    if ref is None:
        ref = (o.clone(), t.clone(), s.clone())
    print(f'{name:22s} {us:9.1f} us  floor {fl:6.1f} us  frac {fl / us:.3f}  supp {s[0, :6].tolist()}  '
          f'maxabs vs first {(o - ref[0]).abs().max().item():.2e}  dtau {(t - ref[1]).abs().max().item():.2e}  '
          f'supp equal {bool((s == ref[2]).all())}')
