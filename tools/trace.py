"""In-graph kernel timeline of one decode step (library built with EXTRA=-DEKV_STAMPS):
first-CTA start / last-CTA end of every kernel, from %globaltimer.
usage: python tools/trace.py [n_tokens] [policy] [k_pages]"""
import ctypes, sys
import torch
sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload, new_tokens
NAMES = ['append', 'score', 'topk', 'mark', 'attend_scores', 'candidates', 'tau_pv', 'delta_bar', 'gauss_select',
         'eval_metrics', 'rebuild']
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20) - 200
policy = sys.argv[2] if len(sys.argv) > 2 else 'topk'
B = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dev = torch.device('cuda')
Hq, Hkv = 32, 8
M = (n + 15) // 16
k = int(sys.argv[3]) if len(sys.argv) > 3 else max(1, -(-M // 100))
import os
wl = make_workload(B, n, Hq, Hkv, seed=1, device=dev, spare_tokens=200, kind=os.environ.get('WORKLOAD', 'llama'))
c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens, bound=os.environ.get('BOUNDS', 'kv'),
                                 stat=os.environ.get('STATS', 'f32'))
ekv.rebuild_page_stats(c)
sel = ekv.select_params('topk' if policy == 'full' else policy, k)
attn = ekv.attn_params(float(__import__('os').environ.get('TRACE_ALPHA', '1.5')),
                       dense_v=__import__('os').environ.get('DENSE', '0') == '1')
ws = ekv.alloc_workspace(c, Hq, sel)
st = ekv.DecodeStats(B, Hq, dev, delta_bar=True, gauss=policy == 'gauss')
_, kn, vn = new_tokens(B, Hq, Hkv, seed=7, device=dev)
q = wl.q.contiguous()
out = torch.empty(B, Hq, 128, dtype=torch.float32, device=dev)
s = torch.cuda.Stream()
L = ekv.lib()
L.entmaxkv_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]


if policy == 'full':
    wsf = ekv.alloc_workspace(c, Hq, None)
    fo = torch.empty(B, Hq, 128, dtype=torch.float32, device=dev)
    ft = torch.empty(B, Hq, dtype=torch.float64, device=dev)
    fs = torch.empty(B, Hq, dtype=torch.int32, device=dev)


def step():
    if policy == 'full':
        ekv.full_attend(c, q, attn, workspace=wsf, out=fo, tau=ft, supp=fs, stream=s)
        return
    ekv.append_kv(c, kn, vn, stream=s)
    ekv.decode(c, q, sel, attn, ws, out=out, stats=st, stream=s)


with torch.cuda.stream(s):
    for _ in range(3):
        step()
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
buf = (ctypes.c_ulonglong * 32)()
for rep in range(3):
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    if not L.entmaxkv_debug_trace(buf, 1):
        sys.exit('library built without -DEKV_STAMPS')
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        g.replay()
        b.record(s)
    torch.cuda.synchronize()
    L.entmaxkv_debug_trace(buf, 0)
    ev = [(buf[2 * i], buf[2 * i + 1], NAMES[i]) for i in range(len(NAMES)) if buf[2 * i + 1]]
    ev.sort()
    t0 = ev[0][0]
    print(f'--- replay {rep}: event time {a.elapsed_time(b) * 1e3:.1f} us, traced span {(max(e[1] for e in ev) - t0) / 1e3:.1f} us')
    prev = t0
    for st_, en, nm in ev:
        print(f'  {nm:14s} start {(st_ - t0) / 1e3:7.2f}  dur {(en - st_) / 1e3:7.2f}  gap {(st_ - prev) / 1e3:6.2f}')
        prev = en

# per-CTA phases of the EKV_PH_KERNEL kernel (last replay)
import numpy as np
L.entmaxkv_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
ph = np.zeros((8, 1024), dtype=np.uint64)
cn = np.zeros((8, 1024), dtype=np.int64)
L.entmaxkv_debug_phases(ph.ctypes.data, cn.ctypes.data)
used = [i for i in range(8) if ph[i].any()]
if used:
    m = ph[0] > 0
    t0 = ph[0][m].min()
    print('per-CTA phases (us from first CTA start): p10 / p50 / p90 / max')
    for i in used:
        x = (ph[i][m].astype(np.float64) - t0) / 1e3
        print(f'  phase {i}: ' + ' / '.join(f'{v:7.2f}' for v in np.percentile(x, [10, 50, 90, 100])))
    last = int(np.argmax(ph[max(used)] * m))
    print('slowest CTA', last, 'phases', [round((int(ph[i][last]) - int(ph[0][last])) / 1e3, 2) for i in used],
          'counters', cn[0][last], cn[1][last])
    for i in range(8):
        if cn[i].any(): print(f'  counter {i}: p50 {np.percentile(cn[i][m], 50):.0f} max {cn[i][m].max()}')
