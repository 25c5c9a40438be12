"""Per-CTA timeline of the instrumented kernel (library built with
EXTRA='-DEKV_STAMPS -DEKV_CTA_KERNEL=k', k = 1 K-score, 2 score_pages)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload
slot = int(sys.argv[1]) if len(sys.argv) > 1 else 3     # block-0 stage stamps: 3 K-score, 4 score_pages
dev = torch.device('cuda')
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 20) - 200
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kp = int(sys.argv[4]) if len(sys.argv) > 4 else 656
Hq, Hkv = 32, 8
wl = make_workload(B, n, Hq, Hkv, seed=1, device=dev, spare_tokens=200)
import os
c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens, bound=os.environ.get('BOUNDS', 'kv'),
                                 stat=os.environ.get('STATS', 'f32')); ekv.rebuild_page_stats(c)
sel = ekv.select_params('topk', kp); attn = ekv.attn_params(1.5); ws = ekv.alloc_workspace(c, Hq, sel)
st = ekv.DecodeStats(B, Hq, dev)
L = ekv.lib(); L.entmaxkv_debug_cta.argtypes = [ctypes.c_void_p]
L.entmaxkv_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 4096)(); sb = (ctypes.c_ulonglong * 256)(); nc = ctypes.c_int()
for it in range(5):
    ekv.decode(c, wl.q, sel, attn, ws, stats=st); torch.cuda.synchronize()
if not L.entmaxkv_debug_cta(buf):
    sys.exit('library built without -DEKV_STAMPS')
L.entmaxkv_debug_stamps(sb, ctypes.byref(nc))
a = np.array(buf[:], dtype=np.float64).reshape(4, 1024)
m = a[0] > 0
s0 = a[0][m].min()
st_, fd, en, cnt = (a[0][m] - s0) / 1e3, (a[1][m] - s0) / 1e3, (a[2][m] - s0) / 1e3, a[3][m]
q = lambda x: np.percentile(x, [0, 10, 50, 90, 100]).round(2).tolist()
print('CTAs', int(m.sum()))
print('start      ', q(st_))
print('first data ', q(fd))
print('end        ', q(en))
print('stages     ', q(cnt))
print('dur/stage  ', q((en - fd) / np.maximum(cnt, 1)))
w = [sb[slot * 32 + i] for i in range(32)]
b0 = a[0][0]
print('blk0 arrivals', [round((x - b0) / 1e3, 2) if x else None for x in w[:16]])
print('blk0 done    ', [round((x - b0) / 1e3, 2) if x else None for x in w[16:32]])
