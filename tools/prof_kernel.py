"""Minimal driver for ncu captures of one decode step's kernels on the C4 workload.
usage: python tools/prof_kernel.py [bounds kv|e4m3] [stats f32|bf16] [what score|decode] [reps]"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload
bounds = sys.argv[1] if len(sys.argv) > 1 else 'kv'
stats = sys.argv[2] if len(sys.argv) > 2 else 'f32'
what = sys.argv[3] if len(sys.argv) > 3 else 'score'
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dev = torch.device('cuda')
wl = make_workload(1, 1 << 20, 32, 8, seed=1000, kind='llama', device=dev)
c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens, bound=bounds, stat=stats)
ekv.rebuild_page_stats(c)
q = wl.q.contiguous()
box = torch.empty(1, 32, c.max_pages, dtype=torch.float32, device=dev)
sel = ekv.select_params('topk', 656)
attn = ekv.attn_params(1.5)
ws = ekv.alloc_workspace(c, 32, sel)
st = ekv.DecodeStats(1, 32, dev, delta_bar=True)
for _ in range(reps):
    if what == 'score':
        ekv.score_pages_into(c, q, box)
    else:
        ekv.decode(c, q, sel, attn, ws, stats=st)
torch.cuda.synchronize()
print('done')
