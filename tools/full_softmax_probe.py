"""Full-cache softmax (a6 baseline) at C5's shape, for a launch list: python tools/full_softmax_probe.py"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload
dev = torch.device('cuda')
wl = make_workload(4, 131072, 32, 8, seed=5, device=dev, kind="llama")
c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens)
ekv.rebuild_page_stats(c)
for _ in range(3):
    ekv.full_attend(c, wl.q, ekv.attn_params(1.5, "softmax"))
torch.cuda.synchronize()
print("ok")
