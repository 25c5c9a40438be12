"""Top-k at C4 size (1M tokens, 32 heads, k=656) against a torch reference (R3: key desc,
then page asc) -- used for debugging and under compute-sanitizer."""
import sys, torch
sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
k = int(sys.argv[2]) if len(sys.argv) > 2 else 656
dev = torch.device('cuda')
wl = make_workload(1, n, 32, 8, seed=5, kind='llama', device=dev)
c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens)
ekv.rebuild_page_stats(c)
box, _, _ = ekv.score_pages(c, wl.q, modes=1)
pi, ns, _ = ekv.select(c, 32, ekv.select_params('topk', k), box=box)
torch.cuda.synchronize()
M = (n + 15) // 16
bad = 0
for h in range(32):
    b = box[0, h, :M].double()
    idx = torch.arange(M, device=dev, dtype=torch.float64)
    order = torch.argsort(b * 1e6 - idx * 0, descending=True, stable=True)   # stable: lower page first on ties
    ref = torch.sort(order[:k]).values.int()
    got = pi[0, h, :int(ns[0, h])]
    if not torch.equal(got, ref):
        bad += 1
        gs, rs = set(got.tolist()), set(ref.tolist())
        print('row', h, 'missing', sorted(rs - gs)[:5], 'extra', sorted(gs - rs)[:5], 'n', len(gs), len(rs),
              'kth', float(b[order[k - 1]]), 'extra box', [float(b[i]) for i in sorted(gs - rs)[:3]])
print('rows', 32, 'bad', bad)
