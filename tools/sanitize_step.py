"""Small decode steps through every C-ABI path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): append, rebuild, top-k / Gaussian (integer and non-integer beta) /
certified decode with statistics, sparse and full attend, softmax.  Prints OK at the end."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload, new_tokens

dev = torch.device('cuda')
for (B, sl, Hq, Hkv, dt) in [(1, 4096, 4, 1, torch.float32), (2, [3000, 1777], 8, 2, torch.bfloat16),
                            (1, 140000, 8, 2, torch.bfloat16)]:
    wl = make_workload(B, sl, Hq, Hkv, dtype=dt, seed=3, kind="planted", spare_tokens=16, device=dev)
    c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens)
    ekv.rebuild_page_stats(c)
    q, kn, vn = new_tokens(B, Hq, Hkv, seed=4, device=dev, dtype=dt)
    ekv.append_kv(c, kn, vn)
    for sel, alpha in [(ekv.select_params("topk", 32), 1.5), (ekv.select_params("gauss"), 2.0),
                       (ekv.select_params("gauss"), 1.7), (ekv.select_params("certified", 8), 1.5)]:
        ws = ekv.alloc_workspace(c, Hq, sel)
        st = ekv.DecodeStats(B, Hq, dev, delta_bar=True, gauss=True, supp_cap=64)
        ekv.decode(c, q, sel, ekv.attn_params(alpha), ws, stats=st)
    ekv.full_attend(c, q, ekv.attn_params(1.5))
    ekv.full_attend(c, q, ekv.attn_params(1.5, dense_v=True))
    ekv.full_attend(c, q, ekv.attn_params(1.5, "softmax"))
    torch.cuda.synchronize()
print("OK")
