"""BASELINE.json configs 2, 3 and 5 on one B200: time per decode step (CUDA-
graph replay, events), the full-cache entmax baseline on the same cache, and the quality
metrics of the selection on the planted Llama-shaped workload (eval_exact: exact delta, support
recall rho = |S cap C_tok| / |S|; R = ||o - o_sparse|| / ||o||).  One JSON line per point.
usage: python tools/sweeps.py [c2|c3|c5|all] [--out file]"""
import json
import math
import sys

import torch

sys.path.insert(0, '.')
from paper_2605_21649_b200 import binding as ekv  # noqa: E402
from paper_2605_21649_b200.workload import make_workload  # noqa: E402

dev = torch.device('cuda')
Hq, Hkv = 32, 8


def time_fn(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(s)
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def point(cache, q, n, sel, alpha, transform="entmax", full=None):
    B = q.shape[0]
    attn = ekv.attn_params(alpha, transform)
    ws = ekv.alloc_workspace(cache, Hq, sel)
    st = ekv.DecodeStats(B, Hq, dev, delta_bar=transform == "entmax", gauss=sel.policy == ekv.EKV_GAUSS)
    out = torch.empty(B, Hq, 128, dtype=torch.float32, device=dev)
    us = time_fn(lambda s: ekv.decode(cache, q, sel, attn, ws, out=out, stats=st, stream=s))
    # quality vs the full-cache distribution of the same transform
    wsf = ekv.alloc_workspace(cache, Hq, None)
    if full is None:
        fo = torch.empty(B, Hq, 128, dtype=torch.float32, device=dev)
        ft = torch.empty(B, Hq, dtype=torch.float64, device=dev)
        fs = torch.empty(B, Hq, dtype=torch.int32, device=dev)
        full_us = time_fn(lambda s: ekv.full_attend(cache, q, attn, workspace=wsf, out=fo, tau=ft, supp=fs, stream=s),
                          reps=5)
        full = {"out": fo, "tau": ft, "supp": fs, "us": full_us}
    del wsf
    res = {"us": us, "full_us": full["us"], "speedup_vs_full": full["us"] / us}
    M = (n + 15) // 16
    res["coverage"] = float(st.n_sel.float().mean().item()) / M
    err = (out - full["out"]).norm(dim=-1) / full["out"].norm(dim=-1).clamp_min(1e-30)
    res["R_mean"] = float(err.mean().item())
    res["maxabs_vs_full"] = float((out - full["out"]).abs().max().item())
    if transform == "entmax":
        ste = ekv.DecodeStats(B, Hq, dev, delta_bar=True, eval_exact=True, gauss=sel.policy == ekv.EKV_GAUSS)
        ekv.decode(cache, q, sel, attn, ekv.alloc_workspace(cache, Hq, sel), stats=ste)
        torch.cuda.synchronize()
        rec, sup = ste.recovered.double(), ste.full_supp.double()
        res.update(delta_mean=float(ste.delta.mean().item()), delta_max=float(ste.delta.max().item()),
                   rho_mean=float((rec / sup).mean().item()), rho_pooled=float((rec.sum() / sup.sum()).item()),
                   rho_min=float((rec / sup).min().item()), supp_mean=float(sup.mean().item()),
                   delta_bar_mean=float(ste.delta_bar.mean().item()))
    else:
        # softmax: dropped mass = 1 - Z_sparse / Z_full (tau holds log Z)
        d = 1.0 - torch.exp(st.tau - full["tau"])
        res.update(delta_mean=float(d.mean().item()), delta_max=float(d.max().item()))
    return res, full


def make(B, n):
    wl = make_workload(B, n, Hq, Hkv, seed=11, kind="planted", device=dev)
    c = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens)
    ekv.rebuild_page_stats(c)
    return c, wl.q


def emit(rec, f):
    line = json.dumps(rec)
    print(line, flush=True)
    if f:
        f.write(line + "\n")


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    f = open(sys.argv[sys.argv.index("--out") + 1], "w") if "--out" in sys.argv else None
    if which in ("c2", "all"):
        c, q = make(16, 32768)
        for k in (64, 128, 256, 512):
            r, _ = point(c, q, 32768, ekv.select_params("topk", k), 1.5)
            emit({"config": "C2", "B": 16, "n": 32768, "alpha": 1.5, "policy": "topk", "k_pages": k, **r}, f)
        del c
    if which in ("c3", "all"):
        c, q = make(16, 131072)
        for alpha in (1.25, 1.5, 2.0):
            for margin in (0.0, 0.1):
                r, _ = point(c, q, 131072, ekv.select_params("gauss", 0, 0.99, margin), alpha)
                emit({"config": "C3", "B": 16, "n": 131072, "alpha": alpha, "policy": "gauss", "q_page": 0.99,
                      "margin": margin, **r}, f)
        del c
    if which in ("c5", "all"):
        c, q = make(4, 131072)
        M = 8192
        fulls = {}
        for pct in (1, 2, 5, 10, 25):
            k = math.ceil(pct / 100 * M)
            for tr in ("entmax", "softmax"):
                r, fulls[tr] = point(c, q, 131072, ekv.select_params("topk", k), 1.5, tr, fulls.get(tr))
                emit({"config": "C5", "B": 4, "n": 131072, "alpha": 1.5, "transform": tr, "budget_pct": pct,
                      "k_pages": k, **r}, f)
    if f:
        f.close()


if __name__ == "__main__":
    main()
