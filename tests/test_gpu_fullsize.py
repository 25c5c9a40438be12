"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(entmaxkv_decode on the whole batch): configs[3] (C4: one 1,048,576-token sequence,
32 q / 8 KV heads, top-k 1 % = 656 pages) and configs[1] (C2: 16 x 32K, top-k 64 pages).
Page scoring here runs its persistent producer over ~220 pages per CTA (several producer
chunks), the top-k radix select over 8-CTA clusters, the tau kernel over 4-CTA clusters.

The oracle re-derives everything (page metadata, scores, top-k, exact entmax) for a
sample of KV groups / (b, head) rows: element by element against the GPU -- box scores
and page sets bit-exact, support sets bit-exact, outputs within 2e-3 (bf16 in, fp32
accumulation), tau within 1e-6 relative.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import gather_head, make_workload

pytestmark = pytest.mark.gpu


def head_cache(wl, b, kv):
    """Oracle cache of ONE (sequence, kv head), pages in logical order (metadata by the oracle)."""
    Kh, Vh = gather_head(wl, b, kv)
    M = Kh.shape[0]
    hc = oracle.HostCache(Kh.float().cpu().numpy()[:, None], Vh.float().cpu().numpy()[:, None],
                          np.arange(M, dtype=np.int32)[None], np.array([int(wl.seq_lens[b])], np.int32))
    hc.build_stats()
    return hc


def run_decode(wl, k, alpha, supp_cap=4096):
    dev = torch.device("cuda")
    dc = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table.to(dev), wl.seq_lens.to(dev))
    ekv.rebuild_page_stats(dc)
    Hq = wl.Hq
    sel = ekv.select_params("topk", k)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(wl.B, Hq, dev, delta_bar=True, supp_cap=supp_cap)
    q = wl.q.to(dev)
    out = ekv.decode(dc, q, sel, ekv.attn_params(alpha), ws, stats=st)
    box, _, _ = ekv.score_pages(dc, q, modes=1)
    pi, ns, _ = ekv.select(dc, Hq, sel, alpha=alpha, box=box)
    torch.cuda.synchronize()
    return dc, out.cpu().numpy(), st, box, pi, ns


def check_row(hc, qrow, alpha, k, out, st, box_row, pi_row, ns_row, b, h, M):
    ref = oracle.decode_head(hc, qrow, 0, 0, alpha, k_pages=k, eval_exact=False)
    # box scores of every page of the row: bit-exact (R1)
    np.testing.assert_array_equal(box_row[:M], ref["box"], err_msg=f"box b={b} h={h}")
    pages = ref["pages"].tolist()
    assert int(ns_row) == len(pages)
    assert pi_row[:len(pages)].tolist() == pages, (b, h)
    assert int(st.n_sel[b, h]) == len(pages)
    np.testing.assert_allclose(out[b, h], ref["o"], atol=2e-3, rtol=0, err_msg=f"b={b} h={h}")
    assert int(st.supp_count[b, h]) == ref["supp"], (b, h)
    assert abs(float(st.tau[b, h]) - ref["tau"]) <= 1e-6 * max(1.0, abs(ref["tau"])), (b, h)
    # support set element by element: the oracle's p over C_tok
    att = hc.attend(qrow, 0, 0, ref["pages"], alpha, want_p=True)
    assert st.support(b, h).cpu().tolist() == np.nonzero(att["p"])[0].tolist(), (b, h)
    return float(np.max(np.abs(out[b, h] - ref["o"])))


@pytest.mark.parametrize("kind,alpha", [("randn", 1.5), ("planted", 1.5), ("planted", 1.25)])
def test_c4_one_million_tokens(kind, alpha):
    """configs[3] on one GPU: n = 2^20, 32q/8kv, k = 656 (1 %); KV groups 0 and 7 checked
    against the oracle (8 query heads: box scores of all 65536 pages, page sets, supports,
    outputs)."""
    dev = torch.device("cuda")
    n, Hq, Hkv, k = 1 << 20, 32, 8, 656
    wl = make_workload(1, n, Hq, Hkv, seed=4242, kind=kind, device=dev)
    dc, out, st, box, pi, ns = run_decode(wl, k, alpha, supp_cap=8192)
    box, pi, ns = box.cpu().numpy(), pi.cpu().numpy(), ns.cpu().numpy()
    qh = wl.q.float().cpu().numpy()
    G = Hq // Hkv
    M = n // 16
    worst = 0.0
    for kv in (0, 7):
        hc = head_cache(wl, 0, kv)
        for g in range(G):
            h = kv * G + g
            worst = max(worst, check_row(hc, qh[0, h], alpha, k, out, st, box[0, h], pi[0, h], ns[0, h], 0, h, M))
    assert worst <= 2e-3


def test_c2_batch16_32k_subsample():
    """configs[1]: 16 x 32K, 32q/8kv, top-k 64 pages, planted; 48 (b, head) rows spread over
    every sequence and KV group are checked against the oracle."""
    dev = torch.device("cuda")
    B, n, Hq, Hkv, k, alpha = 16, 32768, 32, 8, 64, 1.5
    wl = make_workload(B, n, Hq, Hkv, seed=77, kind="planted", device=dev)
    dc, out, st, box, pi, ns = run_decode(wl, k, alpha)
    box, pi, ns = box.cpu().numpy(), pi.cpu().numpy(), ns.cpu().numpy()
    qh = wl.q.float().cpu().numpy()
    G = Hq // Hkv
    rng = np.random.default_rng(0)
    rows = [(b, int(h)) for b in range(B) for h in rng.choice(Hq, size=3, replace=False)]
    caches = {}
    for b, h in rows:
        kv = h // G
        if (b, kv) not in caches:
            caches[b, kv] = head_cache(wl, b, kv)
        check_row(caches[b, kv], qh[b, h], alpha, k, out, st, box[b, h], pi[b, h], ns[b, h], b, h, n // 16)


def test_c2_ragged_batch_last_pages_partial():
    """Batch of ragged 32K-class sequences (partial last pages, different lengths per
    sequence): the flattened (b, page) producer ranges of page scoring straddle sequence
    boundaries inside one CTA."""
    dev = torch.device("cuda")
    lens = [32768 - 5, 20001, 31999, 4097, 32768, 17, 29000, 12345]
    B, Hq, Hkv, k, alpha = len(lens), 32, 8, 64, 2.0
    wl = make_workload(B, lens, Hq, Hkv, seed=91, kind="randn", device=dev)
    dc, out, st, box, pi, ns = run_decode(wl, k, alpha)
    box, pi, ns = box.cpu().numpy(), pi.cpu().numpy(), ns.cpu().numpy()
    qh = wl.q.float().cpu().numpy()
    G = Hq // Hkv
    for b in range(B):
        for h in (0, 13, 31):
            hc = head_cache(wl, b, h // G)
            check_row(hc, qh[b, h], alpha, k, out, st, box[b, h], pi[b, h], ns[b, h], b, h, (lens[b] + 15) // 16)
