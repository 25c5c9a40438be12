"""GPU parity of the compressed stored metadata (DESIGN R24): e4m3 page
bounds rounded outward (kmin down, kmax up) and bf16 kavg/kvar, against the oracle's own
rounding of its own fp32 metadata (oracle.HostCache.build_stats(bound=, stat=)).  Bars as for
the exact layout: stored metadata, box / mu / sigma^2 and page sets bit-exact, supports
bit-exact, outputs within 2e-3 (bf16) / 1e-5 (fp32)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload, new_tokens
from gpu_helpers import device_cache, make_pair, meta_f32, q_host, tol_for

pytestmark = pytest.mark.gpu

FORMS = [("e4m3", "f32"), ("kv", "bf16"), ("e4m3", "bf16")]
CASES = [
    (1, 4096, 4, 1, torch.float32),
    (2, [1000, 777], 8, 2, torch.bfloat16),
    (2, [2048, 1500], 32, 8, torch.bfloat16),
    (1, 300, 16, 2, torch.bfloat16),
]


def ids(c):
    return f"B{c[0]}-{c[2]}q{c[3]}kv-{str(c[4]).split('.')[-1]}"


def _check_meta(dc, hc, B):
    g = meta_f32(dc)
    for name in ("kmin", "kmax", "ksum", "ksumsq", "kavg", "kvar"):
        o = getattr(hc, name)
        for b in range(B):
            for lp in range(hc.n_pages(b)):
                ph = int(hc.page_table[b, lp])
                np.testing.assert_array_equal(g[name][ph], o[ph], err_msg=f"{name} b={b} page={lp}")


@pytest.mark.parametrize("form", FORMS, ids=lambda f: f"{f[0]}-{f[1]}")
@pytest.mark.parametrize("case", CASES, ids=ids)
def test_stored_meta_bit_exact(case, form):
    B, sl, Hq, Hkv, dt = case
    wl, dc, hc = make_pair(B, sl, Hq, Hkv, dtype=dt, seed=11, kind="planted", bound=form[0], stat=form[1])
    torch.cuda.synchronize()
    _check_meta(dc, hc, B)


@pytest.mark.parametrize("form", FORMS, ids=lambda f: f"{f[0]}-{f[1]}")
def test_append_incremental_equals_rebuild(form):
    """Incremental e4m3 bounds: rd(min(rd(m), k)) = rd(min(m, k)) (monotone rounding), so
    single- and multi-token appends give the bulk build's bits."""
    B, Hq, Hkv = 2, 8, 2
    wl = make_workload(B, [40, 15], Hq, Hkv, seed=3, spare_tokens=40)
    dc = device_cache(wl, *form)
    for step in range(20):
        _, k, v = new_tokens(B, Hq, Hkv, seed=100 + step, device="cuda")
        ekv.append_kv(dc, 3.0 * k, v)
    _, k, v = new_tokens(B * 3, Hq, Hkv, seed=999, device="cuda")
    ekv.append_kv(dc, k.view(B, 3, Hkv, 128), v.view(B, 3, Hkv, 128))
    torch.cuda.synchronize()
    hc = oracle.HostCache(dc.K.float().cpu().numpy(), dc.V.float().cpu().numpy(), dc.page_table.cpu().numpy(),
                          dc.seq_lens.cpu().numpy())
    hc.build_stats(bound=form[0], stat=form[1])
    _check_meta(dc, hc, B)


@pytest.mark.parametrize("form", FORMS, ids=lambda f: f"{f[0]}-{f[1]}")
@pytest.mark.parametrize("case", CASES, ids=ids)
def test_score_pages_bit_exact(case, form):
    B, sl, Hq, Hkv, dt = case
    wl, dc, hc = make_pair(B, sl, Hq, Hkv, dtype=dt, seed=5, kind="llama", bound=form[0], stat=form[1])
    G = Hq // Hkv
    box, mu, s2 = ekv.score_pages(dc, wl.q.cuda(), modes=3)
    box1, _, _ = ekv.score_pages(dc, wl.q.cuda(), modes=1)
    _, mu2, s22 = ekv.score_pages(dc, wl.q.cuda(), modes=2)
    torch.cuda.synchronize()
    qh = q_host(wl)
    for b in range(B):
        M = hc.n_pages(b)
        for h in range(Hq):
            ob, om, os2 = hc.score_pages(qh[b, h], b, h // G, modes=3)
            for arr, ref in ((box, ob), (box1, ob), (mu, om), (mu2, om), (s2, os2), (s22, os2)):
                np.testing.assert_array_equal(arr[b, h, :M].cpu().numpy(), ref, err_msg=f"b={b} h={h}")


@pytest.mark.parametrize("alpha", [1.5, 2.0, 1.25])
@pytest.mark.parametrize("case", CASES[1:3], ids=ids)
def test_decode_topk_e4m3(case, alpha):
    B, sl, Hq, Hkv, dt = case
    wl, dc, hc = make_pair(B, sl, Hq, Hkv, dtype=dt, seed=21, kind="llama", bound="e4m3", stat="bf16")
    G, k = Hq // Hkv, 16
    sel = ekv.select_params("topk", k)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(B, Hq, torch.device("cuda"), delta_bar=True, supp_cap=2048)
    out = ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(alpha), ws, stats=st).cpu().numpy()
    torch.cuda.synchronize()
    qh = q_host(wl)
    for b in range(B):
        for h in range(Hq):
            ref = oracle.decode_head(hc, qh[b, h], b, h // G, alpha, k_pages=k)
            assert int(st.n_sel[b, h]) == len(ref["pages"])
            np.testing.assert_allclose(out[b, h], ref["o"], atol=tol_for(dt), rtol=0)
            assert int(st.supp_count[b, h]) == ref["supp"]
            att = hc.attend(qh[b, h], b, h // G, ref["pages"], alpha, want_p=True)
            n = int(st.supp_count[b, h])
            pt = hc.page_table[b]
            # support positions (token order) element by element
            assert st.support(b, h).cpu().tolist() == np.nonzero(att["p"])[0].tolist()


def test_decode_gaussian_bf16_stats():
    B, sl, Hq, Hkv = 2, [3000, 2100], 8, 2
    wl, dc, hc = make_pair(B, sl, Hq, Hkv, seed=8, kind="llama", bound="e4m3", stat="bf16")
    G, alpha = Hq // Hkv, 1.5
    sel = ekv.select_params("gauss", 0, 0.99, 0.0)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(B, Hq, torch.device("cuda"), delta_bar=True, gauss=True)
    out = ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(alpha), ws, stats=st).cpu().numpy()
    torch.cuda.synchronize()
    qh = q_host(wl)
    zq = oracle.zq_table(0.99, 16)
    for b in range(B):
        counts = hc.page_counts(b)
        for h in range(Hq):
            ref = oracle.decode_head(hc, qh[b, h], b, h // G, alpha, policy="gauss")
            tg = float(st.tau_hat[b, h])
            assert abs(tg - ref["tau_hat"]) <= 1e-10 * max(1.0, abs(ref["tau_hat"]))
            pages = oracle.gauss_select(ref["mu"], ref["sigma2"], counts, alpha, tg, 0.0, zq)
            assert int(st.n_sel[b, h]) == len(pages)
            att = hc.attend(qh[b, h], b, h // G, pages, alpha)
            np.testing.assert_allclose(out[b, h], att["o"], atol=2e-3, rtol=0)
            assert int(st.supp_count[b, h]) == att["supp"]


@pytest.mark.parametrize("kind", ["llama"])
def test_c4_one_million_tokens_e4m3(kind):
    """configs[3] with e4m3 bounds and bf16 stats (the N3 layout bench.py times): KV group 3
    against the oracle -- box scores of all 65536 pages, page sets, supports, outputs."""
    from test_gpu_fullsize import check_row, head_cache  # noqa: E402
    dev = torch.device("cuda")
    n, Hq, Hkv, k, alpha = 1 << 20, 32, 8, 656, 1.5
    wl = make_workload(1, n, Hq, Hkv, seed=4243, kind=kind, device=dev)
    dc = device_cache(wl, "e4m3", "bf16")
    sel = ekv.select_params("topk", k)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(1, Hq, dev, delta_bar=True, supp_cap=8192)
    q = wl.q.to(dev)
    out = ekv.decode(dc, q, sel, ekv.attn_params(alpha), ws, stats=st).cpu().numpy()
    box, _, _ = ekv.score_pages(dc, q, modes=1)
    pi, ns, _ = ekv.select(dc, Hq, sel, alpha=alpha, box=box)
    torch.cuda.synchronize()
    box, pi, ns = box.cpu().numpy(), pi.cpu().numpy(), ns.cpu().numpy()
    qh = wl.q.float().cpu().numpy()
    G = Hq // Hkv
    kv = 3
    from paper_2605_21649_b200.workload import gather_head
    Kh, Vh = gather_head(wl, 0, kv)
    M = Kh.shape[0]
    hc = oracle.HostCache(Kh.float().cpu().numpy()[:, None], Vh.float().cpu().numpy()[:, None],
                          np.arange(M, dtype=np.int32)[None], np.array([n], np.int32))
    hc.build_stats(bound="e4m3", stat="bf16")
    for g in range(G):
        h = kv * G + g
        check_row(hc, qh[0, h], alpha, k, out, st, box[0, h], pi[0, h], ns[0, h], 0, h, M)


def test_score_e4m3_query_not_f16_exact():
    """The e4m3 box path runs FHFMA on q converted to f16; query chunks that f16 cannot hold
    exactly (|q_i| < 2^-17, |q_i| > 65504) take the fp32 chain -- the box stays bit-exact."""
    B, sl, Hq, Hkv = 2, [900, 1300], 8, 2
    wl, dc, hc = make_pair(B, sl, Hq, Hkv, seed=12, kind="llama", bound="e4m3", stat="bf16")
    q = wl.q.clone()
    q[0, 1, 5] = 3e-7          # below the f16 subnormal grid for 8 significant bits
    q[1, 6, 100] = -1.1e-6
    q[1, 2, 64] = 7.0e4         # above f16's largest finite value
    q = q.to(torch.bfloat16)
    box, _, _ = ekv.score_pages(dc, q.cuda(), modes=1)
    torch.cuda.synchronize()
    qh = q.float().numpy()
    G = Hq // Hkv
    for b in range(B):
        M = hc.n_pages(b)
        for h in range(Hq):
            ob, _, _ = hc.score_pages(qh[b, h], b, h // G, modes=1)
            np.testing.assert_array_equal(box[b, h, :M].cpu().numpy(), ob, err_msg=f"b={b} h={h}")
