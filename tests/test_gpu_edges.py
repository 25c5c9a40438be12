"""GPU edge cases the parity suite did not reach (round-1 verdict, "untested on GPU"):

* the Gaussian selector's empty-selection fallback (P:432-477 keeps p iff
  a (mu_p + sigma_p zq[c_p]) > tau_hat - Delta; an empty set falls back to argmax mu with
  the lower page index on ties, SURVEY 8(c) step 4 / DESIGN R14), on synthetic page
  statistics where no page passes;
* exact ties at the entmax threshold in the kernels (R9: the support is {j : F(z_j) < 1},
  so tokens with equal scores get the same F and are all in or all out): duplicated key
  rows at the support boundary, support sets compared element by element with the oracle.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload
from gpu_helpers import device_cache, host_cache, q_host, tol_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("alpha", [1.5, 2.0, 1.25])
def test_gaussian_empty_selection_falls_back_to_argmax_mu(alpha):
    """Wide page distributions (sigma = 10) centred low (mu ~ -5): tau_hat sits in the far
    tail, and with q_page = 0.05 (zq[16] ~ +0.95) no page reaches it -> the selection is the
    single page argmax mu; a tie for the maximum goes to the lower page index."""
    B, n, Hq, Hkv = 1, 128 * 16 - 5, 8, 2                  # 128 pages, partial last page
    wl = make_workload(B, n, Hq, Hkv, dtype=torch.bfloat16, seed=71)
    dc, hc = device_cache(wl), host_cache(wl)
    maxp = dc.max_pages
    g = torch.Generator().manual_seed(5)
    mu = (-5.0 + 0.01 * torch.randn(B, Hq, maxp, generator=g)).float()
    s2 = torch.full((B, Hq, maxp), 100.0, dtype=torch.float32)
    expect = {}
    for h in range(Hq):
        if h % 2 == 0:
            mu[0, h, 37 + h] = -1.0                          # unique maximum
            expect[h] = 37 + h
        else:
            mu[0, h, 90] = -1.0                              # tied maximum: lower index wins
            mu[0, h, 50 + h] = -1.0
            expect[h] = 50 + h
    sel = ekv.select_params("gauss", q_page=0.05, margin=0.0)
    pi, ns, th = ekv.select(dc, Hq, sel, alpha=alpha, mu=mu.cuda(), sigma2=s2.cuda())
    torch.cuda.synchronize()
    pi, ns, th = pi.cpu().numpy(), ns.cpu().numpy(), th.cpu().numpy()
    counts = hc.page_counts(0)
    M = len(counts)
    zq = oracle.zq_table(0.05, 16)
    for h in range(Hq):
        m_row, s_row = mu[0, h, :M].numpy(), s2[0, h, :M].numpy()
        t_ref = oracle.gauss_tau(m_row, s_row, counts, alpha)
        assert abs(th[0, h] - t_ref) <= 1e-10 * max(1.0, abs(t_ref)), (h, th[0, h], t_ref)
        # premise: the page rule keeps nothing (every page far below tau_hat)
        a = alpha - 1.0
        keep = a * (m_row.astype(np.float64) + np.sqrt(s_row.astype(np.float64)) * zq[counts]) > th[0, h]
        assert not keep.any()
        ref = oracle.gauss_select(m_row, s_row, counts, alpha, th[0, h], 0.0, zq)
        assert ref.tolist() == [expect[h]]
        assert ns[0, h] == 1 and pi[0, h, 0] == expect[h], (h, ns[0, h], pi[0, h, :2])


def _dup_tokens(wl, b, kvh, src, dsts):
    """Copy token src's key row into the token slots dsts (same sequence and KV head)."""
    P = wl.P
    pt = wl.page_table[b]
    K = wl.K.clone()
    ps, ts = int(pt[src // P]), src % P
    for j in dsts:
        K[int(pt[j // P]), kvh, j % P] = K[ps, kvh, ts]
    wl.K = K.contiguous()


@pytest.mark.parametrize("alpha", [1.5, 2.0, 1.25])
@pytest.mark.parametrize("where", ["last_in", "first_out"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_entmax_ties_at_support_boundary(alpha, where, dtype):
    """Six tokens with one key row (identical scores for every head of the group), placed at
    the support boundary of head 0: the smallest positive p (last_in) or the largest excluded
    z (first_out) of the unmodified row.  Decode over every page (k >= M: the sparse kernels
    see the whole row) must give the oracle's support set element by element, with the tied
    tokens all in or all out, and the outputs within tolerance."""
    B, n, Hq, Hkv = 1, 1024 + 7, 4, 1
    wl = make_workload(B, n, Hq, Hkv, dtype=dtype, seed=83, kind="planted")
    hc0 = host_cache(wl)
    qh = q_host(wl)
    M = hc0.n_pages(0)
    ref0 = hc0.attend(qh[0, 0], 0, 0, np.arange(M, dtype=np.int32), alpha, want_p=True, want_s=True)
    p0, s0 = ref0["p"], ref0["s"]
    if where == "last_in":
        pos = np.nonzero(p0 > 0)[0]
        src = int(pos[np.argmin(p0[pos])])
    else:
        out = np.nonzero(p0 == 0)[0]
        src = int(out[np.argmax(s0[out])])
    rng = np.random.default_rng(3)
    others = np.setdiff1d(np.arange(n), [src])
    dsts = rng.choice(others, size=5, replace=False).tolist()
    _dup_tokens(wl, 0, 0, src, dsts)
    dc, hc = device_cache(wl), host_cache(wl)
    sel = ekv.select_params("topk", M)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(B, Hq, "cuda", supp_cap=4096)
    out = ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(alpha), ws, stats=st)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    tied = sorted([src] + dsts)
    for h in range(Hq):
        ref = hc.attend(qh[0, h], 0, 0, np.arange(M, dtype=np.int32), alpha, want_p=True, want_s=True)
        assert len(set(ref["s"][tied].tolist())) == 1                     # the tie is exact
        sup = st.support(0, h).cpu().tolist()
        assert sup == np.nonzero(ref["p"])[0].tolist(), (h, where)
        ins = [j in set(sup) for j in tied]
        assert all(ins) or not any(ins), (h, ins)
        np.testing.assert_allclose(out[0, h], ref["o"], atol=tol_for(dtype), rtol=0)
        assert abs(float(st.tau[0, h]) - ref["tau"]) <= 1e-6 * max(1.0, abs(ref["tau"]))


@pytest.mark.parametrize("alpha", [1.5, 2.0, 1.25, 1.7])
@pytest.mark.parametrize("ncand", [1, 31, 32, 33, 64])
def test_tau_candidate_count_boundary(alpha, ncand):
    """The tau kernel solves rows with <= 32 candidates (z > z_max - 1) in one warp and larger
    ones on the block path: exactly ncand tokens are placed within 1 / (alpha - 1) of the
    maximum score (the rest far below), so both paths and the switch between them are hit;
    output, tau and the support set against the oracle."""
    B, n, Hq, Hkv = 1, 700, 2, 1
    wl = make_workload(B, n, Hq, Hkv, dtype=torch.float32, seed=91)
    g = torch.Generator().manual_seed(ncand)
    a = alpha - 1.0
    K = torch.zeros_like(wl.K)
    pt = wl.page_table[0]
    near = torch.randperm(n, generator=g)[:ncand].tolist()
    for j in range(n):
        # head 0 scores ~ key[0]: the near tokens spread over (z_max - 0.9 / a, z_max], the rest
        # 5 / a below (z = a s); head 1 sees key[1] (random, unconstrained)
        v = (4.0 - 0.9 * torch.rand(1, generator=g).item() / a) if j in near else (4.0 - 5.0 / a)
        K[int(pt[j // 16]), 0, j % 16, 0] = v
        K[int(pt[j // 16]), 0, j % 16, 1] = torch.randn(1, generator=g).item()
    K[int(pt[near[0] // 16]), 0, near[0] % 16, 0] = 4.0            # the maximum
    wl.K = K.contiguous()
    cd = float(np.float32(1.0 / np.sqrt(128.0)))
    q = torch.zeros(B, Hq, 128, dtype=torch.float32)
    q[0, 0, 0] = 1.0 / cd
    q[0, 1, 1] = 1.0 / cd
    wl.q = q
    dc, hc = device_cache(wl), host_cache(wl)
    qh = q_host(wl)
    M = hc.n_pages(0)
    sel = ekv.select_params("topk", M)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(B, Hq, "cuda", supp_cap=4096)
    out = ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(alpha), ws, stats=st)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    for h in range(Hq):
        ref = hc.attend(qh[0, h], 0, 0, np.arange(M, dtype=np.int32), alpha, want_p=True, want_s=True)
        if h == 0:
            z = a * ref["s"].astype(np.float64)
            assert int(np.sum(z > z.max() - 1.0)) == ncand             # the premise: ncand candidates
        assert st.support(0, h).cpu().tolist() == np.nonzero(ref["p"])[0].tolist(), (h, ncand)
        np.testing.assert_allclose(out[0, h], ref["o"], atol=1e-5, rtol=0)
        assert abs(float(st.tau[0, h]) - ref["tau"]) <= 1e-6 * max(1.0, abs(ref["tau"]))
