"""GPU: capacity limits are surfaced, never silent (SURVEY 8(b) EKV_ERR_CAPACITY + device flag).

* a support larger than the tau kernel's shared-memory list (kTsCap = 10240 candidates): the
  row's out / tau are NaN, supp = -1, and entmaxkv_workspace_status reports EKV_STATUS_CAPACITY
  (EKV_ERR_CAPACITY);
* Gaussian (variable-length) lists run the tau kernel at a reduced capacity (4096); a row whose
  support exceeds it is re-run at the full capacity -- exact result, no flag;
* sequence-sharded: more than 8192 candidates of a row on one rank marks the row on EVERY rank
  in the same round (NaN, supp -1) and the adaptive mode returns EKV_ERR_CAPACITY on all ranks.
"""
import threading

import numpy as np
import pytest
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200 import sharding
from paper_2605_21649_b200.workload import make_workload
from gpu_helpers import device_cache, host_cache, q_host

pytestmark = pytest.mark.gpu


def flat_workload(n, Hq=4, Hkv=1, seed=3, scale=1e-3):
    wl = make_workload(1, n, Hq, Hkv, seed=seed, kind="randn")
    wl.K = (wl.K.float() * scale).to(wl.K.dtype)        # near-equal scores: the support is ~all of C_tok
    return wl


def test_decode_support_over_capacity_is_flagged():
    wl = flat_workload(12000)
    dc = device_cache(wl)
    Hq = 4
    sel = ekv.select_params("topk", 700)                 # 11200 tokens > 10240
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(1, Hq, torch.device("cuda"), delta_bar=True)
    out = ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(1.25), ws, stats=st)
    flags = ekv.workspace_status(dc, Hq, sel, ws)
    assert flags & ekv.EKV_STATUS_CAPACITY
    assert torch.isnan(out).all()
    assert (st.supp_count == -1).all()
    with pytest.raises(ekv.EkvError) as ei:
        ekv.workspace_status(dc, Hq, sel, ws, raise_on_capacity=True)
    assert ei.value.status == ekv.EKV_ERR_CAPACITY
    # a fitting call on the same workspace clears the word
    sel2 = ekv.select_params("topk", 64)
    ws2 = ekv.alloc_workspace(dc, Hq, sel2)
    ekv.decode(dc, wl.q.cuda(), sel2, ekv.attn_params(1.25), ws2, stats=st)
    assert ekv.workspace_status(dc, Hq, sel2, ws2) == 0


def test_gaussian_support_above_reduced_capacity_is_rerun_exactly():
    """6000-token near-flat row, Gaussian selector: every page selected, support ~6000 > 4096."""
    n, Hq, alpha = 6000, 4, 1.25
    wl = flat_workload(n, Hq=Hq)
    dc, hc = device_cache(wl), host_cache(wl)
    sel = ekv.select_params("gauss", 0, 0.99, 0.0)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(1, Hq, torch.device("cuda"), delta_bar=False, gauss=True)
    out = ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(alpha), ws, stats=st).cpu().numpy()
    assert ekv.workspace_status(dc, Hq, sel, ws) == 0
    qh = q_host(wl)
    zq = oracle.zq_table(0.99, 16)
    for h in range(Hq):
        ref = oracle.decode_head(hc, qh[0, h], 0, 0, alpha, policy="gauss")
        pages = oracle.gauss_select(ref["mu"], ref["sigma2"], hc.page_counts(0), alpha, float(st.tau_hat[0, h]), 0.0, zq)
        att = hc.attend(qh[0, h], 0, 0, pages, alpha)
        assert att["supp"] > 4096
        np.testing.assert_allclose(out[0, h], att["o"], atol=2e-3, rtol=0)
        assert int(st.supp_count[0, h]) == att["supp"]


def _run_sharded(wl, world, k, alpha, fixed_rounds=0):
    Hq = wl.q.shape[1]
    grp = sharding.LoopbackGroup(world)
    gl = wl.seq_lens.to(torch.int32).cuda()
    caches = [sharding.shard_cache(wl.K, wl.V, wl.page_table, wl.seq_lens, r, world) for r in range(world)]
    torch.cuda.synchronize()
    sel, attn = ekv.select_params("topk", k), ekv.attn_params(alpha)
    res = [None] * world

    def worker(r):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        ws = ekv.shard_workspace(caches[r], Hq, sel, world)
        st = ekv.DecodeStats(1, Hq, "cuda", delta_bar=False)
        out = torch.full((1, Hq, 128), 7.0, device="cuda")
        err = None
        try:
            with torch.cuda.stream(s):
                ekv.decode_sharded(caches[r], gl, wl.q.cuda(), sel, attn, grp.comm(r), ws, out=out, stats=st,
                                   stream=s, fixed_rounds=fixed_rounds)
        except ekv.EkvError as e:
            err = e
        s.synchronize()
        flags = ekv.workspace_status(caches[r], Hq, sel, ws, stream=s)
        res[r] = (out.cpu().numpy(), st, err, flags)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res


def test_sharded_capacity_overflow_marks_every_rank():
    wl = flat_workload(20000, Hq=4)
    res = _run_sharded(wl, 2, 1100, 1.25)                # ~8800 candidates per rank > 8192
    for out, st, err, flags in res:
        assert err is not None and err.status == ekv.EKV_ERR_CAPACITY
        assert flags & ekv.EKV_STATUS_CAPACITY
        assert np.isnan(out).all()
        assert (st.supp_count == -1).all()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_fixed_rounds_matches_oracle(world):
    """fixed_rounds = 12 (no host read, graph-capturable) gives the adaptive mode's exact result."""
    B, Hq, Hkv, k, alpha = 1, 8, 2, 64, 1.5
    wl = make_workload(B, 20000, Hq, Hkv, seed=43, kind="planted")
    res = _run_sharded(wl, world, k, alpha, fixed_rounds=12)
    hc, qh = host_cache(wl), q_host(wl)
    for h in range(Hq):
        ref = oracle.decode_head(hc, qh[0, h], 0, h // (Hq // Hkv), alpha, k_pages=k)
        for out, st, err, flags in res:
            assert err is None and flags == 0
            np.testing.assert_allclose(out[0, h], ref["o"], atol=2e-3, rtol=0)
            assert int(st.supp_count[0, h]) == ref["supp"]
