"""GPU: certified conservative box selection (Prop. B.2; DESIGN R27)
through entmaxkv_decode with policy CERTIFIED, against the CPU oracle.  Bars: the first pass's
tau~ within 1e-6 relative of the oracle's; |C_page| equal to the oracle's certified set
evaluated at the GPU's tau~ (the fp64 decision at the GPU's threshold, as for tau_hat in R14);
and -- the point of the mode -- the output IS full-cache entmax: out within 2e-3 / 1e-5 of the
oracle's full attend, tau within 1e-6, support size and support token set bit-exact,
delta_bar = 0."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from gpu_helpers import make_pair, q_host, tol_for

pytestmark = pytest.mark.gpu

CASES = [
    (2, [3000, 1777], 8, 2, torch.bfloat16, "planted"),
    (1, 4096, 4, 1, torch.float32, "planted"),
    (2, [2048, 999], 32, 8, torch.bfloat16, "llama"),
    (1, 1500, 8, 8, torch.bfloat16, "randn"),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"B{c[0]}-{c[2]}q{c[3]}kv-{str(c[4]).split('.')[-1]}-{c[5]}")
@pytest.mark.parametrize("alpha", [1.5, 2.0, 1.25])
@pytest.mark.parametrize("k", [4, 16])
def test_certified_decode_is_full_entmax(case, alpha, k):
    B, sl, Hq, Hkv, dt, kind = case
    wl, dc, hc = make_pair(B, sl, Hq, Hkv, dtype=dt, seed=61, kind=kind)
    G = Hq // Hkv
    qh = q_host(wl)
    sel = ekv.select_params("certified", k)
    ws = ekv.alloc_workspace(dc, Hq, sel)
    st = ekv.DecodeStats(B, Hq, "cuda", delta_bar=True, gauss=True, supp_cap=4096)
    out = ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(alpha), ws, stats=st)
    torch.cuda.synchronize()
    out = out.cpu().numpy()
    for b in range(B):
        M = hc.n_pages(b)
        for h in range(Hq):
            box, _, _ = hc.score_pages(qh[b, h], b, h // G, modes=1)
            first = hc.attend(qh[b, h], b, h // G, oracle.topk(box, k), alpha, 0)
            t_gpu = float(st.tau_hat[b, h])
            assert abs(t_gpu - first["tau"]) <= 1e-6 * max(1.0, abs(first["tau"])), (b, h)
            cert = oracle.box_certified(box, alpha, t_gpu)
            assert int(st.n_sel[b, h]) == len(cert), (b, h)
            full = hc.attend(qh[b, h], b, h // G, np.arange(M, dtype=np.int32), alpha, 0, want_p=True)
            np.testing.assert_allclose(out[b, h], full["o"], atol=tol_for(dt), rtol=0, err_msg=f"b={b} h={h}")
            assert int(st.supp_count[b, h]) == full["supp"], (b, h)
            assert abs(float(st.tau[b, h]) - full["tau"]) <= 1e-6 * max(1.0, abs(full["tau"]))
            assert st.support(b, h).cpu().tolist() == np.nonzero(full["p"])[0].tolist(), (b, h)
            assert float(st.delta_bar[b, h]) == 0.0, (b, h)


def test_certified_rejects_softmax():
    wl, dc, hc = make_pair(1, 1000, 4, 1, seed=1)
    sel = ekv.select_params("certified", 4)
    with pytest.raises(ekv.EkvError):
        ekv.decode(dc, wl.q.cuda(), sel, ekv.attn_params(1.5, "softmax"), ekv.alloc_workspace(dc, 4, sel))
