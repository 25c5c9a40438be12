"""Pins for SURVEY 8(f) N4 in the oracle: (1) the certified conservative box selection of
Prop. B.2, C_page = {p : (alpha-1) sbar_box(p) > tau_hat} for tau_hat <= tau, with
tau_hat = the exact threshold of a first top-k pass (DESIGN R27; tau~ <= tau by R13); (2) the
Gaussian selector's truncated moment E[(Y)_+^beta] for non-integer beta, "evaluated
numerically" (DESIGN R28), pinned against arbitrary-precision quadrature (mpmath),
the parabolic-cylinder closed form (scipy), App. D's closed forms at integer beta and the
point-mass limit.

Citations: P:L = PAPER.md line L; R<n> = DESIGN.md reading n."""
import numpy as np
import pytest

import oracle
from test_oracle_pins_r2 import bf16_round


def test_box_certified_hand_case():
    """a = alpha - 1 = 1/2, box = [1, 2, 3, -4, 2.5], tau_hat = 1: a box = [0.5, 1, 1.5, -2, 1.25]
    -> strictly above 1: pages 2 and 4 (page 1 ties: strict >, as P:845; >= would keep it; a
    dropped factor a would keep pages 1, 2, 4; tau_hat = 0.99 adds page 1)."""
    box = np.array([1.0, 2.0, 3.0, -4.0, 2.5], np.float32)
    assert oracle.box_certified(box, 1.5, 1.0).tolist() == [2, 4]
    assert oracle.box_certified(box, 1.5, 0.99).tolist() == [1, 2, 4]
    assert oracle.box_certified(box, 2.0, 2.0).tolist() == [2, 4]        # a = 1: 3 > 2, 2.5 > 2
    assert oracle.box_certified(box, 1.5, 10.0).tolist() == []


def _cache(rng, n, kind):
    P = 16
    M = (n + P - 1) // P
    K = rng.standard_normal((M + 2, 1, P, 128))
    q = rng.standard_normal(128)
    if kind == "planted":                        # a few heavy hitters along q
        for j in rng.choice(n, size=6, replace=False):
            K[j // P, 0, j % P] = 0.5 * K[j // P, 0, j % P] + rng.uniform(2, 5) * q / np.linalg.norm(q) * 1.5
    K = bf16_round(K)
    V = bf16_round(rng.standard_normal((M + 2, 1, P, 128)))
    pt = rng.permutation(M + 2)[:M].astype(np.int32)[None]
    hc = oracle.HostCache(K, V, pt, np.array([n], np.int32))
    hc.build_stats()
    return hc, bf16_round(q * 1.5), M


@pytest.mark.parametrize("alpha", [1.5, 2.0, 1.25])
@pytest.mark.parametrize("kind", ["planted", "randn"])
def test_certified_selection_contains_support_and_is_exact(alpha, kind):
    """Prop. B.2: with tau_hat <= tau every page holding a full-cache support token is selected,
    and then (Prop. 2) sparse entmax over the selection IS full-cache entmax: the
    output, tau and support equal the full pass's (independent: the full pass never looks at
    box scores).  Also tau_lo <= tau (R13)."""
    rng = np.random.default_rng(7 if kind == "planted" else 8)
    for trial in range(3):
        hc, q, M = _cache(rng, int(rng.integers(600, 1500)), kind)
        res = oracle.decode_head(hc, q, 0, 0, alpha, k_pages=4, policy="certified")
        full = hc.attend(q, 0, 0, np.arange(M, dtype=np.int32), alpha, 0, want_p=True)
        assert res["tau_lo"] <= full["tau"] + 1e-12
        sup_pages = {j // 16 for j in np.nonzero(full["p"])[0]}
        assert sup_pages <= set(res["pages"].tolist())
        assert res["supp"] == full["supp"]
        assert abs(res["tau"] - full["tau"]) <= 1e-12 * max(1.0, abs(full["tau"]))
        np.testing.assert_allclose(res["o"], full["o"], atol=1e-12, rtol=0)


def test_certified_with_too_high_tau_can_miss():
    """Sanity of the premise: a tau_hat above tau is not certified -- at tau_hat = the smallest
    (alpha-1) box of a support page (> tau) that page is dropped (strict >), so the inclusion
    checked above is a real property of tau_hat <= tau, not of loose bounds alone."""
    rng = np.random.default_rng(9)
    hc, q, M = _cache(rng, 1200, "planted")
    box, _, _ = hc.score_pages(q, 0, 0, modes=1)
    full = hc.attend(q, 0, 0, np.arange(M, dtype=np.int32), 1.5, 0, want_p=True)
    sup_pages = {j // 16 for j in np.nonzero(full["p"])[0]}
    t_bad = min(0.5 * float(box[p]) for p in sup_pages)
    assert t_bad > full["tau"]
    sel = set(oracle.box_certified(box, 1.5, t_bad).tolist())
    assert not sup_pages <= sel


# ------------------------------------------------------------------ numerical truncated moment
import math  # noqa: E402

BETAS = [0.5, 1.0 / (float(np.float32(1.7)) - 1.0), 2.5, 0.75, 3.3, 6.5]
POINTS = [(-3.0, 1.0), (-1.0, 0.5), (0.0, 1.0), (0.3, 2.0), (2.0, 1.0), (5.0, 0.7), (40.0, 1.5), (-8.0, 1.0)]


@pytest.mark.parametrize("beta", BETAS)
def test_trunc_moment_num_vs_mpmath(beta):
    """E[(Y)_+^beta] = sigY^beta int_0^inf u^beta phi(u - muY/sigY) du, 40-digit mpmath quadrature
    (split at the mode) as the reference: 1e-13 relative.  A dropped sigY^beta, a wrong
    standardisation (m = muY sigY) or integrating from -inf fails."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 40
    for muY, sig in POINTS:
        m = mpmath.mpf(muY) / sig
        ref = float(mpmath.mpf(sig) ** beta * mpmath.quad(lambda u: u ** beta * mpmath.npdf(u - m),
                                                          [0, max(m, 0), max(m, 0) + 40]))
        got = oracle.trunc_moment_num(beta, muY, sig)
        assert abs(got - ref) <= 1e-13 * abs(ref), (beta, muY, sig, got, ref)


@pytest.mark.parametrize("nu", [0.5, 1.4285714, 2.5])
def test_trunc_moment_num_vs_parabolic_cylinder(nu):
    """Closed form through the parabolic cylinder function D (a textbook identity):
    int_0^inf u^nu phi(u - m) du = Gamma(nu+1) e^{-m^2/4} D_{-nu-1}(-m) / sqrt(2 pi)."""
    sp = pytest.importorskip("scipy.special")
    for m in (-3.0, -1.0, 0.0, 0.5, 2.0, 5.0):
        ref = math.gamma(nu + 1) * math.exp(-m * m / 4) * sp.pbdv(-nu - 1, -m)[0] / math.sqrt(2 * math.pi)
        got = oracle.trunc_moment_num(nu, m, 1.0)
        assert abs(got - ref) <= 1e-12 * abs(ref), (nu, m, got, ref)


@pytest.mark.parametrize("beta", [1, 2, 3, 4])
def test_trunc_moment_num_matches_app_d_closed_forms(beta):
    """At integer beta the quadrature reproduces App. D's closed forms (R15).  (Deep
    in the lower tail the closed forms themselves cancel -- muY Phi + sigY phi with muY < 0 --
    and lose up to ~1e-11 relative at m = -3 (beta = 4) and more at m = -8; the quadrature
    matches 40-digit mpmath there, above.  So: 1e-13 for m >= 0, 2e-11 for -5 < m < 0.)"""
    for muY, sig in [x for x in POINTS if x[0] / x[1] > -5]:
        ref = oracle.trunc_moment(beta, muY, sig)
        got = oracle.trunc_moment_num(float(beta), muY, sig)
        tol = 1e-13 if muY >= 0 else 2e-11
        assert abs(got - ref) <= tol * max(abs(ref), 1e-300), (beta, muY, sig, got, ref)


def test_trunc_moment_num_point_mass_limit():
    """sigY -> 0: E[(Y)_+^beta] -> [muY]_+^beta; sigY = 0 is the point mass itself."""
    b = BETAS[1]
    assert oracle.trunc_moment_num(b, 1.3, 0.0) == 1.3 ** b
    assert oracle.trunc_moment_num(b, -0.2, 0.0) == 0.0
    assert abs(oracle.trunc_moment_num(b, 1.3, 1e-4) - 1.3 ** b) <= 1e-6
