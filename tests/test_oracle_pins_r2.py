"""Round-2 pins for the oracle functions that round 1 pinned only one-sidedly (VERDICT r1,
weak 1): each test checks the oracle against a hand-worked value or an independent
computation chosen so that a plausible mistake (a dropped term, sigma^2 for sigma, >= for
>, the wrong count, a V-indexing slip, a Newton step for a Halley step) fails it.

Citations: P:L = PAPER.md line L; R<n> = DESIGN.md reading n.
"""
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest

import oracle

RNG = np.random.default_rng(2024)


def bf16_round(x):
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


# ------------------------------------------------------------------ Gaussian page rule
def test_gauss_select_hand_case():
    """Eq. gaussian-selector-main: keep p iff (alpha-1)(mu_p + sigma_p zq[c_p]) >
    tau_hat - Delta.  alpha = 1.5 (a = 1/2), q_page = 0.99, tau_hat - Delta = 1.375 - 0.125 = 1.25
    (exact).  Hand values of a * sbar (zq[16] = 3.2258715, zq[1] = 2.3263479):
      p0  mu 1.0, sigma^2 0.25, c 16 -> a (1 + 0.5 * 3.2259)  = 1.3065  keep
          (sigma^2 for sigma: 0.903 -> drop)
      p1  mu 2.4, sigma^2 0,    c 16 -> 1.2                   drop  (no factor a: 2.4 -> keep)
      p2  mu 0.2, sigma^2 4,    c 16 -> a (0.2 + 2 * 3.2259)  = 3.326   keep
      p3  mu 2.5, sigma^2 0,    c 16 -> 1.25 == threshold     drop  (strict >, P:145 style; >= keeps)
      p4  mu 3.0, sigma^2 0,    c 16 -> 1.5                   keep  (tau + Delta: 1.5 > 1.5 drops)
      p5  mu 0.0, sigma^2 1,    c 1  -> a * 2.3263 = 1.1632   drop  (zq[16] for c=1: 1.613 -> keep)"""
    mu = np.array([1.0, 2.4, 0.2, 2.5, 3.0, 0.0], np.float32)
    s2 = np.array([0.25, 0.0, 4.0, 0.0, 0.0, 1.0], np.float32)
    cnt = np.array([16, 16, 16, 16, 16, 1], np.int32)
    zq = oracle.zq_table(0.99, 16)
    sel = oracle.gauss_select(mu, s2, cnt, 1.5, 1.375, 0.125, zq)
    assert sel.tolist() == [0, 2, 4]
    # Delta widens the set: Delta = 0.3 -> threshold 1.075 also keeps p1 (1.2), p3 (1.25), p5 (1.163)
    sel = oracle.gauss_select(mu, s2, cnt, 1.5, 1.375, 0.3, zq)
    assert sel.tolist() == [0, 1, 2, 3, 4, 5]


def test_gauss_select_empty_fallback_ties():
    """R6: nothing above the threshold -> argmax mu, lower page index on ties."""
    mu = np.array([1.0, 3.0, 3.0, 2.0], np.float32)
    s2 = np.zeros(4, np.float32)
    cnt = np.full(4, 16, np.int32)
    sel = oracle.gauss_select(mu, s2, cnt, 1.5, 100.0, 0.0, oracle.zq_table(0.99, 16))
    assert sel.tolist() == [1]


def test_gauss_mass_non_integer_beta_is_numerical():
    """App. D's closed forms need an integer beta; alpha = 1.7 (beta = 1.4286) must not be
    silently rounded.  Since N4 (DESIGN R28) the oracle evaluates the
    expectation numerically instead: the mass is the counts-weighted sum of the numerical
    truncated moments (pinned against mpmath in test_oracle_pins_n4.py), not the beta = 1
    (rounded) closed form, and tau_hat is its root."""
    mu = np.array([0.5, 1.0], np.float32)
    s2 = np.array([0.1, 0.2], np.float32)
    cnt = np.array([16, 16], np.int32)
    a = float(np.float32(1.7)) - 1.0
    beta = 1.0 / a
    want = sum(16 * oracle.trunc_moment_num(beta, a * float(m), a * math.sqrt(float(v))) for m, v in zip(mu, s2))
    got = oracle.gauss_mass(mu, s2, cnt, float(np.float32(1.7)), 0.0)
    assert abs(got - want) <= 1e-14 * want
    rounded = sum(16 * oracle.trunc_moment(1, a * float(m), a * math.sqrt(float(v))) for m, v in zip(mu, s2))
    assert abs(got - rounded) > 1e-3 * want                     # not the rounded beta
    t = oracle.gauss_tau(mu, s2, cnt, float(np.float32(1.7)))
    assert abs(oracle.gauss_mass(mu, s2, cnt, float(np.float32(1.7)), t) - 1.0) < 1e-12
    assert not math.isnan(oracle.gauss_mass(mu, s2, cnt, 1.5, 0.0))
    with pytest.raises(ValueError):
        oracle.gauss_tau(mu, s2, cnt, 1.0)                      # alpha <= 1


# ------------------------------------------------------------------ certified delta_bar
@pytest.mark.parametrize("alpha,tau,expect", [
    (2.0, 0.75, (1.0 - 0.75) * 16 + (3.0 - 0.75) * 5),                                  # 15.25
    (1.5, 0.25, (0.5 - 0.25) ** 2 * 16 + (1.5 - 0.25) ** 2 * 5),                        # 8.8125
    (1.25, 0.125, (0.25 - 0.125) ** 4 * 16 + (0.75 - 0.125) ** 4 * 5),                  # 0.766845703125
])
def test_delta_bar_hand_case(alpha, tau, expect):
    """delta_bar = sum_{p not selected} c_p [(alpha-1) box_p - tau~]_+^beta (R16, Prop. B.1 +
    tau~ <= tau).  box = [2, 1, 3, 0.5], counts [16, 16, 5, 16], page 0 selected; page 3 is
    below tau~.  Dyadic values: exact in fp64.  (Counting P instead of c_p for page 2, or not
    skipping page 0, changes the value.)"""
    box = np.array([2.0, 1.0, 3.0, 0.5], np.float32)
    cnt = np.array([16, 16, 5, 16], np.int32)
    got = oracle.delta_bar(box, cnt, [0], alpha, tau)
    assert got == expect


def test_delta_bar_zero_certifies_exactness():
    """delta_bar = 0 => delta = 0 => sparse output == full output (Prop. 2): drop only
    a page whose keys point against q, so its box bound is far below the sparse tau."""
    rng = np.random.default_rng(7)
    n, P = 640, 16
    M = n // P
    K = bf16_round(rng.standard_normal((M, 1, P, 128)))
    V = bf16_round(rng.standard_normal((M, 1, P, 128)))
    q = bf16_round(rng.standard_normal(128) * 2)
    pt = rng.permutation(M).astype(np.int32)[None]
    junk_lp = 17
    K[pt[0, junk_lp], 0, :, :] = bf16_round(-4.0 * np.sign(q))[None, :]
    hc = oracle.HostCache(K, V, pt, np.array([n], np.int32))
    hc.build_stats()
    for alpha in (1.5, 2.0, 1.25):
        res = oracle.decode_head(hc, q, 0, 0, alpha, k_pages=M - 1, eval_exact=True)
        assert junk_lp not in res["pages"].tolist()
        db = oracle.delta_bar(res["box"], hc.page_counts(0), res["pages"], alpha, res["tau"])
        assert db == 0.0
        assert res["metrics"]["delta"] == 0.0
        np.testing.assert_allclose(res["o"], res["full"]["o"], atol=1e-12, rtol=0)


# ------------------------------------------------------------------ o~ = sum p v
@pytest.mark.parametrize("alpha,transform", [(1.5, 0), (1.25, 0), (2.0, 0), (1.5, 1)])
def test_attend_output_is_p_times_v(alpha, transform):
    """o~ = sum_j p~_j v_j.  The oracle's o is compared with its own p (dense over the
    sequence) times V gathered independently in numpy through the page table, for kv head 1
    of 2 (a head- or page-indexing slip in the V read fails)."""
    rng = np.random.default_rng(11)
    n, P, Hkv = 777, 16, 2
    M = (n + P - 1) // P
    K = bf16_round(rng.standard_normal((M + 3, Hkv, P, 128)) * 1.5)
    V = bf16_round(rng.standard_normal((M + 3, Hkv, P, 128)))
    pt = rng.permutation(M + 3)[:M].astype(np.int32)[None]
    hc = oracle.HostCache(K, V, pt, np.array([n], np.int32))
    hc.build_stats()
    q = bf16_round(rng.standard_normal(128) * 2)
    pages = np.sort(rng.choice(M, size=20, replace=False)).astype(np.int32)
    pages[-1] = M - 1                                            # the partial last page
    res = hc.attend(q, 0, 1, pages, alpha, transform, want_p=True)
    j = np.arange(n)
    Vtok = V[pt[0, j // P], 1, j % P].astype(np.float64)        # [n][dv]
    np.testing.assert_allclose(res["o"], res["p"] @ Vtok, atol=1e-12, rtol=0)
    assert abs(res["p"].sum() - 1.0) < 1e-12
    inside = np.zeros(n, bool)
    for lp in pages:
        inside[lp * P:min((lp + 1) * P, n)] = True
    assert np.all(res["p"][~inside] == 0.0)


# ------------------------------------------------------------------ Halley step of the approximate tau
@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0, 4.0 / 3.0])
def test_approx_tau_one_halley_step_decimal(alpha):
    """R23 / P:485: tau_1 = tau_0 - 2 f f' / (2 f'^2 - f f''), f(t) = sum_{z>t} (z - t)^beta - 1,
    f' = -beta S_{beta-1}, f'' = beta (beta-1) S_{beta-2}, evaluated here in 50-digit decimal
    from the oracle's tau_0 (h = 0).  A Newton step (t - f / f') differs at this distance from
    the root, so it fails."""
    getcontext().prec = 50
    beta = round(1.0 / (alpha - 1.0))
    rng = np.random.default_rng(5)
    for trial in range(6):
        z = (alpha - 1.0) * rng.standard_normal(int(rng.integers(20, 300))) * 2.0
        _, t0, _ = oracle.entmax_approx(z, alpha, 0)
        _, t1, _ = oracle.entmax_approx(z, alpha, 1)
        T = Decimal(repr(t0))
        w = [Decimal(repr(float(v))) - T for v in z]
        w = [x for x in w if x > 0]
        S = lambda m: sum(x ** m for x in w) if m > 0 else (Decimal(len(w)) if m == 0 else Decimal(0))
        f = S(beta) - 1
        fp = -beta * S(beta - 1)
        fpp = beta * (beta - 1) * S(beta - 2)
        ref = T - 2 * f * fp / (2 * fp * fp - f * fpp)
        assert abs(t1 - float(ref)) <= 1e-13 * max(1.0, abs(float(ref))), (alpha, trial, t1, float(ref))
        newton = T - f / fp
        if abs(float(newton - ref)) > 1e-9:
            assert abs(t1 - float(newton)) > 1e-12


# ------------------------------------------------------------------ Gaussian page moments
def test_gaussian_moments_equal_token_score_moments_on_orthogonal_design():
    """mu = q^T kavg / sqrt(d), sigma^2 = (1/d) sum_i q_i^2 Var(k_i) is the variance of
    the token score s = q^T k / sqrt(d) when the key coordinates are uncorrelated.  A 2^4 full
    factorial page (16 tokens, dims 0..3 = +-c_i, the others constant) has exactly
    uncorrelated coordinates, so sigma^2 must equal the population variance of the 16 token
    scores (computed here from the scores themselves, in fp64) and mu their mean."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        c = np.array([0.5, 1.0, 1.5, 2.0]) * rng.uniform(0.5, 2.0)
        keys = np.zeros((16, 128), np.float32)
        keys[:, 4:] = bf16_round(rng.standard_normal(124))[None, :]      # constant dims
        for t in range(16):
            for i in range(4):
                keys[t, i] = c[i] if (t >> i) & 1 else -c[i]
        keys = bf16_round(keys)
        K = np.zeros((1, 1, 16, 128), np.float32)
        K[0, 0] = keys
        hc = oracle.HostCache(K, np.zeros_like(K), np.array([[0]], np.int32), np.array([16], np.int32))
        hc.build_stats()
        q = bf16_round(rng.standard_normal(128))
        _, mu, s2 = hc.score_pages(q, 0, 0, modes=2)
        s = keys.astype(np.float64) @ q.astype(np.float64) / math.sqrt(128)
        var_s = float(np.mean((s - s.mean()) ** 2))
        assert abs(float(s2[0]) - var_s) <= 2e-6 * max(1e-3, var_s), (trial, float(s2[0]), var_s)
        assert abs(float(mu[0]) - s.mean()) <= 1e-5 * max(1.0, abs(s.mean()))


# ------------------------------------------------------------------ tau_hat-initialised Halley (R25)
@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0, 4.0 / 3.0])
def test_approx_init_one_halley_step_decimal(alpha):
    """P:488 (Gaussian variant): tau_1 = one Halley step from the given tau_hat, the same update
    as P:485's, here recomputed in 50-digit decimal from an arbitrary start inside
    [z_max - 1, z_max) (DESIGN R25)."""
    getcontext().prec = 50
    beta = round(1.0 / (alpha - 1.0))
    rng = np.random.default_rng(15)
    for trial in range(6):
        z = (alpha - 1.0) * rng.standard_normal(int(rng.integers(20, 300))) * 2.0
        zmax = float(z.max())
        _, tex, _ = oracle.entmax(z, alpha)
        t0 = tex - rng.uniform(0.05, 0.9) * (tex - (zmax - 1.0))        # left of the root, in range
        _, t1, _ = oracle.entmax_approx_init(z, alpha, t0, 1)
        T = Decimal(repr(t0))
        w = [Decimal(repr(float(v))) - T for v in z]
        w = [x for x in w if x > 0]
        S = lambda m: sum(x ** m for x in w) if m > 0 else (Decimal(len(w)) if m == 0 else Decimal(0))
        f, fp, fpp = S(beta) - 1, -beta * S(beta - 1), beta * (beta - 1) * S(beta - 2)
        ref = T - 2 * f * fp / (2 * fp * fp - f * fpp)
        assert abs(t1 - float(ref)) <= 1e-13 * max(1.0, abs(float(ref))), (alpha, trial)


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_approx_init_fixed_point_range_and_convergence(alpha):
    """The exact tau is a fixed point of the refinement; a start outside [z_max - 1, z_max) is
    replaced by z_max - 1 (R25); iterates never fall below z_max - 1; many steps reach the exact
    tau (pinned to the closed forms / brute force in test_oracle_pins.py)."""
    rng = np.random.default_rng(16)
    for trial in range(8):
        z = (alpha - 1.0) * rng.standard_normal(int(rng.integers(10, 400))) * 3.0
        zmax = float(z.max())
        p_ex, tex, kex = oracle.entmax(z, alpha)
        _, t1, k1 = oracle.entmax_approx_init(z, alpha, tex, 1)
        assert abs(t1 - tex) <= 1e-12 * max(1.0, abs(tex)) and k1 == kex
        for bad in (zmax, zmax + 3.0, zmax - 1.5, float("inf")):
            _, tb, _ = oracle.entmax_approx_init(z, alpha, bad, 2)
            _, tr, _ = oracle.entmax_approx_init(z, alpha, zmax - 1.0, 2)
            assert tb == tr
        for h in (1, 2, 3):
            _, th, _ = oracle.entmax_approx_init(z, alpha, zmax - 0.999, h)
            assert th >= zmax - 1.0
        _, t12, k12 = oracle.entmax_approx_init(z, alpha, zmax - 0.5, 12)
        assert abs(t12 - tex) <= 1e-10 * max(1.0, abs(tex)) and k12 == kex
