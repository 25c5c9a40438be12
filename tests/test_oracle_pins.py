"""Pins for the CPU oracle: each test checks the oracle against something other
than itself -- a value the paper/SPEC prints, a textbook closed form, an
independent algorithm (brute-force support enumeration, exact rational
arithmetic, numerical quadrature), or an invariant the paper proves.

Citations: P:L = PAPER.md line L, S:L = SPEC.md line L, R<n> = DESIGN.md reading.
"""
import itertools
import json
import math
import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest
from scipy import integrate, special

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(1234)


def bf16_round(x):
    """Round fp32 values to bf16 (RNE) and return them as fp32 (exact)."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


# ----------------------------------------------------------------------------- R1 dot order
def test_dot_canon_exact_on_small_integers():
    # integer-valued products/sums below 2^24 are exact in any order -> exact integer result
    for _ in range(50):
        x = RNG.integers(-20, 21, 128).astype(np.float32)
        y = RNG.integers(-20, 21, 128).astype(np.float32)
        assert float(oracle.dot_canon(x, y)) == float(np.dot(x.astype(np.int64), y.astype(np.int64)))


def test_dot_canon_tree_structure():
    # R1: chunks of 8 (fma chains), then pairwise c+(c+8), c+(c+4), c+(c+2), c0+c1.
    # x0 = 2^24 and 1.0 in chunks 1 and 9: the tree adds 1+1 first (chunk 1 + chunk 9 at
    # level 1) and returns 2^24+2, whereas left-to-right summation would lose both ones.
    x = np.zeros(128, np.float32)
    y = np.ones(128, np.float32)
    x[0], x[8], x[72] = 2.0 ** 24, 1.0, 1.0
    assert float(oracle.dot_canon(x, y)) == 2.0 ** 24 + 2.0
    # a transposed tree (c + (c+1) first) would give 2^24 here: chunks 0 and 1 meet first
    x2 = np.zeros(128, np.float32)
    x2[0], x2[8], x2[16] = 2.0 ** 24, 1.0, 1.0   # chunks 0,1,2: level1 none, level2 (0,4),(1,5),(2,6)
    # level 3: c0+c2 = 2^24+1 -> 2^24 (tie to even); c1 = 1; level 4: 2^24 + 1 -> 2^24
    assert float(oracle.dot_canon(x2, y)) == 2.0 ** 24


def test_dot_canon_error_bound():
    # |fl(dot) - dot| <= gamma_{12} * sum|x_i y_i| (8-term chains + 4 tree levels), u = 2^-24
    u = 2.0 ** -24
    gam = 12 * u / (1 - 12 * u)
    for _ in range(200):
        x = bf16_round(RNG.standard_normal(128) * 3)
        y = bf16_round(RNG.standard_normal(128) * 3)
        exact = math.fsum(float(a) * float(b) for a, b in zip(x, y))
        got = float(oracle.dot_canon(x, y))
        assert abs(got - exact) <= gam * float(np.sum(np.abs(x.astype(np.float64) * y))) + 1e-30


# ----------------------------------------------------------------------------- entmax
def test_golden_entmax_cases():
    cases = json.load(open(os.path.join(GOLD, "entmax_cases.json")))["cases"]
    for c in cases:
        p, tau, k = oracle.entmax_scores(c["s"], c["alpha"])
        assert abs(tau - c["tau"]) <= 1e-10, c
        np.testing.assert_allclose(p, c["p"], atol=1e-10, rtol=0)
        assert k == len(c["support"]) and sorted(np.nonzero(p)[0].tolist()) == c["support"], c


def sparsemax_textbook(z):
    """Martins & Astudillo (2016) sort-based sparsemax in exact rational arithmetic:
    k(z) = max{k : 1 + k z_(k) > sum_{j<=k} z_(j)},  tau = (sum_{j<=k(z)} z_(j) - 1)/k(z)."""
    zs = sorted(z, reverse=True)
    kz, csum = 0, Fraction(0)
    for k in range(1, len(zs) + 1):
        csum += zs[k - 1]
        if 1 + k * zs[k - 1] > csum:
            kz = k
    tau = (sum(zs[:kz]) - 1) / kz
    return tau, [max(zi - tau, 0) for zi in z]


def test_sparsemax_matches_textbook_exact():
    # alpha = 2 (P:149 special case): oracle (F-criterion) vs the textbook algorithm
    for n in range(1, 25):
        for _ in range(20):
            # dyadic rationals so that the fp64 oracle sees the exact inputs
            z = [Fraction(int(v), 64) for v in RNG.integers(-200, 200, n)]
            tau, p = sparsemax_textbook(z)
            po, to, k = oracle.entmax([float(v) for v in z], 2.0)
            assert abs(to - float(tau)) <= 1e-12
            assert [bool(x > 0) for x in p] == [bool(x > 0) for x in po]
            np.testing.assert_allclose(po, [float(x) for x in p], atol=1e-12)


def brute_force_entmax(z, beta, prec=60):
    """Enumerate every candidate support S (2^n subsets); solve sum_{S}(z_i - tau)^beta = 1
    by high-precision bisection on (min_S z - 1, min_S z); keep the S consistent with
    Eq. entmax-support: z_i > tau for i in S and z_j <= tau otherwise."""
    getcontext().prec = prec
    zd = [Decimal(repr(float(v))) for v in z]
    n = len(z)
    found = []
    for r in range(1, n + 1):
        for S in itertools.combinations(range(n), r):
            zmin = min(zd[i] for i in S)
            lo, hi = zmin - 1, zmin
            for _ in range(200):
                mid = (lo + hi) / 2
                F = sum((zd[i] - mid) ** beta for i in S)
                if F >= 1:
                    lo = mid
                else:
                    hi = mid
            tau = (lo + hi) / 2
            if all(zd[j] <= tau for j in range(n) if j not in S):
                F = sum((zd[i] - tau) ** beta for i in S)
                if abs(F - 1) < Decimal(10) ** -30:
                    found.append((set(S), tau))
    assert len(found) == 1, found
    return found[0]


@pytest.mark.parametrize("alpha,beta", [(2.0, 1), (1.5, 2), (4.0 / 3.0, 3), (1.25, 4)])
def test_entmax_brute_force_small(alpha, beta):
    # S:62, AC1 S:522: equivalence with support enumeration on tiny inputs
    for n in range(1, 8):
        for _ in range(4):
            z = RNG.uniform(-1.5, 1.5, n)
            S, tau = brute_force_entmax(z, beta)
            p, to, k = oracle.entmax(z, alpha)
            assert set(np.nonzero(p)[0].tolist()) == S
            assert abs(to - float(tau)) <= 1e-12 * max(1.0, abs(float(tau)))


def entmax15_sort_closed_form(z):
    """Peters et al. (2019) exact sort-based 1.5-entmax (beta = 2): for each prefix k of the
    descending sort, tau_k = mean_k - sqrt((1 - ss_k)/k); the support is the largest k with
    tau_k <= z_(k).  Evaluated in 50-digit decimal."""
    getcontext().prec = 50
    zs = sorted((Decimal(repr(float(v))) for v in z), reverse=True)
    best = None
    for k in range(1, len(zs) + 1):
        m = sum(zs[:k]) / k
        ss = sum((v - m) ** 2 for v in zs[:k])
        if ss > 1:
            break
        tau = m - ((1 - ss) / k).sqrt()
        if tau <= zs[k - 1]:
            best = (k, tau)
    return best


def test_entmax15_matches_sort_closed_form():
    for n in [2, 5, 16, 64, 200]:
        for _ in range(10):
            z = 0.5 * RNG.uniform(-2, 2, n) * (3 if n > 50 else 1)
            k, tau = entmax15_sort_closed_form(z)
            p, to, ko = oracle.entmax(z, 1.5)
            assert ko == k
            assert abs(to - float(tau)) <= 1e-12


def test_entmax_invariants():
    # normalization, exact zeros, permutation equivariance, shift behaviour
    for alpha in [1.25, 1.5, 2.0, 1.7]:
        for _ in range(20):
            s = RNG.standard_normal(int(RNG.integers(1, 300))) * 2
            p, tau, k = oracle.entmax_scores(s, alpha)
            assert abs(p.sum() - 1) < 1e-9
            z = (alpha - 1) * s
            assert np.all(p[z <= tau] == 0.0) and np.all(p[z > tau] > 0)
            perm = RNG.permutation(s.shape[0])
            p2, tau2, _ = oracle.entmax_scores(s[perm], alpha)
            np.testing.assert_allclose(p2, p[perm], atol=1e-12)
            c = 0.375
            p3, tau3, _ = oracle.entmax_scores(s + c, alpha)
            np.testing.assert_allclose(p3, p, atol=1e-10)
            assert abs(tau3 - (tau + (alpha - 1) * c)) < 1e-10


def test_entmax_softmax_limit_and_softmax_pins():
    p, _ = oracle.softmax([0.0, 0.0, 0.0])
    np.testing.assert_allclose(p, [1 / 3] * 3, atol=1e-15)
    p, _ = oracle.softmax([math.log(2.0), 0.0])
    np.testing.assert_allclose(p, [2 / 3, 1 / 3], atol=1e-15)
    s = RNG.standard_normal(32)
    pe, _, _ = oracle.entmax_scores(s, 1 + 1e-4)
    ps, _ = oracle.softmax(s)
    assert np.max(np.abs(pe - ps)) < 1e-2
    p, tau, k = oracle.entmax_scores([7.0], 1.5)                    # S:96 n = 1
    assert k == 1 and p[0] == 1.0


# ----------------------------------------------------------------------------- page stats
def test_page_stats_against_numpy():
    for c in [1, 2, 7, 16]:
        keys = bf16_round(RNG.standard_normal((c, 128)) * 2)
        st = oracle.page_stats(keys)
        np.testing.assert_array_equal(st["kmin"], keys.min(0))
        np.testing.assert_array_equal(st["kmax"], keys.max(0))
        k64 = keys.astype(np.float64)
        np.testing.assert_allclose(st["kavg"], k64.mean(0), rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(st["kvar"], k64.var(0), rtol=1e-4, atol=1e-5)
        assert np.all(st["kvar"] >= 0)
        assert np.all(st["kmin"] <= st["kavg"] + 1e-6) and np.all(st["kavg"] <= st["kmax"] + 1e-6)
        if c == 1:
            assert np.all(st["kvar"] == 0)
    same = np.tile(bf16_round(RNG.standard_normal(128)), (2, 1))
    assert np.all(oracle.page_stats(same)["kvar"] == 0)


# ----------------------------------------------------------------------------- page scores
def _single_page_cache(keys, Hkv=1):
    c = keys.shape[0]
    K = np.zeros((1, Hkv, 16, 128), np.float32)
    K[0, 0, :c] = keys
    hc = oracle.HostCache(K, np.zeros((1, Hkv, 16, 128), np.float32), np.array([[0]], np.int32),
                          np.array([c], np.int32))
    hc.build_stats()
    return hc


def test_box_bound_pins():
    # S:207 example embedded in d = 128: q = (1,-1,0,...), kmin = (-1,-1,..), kmax = (1,1,..)
    keys = np.zeros((2, 128), np.float32)
    keys[0, :2] = [-1, -1]
    keys[1, :2] = [1, 1]
    hc = _single_page_cache(keys)
    q = np.zeros(128, np.float32)
    q[:2] = [1, -1]
    box, _, _ = hc.score_pages(q, 0, 0, modes=1)
    assert float(box[0]) == float(np.float32(2.0) * np.float32(1 / math.sqrt(128)))
    # single-token page: box equals the token's score exactly
    k1 = bf16_round(RNG.standard_normal((1, 128)))
    hc = _single_page_cache(k1)
    q = bf16_round(RNG.standard_normal(128))
    box, mu, s2 = hc.score_pages(q, 0, 0, modes=3)
    assert box[0] == oracle.token_score(q, k1[0]) == mu[0] and s2[0] == 0.0


def test_box_bound_soundness_fp32():
    # Prop. B.1; holds in fp32 under the shared canonical order (R1, monotone rounding)
    for trial in range(300):
        c = int(RNG.integers(1, 17))
        keys = bf16_round(RNG.standard_normal((c, 128)) * RNG.uniform(0.1, 4))
        hc = _single_page_cache(keys)
        q = bf16_round(RNG.standard_normal(128) * RNG.uniform(0.1, 4))
        box, _, _ = hc.score_pages(q, 0, 0, modes=1)
        for t in range(c):
            assert oracle.token_score(q, keys[t]) <= box[0]


def test_gaussian_moments_pins():
    # single-token page -> sigma2 = 0; q = 0 -> (0, 0);
    # Monte Carlo: for a page of many iid keys, mu and sigma2 match the token-score moments
    keys = bf16_round(RNG.standard_normal((1, 128)))
    hc = _single_page_cache(keys)
    _, mu, s2 = hc.score_pages(np.zeros(128, np.float32), 0, 0, modes=2)
    assert mu[0] == 0 and s2[0] == 0
    # diagonal model: sigma^2 = (1/d) sum q_i^2 var_i equals Var(s) when coordinates are independent
    c = 16
    keys = bf16_round(RNG.standard_normal((c, 128)) * np.linspace(0.2, 3, 128))
    hc = _single_page_cache(keys)
    q = bf16_round(RNG.standard_normal(128))
    _, mu, s2 = hc.score_pages(q, 0, 0, modes=2)
    s = (keys.astype(np.float64) @ q.astype(np.float64)) / math.sqrt(128)
    assert abs(mu[0] - s.mean()) < 1e-5
    # sigma2 is the diagonal part of Var(s): compare with sum_i q_i^2 var_i / d exactly in fp64
    var_i = keys.astype(np.float64).var(0)
    assert abs(s2[0] - float(np.sum(q.astype(np.float64) ** 2 * var_i)) / 128) < 1e-4 * (1 + s2[0])


# ----------------------------------------------------------------------------- top-k
def test_topk_pins():
    assert oracle.topk([1, 5, 3], 1).tolist() == [1]
    assert oracle.topk([1, 5, 3], 7).tolist() == [0, 1, 2]
    assert oracle.topk([7, 7, 2], 1).tolist() == [0]                # S:265 (R3)
    for _ in range(50):
        M = int(RNG.integers(1, 400))
        s = np.round(RNG.standard_normal(M) * 4) / 4            # many ties
        k = int(RNG.integers(1, M + 3))
        got = oracle.topk(s, k)
        ref = np.sort(np.lexsort((np.arange(M), -s))[:min(k, M)])
        assert got.tolist() == ref.tolist()


# ----------------------------------------------------------------------------- propositions
def _rand_cache(n, seed, Hkv=1, scale=1.0):
    rng = np.random.default_rng(seed)
    P = 16
    M = (n + P - 1) // P
    K = bf16_round(rng.standard_normal((M, Hkv, P, 128)) * scale)
    V = bf16_round(rng.standard_normal((M, Hkv, P, 128)))
    pt = rng.permutation(M).astype(np.int32)[None]
    hc = oracle.HostCache(K, V, pt, np.array([n], np.int32))
    hc.build_stats()
    return hc, rng


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_prop2_exactness(alpha):
    # Prop. 2 (AC3 S:524): kept set containing the support -> delta = 0, o~ = o
    for seed in range(6):
        hc, rng = _rand_cache(700, seed, scale=2.0)
        q = bf16_round(rng.standard_normal(128) * 2)
        M = hc.n_pages(0)
        full = hc.attend(q, 0, 0, np.arange(M), alpha, want_p=True)
        supp_pages = sorted({j // 16 for j in np.nonzero(full["p"])[0]})
        extra = rng.choice(M, size=min(3, M), replace=False).tolist()
        keep_pages = np.array(sorted(set(supp_pages) | set(extra)), np.int32)
        sp = hc.attend(q, 0, 0, keep_pages, alpha, want_p=True)
        keep = np.zeros(700, np.uint8)
        for lp in keep_pages:
            keep[lp * 16:(lp + 1) * 16] = 1
        m = oracle.metrics(full["p"], keep)
        assert m["delta"] == 0.0 and m["rho"] == 1.0
        np.testing.assert_allclose(sp["o"], full["o"], atol=1e-10, rtol=0)


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_prop1_bound_deployed_path(alpha):
    # Prop. 1 and R13: ||o - o~|| <= 2 B delta also for entmax recomputed on C_tok
    for seed in range(10):
        hc, rng = _rand_cache(480, 100 + seed, scale=2.5)
        q = bf16_round(rng.standard_normal(128) * 2)
        M = hc.n_pages(0)
        full = hc.attend(q, 0, 0, np.arange(M), alpha, want_p=True)
        keep_pages = np.sort(rng.choice(M, size=int(rng.integers(1, M)), replace=False)).astype(np.int32)
        keep = np.zeros(480, np.uint8)
        for lp in keep_pages:
            keep[lp * 16:(lp + 1) * 16] = 1
        sp = hc.attend(q, 0, 0, keep_pages, alpha)
        m = oracle.metrics(full["p"], keep)
        Bv = float(np.max(np.linalg.norm(hc.V.reshape(-1, 128).astype(np.float64), axis=1)))
        err = float(np.linalg.norm(sp["o"] - full["o"]))
        assert err <= 2 * Bv * m["delta"] + 1e-9
        assert sp["tau"] <= full["tau"] + 1e-12                   # tau~ <= tau (R13)


def test_prop1_tightness():
    # p = (1-delta, delta), v = +-B u, keep token 0 -> ||o - o~|| = 2 B delta
    B, delta = 3.0, 0.125
    p = np.array([1 - delta, delta])
    u = np.zeros(4); u[0] = 1
    V = np.stack([B * u, -B * u])
    o = p @ V
    pt = np.array([1.0, 0.0])
    assert abs(np.linalg.norm(o - pt @ V) - 2 * B * delta) < 1e-12


@pytest.mark.parametrize("alpha", [1.5, 2.0, 1.25])
def test_delta_bar_certificate(alpha):
    # R16: delta <= delta_bar (Prop. B.1 + tau~ <= tau)
    for seed in range(5):
        hc, rng = _rand_cache(800, 300 + seed, scale=2.0)
        q = bf16_round(rng.standard_normal(128) * 2)
        res = oracle.decode_head(hc, q, 0, 0, alpha, k_pages=8, eval_exact=True)
        counts = hc.page_counts(0)
        db = oracle.delta_bar(res["box"], counts, res["pages"], alpha, res["tau"])
        assert res["metrics"]["delta"] <= db + 1e-12


# ----------------------------------------------------------------------------- Gaussian selector
def quad_moment(beta, muY, sigY):
    f = lambda y: y ** beta * math.exp(-0.5 * ((y - muY) / sigY) ** 2) / (sigY * math.sqrt(2 * math.pi))
    v, _ = integrate.quad(f, 0, max(muY, 0) + 40 * sigY, epsabs=1e-14, epsrel=1e-12, limit=200)
    return v


@pytest.mark.parametrize("beta", [1, 2, 3, 4])
def test_trunc_moments_vs_quadrature(beta):
    # App. D closed forms vs independent numerical integration
    for _ in range(40):
        muY = RNG.uniform(-3, 3)
        sigY = RNG.uniform(0.05, 2)
        got = oracle.trunc_moment(beta, muY, sigY)
        ref = quad_moment(beta, muY, sigY)
        assert abs(got - ref) <= 1e-9 * max(1.0, abs(ref)), (beta, muY, sigY, got, ref)


def test_trunc_moment_pins():
    assert abs(oracle.trunc_moment(1, 0.0, 1.0) - 1 / math.sqrt(2 * math.pi)) < 1e-15
    assert oracle.trunc_moment(1, 0.25, 0.0) == 0.25
    assert oracle.trunc_moment(2, -0.5, 0.0) == 0.0


def test_norm_ppf_and_zq_pins():
    for u in [1e-10, 0.001, 0.3, 0.5, 0.9, 0.99, 0.999999]:
        assert abs(oracle.norm_ppf(u) - special.ndtri(u)) < 1e-12
    gold = json.load(open(os.path.join(GOLD, "zq_099.json")))
    zq = oracle.zq_table(0.99, 16)
    for c, v in gold["zq"].items():
        assert abs(zq[int(c)] - v) < 1e-11
    for c in range(1, 17):
        assert abs(zq[c] - special.ndtri(0.99 ** (1.0 / c))) < 1e-11
    assert oracle.norm_ppf(0.5) == pytest.approx(0.0, abs=1e-15)   # S:293 (c=1, q=0.5 -> mu)


def test_gauss_tau_point_mass_reductions():
    # one page sigma=0, c=1, alpha=2, mu=3 -> tau_hat = 2; pages mu={3,0} -> 2
    t = oracle.gauss_tau([3.0], [0.0], [1], 2.0)
    assert abs(t - 2.0) < 1e-12
    t = oracle.gauss_tau([3.0, 0.0], [0.0, 0.0], [1, 1], 2.0)
    assert abs(t - 2.0) < 1e-12
    # with every sigma = 0 the equation is exact entmax over the page scores with
    # multiplicities: compare with brute-force support enumeration
    for beta, alpha in [(1, 2.0), (2, 1.5), (4, 1.25)]:
        mu = RNG.uniform(-2, 2, 5).astype(np.float32)
        cnt = RNG.integers(1, 4, 5)
        z = np.repeat((alpha - 1) * mu.astype(np.float64), cnt)
        S, tau = brute_force_entmax(z, beta)
        t = oracle.gauss_tau(mu, np.zeros(5, np.float32), cnt, alpha)
        assert abs(t - float(tau)) < 1e-10


@pytest.mark.parametrize("alpha", [2.0, 1.5, 1.25])
def test_gauss_tau_solves_mass_equation_by_quadrature(alpha):
    # Eq. gaussian-threshold-main: at tau_hat the mass, recomputed by quadrature, is 1
    beta = round(1 / (alpha - 1))
    a = alpha - 1
    M = 12
    mu = RNG.normal(0, 1, M).astype(np.float32)
    s2 = RNG.uniform(0.05, 1.5, M).astype(np.float32)
    cnt = np.full(M, 16)
    t = oracle.gauss_tau(mu, s2, cnt, alpha)
    mass = sum(16 * quad_moment(beta, a * float(m) - t, a * math.sqrt(float(v))) for m, v in zip(mu, s2))
    assert abs(mass - 1.0) < 1e-8


def test_gauss_select_properties():
    M = 40
    mu = RNG.normal(0, 1, M).astype(np.float32)
    s2 = RNG.uniform(0.05, 1.0, M).astype(np.float32)
    cnt = np.full(M, 16)
    zq = oracle.zq_table(0.99, 16)
    t = oracle.gauss_tau(mu, s2, cnt, 1.5)
    prev = set()
    for margin in [0.0, 0.05, 0.1, 0.5, 1e9]:                      # S:322 monotone in Delta
        sel = set(oracle.gauss_select(mu, s2, cnt, 1.5, t, margin, zq).tolist())
        assert prev <= sel
        prev = sel
    assert prev == set(range(M))                                     # S:304 Delta -> inf
    # empty -> argmax mu fallback (R6)
    sel = oracle.gauss_select(mu, s2, cnt, 1.5, 1e9, 0.0, zq)
    assert sel.tolist() == [int(np.argmax(mu))]
    # q_page = 0.5, c = 1 -> sbar = mu exactly
    zq5 = oracle.zq_table(0.5, 16)
    assert abs(zq5[1]) < 1e-15


# --------------------------------------------------------------------------- approximate tau (N1)
@pytest.mark.parametrize("alpha", [1.25, 1.5, 1.75, 2.0])
def test_approx_tau_converges_to_exact(alpha):
    """The paper's kernel recipe (histogram init + Halley; DESIGN R23): with enough
    Halley steps it reaches the exact threshold, which is itself pinned to the closed forms
    and to brute force above."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        z = (alpha - 1.0) * rng.standard_normal(int(rng.integers(2, 400))) * rng.uniform(0.3, 3.0)
        _, t_ex, k_ex = oracle.entmax(z, alpha)
        p, t, k = oracle.entmax_approx(z, alpha, 8)
        assert abs(t - t_ex) <= 1e-12 * max(1.0, abs(t_ex))
        assert k == k_ex
        assert abs(p.sum() - 1.0) <= 1e-10


@pytest.mark.parametrize("alpha", [1.25, 1.5, 2.0])
def test_approx_tau_initialisation_is_a_lower_bound(alpha):
    """h = 0: tau_0 is a bin edge whose certified lower bound of F reaches 1, so F(tau_0) >= 1,
    tau_0 <= tau and {z > tau_0} contains the exact support (nothing is dropped before the
    Halley steps); tau_0 >= z_max - 1."""
    beta = 1.0 / (alpha - 1.0)
    rng = np.random.default_rng(12)
    for trial in range(30):
        z = (alpha - 1.0) * rng.standard_normal(int(rng.integers(1, 500)))
        _, t_ex, k_ex = oracle.entmax(z, alpha)
        _, t0, k0 = oracle.entmax_approx(z, alpha, 0)
        F0 = np.sum(np.maximum(z - t0, 0.0) ** beta)
        assert F0 >= 1.0 - 1e-12
        assert z.max() - 1.0 - 1e-12 <= t0 <= t_ex + 1e-12
        assert k0 >= k_ex
