"""Pins of the oracle's compressed-metadata forms (DESIGN R24), each
against something other than the oracle itself:

* e4m3 outward rounding against torch's float8_e4m3fn value set (an independent
  implementation of the OCP FN format): round-down = the largest representable value <= x,
  round-up = the smallest >= x; fixed points on every representable value; adjacent
  grid points bracket every x;
* bf16 rounding against torch's fp32 -> bfloat16 conversion (round to nearest even);
* Prop. B.1 with the stored e4m3 bounds: every token score of a page is
  <= its box bound (fp32, canonical order), and the e4m3 box is >= the exact box.
"""
import numpy as np
import torch

import oracle


def e4m3_values():
    codes = torch.arange(256, dtype=torch.uint8)
    v = codes.view(torch.float8_e4m3fn).float().numpy()
    v = v[np.isfinite(v)]
    return np.unique(v.astype(np.float64))


def test_e4m3_rounding_against_torch_value_set():
    vals = e4m3_values()
    assert vals.size == 253 and vals.max() == 448.0 and vals.min() == -448.0
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-448, 448, 4000), rng.normal(0, 2, 4000), rng.normal(0, 0.01, 2000),
                         vals, vals[1:-1] + 1e-7, vals[1:-1] - 1e-7, [0.0, -0.0]]).astype(np.float32)
    for x in xs:
        lo, hi = oracle.e4m3_round_down(x), oracle.e4m3_round_up(x)
        ref_lo = vals[vals <= float(x)].max()
        ref_hi = vals[vals >= float(x)].min()
        assert float(lo) == ref_lo and float(hi) == ref_hi, (x, lo, hi, ref_lo, ref_hi)


def test_e4m3_fixed_points_and_bracketing():
    vals = e4m3_values()
    for v in vals:
        assert float(oracle.e4m3_round_down(v)) == v and float(oracle.e4m3_round_up(v)) == v
    # between two adjacent grid points every x rounds down to the lower and up to the upper one
    for a, b in zip(vals[:-1], vals[1:]):
        x = np.float32(0.5 * (a + b))
        if a < float(x) < b:
            assert float(oracle.e4m3_round_down(x)) == a and float(oracle.e4m3_round_up(x)) == b


def test_bf16_round_against_torch():
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.normal(0, 1, 20000), rng.normal(0, 1e-3, 5000), rng.uniform(-300, 300, 5000)])
    xs = xs.astype(np.float32)
    # exact ties: 1 + (2j+1) 2^-8 are halfway between bf16 neighbours
    ties = (1.0 + (2 * np.arange(64) + 1) * 2.0 ** -8).astype(np.float32)
    xs = np.concatenate([xs, ties, -ties])
    ref = torch.from_numpy(xs).to(torch.bfloat16).float().numpy()
    got = np.array([oracle.bf16_round(x) for x in xs], np.float32)
    np.testing.assert_array_equal(got, ref)


def test_store_meta_composes_rounding_with_build_stats():
    rng = np.random.default_rng(2)
    K = rng.normal(0, 3, size=(6, 2, 16, 128)).astype(np.float32)
    V = np.zeros_like(K)
    pt = np.arange(6, dtype=np.int32)[None]
    exact = oracle.HostCache(K, V, pt, np.array([90], np.int32))
    exact.build_stats()
    st = oracle.HostCache(K, V, pt, np.array([90], np.int32))
    st.build_stats(bound="e4m3", stat="bf16")
    for i in range(0, exact.kmin.size, 97):
        assert st.kmin.flat[i] == oracle.e4m3_round_down(exact.kmin.flat[i])
        assert st.kmax.flat[i] == oracle.e4m3_round_up(exact.kmax.flat[i])
        assert st.kavg.flat[i] == oracle.bf16_round(exact.kavg.flat[i])
        assert st.kvar.flat[i] == oracle.bf16_round(exact.kvar.flat[i])
    np.testing.assert_array_equal(st.ksum, exact.ksum)       # accumulators stay fp32


def test_prop_b1_soundness_with_e4m3_bounds():
    """Every token score <= its page's e4m3 box bound, and the e4m3 box >= the exact box
    (outward rounding only loosens the bound; Prop. B.1)."""
    rng = np.random.default_rng(3)
    for trial in range(4):
        M, c_last = 40, 1 + trial * 5
        n = (M - 1) * 16 + c_last
        K = (rng.normal(0, 1, size=(M, 1, 16, 128)) * np.exp(rng.uniform(-1.4, 1.4, 128))).astype(np.float32)
        K = torch.from_numpy(K).to(torch.bfloat16).float().numpy()
        V = np.zeros_like(K)
        pt = rng.permutation(M).astype(np.int32)[None]
        hx = oracle.HostCache(K, V, pt, np.array([n], np.int32))
        hx.build_stats()
        h8 = oracle.HostCache(K, V, pt, np.array([n], np.int32))
        h8.build_stats(bound="e4m3")
        q = torch.from_numpy(rng.normal(0, 1, 128).astype(np.float32)).to(torch.bfloat16).float().numpy()
        bx, _, _ = hx.score_pages(q, 0, 0, modes=1)
        b8, _, _ = h8.score_pages(q, 0, 0, modes=1)
        assert np.all(b8 >= bx)
        for lp in range(M):
            ph = int(pt[0, lp])
            cnt = 16 if lp < M - 1 else c_last
            for t in range(cnt):
                s = oracle.token_score(q, K[ph, 0, t])
                assert s <= b8[lp], (trial, lp, t, s, b8[lp])
