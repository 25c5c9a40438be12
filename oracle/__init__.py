"""CPU oracle for the EntmaxKV decode step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``)
and ``__graft_entry__.smoke()`` may import this package.  The product package
``paper_2605_21649_b200`` never imports it, and it never imports the product.

This module is argument marshalling (numpy <-> ctypes) over
``oracle/entmaxkv_oracle.c``, a plain, slow, single-threaded C implementation
written from PAPER.md (see the citations in that file).  A few pure-Python
helpers below compose those C calls for a whole paged cache; they add no
arithmetic of the method.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "entmaxkv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

D = 128


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, IEEE semantics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-fPIC", "-shared",
               "-ffp-contract=off", "-fno-fast-math", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        i32p = ctypes.POINTER(ctypes.c_int32)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        c_int, c_double = ctypes.c_int, ctypes.c_double
        L.orc_dot_canon.argtypes = [f32p, f32p]
        L.orc_dot_canon.restype = ctypes.c_float
        L.orc_token_score.argtypes = [f32p, f32p]
        L.orc_token_score.restype = ctypes.c_float
        L.orc_page_stats.argtypes = [f32p, c_int, c_int] + [f32p] * 6
        L.orc_build_stats.argtypes = [f32p, c_int, c_int, c_int, i32p, i32p, c_int, c_int] + [f32p] * 6
        L.orc_score_pages.argtypes = [f32p, c_int, c_int, f32p, f32p, f32p, f32p,
                                      i32p, c_int, c_int, f32p, f32p, f32p]
        L.orc_topk.argtypes = [f32p, c_int, c_int, i32p]
        L.orc_topk.restype = c_int
        L.orc_entmax.argtypes = [f64p, c_int, c_double, f64p, f64p]
        L.orc_entmax.restype = c_int
        L.orc_softmax.argtypes = [f64p, c_int, f64p]
        L.orc_softmax.restype = c_double
        L.orc_attend.argtypes = [f32p, f32p, f32p, i32p, c_int, c_int, c_int, c_int,
                                 c_int, i32p, c_int, c_double, c_int, f64p, f64p,
                                 f64p, f32p, c_int, c_double]
        L.orc_entmax_approx_init.argtypes = [f64p, c_int, c_double, c_double, c_int, f64p, f64p]
        L.orc_entmax_approx_init.restype = c_int
        L.orc_entmax_approx.argtypes = [f64p, c_int, c_double, c_int, f64p, f64p]
        L.orc_entmax_approx.restype = c_int
        L.orc_attend.restype = c_int
        L.orc_metrics.argtypes = [f64p, u8p, c_int, f64p, f64p, i32p, i32p]
        L.orc_trunc_moment.argtypes = [c_int, c_double, c_double]
        L.orc_trunc_moment.restype = c_double
        L.orc_gauss_mass.argtypes = [f32p, f32p, i32p, c_int, c_double, c_double]
        L.orc_gauss_mass.restype = c_double
        L.orc_gauss_tau.argtypes = [f32p, f32p, i32p, c_int, c_double, f64p]
        L.orc_gauss_tau.restype = c_int
        L.orc_norm_ppf.argtypes = [c_double]
        L.orc_norm_ppf.restype = c_double
        L.orc_gauss_select.argtypes = [f32p, f32p, i32p, c_int, c_double, c_double,
                                       c_double, f64p, i32p]
        L.orc_gauss_select.restype = c_int
        L.orc_delta_bar.argtypes = [f32p, i32p, u8p, c_int, c_double, c_double]
        L.orc_delta_bar.restype = c_double
        L.orc_trunc_moment_num.argtypes = [c_double, c_double, c_double]
        L.orc_trunc_moment_num.restype = c_double
        L.orc_box_certified.argtypes = [f32p, c_int, c_double, c_double, i32p]
        L.orc_box_certified.restype = c_int
        L.orc_e4m3_round_down.argtypes = [ctypes.c_float]
        L.orc_e4m3_round_down.restype = ctypes.c_float
        L.orc_e4m3_round_up.argtypes = [ctypes.c_float]
        L.orc_e4m3_round_up.restype = ctypes.c_float
        L.orc_bf16_round.argtypes = [ctypes.c_float]
        L.orc_bf16_round.restype = ctypes.c_float
        L.orc_store_meta.argtypes = [f32p, f32p, f32p, f32p, ctypes.c_size_t, c_int, c_int]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# --------------------------------------------------------------------------- scalar pieces
def dot_canon(x, y) -> np.float32:
    x, y = _f32(x), _f32(y)
    assert x.shape == (D,) and y.shape == (D,)
    return np.float32(lib().orc_dot_canon(_p(x, ctypes.c_float), _p(y, ctypes.c_float)))


def token_score(q, k) -> np.float32:
    q, k = _f32(q), _f32(k)
    return np.float32(lib().orc_token_score(_p(q, ctypes.c_float), _p(k, ctypes.c_float)))


def page_stats(keys):
    """keys [c][d] of one page in append order -> dict of the six fp32 vectors."""
    keys = _f32(keys)
    c, d = keys.shape
    out = {n: np.zeros(d, np.float32) for n in ("kmin", "kmax", "ksum", "ksumsq", "kavg", "kvar")}
    lib().orc_page_stats(_p(keys, ctypes.c_float), c, d,
                         *[_p(out[n], ctypes.c_float) for n in ("kmin", "kmax", "ksum", "ksumsq", "kavg", "kvar")])
    return out


def entmax(z, alpha: float):
    """alpha-entmax of already-scaled z = (alpha-1)*s. Returns (p, tau, support_size)."""
    z = _f64(z)
    n = z.shape[0]
    if n == 0:
        raise ValueError("empty scores")
    p = np.zeros(n, np.float64)
    tau = np.zeros(1, np.float64)
    k = lib().orc_entmax(_p(z, ctypes.c_double), n, float(alpha), _p(p, ctypes.c_double), _p(tau, ctypes.c_double))
    return p, float(tau[0]), int(k)


def entmax_approx(z, alpha: float, halley: int):
    """The paper's approximate threshold (histogram init + Halley steps; DESIGN R23)
    on already-scaled z.  Returns (unnormalised p, tau, |{z > tau}|)."""
    z = _f64(z)
    n = z.shape[0]
    p = np.zeros(max(n, 1), np.float64)
    tau = np.zeros(1, np.float64)
    k = lib().orc_entmax_approx(_p(z, ctypes.c_double), n, float(alpha), int(halley), _p(p, ctypes.c_double),
                                _p(tau, ctypes.c_double))
    return p[:n], float(tau[0]), int(k)


def entmax_approx_init(z, alpha: float, tau0: float, halley: int):
    """The Gaussian variant's approximate threshold (tau_hat start + Halley steps; R25) on
    already-scaled z.  Returns (unnormalised p, tau, |{z > tau}|)."""
    z = _f64(z)
    n = z.shape[0]
    p = np.zeros(max(n, 1), np.float64)
    tau = np.zeros(1, np.float64)
    k = lib().orc_entmax_approx_init(_p(z, ctypes.c_double), n, float(alpha), float(tau0), int(halley),
                                     _p(p, ctypes.c_double), _p(tau, ctypes.c_double))
    return p[:n], float(tau[0]), int(k)


def entmax_scores(s, alpha: float):
    """alpha-entmax of raw scores s (z = (alpha-1)*s in fp64)."""
    return entmax((float(alpha) - 1.0) * _f64(s), alpha)


def softmax(s):
    s = _f64(s)
    p = np.zeros_like(s)
    lz = lib().orc_softmax(_p(s, ctypes.c_double), s.shape[0], _p(p, ctypes.c_double))
    return p, float(lz)


def topk(score, k: int):
    score = _f32(score)
    M = score.shape[0]
    out = np.zeros(max(min(k, M), 1), np.int32)
    n = lib().orc_topk(_p(score, ctypes.c_float), M, int(k), _p(out, ctypes.c_int32))
    return out[:n].copy()


def trunc_moment(beta: int, muY: float, sigY: float) -> float:
    return float(lib().orc_trunc_moment(int(beta), float(muY), float(sigY)))


def trunc_moment_num(beta: float, muY: float, sigY: float) -> float:
    """E[(Y)_+^beta], Y ~ N(muY, sigY^2), any real beta > 0, by quadrature (R28)."""
    return float(lib().orc_trunc_moment_num(float(beta), float(muY), float(sigY)))


def gauss_mass(mu, sigma2, counts, alpha, tau):
    mu, sigma2, counts = _f32(mu), _f32(sigma2), _i32(counts)
    return float(lib().orc_gauss_mass(_p(mu, ctypes.c_float), _p(sigma2, ctypes.c_float),
                                      _p(counts, ctypes.c_int32), mu.shape[0], float(alpha), float(tau)))


def gauss_tau(mu, sigma2, counts, alpha):
    mu, sigma2, counts = _f32(mu), _f32(sigma2), _i32(counts)
    t = np.zeros(1, np.float64)
    rc = lib().orc_gauss_tau(_p(mu, ctypes.c_float), _p(sigma2, ctypes.c_float), _p(counts, ctypes.c_int32),
                             mu.shape[0], float(alpha), _p(t, ctypes.c_double))
    if rc == -2:
        raise ValueError(f"Gaussian tau_hat needs alpha > 1 (alpha={alpha})")
    if rc != 0:
        raise RuntimeError("tau_hat bracket failure")
    return float(t[0])


def norm_ppf(u: float) -> float:
    return float(lib().orc_norm_ppf(float(u)))


def zq_table(q_page: float, P: int):
    """zq[c] = Phi^{-1}(q_page^{1/c}) for c = 0..P (zq[0] unused)."""
    z = np.zeros(P + 1, np.float64)
    for c in range(1, P + 1):
        z[c] = norm_ppf(q_page ** (1.0 / c))
    return z


def gauss_select(mu, sigma2, counts, alpha, tau_hat, margin, zq):
    mu, sigma2, counts, zq = _f32(mu), _f32(sigma2), _i32(counts), _f64(zq)
    M = mu.shape[0]
    out = np.zeros(max(M, 1), np.int32)
    n = lib().orc_gauss_select(_p(mu, ctypes.c_float), _p(sigma2, ctypes.c_float), _p(counts, ctypes.c_int32),
                               M, float(alpha), float(tau_hat), float(margin), _p(zq, ctypes.c_double),
                               _p(out, ctypes.c_int32))
    return out[:n].copy()


def box_certified(box, alpha, tau_hat):
    """Prop. B.2: pages with (alpha-1) box > tau_hat, ascending."""
    box = _f32(box)
    out = np.zeros(max(box.shape[0], 1), np.int32)
    n = lib().orc_box_certified(_p(box, ctypes.c_float), box.shape[0], float(alpha), float(tau_hat),
                                _p(out, ctypes.c_int32))
    return out[:n].copy()


def e4m3_round_down(x) -> np.float32:
    return np.float32(lib().orc_e4m3_round_down(float(x)))


def e4m3_round_up(x) -> np.float32:
    return np.float32(lib().orc_e4m3_round_up(float(x)))


def bf16_round(x) -> np.float32:
    return np.float32(lib().orc_bf16_round(float(x)))


def delta_bar(box, counts, selected_pages, alpha, tau_sparse):
    box, counts = _f32(box), _i32(counts)
    sel = np.zeros(box.shape[0], np.uint8)
    sel[np.asarray(selected_pages, dtype=np.int64)] = 1
    return float(lib().orc_delta_bar(_p(box, ctypes.c_float), _p(counts, ctypes.c_int32), _p(sel, ctypes.c_uint8),
                                     box.shape[0], float(alpha), float(tau_sparse)))


# --------------------------------------------------------------------------- paged-cache pieces
class HostCache:
    """fp32 host copy of a paged cache (values exactly those stored on the device).

    K, V: [n_phys][Hkv][P][d]; kmin/kmax/kavg/kvar: [n_phys][Hkv][d];
    page_table: [B][max_pages]; seq_lens: [B].
    """

    def __init__(self, K, V, page_table, seq_lens, kmin=None, kmax=None, kavg=None, kvar=None):
        self.K, self.V = _f32(K), _f32(V)
        self.page_table = _i32(page_table)
        self.seq_lens = _i32(seq_lens)
        self.n_phys, self.Hkv, self.P, self.d = self.K.shape
        self.dv = self.V.shape[3]
        self.kmin = None if kmin is None else _f32(kmin)
        self.kmax = None if kmax is None else _f32(kmax)
        self.kavg = None if kavg is None else _f32(kavg)
        self.kvar = None if kvar is None else _f32(kvar)

    def n_pages(self, b):
        return (int(self.seq_lens[b]) + self.P - 1) // self.P

    def page_counts(self, b):
        n = int(self.seq_lens[b])
        M = self.n_pages(b)
        c = np.full(M, self.P, np.int32)
        if M:
            c[-1] = n - (M - 1) * self.P
        return c

    def build_stats(self, bound="kv", stat="f32"):
        """Recompute every page's metadata from its tokens (orc_page_stats), then round it to the
        stored form (orc_store_meta): bound "e4m3" = outward-rounded fp8 kmin/kmax, stat "bf16" =
        nearest-even bf16 kavg/kvar (DESIGN R24)."""
        shp = (self.n_phys, self.Hkv, self.d)
        self.kmin, self.kmax = np.zeros(shp, np.float32), np.zeros(shp, np.float32)
        self.ksum, self.ksumsq = np.zeros(shp, np.float32), np.zeros(shp, np.float32)
        self.kavg, self.kvar = np.zeros(shp, np.float32), np.zeros(shp, np.float32)
        lib().orc_build_stats(_p(self.K, ctypes.c_float), self.Hkv, self.P, self.d, _p(self.page_table, ctypes.c_int32),
                              _p(self.seq_lens, ctypes.c_int32), self.page_table.shape[0], self.page_table.shape[1],
                              *[_p(getattr(self, n), ctypes.c_float)
                                for n in ("kmin", "kmax", "ksum", "ksumsq", "kavg", "kvar")])
        if bound != "kv" or stat != "f32":
            lib().orc_store_meta(_p(self.kmin, ctypes.c_float), _p(self.kmax, ctypes.c_float),
                                 _p(self.kavg, ctypes.c_float), _p(self.kvar, ctypes.c_float), self.kmin.size,
                                 1 if bound == "e4m3" else 0, 1 if stat == "bf16" else 0)

    def score_pages(self, q, b, kvh, modes=1):
        q = _f32(q)
        M = self.n_pages(b)
        box, mu, s2 = (np.zeros(max(M, 1), np.float32) for _ in range(3))
        row = _i32(self.page_table[b])
        dummy = self.kmin if self.kmin is not None else self.kavg
        L = lib()
        L.orc_score_pages(_p(q, ctypes.c_float), int(kvh), self.Hkv,
                          _p(self.kmin if self.kmin is not None else dummy, ctypes.c_float),
                          _p(self.kmax if self.kmax is not None else dummy, ctypes.c_float),
                          _p(self.kavg if self.kavg is not None else dummy, ctypes.c_float),
                          _p(self.kvar if self.kvar is not None else dummy, ctypes.c_float),
                          _p(row, ctypes.c_int32), M, int(modes),
                          _p(box, ctypes.c_float), _p(mu, ctypes.c_float), _p(s2, ctypes.c_float))
        return box[:M], mu[:M], s2[:M]

    def attend(self, q, b, kvh, pages, alpha, transform=0, want_p=False, want_s=False, approx_halley=0,
               tau_init=None):
        """Attention of one query head over the given logical pages of sequence b."""
        q = _f32(q)
        pages = _i32(pages)
        n = int(self.seq_lens[b])
        o = np.zeros(self.dv, np.float64)
        tau = np.zeros(1, np.float64)
        p_tok = np.zeros(n, np.float64) if want_p else None
        s_tok = np.full(n, np.nan, np.float32) if want_s else None
        row = _i32(self.page_table[b])
        k = lib().orc_attend(_p(q, ctypes.c_float), _p(self.K, ctypes.c_float), _p(self.V, ctypes.c_float),
                             _p(row, ctypes.c_int32), n, int(kvh), self.Hkv, self.P, self.dv,
                             _p(pages, ctypes.c_int32), pages.shape[0], float(alpha), int(transform),
                             _p(o, ctypes.c_double), _p(tau, ctypes.c_double),
                             None if p_tok is None else _p(p_tok, ctypes.c_double),
                             None if s_tok is None else _p(s_tok, ctypes.c_float), int(approx_halley),
                             float("nan") if tau_init is None else float(tau_init))
        return {"o": o, "tau": float(tau[0]), "supp": int(k), "p": p_tok, "s": s_tok}


def metrics(p_full, keep_mask):
    p_full = _f64(p_full)
    keep = np.ascontiguousarray(keep_mask, dtype=np.uint8)
    dl, rho = np.zeros(1), np.zeros(1)
    rec, sup = np.zeros(1, np.int32), np.zeros(1, np.int32)
    lib().orc_metrics(_p(p_full, ctypes.c_double), _p(keep, ctypes.c_uint8), p_full.shape[0],
                      _p(dl, ctypes.c_double), _p(rho, ctypes.c_double), _p(rec, ctypes.c_int32),
                      _p(sup, ctypes.c_int32))
    return {"delta": float(dl[0]), "rho": float(rho[0]), "recovered": int(rec[0]), "full_supp": int(sup[0])}


def decode_head(cache: HostCache, q, b, kvh, alpha, k_pages=None, policy="topk", q_page=0.99,
                margin=0.0, transform=0, eval_exact=False):
    """One query head's full decode step, composed from the steps above in the paper's order
    (P:275-303): score pages -> select (top-k P:369-381 or Gaussian P:386-477) -> attend."""
    M = cache.n_pages(b)
    counts = cache.page_counts(b)
    res = {}
    if policy == "topk":
        box, _, _ = cache.score_pages(q, b, kvh, modes=1)
        pages = topk(box, k_pages)
        res["box"] = box
    elif policy == "all":
        pages = np.arange(M, dtype=np.int32)
    elif policy == "certified":
        # N4 (Prop. B.2; DESIGN R27): a top-k pass gives the exact sparse threshold
        # tau~ <= tau (R13); every page with (alpha-1) box > tau~ is then selected
        box, _, _ = cache.score_pages(q, b, kvh, modes=1)
        first = cache.attend(q, b, kvh, topk(box, k_pages), alpha, transform)
        tau_lo = first["tau"]
        pages = box_certified(box, alpha, tau_lo)
        res.update(box=box, tau_lo=tau_lo)
    else:
        _, mu, s2 = cache.score_pages(q, b, kvh, modes=2)
        tau_hat = gauss_tau(mu, s2, counts, alpha)
        zq = zq_table(q_page, cache.P)
        pages = gauss_select(mu, s2, counts, alpha, tau_hat, margin, zq)
        res.update(mu=mu, sigma2=s2, tau_hat=tau_hat)
    att = cache.attend(q, b, kvh, pages, alpha, transform, want_p=eval_exact)
    res.update(pages=pages, **att)
    if eval_exact:
        full = cache.attend(q, b, kvh, np.arange(M, dtype=np.int32), alpha, 0, want_p=True)
        keep = np.zeros(int(cache.seq_lens[b]), np.uint8)
        for lp in pages:
            keep[lp * cache.P: min((lp + 1) * cache.P, int(cache.seq_lens[b]))] = 1
        res["metrics"] = metrics(full["p"], keep)
        res["full"] = full
    return res
