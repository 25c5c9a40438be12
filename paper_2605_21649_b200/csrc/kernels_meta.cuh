// kernels_meta.cuh -- a0 (append + page statistics) and a1 (page scoring).
#pragma once
#include "common.cuh"

namespace ekv {

// ============================================================================ a0: append_kv
// One CTA per sequence; thread (h, i) owns dimension i of kv head h (loops when
// Hkv*D > blockDim).  Token t of the call goes to position L + t.  Statistics are
// updated in append order (R5): kmin/kmax by comparison, ksum += k, ksumsq =
// fma(k, k, ksumsq), kavg = ksum / c, kvar = max(0, ksumsq/c - kavg*kavg), all with
// explicit round-to-nearest intrinsics (no contraction).  seq_lens[b] is bumped after
// a CTA barrier.
template <typename T>
__global__ void __launch_bounds__(1024) k_append(CacheView c, const T *__restrict__ k_new,
                                                 const T *__restrict__ v_new, int n_tokens) {
    const int b = blockIdx.x;
    const int L = c.seq_lens[b];
    T *K = reinterpret_cast<T *>(c.Kw);
    T *V = reinterpret_cast<T *>(c.Vw);
    T *kmin = reinterpret_cast<T *>(c.kmin);
    T *kmax = reinterpret_cast<T *>(c.kmax);
    const int HD = c.Hkv * kD;
    for (int t = 0; t < n_tokens; ++t) {
        const int pos = L + t;
        const int page = c.page_table[(size_t)b * c.maxp + pos / kP];
        const int slot = pos % kP;
        for (int e = threadIdx.x; e < HD; e += blockDim.x) {
            const int h = e / kD, i = e % kD;
            const size_t src = ((size_t)(b * n_tokens + t) * c.Hkv + h) * kD + i;
            const T kv = k_new[src];
            const size_t dst = (((size_t)page * c.Hkv + h) * kP + slot) * kD + i;
            K[dst] = kv;
            V[dst] = v_new[src];
            const size_t m = ((size_t)page * c.Hkv + h) * kD + i;
            const float kf = Elem<T>::to_f(kv);
            float mn, mx, s, ss;
            if (slot == 0) {
                mn = kf; mx = kf; s = __fadd_rn(0.0f, kf); ss = __fmaf_rn(kf, kf, 0.0f);
            } else {
                mn = Elem<T>::to_f(kmin[m]); mx = Elem<T>::to_f(kmax[m]);
                if (kf < mn) mn = kf;
                if (kf > mx) mx = kf;
                s = __fadd_rn(c.ksum[m], kf);
                ss = __fmaf_rn(kf, kf, c.ksumsq[m]);
            }
            const float cf = (float)(slot + 1);
            const float avg = __fdiv_rn(s, cf);
            const float m2 = __fdiv_rn(ss, cf);
            float var = __fsub_rn(m2, __fmul_rn(avg, avg));
            if (!(var > 0.0f)) var = 0.0f;
            kmin[m] = Elem<T>::from_f(mn); kmax[m] = Elem<T>::from_f(mx);
            c.ksum[m] = s; c.ksumsq[m] = ss; c.kavg[m] = avg; c.kvar[m] = var;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) c.seq_lens[b] = L + n_tokens;
}

// ============================================================================ a0 bulk: rebuild
// One thread per (page, kv head, dim): sequential over the page's c <= P tokens,
// identical arithmetic to the incremental append (R5).
template <typename T>
__global__ void __launch_bounds__(256) k_rebuild(CacheView c) {
    const int b = blockIdx.y;
    const int L = c.seq_lens[b];
    const int M = n_pages_of(L);
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int per_page = c.Hkv * kD;
    const int p = (int)(e / per_page);
    if (p >= M) return;
    const int h = (int)(e % per_page) / kD, i = (int)(e % kD);
    const int page = c.page_table[(size_t)b * c.maxp + p];
    const int cnt = min(kP, L - p * kP);
    const T *K = reinterpret_cast<const T *>(c.K);
    const size_t base = (((size_t)page * c.Hkv + h) * kP) * kD + i;
    float mn = Elem<T>::to_f(K[base]), mx = mn, s = 0.0f, ss = 0.0f;
    for (int t = 0; t < cnt; ++t) {
        const float kf = Elem<T>::to_f(K[base + (size_t)t * kD]);
        if (kf < mn) mn = kf;
        if (kf > mx) mx = kf;
        s = __fadd_rn(s, kf);
        ss = __fmaf_rn(kf, kf, ss);
    }
    const float cf = (float)cnt;
    const float avg = __fdiv_rn(s, cf);
    const float m2 = __fdiv_rn(ss, cf);
    float var = __fsub_rn(m2, __fmul_rn(avg, avg));
    if (!(var > 0.0f)) var = 0.0f;
    const size_t m = ((size_t)page * c.Hkv + h) * kD + i;
    reinterpret_cast<T *>(c.kmin)[m] = Elem<T>::from_f(mn);
    reinterpret_cast<T *>(c.kmax)[m] = Elem<T>::from_f(mx);
    c.ksum[m] = s; c.ksumsq[m] = ss; c.kavg[m] = avg; c.kvar[m] = var;
}

// ============================================================================ a1: score_pages
// CTA = (chunk of PPC pages) x (sequence b), 256 threads = 16 half-warps.  Half-warp
// hw serves kv head hw / (16/Hkv) and pages p0 + sub, p0 + sub + 16/Hkv, ...; lane c
// of the half-warp owns dims [8c, 8c+8) and keeps q for the G query heads of its kv
// group in registers.  kmin/kmax (and kavg/kvar) rows are read straight from HBM as
// 16-byte loads (each half-warp reads one contiguous 256/512-byte row: coalesced);
// the per-lane fma chains and the 16-lane reduce-scatter tree realise dot16x8 (R1).
// Box: max(q_i kmin_i, q_i kmax_i) = q_i kext_i is evaluated as two fmas with
// qneg = (q_i >= 0 ? 0 : q_i) and qpos = (q_i >= 0 ? q_i : 0); one of the two adds an
// exact zero, so the chain equals the canonical fma(q_i, kext_i, acc).
template <typename T, int G, int MODES, int UNR>
__global__ void __launch_bounds__(256) k_score(CacheView c, const T *__restrict__ q, int Hq, int ppc,
                                                float *__restrict__ box, float *__restrict__ mu,
                                                float *__restrict__ sigma2) {
    const int b = blockIdx.y;
    const int L = c.seq_lens[b];
    const int M = n_pages_of(L);
    const int p0 = blockIdx.x * ppc;
    if (p0 >= M) return;
    const int lane = threadIdx.x & 31;
    const int l16 = threadIdx.x & 15;
    const int hw = threadIdx.x >> 4;
    const int hwpk = 16 / c.Hkv;
    const int kvh = hw / hwpk, sub = hw % hwpk;
    const int hq0 = kvh * G;

    float qp[G][8], qn[G][8], qa[G][8], q2[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float x[8];
        Elem<T>::load8(q + ((size_t)b * Hq + hq0 + g) * kD + 8 * l16, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const bool nn = x[i] >= 0.0f;
            qp[g][i] = nn ? x[i] : 0.0f;
            qn[g][i] = nn ? 0.0f : x[i];
            qa[g][i] = x[i];
            q2[g][i] = __fmul_rn(x[i], x[i]);
        }
    }
    const int pend = min(p0 + ppc, M);
    const T *kmin = reinterpret_cast<const T *>(c.kmin);
    const T *kmax = reinterpret_cast<const T *>(c.kmax);
    const int h_out = hq0 + rs_head<G>(lane);
    const bool writer = rs_writer<G>(lane);
    // warp-uniform trip count: both half-warps of a warp run the same iterations
    for (int base = p0; base < pend; base += UNR * hwpk) {
        float mn[UNR][8], mx[UNR][8], av[UNR][8], vr[UNR][8];
        int pp[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            pp[u] = base + sub + u * hwpk;
            const int p = min(pp[u], pend - 1);
            const int page = __ldg(c.page_table + (size_t)b * c.maxp + p);
            const size_t off = ((size_t)page * c.Hkv + kvh) * kD + 8 * l16;
            if (MODES & 1) {
                Elem<T>::load8_nc(kmin + off, mn[u]);
                Elem<T>::load8_nc(kmax + off, mx[u]);
            }
            if (MODES & 2) {
                Elem<float>::load8_nc(c.kavg + off, av[u]);
                Elem<float>::load8_nc(c.kvar + off, vr[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const bool valid = pp[u] < pend;
            if (MODES & 1) {
                float acc[G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float a = 0.0f;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        a = __fmaf_rn(qn[g][i], mn[u][i], a);
                        a = __fmaf_rn(qp[g][i], mx[u][i], a);
                    }
                    acc[g] = a;
                }
                const float r = __fmul_rn(rs_reduce16<G>(acc, lane), kCd);
                if (writer && valid) box[((size_t)b * Hq + h_out) * c.maxp + pp[u]] = r;
            }
            if (MODES & 2) {
                float am[G], as[G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float a = 0.0f, s = 0.0f;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        a = __fmaf_rn(qa[g][i], av[u][i], a);
                        s = __fmaf_rn(q2[g][i], vr[u][i], s);
                    }
                    am[g] = a; as[g] = s;
                }
                const float rm = __fmul_rn(rs_reduce16<G>(am, lane), kCd);
                const float rs = __fmul_rn(rs_reduce16<G>(as, lane), 1.0f / (float)kD);
                if (writer && valid) {
                    mu[((size_t)b * Hq + h_out) * c.maxp + pp[u]] = rm;
                    sigma2[((size_t)b * Hq + h_out) * c.maxp + pp[u]] = rs;
                }
            }
        }
    }
}

}  // namespace ekv
