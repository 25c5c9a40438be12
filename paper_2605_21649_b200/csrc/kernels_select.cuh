// kernels_select.cuh -- a2 (top-k page selection), a2' (Gaussian-aware selection)
// and the per-KV-group union of the selected pages (R17).
#pragma once
#include "common.cuh"

namespace ekv {

// ============================================================================ a2: top-k
// One CTA (NT threads) per (b, q-head) row (R3: key desc, then lower page
// index).  Keys are the ordered-int encodings of the fp32 box scores (-0 == +0).
//  1. Partition bound: thread t reads the keys {4(t + NT j) .. +3} (float4, coalesced,
//     4 loads in flight per thread) and keeps their max m_t.  L = the k-th largest
//     m_t, found MSB-first with __syncthreads_count.  At least k keys are >= L, so the
//     k-th largest key T* >= L and every selected key is a candidate {key >= L}.
//  2. Candidates are compacted into shared memory (warp ballot + one shared atomic per
//     warp; their order does not matter: the selection is defined by (key, index)).
//  3. T* by an MSB-first search over the candidates (__syncthreads_count per slot);
//     ties at T* are broken by the smallest page indices (MSB-first over the index).
//  4. The selection is marked in a shared bitmap and written ascending (block scan).
// Overflow (more than kTopkCap candidates): the same searches run over all keys read
// from global memory (L2) -- exact, slower.
constexpr int kTopkCap = 8192;
__device__ int ekv_dbg_nc;

__device__ __forceinline__ void topk_key4(const float *x, int i4, int M, bool vec, uint32_t (&kk)[4]) {
    if (vec && i4 + 3 < M) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(x + i4));
        kk[0] = f2key(v.x); kk[1] = f2key(v.y); kk[2] = f2key(v.z); kk[3] = f2key(v.w);
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) kk[e] = (i4 + e < M) ? f2key(__ldg(x + i4 + e)) : 0u;
    }
}
// #(candidates with key >= Tt) (or over all keys on overflow), block-wide
template <int NT>
__device__ __forceinline__ int topk_cnt_ge(uint32_t Tt, bool ovf, int nc, int slots, const uint32_t *ckey,
                                           const float *x, int M, int *sh) {
    if (!ovf) {
        int c = 0;
        for (int s2 = 0; s2 < slots; ++s2) {
            const int j = s2 * NT + threadIdx.x;
            c += __syncthreads_count(j < nc && ckey[j] >= Tt);
        }
        return c;
    }
    int c = 0;
    for (int i = threadIdx.x; i < M; i += NT) c += f2key(__ldg(x + i)) >= Tt;
    return block_sum_i<NT>(c, sh);
}
// #(key == T && idx < I), block-wide
template <int NT>
__device__ __forceinline__ int topk_cnt_eq_lt(uint32_t T, int I, bool ovf, int nc, int slots, const uint32_t *ckey,
                                              const int32_t *cidx, const float *x, int M, int *sh) {
    if (!ovf) {
        int c = 0;
        for (int s2 = 0; s2 < slots; ++s2) {
            const int j = s2 * NT + threadIdx.x;
            c += __syncthreads_count(j < nc && ckey[j] == T && cidx[j] < I);
        }
        return c;
    }
    int c = 0;
    for (int i = threadIdx.x; i < min(M, I); i += NT) c += f2key(__ldg(x + i)) == T;
    return block_sum_i<NT>(c, sh);
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_topk(const float *__restrict__ box, int Hq, int maxp,
                                             const int32_t *__restrict__ seq_lens, int k,
                                             int32_t *__restrict__ page_idx, int32_t *__restrict__ n_sel,
                                             int sel_stride) {
    extern __shared__ __align__(16) unsigned char tk_smem[];
    uint32_t *ckey = reinterpret_cast<uint32_t *>(tk_smem);                 // [kTopkCap]
    int32_t *cidx = reinterpret_cast<int32_t *>(tk_smem + 4 * kTopkCap);    // [kTopkCap]
    uint32_t *bits = reinterpret_cast<uint32_t *>(tk_smem + 8 * kTopkCap);  // [maxp/32]
    __shared__ int sh[NT / 32 + 1];
    __shared__ int s_cnt;
    const int row = blockIdx.x;
    const int b = row / Hq;
    const int M = n_pages_of(seq_lens[b]);
    const int keff = min(k, M);
    int32_t *out = page_idx + (size_t)row * sel_stride;
    if (keff >= M) {
        for (int p = threadIdx.x; p < M; p += NT) out[p] = p;
        if (threadIdx.x == 0) n_sel[row] = M;
        return;
    }
    stamp(1, 0);
    const float *x = box + (size_t)row * maxp;
    const int W = (M + 31) / 32;
    for (int w = threadIdx.x; w < W; w += NT) bits[w] = 0u;
    if (threadIdx.x == 0) s_cnt = 0;
    const bool vec = (maxp & 3) == 0;
    // 1. partition maxima: thread t owns the float4 groups {t + NT*j}; the max of each
    //    group is kept (fp32 max == key max: f2key is monotone) for the second pass.
    constexpr int GPT = 16;                  // groups per thread (M <= 16 * 4 * NT)
    float gmax[GPT];
    uint32_t mt = 0u;
#pragma unroll
    for (int j0 = 0; j0 < GPT; j0 += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i4 = 4 * (threadIdx.x + (j0 + u) * NT);
            if (vec && i4 + 3 < M) v[u] = __ldg(reinterpret_cast<const float4 *>(x + i4));
            else {
                v[u].x = (i4 < M) ? __ldg(x + i4) : -INFINITY;
                v[u].y = (i4 + 1 < M) ? __ldg(x + i4 + 1) : -INFINITY;
                v[u].z = (i4 + 2 < M) ? __ldg(x + i4 + 2) : -INFINITY;
                v[u].w = (i4 + 3 < M) ? __ldg(x + i4 + 3) : -INFINITY;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i4 = 4 * (threadIdx.x + (j0 + u) * NT);
            gmax[j0 + u] = (i4 < M) ? fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)) : NAN;
            if (i4 < M) mt = max(mt, f2key(gmax[j0 + u]));
        }
    }
    __syncthreads();
    stamp(1, 1);
    uint32_t Lb = 1u;
    if (keff <= NT) {
        uint32_t T = 0u;
        for (int bit = 31; bit >= 0; --bit) {
            const uint32_t Tt = T | (1u << bit);
            if (__syncthreads_count(mt >= Tt) >= keff) T = Tt;
        }
        Lb = T > 1u ? T : 1u;
    }
    stamp(1, 2);
    // 2. candidates: only groups whose max reaches L are re-read
#pragma unroll
    for (int j = 0; j < GPT; ++j) {
        const int i4 = 4 * (threadIdx.x + j * NT);
        const bool hit = (i4 < M) && f2key(gmax[j]) >= Lb;
        if (__ballot_sync(0xffffffffu, hit) == 0u) continue;
        uint32_t kk[4] = {0u, 0u, 0u, 0u};
        if (hit) topk_key4(x, i4, M, vec, kk);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const bool c = hit && kk[e] >= Lb;
            const unsigned m = __ballot_sync(0xffffffffu, c);
            if (!m) continue;
            int pos = 0;
            if ((threadIdx.x & 31) == 0) pos = atomicAdd(&s_cnt, __popc(m));
            pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
            if (c && pos < kTopkCap) { ckey[pos] = kk[e]; cidx[pos] = i4 + e; }
        }
    }
    __syncthreads();
    const int nc = s_cnt;
    const bool ovf = nc > kTopkCap;
    stamp(1, 3);
    if (threadIdx.x == 0 && blockIdx.x == 0) ekv_dbg_nc = nc;
    const int slots = (nc + NT - 1) / NT;
    // 3. T* = k-th largest candidate key (or key, on overflow)
    uint32_t T = 0u;        // largest T with #(key >= T) >= k; holds for T <= L by step 1
    for (int bit = 31; bit >= 0; --bit) {
        const uint32_t Tt = T | (1u << bit);
        if (Tt <= Lb || topk_cnt_ge<NT>(Tt, ovf, nc, slots, ckey, x, M, sh) >= keff) T = Tt;
    }
    const int n_gt = (T == 0xffffffffu) ? 0 : topk_cnt_ge<NT>(T + 1u, ovf, nc, slots, ckey, x, M, sh);
    const int need = keff - n_gt;
    stamp(1, 4);
    int Ithr = M;                                    // select equal keys with idx < Ithr
    if (topk_cnt_eq_lt<NT>(T, M, ovf, nc, slots, ckey, cidx, x, M, sh) > need) {
        int I = 0;                                   // largest I with #(eq, idx < I) <= need
        for (int bit = 17; bit >= 0; --bit) {
            const int It = I + (1 << bit);
            if (It <= M && topk_cnt_eq_lt<NT>(T, It, ovf, nc, slots, ckey, cidx, x, M, sh) <= need) I = It;
        }
        Ithr = I;
    }
    stamp(1, 5);
    // 4. mark + ascending output
    if (!ovf) {
        for (int j = threadIdx.x; j < nc; j += NT) {
            const uint32_t kk = ckey[j];
            const int i = cidx[j];
            if (kk > T || (kk == T && i < Ithr)) atomicOr(&bits[i >> 5], 1u << (i & 31));
        }
    } else {
        for (int i = threadIdx.x; i < M; i += NT) {
            const uint32_t kk = f2key(__ldg(x + i));
            if (kk > T || (kk == T && i < Ithr)) atomicOr(&bits[i >> 5], 1u << (i & 31));
        }
    }
    __syncthreads();
    const int wpt = (W + NT - 1) / NT;
    int cnt = 0;
    for (int w = 0; w < wpt; ++w) {
        const int wi = threadIdx.x * wpt + w;
        if (wi < W) cnt += __popc(bits[wi]);
    }
    int tot;
    int o = block_excl_scan<NT>(cnt, sh, &tot);
    for (int w = 0; w < wpt; ++w) {
        const int wi = threadIdx.x * wpt + w;
        if (wi >= W) break;
        uint32_t v = bits[wi];
        while (v) {
            const int bpos = __ffs(v) - 1;
            v &= v - 1;
            out[o++] = wi * 32 + bpos;
        }
    }
    if (threadIdx.x == 0) n_sel[row] = keff;
    stamp(1, 6);
}

// ============================================================================ union per KV group
// The union of the G selections of a KV group (R17): umask[b][kvh][page] bytes (4 per
// u32, bit g = selected by query head g of the group), zeroed by the host and filled
// with atomicOr from the page lists; the head that sets a page's first bit also appends
// the page to the group's compact list ulist[b][kvh][0..ucount) (order irrelevant: the
// K-score kernel's result does not depend on the order in which pages are processed).
__global__ void __launch_bounds__(256) k_mark(int Hq, int G, const int32_t *__restrict__ page_idx,
                                              const int32_t *__restrict__ n_sel, int sel_stride,
                                              uint32_t *__restrict__ umask, int W, int32_t *__restrict__ ulist,
                                              int32_t *__restrict__ ucount, int ucap) {
    const int row = blockIdx.x;
    const int b = row / Hq, h = row % Hq;
    const int kvh = h / G, g = h % G;
    const int Hkv = Hq / G;
    const int unit = b * Hkv + kvh;
    const int n = n_sel[row];
    const int32_t *pl = page_idx + (size_t)row * sel_stride;
    uint32_t *um = umask + (size_t)unit * W;
    for (int i = threadIdx.x; i < n; i += 256) {
        const int p = pl[i];
        const uint32_t old = atomicOr(um + (p >> 2), 1u << ((p & 3) * 8 + g));
        if (((old >> ((p & 3) * 8)) & 0xffu) == 0u) {
            const int pos = atomicAdd(ucount + unit, 1);
            if (pos < ucap) ulist[(size_t)unit * ucap + pos] = p;
        }
    }
}

// ============================================================================ a2': Gaussian selector
// One CTA per (b, q-head).  tau_hat solves  sum_p c_p E[(a S_p - tau)_+^beta] = 1
// (Eq. gaussian-threshold-main) with the App. D closed forms in fp64
// (beta = 4 by the truncated-moment recursion, R15).  Bracket [lo, hi] with
// mass(lo) >= 1 > mass(hi), then safeguarded Newton (dE/dtau = -beta * M_{beta-1}),
// falling back to bisection when a Newton step leaves the bracket.  Page rule
// (Eq. gaussian-selector-main, R14): keep p iff
// (double)a * fmaf(sqrtf(sigma2), zq[c], mu) > tau_hat - margin; empty -> argmax mu.
struct GaussMoments { double m, dm; };   // M_beta and M_{beta-1}

__device__ __forceinline__ GaussMoments trunc_moments(int beta, double muY, double sigY) {
    if (!(sigY > 0.0)) {
        const double x = muY > 0.0 ? muY : 0.0;
        double r = 1.0, rm = 1.0;
        for (int i = 0; i < beta; ++i) { rm = r; r *= x; }
        if (beta == 0) rm = 0.0;
        return {r, rm};
    }
    const double t = muY / sigY;
    const double Ph = normcdf(t);
    const double ph = exp(-0.5 * t * t) * 0.39894228040143267794;   // 1/sqrt(2 pi)
    double m0 = Ph, m1 = muY * Ph + sigY * ph;
    if (beta == 1) return {m1, m0};
    double prev = m0, cur = m1;
    for (int k = 2; k <= beta; ++k) {
        const double nx = muY * cur + (double)(k - 1) * sigY * sigY * prev;
        prev = cur; cur = nx;
    }
    return {cur, prev};
}

template <int NT>
__device__ void gauss_mass(const float *mu, const float *s2, int M, int Lseq, double a, int beta,
                           double tau, double &mass, double &dmass, double *shd) {
    double m = 0.0, dm = 0.0;
    for (int p = threadIdx.x; p < M; p += NT) {
        const double cnt = (double)min(kP, Lseq - p * kP);
        const double sg = sqrt((double)s2[p]);
        GaussMoments g = trunc_moments(beta, a * (double)mu[p] - tau, a * sg);
        m += cnt * g.m;
        dm += cnt * (double)beta * g.dm;      // -d mass / d tau
    }
    block_sum2_d<NT>(m, dm, shd);
    mass = m; dmass = dm;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_gauss_select(const float *__restrict__ mu, const float *__restrict__ sigma2,
                                                     int Hq, int maxp, const int32_t *__restrict__ seq_lens,
                                                     float alpha, double margin, double q_page,
                                                     int32_t *__restrict__ page_idx, int32_t *__restrict__ n_sel,
                                                     int sel_stride, double *__restrict__ tau_hat_out) {
    __shared__ double shd[2 * (NT / 32) + 2];
    __shared__ int shi[NT / 32 + 1];
    __shared__ float shf[NT / 32 + 1];
    __shared__ float zq[kP + 1];
    // zq[c] = Phi^{-1}(q_page^{1/c}), fp64 normcdfinv rounded to fp32 (R14)
    if (threadIdx.x >= 1 && threadIdx.x <= kP)
        zq[threadIdx.x] = (float)normcdfinv(pow(q_page, 1.0 / (double)threadIdx.x));
    const int row = blockIdx.x;
    const int b = row / Hq;
    const int Lseq = seq_lens[b];
    const int M = n_pages_of(Lseq);
    const float *m_ = mu + (size_t)row * maxp;
    const float *s_ = sigma2 + (size_t)row * maxp;
    const double a = (double)alpha - 1.0;
    const int beta = (int)llrint(1.0 / a);
    // bracket: top = a * max_p (mu + 8 sigma)
    float tmax = -INFINITY;
    for (int p = threadIdx.x; p < M; p += NT) tmax = fmaxf(tmax, m_[p] + 8.0f * sqrtf(s_[p]));
    tmax = block_max_f<NT>(tmax, shf);
    double hi = a * (double)tmax, w = 1.0, mass, dmass;
    for (int it = 0; it < 200; ++it) {
        gauss_mass<NT>(m_, s_, M, Lseq, a, beta, hi, mass, dmass, shd);
        if (mass < 1.0) break;
        hi += w; w *= 2.0;
    }
    double lo = hi - 1.0;
    w = 1.0;
    for (int it = 0; it < 200; ++it) {
        gauss_mass<NT>(m_, s_, M, Lseq, a, beta, lo, mass, dmass, shd);
        if (mass >= 1.0) break;
        lo -= w; w *= 2.0;
    }
    // safeguarded Newton from lo (mass convex decreasing -> monotone from the left)
    double tau = lo;
    for (int it = 0; it < 200; ++it) {
        gauss_mass<NT>(m_, s_, M, Lseq, a, beta, tau, mass, dmass, shd);
        if (mass >= 1.0) lo = tau; else hi = tau;
        double nt = (dmass > 0.0) ? tau + (mass - 1.0) / dmass : 0.5 * (lo + hi);
        if (!(nt > lo && nt < hi)) nt = 0.5 * (lo + hi);
        if (fabs(nt - tau) <= 1e-15 * fmax(1.0, fabs(tau)) || hi - lo <= 1e-15 * fmax(1.0, fabs(hi))) {
            tau = nt;
            break;
        }
        tau = nt;
    }
    // page rule + ordered compaction (NT pages per round)
    int32_t *out = page_idx + (size_t)row * sel_stride;
    int base = 0;
    for (int r0 = 0; r0 < M; r0 += NT) {
        const int p = r0 + threadIdx.x;
        int keep = 0;
        if (p < M) {
            const int cnt = min(kP, Lseq - p * kP);
            const float sg = __fmaf_rn(sqrtf(s_[p]), zq[cnt], m_[p]);
            keep = (a * (double)sg > tau - margin) ? 1 : 0;
        }
        int tot;
        const int pos = block_excl_scan<NT>(keep, shi, &tot);
        if (keep) out[base + pos] = p;
        base += tot;
    }
    if (base == 0 && M > 0) {
        // argmax mu, lower index on ties (R6)
        uint64_t best = 0;
        for (int p = threadIdx.x; p < M; p += NT) {
            const uint64_t k = ((uint64_t)f2key(m_[p]) << 32) | (uint32_t)(0xffffffffu - (uint32_t)p);
            best = best > k ? best : k;
        }
        // block max of u64 via two passes on shared memory
        __shared__ unsigned long long shb[NT / 32];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const uint64_t y = __shfl_xor_sync(0xffffffffu, best, o);
            best = best > y ? best : y;
        }
        if ((threadIdx.x & 31) == 0) shb[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t r = 0;
            for (int i = 0; i < NT / 32; ++i) r = r > shb[i] ? r : shb[i];
            out[0] = (int)(0xffffffffu - (uint32_t)(r & 0xffffffffu));
        }
        base = 1;
    }
    if (threadIdx.x == 0) {
        n_sel[row] = base;
        if (tau_hat_out) tau_hat_out[row] = tau;
    }
}

}  // namespace ekv
