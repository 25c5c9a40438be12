// kernels_select.cuh -- a2 (top-k page selection), a2' (Gaussian-aware selection)
// and the per-KV-group union of the selected pages (R17).
#pragma once
#include "common.cuh"

namespace ekv {

// ============================================================================ a2: top-k
// One CTA (NT threads) per (b, q-head) row (R3: key desc, then lower page
// index).  Keys are the ordered-int encodings of the fp32 box scores (-0 == +0).
//  1. Partition bound: thread t reads the float4 groups {t + NT j} (coalesced, 8 loads in
//     flight) and keeps each group's max; L = the k-th largest per-thread max (MSB-first
//     with __syncthreads_count).  At least k keys are >= L, so T* (the k-th largest key)
//     >= L and every selected key is a candidate {key >= L}.
//  2. Groups whose max reaches L are listed in shared memory and re-read in parallel; the
//     keys >= L are compacted into shared memory (order irrelevant: the selection is
//     defined by (key, index)).
//  3. T* and the tie cut (smallest indices first) by MSB-first searches run by warp 0
//     alone over the shared candidates (warp reductions, no block barriers).
//  4. The selection is marked in a shared bitmap, written ascending (block scan), and --
//     if umask != NULL -- merged into the KV-group union (mask bits + compact list).
// Overflow (more than kTopkCap candidates): exact block-wide searches over all keys.
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

// union mark of one selected page: bit g of the page's byte (fire-and-forget atomic)
__device__ __forceinline__ void union_mark(uint32_t *um, int p, int g) {
    atomicOr(um + (p >> 2), 1u << ((p & 3) * 8 + g));
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_topk(const float *__restrict__ box, int Hq, int maxp,
                                                const int32_t *__restrict__ seq_lens, int k,
                                                int32_t *__restrict__ page_idx, int32_t *__restrict__ n_sel,
                                                int sel_stride, int G, uint32_t *__restrict__ umask, int W) {
    constexpr int CPT = kTopkCap / NT;       // candidate slots per thread
    extern __shared__ __align__(16) unsigned char tk_smem[];
    uint32_t *ckey = reinterpret_cast<uint32_t *>(tk_smem);                 // [kTopkCap]
    int32_t *cidx = reinterpret_cast<int32_t *>(tk_smem + 4 * kTopkCap);    // [kTopkCap]
    __shared__ uint32_t bits[2048];
    __shared__ uint32_t hist[256];
    __shared__ int sh[NT / 32 + 2];
    const int row = blockIdx.x;
    const int b = row / Hq;
    const int M = n_pages_of(seq_lens[b]);
    const int keff = min(k, M);
    int32_t *out = page_idx + (size_t)row * sel_stride;
    const int unit = b * (Hq / G) + (row % Hq) / G, gh = (row % Hq) % G;
    uint32_t *um = umask ? umask + (size_t)unit * W : nullptr;
    stamp(1, 0);
    if (keff >= M) {
        for (int p = threadIdx.x; p < M; p += NT) {
            out[p] = p;
            if (um) union_mark(um, p, gh);
        }
        if (threadIdx.x == 0) n_sel[row] = M;
        return;
    }
    const float *x = box + (size_t)row * maxp;
    const int Wb = (M + 31) / 32;
    for (int w = threadIdx.x; w < Wb; w += NT) bits[w] = 0u;
    const bool vec = (maxp & 3) == 0;
    // 1. partition maxima: thread t owns the float4 groups {t + NT j}, j < GPT
    constexpr int GPT = 16;                  // groups per thread (M <= 64 NT)
    uint32_t gkey[GPT];
    uint32_t mt = 0u;
#pragma unroll
    for (int j0 = 0; j0 < GPT; j0 += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
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
        for (int u = 0; u < 8; ++u) {
            const int i4 = 4 * (threadIdx.x + (j0 + u) * NT);
            gkey[j0 + u] = (i4 < M) ? f2key(fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w))) : 0u;
            mt = max(mt, gkey[j0 + u]);
        }
    }
    stamp(1, 1);
    uint32_t Lb = 1u;
    int dummy;
    // the bound needs at least k non-empty partitions (block_kth_largest requires k <= #keys)
    if (keff <= NT && __syncthreads_count(mt != 0u) >= keff) {
        const uint32_t km[1] = {mt};
        Lb = block_kth_largest<NT, 1>(km, keff, hist, sh, &dummy);
        if (Lb == 0u) Lb = 1u;
    }
    stamp(1, 2);
    // 2. candidates {key >= L}: re-read the hit groups (8 in flight), block-scan compaction
    int nc = 0;
    bool ovf = false;
#pragma unroll
    for (int j0 = 0; j0 < GPT; j0 += 8) {
        uint32_t kk[8][4];
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i4 = 4 * (threadIdx.x + (j0 + u) * NT);
            if (gkey[j0 + u] >= Lb) topk_key4(x, i4, M, vec, kk[u]);
            else { kk[u][0] = kk[u][1] = kk[u][2] = kk[u][3] = 0u; }
#pragma unroll
            for (int e = 0; e < 4; ++e) cnt += kk[u][e] >= Lb;
        }
        int tot;
        int pos = nc + block_excl_scan<NT>(cnt, sh, &tot);
        if (nc + tot > kTopkCap) { ovf = true; break; }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (kk[u][e] >= Lb) { ckey[pos] = kk[u][e]; cidx[pos] = 4 * (threadIdx.x + (j0 + u) * NT) + e; ++pos; }
        nc += tot;
    }
    __syncthreads();
    stamp(1, 3);
    if (threadIdx.x == 0 && blockIdx.x == 0) ekv_dbg_nc = nc;
    uint32_t T;
    int n_gt, Ithr = M;
    if (!ovf) {
        // 3. T* = k-th largest candidate (radix select), then the tie cut by index
        uint32_t ck[CPT];
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int e = j * NT + threadIdx.x;
            ck[j] = e < nc ? ckey[e] : 0u;
        }
        T = block_kth_largest<NT, CPT>(ck, keff, hist, sh, &n_gt);
        const int need = keff - n_gt;
        int ceq = 0;
#pragma unroll
        for (int j = 0; j < CPT; ++j) ceq += ck[j] == T;
        if (block_sum_i<NT>(ceq, sh) > need) {
            int I = 0;                       // largest I with #(eq, idx < I) <= need
            for (int bit = 17; bit >= 0; --bit) {
                const int It = I + (1 << bit);
                if (It > M) continue;
                int c = 0;
#pragma unroll
                for (int j = 0; j < CPT; ++j) {
                    const int e = j * NT + threadIdx.x;
                    c += (ck[j] == T && e < nc && cidx[e] < It);
                }
                if (block_sum_i<NT>(c, sh) <= need) I = It;
            }
            Ithr = I;
        }
        for (int e = threadIdx.x; e < nc; e += NT) {
            const uint32_t kv = ckey[e];
            const int i = cidx[e];
            if (kv > T || (kv == T && i < Ithr)) atomicOr(&bits[i >> 5], 1u << (i & 31));
        }
    } else {
        // exact fallback over all keys (bitwise threshold search, block-wide counts)
        T = 0u;
        for (int bit = 31; bit >= 0; --bit) {
            const uint32_t Tt = T | (1u << bit);
            int c = 0;
            for (int i = threadIdx.x; i < M; i += NT) c += f2key(__ldg(x + i)) >= Tt;
            if (block_sum_i<NT>(c, sh) >= keff) T = Tt;
        }
        int c = 0;
        for (int i = threadIdx.x; i < M; i += NT) c += f2key(__ldg(x + i)) > T;
        const int need = keff - block_sum_i<NT>(c, sh);
        c = 0;
        for (int i = threadIdx.x; i < M; i += NT) c += f2key(__ldg(x + i)) == T;
        if (block_sum_i<NT>(c, sh) > need) {
            int I = 0;
            for (int bit = 17; bit >= 0; --bit) {
                const int It = I + (1 << bit);
                if (It > M) continue;
                int c2 = 0;
                for (int i = threadIdx.x; i < It; i += NT) c2 += f2key(__ldg(x + i)) == T;
                if (block_sum_i<NT>(c2, sh) <= need) I = It;
            }
            Ithr = I;
        }
        for (int i = threadIdx.x; i < M; i += NT) {
            const uint32_t kv = f2key(__ldg(x + i));
            if (kv > T || (kv == T && i < Ithr)) atomicOr(&bits[i >> 5], 1u << (i & 31));
        }
    }
    __syncthreads();
    stamp(1, 5);
    // 4. ascending output (+ union marks)
    const int wpt = (Wb + NT - 1) / NT;
    int cnt = 0;
    for (int w = 0; w < wpt; ++w) {
        const int wi = threadIdx.x * wpt + w;
        if (wi < Wb) cnt += __popc(bits[wi]);
    }
    int tot;
    int o = block_excl_scan<NT>(cnt, sh, &tot);
    for (int w = 0; w < wpt; ++w) {
        const int wi = threadIdx.x * wpt + w;
        if (wi >= Wb) break;
        uint32_t v = bits[wi];
        while (v) {
            const int bpos = __ffs(v) - 1;
            v &= v - 1;
            out[o++] = wi * 32 + bpos;
            if (um) union_mark(um, wi * 32 + bpos, gh);
        }
    }
    if (threadIdx.x == 0) n_sel[row] = keff;
    stamp(1, 6);
}

// ============================================================================ union per KV group
// The union of the G selections of a KV group (R17): umask[b][kvh][page] bytes (4 per
// u32, bit g = selected by query head g of the group), zeroed by the host and filled
// with atomicOr from the page lists.  The K-score kernel walks the G page lists of a
// group and keeps a page only from its lowest selecting head (one read per union page).
__global__ void __launch_bounds__(256) k_mark(int Hq, int G, const int32_t *__restrict__ page_idx,
                                              const int32_t *__restrict__ n_sel, int sel_stride,
                                              uint32_t *__restrict__ umask, int W) {
    const int row = blockIdx.x;
    const int b = row / Hq, h = row % Hq;
    const int unit = b * (Hq / G) + h / G, g = h % G;
    const int n = n_sel[row];
    const int32_t *pl = page_idx + (size_t)row * sel_stride;
    uint32_t *um = umask + (size_t)unit * W;
    for (int i = threadIdx.x; i < n; i += 256) union_mark(um, pl[i], g);
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
