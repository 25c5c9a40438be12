// kernels_select.cuh -- a2 (top-k page selection), a2' (Gaussian-aware selection)
// and the per-KV-group union of the selected pages (R17).
#pragma once
#include "common.cuh"
#include <cooperative_groups.h>

namespace ekv {

// ============================================================================ a2: top-k
// A thread-block cluster of CL CTAs (CL = 1, 2, 4 or 8) per (b, q-head) row (
// R3: key desc, then lower page index).  Keys are the ordered-int encodings of the fp32
// box scores (-0 == +0; pages past the sequence end get key 0, below every real key).
// CTA r of the cluster owns pages [8192 r, 8192 (r + 1)); thread t (of 512) holds the 16
// keys of pages 8192 r + 4 (t + 512 j) + e (j < 4, e < 4: coalesced float4 loads, issued
// together with the sequence-length load) in registers.  Many threads per CTA: every
// step below is a chain of dependent warp-synchronous instructions, hidden only by TLP.
//  1. MSB-first radix select of T* = the k-th largest key with 8-bit digits: each CTA
//     histograms the digit of its keys that match the prefix so far (per-warp private
//     shared histograms, one atomic per warp when the active lanes agree -- the usual case
//     for the leading digits -- then summed), the cluster barrier publishes the CTA
//     histograms, every CTA sums the CL histograms through distributed shared memory and
//     locates the digit holding the k-th key (warp suffix scan).  The CTA histogram buffers
//     alternate: one cluster barrier per digit.  A digit whose whole bin is taken ends the search early (no tie cut needed).
//  2. Ties at T* (only if the bin of T* is split): CTA r takes the first
//     clamp(need - #eq in CTAs < r, 0, #eq in r) equal keys in page order.
//  3. Selection bitmap (bit = page), one word per thread (t < 256), block scan + cluster
//     offsets: ascending page ids, and -- if umask != NULL -- the KV-group union marks.
//     (512 threads, 2 CTAs per SM: the 256 CTAs of a 32-row, 65536-page launch are one wave.)
constexpr int kTkKPT = 16;                  // keys per thread; NT = 512 (8192 pages per CTA,
                                            // <= 8 CTAs -> 65536 pages) or 256 for short rows

// union mark of one selected page: bit g of the page's byte (fire-and-forget atomic)
__device__ __forceinline__ void union_mark(uint32_t *um, int p, int g) {
    atomicOr(um + (p >> 2), 1u << ((p & 3) * 8 + g));
}

// bitmap word of the CTA-local pages 2048 j + 4 t + e (e < 4) of a 4-bit nibble per thread:
// 8 consecutive lanes share a word (index 64 j + t / 8); lane t % 8 == 0 returns it
__device__ __forceinline__ uint32_t nibble_word(uint32_t nib, int lane) {
    uint32_t w = nib << (4 * (lane & 7));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    return w;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_topk(const float *__restrict__ box, int Hq, int maxp,
                                                const int32_t *__restrict__ seq_lens, int k,
                                                int32_t *__restrict__ page_idx, int32_t *__restrict__ n_sel,
                                                int sel_stride, int G, uint32_t *__restrict__ umask, int W) {
    EKV_TRACE(2);
    pdl_wait();
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int CL = (int)cl.num_blocks(), r = (int)cl.block_rank();
    const int row = blockIdx.x / CL;
    const int t = threadIdx.x, lane = t & 31;
    constexpr int NWp = NT / 32;
    __shared__ uint32_t whist[NWp][256];     // per-warp private histograms (no cross-warp contention)
    __shared__ uint32_t hist[2][256];        // the CTA's histogram of the current digit (published)
    __shared__ uint32_t bits[256];
    __shared__ int xch[2];                   // published to the cluster: [0] #eq, [1] #selected
    __shared__ int sh[(NT / 32 + 2)];
    const int b = row / Hq;
    const int base = r * (NT * kTkKPT);
    const float *x = box + (size_t)row * maxp;
    const bool vec = (maxp & 3) == 0;
    // keys and the sequence length in one round trip (masked below)
    const int Lb = __ldg(seq_lens + b);
    float4 kv[kTkKPT / 4];
#pragma unroll
    for (int j = 0; j < kTkKPT / 4; ++j) {
        const int i4 = base + 4 * (t + NT * j);
        if (vec && i4 + 3 < maxp) kv[j] = __ldg(reinterpret_cast<const float4 *>(x + i4));
        else {
            kv[j].x = (i4 < maxp) ? __ldg(x + i4) : 0.f;
            kv[j].y = (i4 + 1 < maxp) ? __ldg(x + i4 + 1) : 0.f;
            kv[j].z = (i4 + 2 < maxp) ? __ldg(x + i4 + 2) : 0.f;
            kv[j].w = (i4 + 3 < maxp) ? __ldg(x + i4 + 3) : 0.f;
        }
    }
    const int M = n_pages_of(Lb);
    const int keff = min(k, M);
    int32_t *out = page_idx + (size_t)row * sel_stride;
    const int unit = b * (Hq / G) + (row % Hq) / G, gh = (row % Hq) % G;
    uint32_t *um = umask ? umask + (size_t)unit * W : nullptr;
    stamp(1, 0);
    ph_stamp<2>(0);
    if (keff >= M) {                         // every page (uniform over the cluster)
        for (int p = base + t; p < min(M, base + (NT * kTkKPT)); p += NT) {
            out[p] = p;
            if (um) union_mark(um, p, gh);
        }
        if (r == 0 && t == 0) n_sel[row] = M;
        return;
    }
    uint32_t key[kTkKPT];
#pragma unroll
    for (int j = 0; j < kTkKPT / 4; ++j) {
        const int i4 = base + 4 * (t + NT * j);
        key[4 * j] = (i4 < M) ? f2key(kv[j].x) : 0u;
        key[4 * j + 1] = (i4 + 1 < M) ? f2key(kv[j].y) : 0u;
        key[4 * j + 2] = (i4 + 2 < M) ? f2key(kv[j].z) : 0u;
        key[4 * j + 3] = (i4 + 3 < M) ? f2key(kv[j].w) : 0u;
    }
    for (int i = t; i < NWp * 256; i += NT) (&whist[0][0])[i] = 0u;
    __syncthreads();
    stamp(1, 1);
    ph_stamp<2>(1);
    // 1. radix select over the cluster
    uint32_t prefix = 0u, pmask = 0u;
    int kk = keff;                           // keys still to take among those matching prefix
    bool whole = false;                      // the last digit's bin is taken entirely
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        uint32_t *hb = hist[pass & 1];
        uint32_t *wh = whist[t >> 5];
#pragma unroll
        for (int j = 0; j < kTkKPT; ++j) {
            const uint32_t v = key[j];
            const bool act = v != 0u && (v & pmask) == prefix;
            const unsigned bal = __ballot_sync(0xffffffffu, act);
            if (bal == 0u) continue;                                   // warp-uniform skip
            // the common case (every active lane in one bin) costs one atomic; otherwise the
            // lanes add one each (shared atomics serialise only equal addresses)
            const uint32_t d = (v >> shift) & 255u;
            const int leader = __ffs(bal) - 1;
            const uint32_t dl = __shfl_sync(0xffffffffu, d, leader);
            const unsigned same = __ballot_sync(0xffffffffu, act && d == dl);
            if (same == bal) {
                if (lane == leader) atomicAdd(&wh[dl], (uint32_t)__popc(bal));
            } else if (act) {
                atomicAdd(&wh[d], 1u);
            }
        }
        __syncthreads();
        if (t < 256) {                       // CTA histogram = sum of the warp histograms (then cleared)
            uint32_t sum = 0u;
#pragma unroll
            for (int w = 0; w < NWp; ++w) { sum += whist[w][t]; whist[w][t] = 0u; }
            hb[t] = sum;
        }
        ph_stamp<2>(2 + pass);
        cl.sync();                           // histograms of this digit visible cluster-wide
        // the other buffer was last read remotely before this barrier: clear it for the next digit
        if (t < 256) {
            uint32_t g = 0u;
            for (int q = 0; q < CL; ++q) g += cl.map_shared_rank(hb, q)[t];
            bits[t] = g;                     // global histogram (bits[] is free until step 3)
        }
        __syncthreads();
        if (t < 32) {
            int v[8], s = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) { v[e] = (int)bits[255 - 8 * lane - e]; s += v[e]; }
            int incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int excl = incl - s;
            int D = -1, cab = 0, cum = excl, cnt = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (D < 0 && cum + v[e] >= kk) { D = 255 - 8 * lane - e; cab = cum; cnt = v[e]; }
                cum += v[e];
            }
            const unsigned bm = __ballot_sync(0xffffffffu, D >= 0 && excl < kk);
            const int src = __ffs(bm) - 1;
            D = __shfl_sync(0xffffffffu, D, src);
            cab = __shfl_sync(0xffffffffu, cab, src);
            cnt = __shfl_sync(0xffffffffu, cnt, src);
            if (lane == 0) { sh[0] = D; sh[1] = cab; sh[2] = cnt; }
        }
        __syncthreads();
        prefix |= (uint32_t)sh[0] << shift;
        pmask |= 255u << shift;
        kk -= sh[1];
        const int cnt = sh[2];
        if (kk == cnt) { whole = true; break; }
    }
    stamp(1, 2);
    ph_stamp<2>(6);
    // selected: (key & pmask) > prefix, or (key & pmask) == prefix and (whole, or one of the
    // first kk equal keys in page order)
    int take = 0;
    if (!whole) {
        int ceq = 0;
#pragma unroll
        for (int j = 0; j < kTkKPT; ++j) ceq += key[j] == prefix;
        ceq = block_sum_i<NT>(ceq, sh);
        if (t == 0) xch[0] = ceq;
        cl.sync();
        int before = 0;
        for (int q = 0; q < r; ++q) before += *cl.map_shared_rank(&xch[0], q);
        take = min(max(kk - before, 0), ceq);
        // equal keys of this CTA in page order: bitmap, word w = pages 32 w .. 32 w + 31
#pragma unroll
        for (int j = 0; j < kTkKPT / 4; ++j) {
            uint32_t nib = 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e) nib |= (key[4 * j + e] == prefix ? 1u : 0u) << e;
            const uint32_t w = nibble_word(nib, lane);
            if ((lane & 7) == 0) bits[(NT / 8) * j + (t >> 3)] = w;
        }
        __syncthreads();
        uint32_t w = t < NT / 2 ? bits[t] : 0u;
        int tot;
        int rank = block_excl_scan<NT>(__popc(w), sh, &tot);
        uint32_t keep = 0u;
        while (w) {
            const uint32_t lb = w & (0u - w);
            if (rank < take) keep |= lb;
            ++rank;
            w ^= lb;
        }
        __syncthreads();
        if (t < NT / 2) bits[t] = keep;      // chosen equal keys
        __syncthreads();
    }
    // 3. selection bitmap and ascending output
#pragma unroll
    for (int j = 0; j < kTkKPT / 4; ++j) {
        uint32_t nib = 0u;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t v = key[4 * j + e] & pmask;
            const bool s = v > prefix || (whole && v == prefix);
            nib |= (s ? 1u : 0u) << e;
        }
        const uint32_t w = nibble_word(nib, lane);
        if ((lane & 7) == 0) {
            const int wi = (NT / 8) * j + (t >> 3);
            bits[wi] = whole ? w : (w | bits[wi]);
        }
    }
    __syncthreads();
    const uint32_t w = t < NT / 2 ? bits[t] : 0u;
    int tot;
    const int pos = block_excl_scan<NT>(__popc(w), sh, &tot);
    if (t == 0) xch[1] = tot;
    cl.sync();
    int o = pos;
    for (int q = 0; q < r; ++q) o += *cl.map_shared_rank(&xch[1], q);
    uint32_t v = w;
    while (v) {
        const int p = base + 32 * t + __ffs(v) - 1;
        v &= v - 1;
        out[o++] = p;
        if (um) union_mark(um, p, gh);
    }
    if (r == 0 && t == 0) n_sel[row] = keff;
    stamp(1, 6);
    ph_stamp<2>(7);
    cl.sync();                               // keep shared memory alive for remote readers
}

// ============================================================================ union per KV group
// The union of the G selections of a KV group (R17): umask[b][kvh][page] bytes (4 per
// u32, bit g = selected by query head g of the group), zeroed by the host and filled
// with atomicOr from the page lists.  The K-score kernel walks the G page lists of a
// group and keeps a page only from its lowest selecting head (one read per union page).
__global__ void __launch_bounds__(256) k_mark(int Hq, int G, const int32_t *__restrict__ page_idx,
                                              const int32_t *__restrict__ n_sel, int sel_stride,
                                              uint32_t *__restrict__ umask, int W) {
    EKV_TRACE(3);
    pdl_wait();
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

// mass(tau) = sum_p c_p M_beta(a mu_p - tau, a sigma_p) and -d mass / d tau, in fp64 (FP64 = 1)
// or fp32 (steering only).  Pages whose standardised t = (a mu - tau) / (a sigma) < -9 are
// skipped: their terms are below Phi(-9) ~ 1e-19 relative (the fp64 sum's own rounding is
// ~1e-16), decided by a conservative fp32 pre-test.
template <int NT, bool FP64>
__device__ void gauss_mass2(const float *mu, const float *s2, int M, int Lseq, float af, int beta, double tau,
                            double &mass, double &dmass, double *shd) {
    double m = 0.0, dm = 0.0;
    const float tf = (float)tau;
    for (int p = threadIdx.x; p < M; p += NT) {
        const float mp = __ldg(mu + p), sp = sqrtf(__ldg(s2 + p));
        const float num = af * mp - tf, den = af * sp;
        if (den > 0.f ? (num < -9.5f * den) : (num <= 0.f)) continue;
        const double cnt = (double)min(kP, Lseq - p * kP);
        if constexpr (FP64) {
            const double a = (double)af;
            const double sg = sqrt((double)s2[p]);
            GaussMoments g = trunc_moments(beta, a * (double)mp - tau, a * sg);
            m += cnt * g.m;
            dm += cnt * (double)beta * g.dm;
        } else {
            float r, rm;
            if (!(den > 0.f)) {
                const float x = num > 0.f ? num : 0.f;
                r = 1.f; rm = 1.f;
                for (int i = 0; i < beta; ++i) { rm = r; r *= x; }
            } else {
                const float t = num / den;
                const float Ph = normcdff(t), ph = __expf(-0.5f * t * t) * 0.39894228f;
                float m0 = Ph, m1 = num * Ph + den * ph;
                if (beta == 1) { r = m1; rm = m0; }
                else {
                    float pr = m0, cu = m1;
                    for (int k = 2; k <= beta; ++k) { const float nx = num * cu + (float)(k - 1) * den * den * pr; pr = cu; cu = nx; }
                    r = cu; rm = pr;
                }
            }
            m += cnt * (double)r;
            dm += cnt * (double)beta * (double)rm;
        }
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
    EKV_TRACE(8);
    pdl_wait();
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
    const float af = (float)a;
    const int beta = (int)llrint(1.0 / a);
    // (1) fp32 steering: bracket from a max_p (mu + 8 sigma), then safeguarded Newton
    float tmax = -INFINITY;
    for (int p = threadIdx.x; p < M; p += NT) tmax = fmaxf(tmax, m_[p] + 8.0f * sqrtf(s_[p]));
    tmax = block_max_f<NT>(tmax, shf);
    double hi = a * (double)tmax, w = 1.0, mass, dmass;
    for (int it = 0; it < 200; ++it) {
        gauss_mass2<NT, false>(m_, s_, M, Lseq, af, beta, hi, mass, dmass, shd);
        if (mass < 1.0) break;
        hi += w; w *= 2.0;
    }
    double lo = hi - 1.0;
    w = 1.0;
    for (int it = 0; it < 200; ++it) {
        gauss_mass2<NT, false>(m_, s_, M, Lseq, af, beta, lo, mass, dmass, shd);
        if (mass >= 1.0) break;
        lo -= w; w *= 2.0;
    }
    double tau = lo;
    for (int it = 0; it < 60; ++it) {
        gauss_mass2<NT, false>(m_, s_, M, Lseq, af, beta, tau, mass, dmass, shd);
        if (mass >= 1.0) lo = tau; else hi = tau;
        double nt = (dmass > 0.0) ? tau + (mass - 1.0) / dmass : 0.5 * (lo + hi);
        if (!(nt > lo && nt < hi)) nt = 0.5 * (lo + hi);
        const bool stop = fabs(nt - tau) <= 2e-7 * fmax(1.0, fabs(tau)) || hi - lo <= 2e-7 * fmax(1.0, fabs(hi));
        tau = nt;
        if (stop) break;
    }
    // (2) fp64 Newton straight from the fp32 root (mass is convex and decreasing: quadratic
    // convergence from ~1e-6 takes two or three passes); any large or non-finite step falls
    // back to a verified bracket + safeguarded Newton
    bool done64 = false;
    {
        double t = tau;
        for (int it = 0; it < 4; ++it) {
            gauss_mass2<NT, true>(m_, s_, M, Lseq, af, beta, t, mass, dmass, shd);
            if (!(dmass > 0.0)) break;
            const double step = (mass - 1.0) / dmass;
            if (!(fabs(step) <= 1e-3 * fmax(1.0, fabs(t)))) break;
            t += step;
            if (fabs(step) <= 1e-14 * fmax(1.0, fabs(t))) { done64 = true; break; }
        }
        if (done64) tau = t;
    }
    double dl = 1e-4 * fmax(1.0, fabs(tau));
    if (!done64) {
    lo = tau - dl;
    for (int it = 0; it < 200; ++it) {
        gauss_mass2<NT, true>(m_, s_, M, Lseq, af, beta, lo, mass, dmass, shd);
        if (mass >= 1.0) break;
        dl *= 4.0; lo = tau - dl;
    }
    double dh = 1e-4 * fmax(1.0, fabs(tau));
    hi = tau + dh;
    for (int it = 0; it < 200; ++it) {
        gauss_mass2<NT, true>(m_, s_, M, Lseq, af, beta, hi, mass, dmass, shd);
        if (mass < 1.0) break;
        dh *= 4.0; hi = tau + dh;
    }
    tau = fmin(fmax(tau, lo), hi);
    for (int it = 0; it < 100; ++it) {
        gauss_mass2<NT, true>(m_, s_, M, Lseq, af, beta, tau, mass, dmass, shd);
        if (mass >= 1.0) lo = tau; else hi = tau;
        double nt = (dmass > 0.0) ? tau + (mass - 1.0) / dmass : 0.5 * (lo + hi);
        if (!(nt > lo && nt < hi)) nt = 0.5 * (lo + hi);
        if (fabs(nt - tau) <= 1e-15 * fmax(1.0, fabs(tau)) || hi - lo <= 1e-15 * fmax(1.0, fabs(hi))) {
            tau = nt;
            break;
        }
        tau = nt;
    }
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
