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

// bitmap word of the CTA-local pages 2048 j + 4 t + e (e < 4) of a 4-bit nibble per thread:
// 8 consecutive lanes share a word (index 64 j + t / 8); lane t % 8 == 0 returns it
__device__ __forceinline__ uint32_t nibble_word(uint32_t nib, int lane) {
    uint32_t w = nib << (4 * (lane & 7));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    return w;
}

// One histogram increment per active lane, aggregated to one shared atomic when all active
// lanes of the warp hit the same bin (the usual case for leading digits).  (__match_any_sync
// was measured at ~12 us for a 4-pass select over 4096 keys: far slower than this.)
__device__ __forceinline__ void hist_add_agg(uint32_t *hist, uint32_t d, bool act, int lane) {
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (bal == 0u) return;
    const int leader = __ffs(bal) - 1;
    const uint32_t dl = __shfl_sync(0xffffffffu, d, leader);
    const unsigned same = __ballot_sync(0xffffffffu, act && d == dl);
    if (same == bal) {
        if (lane == leader) atomicAdd(&hist[dl], (uint32_t)__popc(bal));
    } else if (act) {
        atomicAdd(&hist[d], 1u);
    }
}

// Block-wide k-th largest of per-thread uint32 keys (CPT per thread, 0 = no key; 1 <= k <= #keys):
// MSB-first radix select, 8-bit digits, one shared 256-bin histogram per digit.
// Per-warp private histograms whist[NT/32][256] (zero on entry, left zero on exit): no
// cross-warp contention on the leading digits' single hot bin.
template <int NT>
__device__ __forceinline__ void hist_merge(uint32_t (*whist)[256], uint32_t *hist) {
    for (int i = threadIdx.x; i < 256; i += NT) {
        uint32_t g = 0u;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) { g += whist[w][i]; whist[w][i] = 0u; }
        hist[i] = g;
    }
}
template <int NT, int CPT>
__device__ uint32_t block_kth_largest_agg(const uint32_t (&key)[CPT], int k, uint32_t (*whist)[256], uint32_t *hist,
                                          int *sh) {
    uint32_t prefix = 0u, pmask = 0u;
    int kk = k;
    const int t = threadIdx.x, lane = t & 31;
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const bool act = key[j] != 0u && (key[j] & pmask) == prefix;
            hist_add_agg(whist[t >> 5], (key[j] >> shift) & 255u, act, lane);
        }
        __syncthreads();
        hist_merge<NT>(whist, hist);
        __syncthreads();
        if (t < 32) {
            int v[8], s = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) { v[e] = (int)hist[255 - 8 * lane - e]; s += v[e]; }
            int incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int excl = incl - s;
            int D = -1, cab = 0, cum = excl;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (D < 0 && cum + v[e] >= kk) { D = 255 - 8 * lane - e; cab = cum; }
                cum += v[e];
            }
            const unsigned bm = __ballot_sync(0xffffffffu, D >= 0 && excl < kk);
            const int src = __ffs(bm) - 1;
            D = __shfl_sync(0xffffffffu, D, src);
            cab = __shfl_sync(0xffffffffu, cab, src);
            if (lane == 0) { sh[0] = D; sh[1] = cab; }
        }
        __syncthreads();
        prefix |= (uint32_t)sh[0] << shift;
        pmask |= 255u << shift;
        kk -= sh[1];
        __syncthreads();
    }
    return prefix;
}


// ---- value-domain (linear) histogram helpers of the sample-pivot top-k
constexpr int kLinNB = 1024;
template <int NT> __device__ __forceinline__ uint32_t block_max_u32(uint32_t v, uint32_t *shu) {
    v = __reduce_max_sync(0xffffffffu, v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) shu[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t r = 0u;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) r = max(r, shu[w]);
    return r;
}
template <int NT> __device__ __forceinline__ uint32_t block_min_u32(uint32_t v, uint32_t *shu) {
    v = __reduce_min_sync(0xffffffffu, v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) shu[threadIdx.x >> 5] = v;
    __syncthreads();
    uint32_t r = 0xffffffffu;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) r = min(r, shu[w]);
    return r;
}
// bin of an ordered key in [klo, khi]: floor((v - vlo) * sc), monotone non-decreasing in the key
__device__ __forceinline__ int lin_bin(uint32_t key, float vlo, float sc) {
    return min(kLinNB - 1, max(0, (int)((key2f(key) - vlo) * sc)));
}
// Locate the bin holding the r-th largest element of a kLinNB-bin histogram: out[0] = bin,
// out[1] = #elements in higher bins, out[2] = the bin's count.  1 <= r <= total.
// Sample-pivot variant: r is derived from the histogram's total (the valid samples Sv):
// r = min(Sv, ceil(1.25 k Sv / M) + 16); out[3] = r (0: no valid sample, out[0] = -1).
template <int NT> __device__ __forceinline__ void lin_find_rp(const uint32_t *lin, int keff, int M, int *sh, int *out) {
    constexpr int PER = kLinNB / NT;
    const int t = threadIdx.x;
    int loc = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) loc += (int)lin[kLinNB - 1 - (t * PER + i)];
    if (t == 0) out[0] = -1;                 // (ordered before the finder's write by the scan's barrier)
    int tot;
    const int ex = block_excl_scan1<NT>(loc, sh, &tot);
    const int r = min(tot, (int)ceil(1.25 * (double)keff * (double)tot / (double)M) + 16);
    if (t == 0) out[3] = r;
    if (r >= 1 && ex < r && r <= ex + loc) {
        int cum = ex;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int bn = kLinNB - 1 - (t * PER + i);
            const int c = (int)lin[bn];
            if (cum + c >= r) { out[0] = bn; out[1] = cum; out[2] = c; break; }
            cum += c;
        }
    }
    __syncthreads();
}
template <int NT> __device__ __forceinline__ void lin_find(const uint32_t *lin, int r, int *sh, int *out) {
    constexpr int PER = kLinNB / NT;                  // bins per thread, from the top down
    const int t = threadIdx.x;
    int loc = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) loc += (int)lin[kLinNB - 1 - (t * PER + i)];
    int tot;
    const int ex = block_excl_scan1<NT>(loc, sh, &tot);
    if (ex < r && r <= ex + loc) {
        int cum = ex;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int bn = kLinNB - 1 - (t * PER + i);
            const int c = (int)lin[bn];
            if (cum + c >= r) { out[0] = bn; out[1] = cum; out[2] = c; break; }
            cum += c;
        }
    }
    __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_topk(const float *__restrict__ box, int Hq, int maxp,
                                                const int32_t *__restrict__ seq_lens, int k,
                                                int32_t *__restrict__ page_idx, int32_t *__restrict__ n_sel,
                                                int sel_stride, int G, uint32_t *__restrict__ umask, int W) {
    EKV_TRACE(2);
    pdl_enter();
    pdl_trigger<2>();
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
    __shared__ int wsc2[2][NT / 32];
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
    // 1a. Sample pivot (exact; the cluster radix select below is the fallback).  Every CTA
    //     publishes NT sampled keys (one per thread, spread over its range); every CTA gathers
    //     the cluster's samples and takes, by a block radix select, the pivot T_p = the r_p-th
    //     largest sample, r_p ~ 1.25 k / M of the samples + 16 (so that about 1.25 k keys and
    //     always at least k, barring a 4-sigma sampling event, are >= T_p).  The candidates
    //     key >= T_p are collected as unique composites (key << 32 | ~page: larger key first,
    //     then the lower page, R3) -- if there are between k and kTkCap of them, every CTA
    //     gathers them all and finds T* = the k-th largest composite (MSB-first radix select
    //     with 8-bit digits, stopping when a digit's bin is taken whole); the selection is
    //     composite >= T*.  Two cluster barriers instead of one per digit and a tie round.
    extern __shared__ __align__(16) unsigned long long tk_dyn[];
    bool fast = false;
    int nfast = 0;
    unsigned long long tcomp = 0ull;
    uint32_t tpiv = 0xffffffffu;
    {
        unsigned long long *lc = tk_dyn;               // [kTkCap] this CTA's candidates
        unsigned long long *gc = tk_dyn + kTkCap;      // [kTkCap] the cluster's candidates
        __shared__ uint32_t samp[NT];
        __shared__ uint32_t lin[kLinNB];
        __shared__ int lincnt, linres[4];
        __shared__ uint32_t xmax, cmax_sh;           // published: max candidate key of the CTA
        __shared__ unsigned long long tcomp_sh;
        __shared__ int qoff[8], qcnt[8];
        {
            const int si = (t & 3) * 4 + ((t >> 2) & 3);      // (keeps key[] in registers)
            uint32_t sv0 = 0u;
#pragma unroll
            for (int j = 0; j < kTkKPT; ++j) sv0 = (j == si) ? key[j] : sv0;
            samp[t] = sv0;
        }
        for (int i = t; i < NWp * 256; i += NT) (&whist[0][0])[i] = 0u;
        for (int i = t; i < kLinNB; i += NT) lin[i] = 0u;
        if (t == 0) { xmax = 0u; lincnt = 0; }
        cl.sync();                                     // (1) samples published (and whist, lin zero)
        ph_stamp<2>(2);
        uint32_t sk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) sk[i] = (i < CL) ? cl.map_shared_rank(samp, i)[t] : 0u;
        // pivot: tp with #{samples >= tp} >= rp -- the lower edge of the linear-histogram bin
        // (1024 bins over the samples' value range) holding the rp-th largest sample; rp from
        // the valid-sample count the histogram's scan yields
        uint32_t tp = 0xffffffffu;
        int rp = 0;
        {
            uint32_t smax = 0u, smin = 0xffffffffu;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (sk[i]) { smax = max(smax, sk[i]); smin = min(smin, sk[i]); }
            {
                const uint32_t a = __reduce_max_sync(0xffffffffu, smax), b2 = __reduce_min_sync(0xffffffffu, smin);
                if (lane == 0) { bits[t >> 5] = a; bits[32 + (t >> 5)] = b2; }
                __syncthreads();
#pragma unroll
                for (int w = 0; w < NWp; ++w) { smax = max(smax, bits[w]); smin = min(smin, bits[32 + w]); }
            }
            const float vlo = key2f(smin), sc = (float)kLinNB / (key2f(smax) - vlo);
            if (smin == 0xffffffffu) {
                // no valid sample: no pivot (radix fallback)
            } else if (smax == smin) {
                tp = smax;
                rp = 1;
            } else if (!(sc > 0.0f && sc < INFINITY)) {
                int sv = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) sv += sk[i] != 0u;
                const int Sv = block_sum_i<NT>(sv, sh);
                rp = min(Sv, (int)ceil(1.25 * (double)keff * (double)Sv / (double)M) + 16);
                tp = block_kth_largest_agg<NT, 8>(sk, rp, whist, hist[0], sh);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (sk[i]) atomicAdd(&lin[lin_bin(sk[i], vlo, sc)], 1u);
                __syncthreads();
                lin_find_rp<NT>(lin, keff, M, sh, linres);
                const int B = linres[0];
                rp = linres[3];
                if (B == 0) tp = smin;
                else if (B > 0) {
                    // every sample of bins >= B is >= the bin's lower edge, less a relative margin
                    // for lin_bin's two roundings
                    const float e = vlo + (float)B / sc;
                    tp = max(f2key(e - (fabsf(e) + fabsf(vlo)) * 1.0e-5f), smin);
                }
                for (int i = t; i < kLinNB; i += NT) lin[i] = 0u;     // (read before lin_find's barrier)
            }
        }
        tpiv = tp;
        ph_stamp<2>(3);
        int nc = 0;
        uint32_t kmx = 0u;
#pragma unroll
        for (int j = 0; j < kTkKPT; ++j) {
            const bool cnd = key[j] != 0u && key[j] >= tp;
            nc += cnd ? 1 : 0;
            kmx = cnd ? max(kmx, key[j]) : kmx;
        }
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        if (lane == 0 && kmx) atomicMax(&xmax, kmx);
        int ntot;
        int pos = block_excl_scan1<NT>(nc, sh, &ntot);
#pragma unroll
        for (int j = 0; j < kTkKPT; ++j) {
            if (key[j] != 0u && key[j] >= tp) {
                if (pos < kTkCap) {
                    const uint32_t page = (uint32_t)(base + 4 * (t + NT * (j >> 2)) + (j & 3));
                    lc[pos] = ((unsigned long long)key[j] << 32) | (unsigned long long)(0xffffffffu - page);
                }
                ++pos;
            }
        }
        if (t == 0) xch[0] = ntot;
        cl.sync();                                     // (2) candidate lists published
        ph_stamp<2>(4);
        // the CTAs' counts in one round of parallel remote loads (lane q reads CTA q)
        if (t < 32) {
            const int nq = t < CL ? *cl.map_shared_rank(&xch[0], t) : 0;
            const uint32_t mq = __reduce_max_sync(0xffffffffu, t < CL ? *cl.map_shared_rank(&xmax, t) : 0u);
            int inc = nq;
#pragma unroll
            for (int o2 = 1; o2 < 8; o2 <<= 1) { const int y = __shfl_up_sync(0xffffffffu, inc, o2); if (t >= o2) inc += y; }
            if (t < 8) { qoff[t] = inc - nq; qcnt[t] = nq; }
            if (t == 0) cmax_sh = mq;
        }
        __syncthreads();
        const int C = qoff[CL - 1] + qcnt[CL - 1];
        fast = rp >= 1 && C >= keff && C <= kTkCap;    // uniform over the cluster
        nfast = C;
        ph_count<2>(0, C);
        ph_count<2>(1, (long long)rp * 10 + (fast ? 1 : 0));
        if (fast) {
            // gather: element i comes from the CTA q with qoff[q] <= i < qoff[q] + qcnt[q]; all of a
            // thread's remote loads are issued before any is used
            constexpr int GPT = kTkCap / NT;
            unsigned long long tmp[GPT];
#pragma unroll
            for (int u = 0; u < GPT; ++u) {
                const int i = t + NT * u;
                int q = 0;
#pragma unroll
                for (int z = 1; z < 8; ++z) q += (z < CL && qoff[z] <= i) ? 1 : 0;
                tmp[u] = i < C ? cl.map_shared_rank(lc, q)[i - qoff[q]] : 0ull;
            }
            // T* = the keff-th largest composite: linear histogram of the candidates' values over
            // [tp, max] (built from the gathered registers), then a brute-force rank among the
            // (few) composites of the boundary bin.  Every later pass over gc reads only the
            // thread's own entries i = t + NT u: no barrier for gc itself.
            const uint32_t cmax = cmax_sh;           // (lin and lincnt were zeroed before barrier (2))
            const float vlo = key2f(tp), sc = (float)kLinNB / (key2f(cmax) - vlo);
            const bool linok = cmax != tp && sc > 0.0f && sc < INFINITY;
#pragma unroll
            for (int u = 0; u < GPT; ++u) {
                const int i = t + NT * u;
                if (i < C) {
                    gc[i] = tmp[u];
                    if (linok) atomicAdd(&lin[lin_bin((uint32_t)(tmp[u] >> 32), vlo, sc)], 1u);
                }
            }
            // this thread's remote reads are done: arrive on the cluster barrier now, wait only at
            // exit (the other CTAs' lists stay alive until every CTA has gathered)
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            bool done = false;
            {
                if (linok) {
                    __syncthreads();
                    lin_find<NT>(lin, keff, sh, linres);
                    const int B = linres[0], need = keff - linres[1], cB = linres[2];
                    unsigned long long *bb = reinterpret_cast<unsigned long long *>(&whist[0][0]);
                    constexpr int BBCAP = NWp * 256 / 2;
                    if (cB <= BBCAP) {
                        for (int i = t; i < C; i += NT)
                            if (lin_bin((uint32_t)(gc[i] >> 32), vlo, sc) == B) bb[atomicAdd(&lincnt, 1)] = gc[i];
                        __syncthreads();
                        for (int i = t; i < cB; i += NT) {
                            int rk = 0;
                            const unsigned long long me = bb[i];
                            for (int j2 = 0; j2 < cB; ++j2) rk += bb[j2] > me;
                            if (rk == need - 1) tcomp_sh = me;
                        }
                        __syncthreads();
                        tcomp = tcomp_sh;
                        done = true;
                    }
                }
            }
            unsigned long long pre = 0ull, pm = 0ull;
            int kk = keff;
            if (!done) {
#pragma unroll 1
            for (int pass = 0; pass < 8; ++pass) {
                const int shift = 56 - 8 * pass;
                for (int i0 = 0; i0 < C; i0 += NT) {   // uniform trip count (warp votes below)
                    const int i = i0 + t;
                    const unsigned long long xv = i < C ? gc[i] : 0ull;
                    const bool act = i < C && (xv & pm) == pre;
                    hist_add_agg(whist[t >> 5], (uint32_t)((xv >> shift) & 255ull), act, lane);
                }
                __syncthreads();
                hist_merge<NT>(whist, hist[0]);
                __syncthreads();
                if (t < 32) {
                    int v[8], s8 = 0;
#pragma unroll
                    for (int e = 0; e < 8; ++e) { v[e] = (int)hist[0][255 - 8 * lane - e]; s8 += v[e]; }
                    int incl = s8;
#pragma unroll
                    for (int o2 = 1; o2 < 32; o2 <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o2);
                        if (lane >= o2) incl += y;
                    }
                    const int excl = incl - s8;
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
                pre |= (unsigned long long)sh[0] << shift;
                pm |= 255ull << shift;
                kk -= sh[1];
                const int cnt = sh[2];
                __syncthreads();
                if (kk == cnt) break;                  // the bin is taken whole (composites are unique)
            }
            tcomp = pre;
            }
        }
#ifdef EKV_DBG_TOPK
        if (t == 0 && row == EKV_DBG_TOPK)
            printf("row %d r %d CL %d M %d keff %d rp %d tp %08x C %d nloc %d fast %d tcomp %016llx\n", row, r, CL, M,
                   keff, rp, tp, C, xch[0], (int)fast, tcomp);
#endif
        ph_stamp<2>(5);
    }
    stamp(1, 1);
    ph_stamp<2>(1);
    // 1. radix select over the cluster (fallback)
    uint32_t prefix = 0u, pmask = 0u;
    int kk = keff;                           // keys still to take among those matching prefix
    bool whole = fast;                       // the last digit's bin is taken entirely
    if (!fast) {
    for (int i = t; i < NWp * 256; i += NT) (&whist[0][0])[i] = 0u;
    __syncthreads();
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
            bool s;
            if (fast) {
                const uint32_t page = (uint32_t)(base + 4 * (t + NT * j) + e);
                s = key[4 * j + e] != 0u && key[4 * j + e] >= tpiv &&          // a candidate, and
                    (((unsigned long long)key[4 * j + e] << 32) | (unsigned long long)(0xffffffffu - page)) >= tcomp;
            } else {
                const uint32_t v = key[4 * j + e] & pmask;
                s = v > prefix || (whole && v == prefix);
            }
            nib |= (s ? 1u : 0u) << e;
        }
        const uint32_t w = nibble_word(nib, lane);
        if ((lane & 7) == 0) {
            const int wi = (NT / 8) * j + (t >> 3);
            bits[wi] = whole ? w : (w | bits[wi]);
        }
    }
    // the lower ranks' selected pages (fast: counted from this CTA's copy of the candidate list --
    // every selected page is a candidate -- no cluster exchange), folded into the one-barrier scan
    int clow = 0;
    if (fast && r > 0) {
        const unsigned long long *gc = tk_dyn + kTkCap;
        const uint32_t inv_base = 0xffffffffu - (uint32_t)base;   // page < base <=> low word > inv_base
        for (int i = t; i < nfast; i += NT) {
            const unsigned long long x = gc[i];
            clow += (x >= tcomp && (uint32_t)(x & 0xffffffffu) > inv_base) ? 1 : 0;
        }
    }
    __syncthreads();
    const uint32_t w = t < NT / 2 ? bits[t] : 0u;
    int tot, o;
    {
        const int pc = __popc(w);
        int x = pc;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o2); if (lane >= o2) x += y; }
        const int cw = __reduce_add_sync(0xffffffffu, clow);
        if (lane == 31) { wsc2[0][t >> 5] = x; wsc2[1][t >> 5] = cw; }
        __syncthreads();
        const int wv = lane < NWp ? wsc2[0][lane] : 0, cv = lane < NWp ? wsc2[1][lane] : 0;
        tot = __reduce_add_sync(0xffffffffu, wv);
        o = __reduce_add_sync(0xffffffffu, lane < (t >> 5) ? wv : 0) + x - pc + __reduce_add_sync(0xffffffffu, cv);
    }
    if (!fast) {
        if (t == 0) xch[1] = tot;
        cl.sync();
        if (r > 0) {                                         // sum of the lower ranks' counts
            int c = (lane < r) ? *cl.map_shared_rank(&xch[1], lane) : 0;
            c = __reduce_add_sync(0xffffffffu, c);
            o += c;
        }
    }
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
    if (fast) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // (arrived after the gather)
    else cl.sync();                          // keep shared memory alive for remote readers
}

// ============================================================================ union per KV group
// The union of the G selections of a KV group (R17): umask[b][kvh][page] bytes (4 per
// u32, bit g = selected by query head g of the group), zeroed by the host and filled
// with atomicOr from the page lists.  The K-score kernel walks the G page lists of a
// group and keeps a page only from its lowest selecting head (one read per union page).
static __global__ void __launch_bounds__(256) k_mark(int Hq, int G, const int32_t *__restrict__ page_idx,
                                              const int32_t *__restrict__ n_sel, int sel_stride,
                                              uint32_t *__restrict__ umask, int W) {
    EKV_TRACE(3);
    pdl_enter();
    const int row = blockIdx.x;
    const int b = row / Hq, h = row % Hq;
    const int unit = b * (Hq / G) + h / G, g = h % G;
    const int n = n_sel[row];
    const int32_t *pl = page_idx + (size_t)row * sel_stride;
    uint32_t *um = umask + (size_t)unit * W;
    for (int i = threadIdx.x; i < n; i += 256) union_mark(um, pl[i], g);
}

// ============================================================================ N4: certified selection
// Prop. B.2: C_page = {p : (alpha-1) sbar_box(p) > tau_hat} with tau_hat <= tau
// (here the exact threshold of a first top-k pass, R13 / R27); the fp64 decision of R9.
// One CTA per (b, q-head), 512 threads x 4 consecutive pages per chunk, ascending output by
// block scan, union marks for the group (umask zeroed by the host).  A NaN tau_hat (the
// first pass overflowed) selects every page -- still a superset.
static __global__ void __launch_bounds__(512) k_box_certified(const float *__restrict__ box, int Hq, int G, int maxp,
                                                              const int32_t *__restrict__ seq_lens,
                                                              const double *__restrict__ tau_hat, float alpha,
                                                              int32_t *__restrict__ page_idx,
                                                              int32_t *__restrict__ n_sel, int stride,
                                                              uint32_t *__restrict__ umask, int W) {
    pdl_enter();
    __shared__ int sh[18];
    const int row = blockIdx.x, b = row / Hq;
    const int M = n_pages_of(seq_lens[b]);
    const double a = (double)alpha - 1.0, t = tau_hat[row];
    const bool all = !(t == t);
    const float *x = box + (size_t)row * maxp;
    int32_t *out = page_idx + (size_t)row * stride;
    uint32_t *um = umask + (size_t)(b * (Hq / G) + (row % Hq) / G) * W;
    const int g = (row % Hq) % G;
    int base = 0;
    for (int p0 = 0; p0 < M; p0 += 512 * 4) {
        uint32_t bits = 0u;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int p = p0 + 4 * threadIdx.x + e;
            if (p < M && (all || a * (double)__ldg(x + p) > t)) bits |= 1u << e;
        }
        int tot;
        int pos = base + block_excl_scan<512>(__popc(bits), sh, &tot);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if ((bits >> e) & 1u) {
                const int p = p0 + 4 * threadIdx.x + e;
                out[pos++] = p;
                union_mark(um, p, g);
            }
        base += tot;
    }
    if (threadIdx.x == 0) n_sel[row] = base;
}

// ============================================================================ a2': Gaussian selector
struct GaussMoments { double m, dm, d2; };   // M_beta, M_{beta-1}, and the d^2/dtau^2 term

// truncated moments of Y ~ N(muY, sigY^2): M_k = E[(Y)_+^k] by the App. D recursion
// M_k = muY M_{k-1} + (k-1) sigY^2 M_{k-2} (M_0 = Phi(t), M_1 = muY Phi + sigY phi).
// d2 = M_{beta-2} (beta >= 2) or phi(t) / sigY (beta = 1): with it
// mass'' = beta (beta-1) sum c M_{beta-2}  (beta = 1: sum c phi / sigY), for Halley steps.
__device__ __forceinline__ GaussMoments trunc_moments(int beta, double muY, double sigY) {
    if (!(sigY > 0.0)) {
        if (!(muY > 0.0)) return {0.0, 0.0, 0.0};
        double r = 1.0, rm = 1.0, rm2 = 1.0;
        for (int i = 0; i < beta; ++i) { rm2 = rm; rm = r; r *= muY; }
        return {r, rm, beta == 1 ? 0.0 : rm2};
    }
    const double t = muY / sigY;
    const double Ph = normcdf(t);
    const double ph = exp(-0.5 * t * t) * 0.39894228040143267794;   // 1/sqrt(2 pi)
    const double m0 = Ph, m1 = muY * Ph + sigY * ph;
    if (beta == 1) return {m1, m0, ph / sigY};
    double pp = m0, prev = m0, cur = m1;
    for (int k = 2; k <= beta; ++k) {
        const double nx = muY * cur + (double)(k - 1) * sigY * sigY * prev;
        pp = prev; prev = cur; cur = nx;
    }
    return {cur, prev, pp};
}

// ---------------------------------------------------------------- non-integer beta (N4, R28)
// E[(Y)_+^beta] = sigY^beta h(m), m = muY / sigY, h(m) = int_0^inf u^beta phi(u - m) du ("the
// expectation can be evaluated numerically").  Per call, k_gauss_table fills a table
// of g = log h on [-10, 22) -- 64 intervals of width 1/2, a degree-15 Chebyshev series each,
// from tanh-sinh quadrature at the Chebyshev nodes -- plus the series of g' and g''; pages
// then get h = e^g, h' = g' h (= beta h_{beta-1}), h'' = (g'' + g'^2) h (= beta (beta-1)
// h_{beta-2}) from three Clenshaw sums.  m < -10: 0 (such pages are skipped, t < -9.5);
// m >= 22: the asymptotic series E[(m + Z)^b] = m^b sum_k C(b, 2k) (2k-1)!! m^-2k.
constexpr int kGtN = 16, kGtI = 64, kGtStride = 48;
constexpr double kGtLo = -10.0, kGtW = 0.5;
__device__ double gt_quad(double beta, double m) {
    const double L = fmax(0.0, m - 12.0), U = fmax(m, 0.0) + 12.0, hw = 0.5 * (U - L);
    double prev = NAN, s = 0.0;
    for (double h = 0.125; h > 0.0009; h *= 0.5) {
        s = 0.0;
        const int K = (int)ceil(4.5 / h);
        for (int k = -K; k <= K; ++k) {
            const double t = k * h, y = 1.5707963267948966 * sinh(t);
            const double e = exp(-2.0 * fabs(y));
            const double dn = 2.0 * hw * e / (1.0 + e);
            const double u = t < 0.0 ? L + dn : U - dn;
            const double ch = cosh(y);
            const double w = hw * 1.5707963267948966 * cosh(t) / (ch * ch);
            if (!(w > 0.0) || !(u > 0.0)) continue;
            s += w * pow(u, beta) * exp(-0.5 * (u - m) * (u - m));
        }
        s *= h * 0.39894228040143267794;
        if (fabs(s - prev) <= 1e-13 * fabs(s)) break;   // (the DE rule's error ~squares per halving)
        prev = s;
    }
    return s;
}
// one CTA per interval, kGtN threads (one Chebyshev node each)
static __global__ void __launch_bounds__(kGtN) k_gauss_table(double beta, double *__restrict__ tab) {
    pdl_enter();
    __shared__ double gv[kGtN], cf[kGtN];
    const int iv = blockIdx.x, j = threadIdx.x;
    const double a0 = kGtLo + kGtW * iv, c = a0 + 0.5 * kGtW, r = 0.5 * kGtW;
    const double x = cos(3.141592653589793 * (j + 0.5) / kGtN);
    gv[j] = log(gt_quad(beta, c + r * x));
    __syncthreads();
    double sum = 0.0;
    for (int k = 0; k < kGtN; ++k) sum += gv[k] * cos(3.141592653589793 * j * (k + 0.5) / kGtN);
    cf[j] = sum * (2.0 / kGtN);
    __syncthreads();
    if (j == 0) {
        // derivative series (Chebyshev recurrence), scaled by 1 / r per derivative
        double *t = tab + (size_t)iv * kGtStride;
        double d1[kGtN], d2[kGtN];
        for (int k = 0; k < kGtN; ++k) t[k] = cf[k];
        d1[kGtN - 1] = 0.0;
        d1[kGtN - 2] = 2.0 * (kGtN - 1) * cf[kGtN - 1];
        for (int k = kGtN - 3; k >= 0; --k) d1[k] = d1[k + 2] + 2.0 * (k + 1) * cf[k + 1];
        d2[kGtN - 1] = 0.0;
        d2[kGtN - 2] = 2.0 * (kGtN - 1) * d1[kGtN - 1];
        for (int k = kGtN - 3; k >= 0; --k) d2[k] = d2[k + 2] + 2.0 * (k + 1) * d1[k + 1];
        for (int k = 0; k < kGtN; ++k) { t[kGtN + k] = d1[k] / r; t[2 * kGtN + k] = d2[k] / (r * r); }
    }
}
// Chebyshev sum sum_k c_k T_k(y) - c_0 / 2 (Clenshaw)
__device__ __forceinline__ double gt_cheb(const double *c, double y) {
    double b1 = 0.0, b2 = 0.0;
    for (int k = kGtN - 1; k >= 1; --k) { const double t = 2.0 * y * b1 - b2 + __ldg(c + k); b2 = b1; b1 = t; }
    return y * b1 - b2 + 0.5 * __ldg(c);
}
// E[(m + Z)_+^b] for large m (asymptotic series; the cut lower tail is below phi(22))
__device__ __forceinline__ double gt_asym(double b, double m) {
    double term = 1.0, s = 1.0;
    const double im2 = 1.0 / (m * m);
    for (int k = 0; k < 40; ++k) {
        term *= (b - 2 * k) * (b - 2 * k - 1) * im2 / (2.0 * (k + 1));   // C(b,2k+2)(2k+1)!!/(C(b,2k)(2k-1)!!)
        s += term;
        if (fabs(term) <= 1e-17 * fabs(s)) break;
    }
    return pow(m, b) * s;
}
// h, h', h'' at m (h' = dh/dm, h'' = d2h/dm2)
__device__ __forceinline__ void gt_eval(const double *tab, double beta, double m, double &h, double &h1, double &h2) {
    if (m < kGtLo) { h = h1 = h2 = 0.0; return; }
    if (m >= kGtLo + kGtI * kGtW) {
        h = gt_asym(beta, m);
        h1 = beta * gt_asym(beta - 1.0, m);
        h2 = beta * (beta - 1.0) * gt_asym(beta - 2.0, m);
        return;
    }
    const int iv = min(kGtI - 1, (int)((m - kGtLo) / kGtW));
    const double c = kGtLo + kGtW * iv + 0.5 * kGtW;
    const double y = (m - c) / (0.5 * kGtW);
    const double *t = tab + (size_t)iv * kGtStride;
    const double g = gt_cheb(t, y), g1 = gt_cheb(t + kGtN, y), g2 = gt_cheb(t + 2 * kGtN, y);
    h = exp(g);
    h1 = g1 * h;
    h2 = (g2 + g1 * g1) * h;
}
// the moments of trunc_moments for a non-integer beta, already multiplied as the mass needs:
// m = E[Y_+^b], dm = -dE/dtau = b E[Y_+^(b-1)], d2 = d2E/dtau2 = b (b-1) E[Y_+^(b-2)]
__device__ __forceinline__ GaussMoments trunc_moments_tab(const double *tab, double beta, double muY, double sigY) {
    if (!(sigY > 0.0)) {
        if (!(muY > 0.0)) return {0.0, 0.0, 0.0};
        return {pow(muY, beta), beta * pow(muY, beta - 1.0), beta * (beta - 1.0) * pow(muY, beta - 2.0)};
    }
    double h, h1, h2;
    gt_eval(tab, beta, muY / sigY, h, h1, h2);
    const double sb = pow(sigY, beta);
    return {sb * h, sb / sigY * h1, sb / (sigY * sigY) * h2};
}

template <int NT> __device__ __forceinline__ void block_sum3_d(double &a, double &b, double &c, double *sh) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { sh[3 * w] = a; sh[3 * w + 1] = b; sh[3 * w + 2] = c; }
    __syncthreads();
    if (w == 0) {
        double x = 0.0, y = 0.0, z = 0.0;
        if (l < NT / 32) { x = sh[3 * l]; y = sh[3 * l + 1]; z = sh[3 * l + 2]; }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            x += __shfl_xor_sync(0xffffffffu, x, o);
            y += __shfl_xor_sync(0xffffffffu, y, o);
            z += __shfl_xor_sync(0xffffffffu, z, o);
        }
        if (l == 0) { sh[0] = x; sh[1] = y; sh[2] = z; }
    }
    __syncthreads();
    a = sh[0]; b = sh[1]; c = sh[2];
}

// Pages whose standardised t = (a mu - tau) / (a sigma) < -9.5 are skipped: their terms are
// below Phi(-9.5) ~ 1e-21 relative (the fp64 sum's own rounding is ~1e-16), decided by a
// conservative fp32 pre-test.  sg = sqrtf(sigma2) (cached) or nullptr (computed).
#define EKV_GAUSS_SKIP(num, den) ((den) > 0.f ? ((num) < -9.5f * (den)) : ((num) <= 0.f))

// Cluster-split rows (CL > 1 CTAs per row, page slice [p0, p1) each): the CTA's partial sums
// are published in a double-buffered shared slot and every CTA adds the CL slots in rank order
// -- identical totals (and so identical Newton / Halley control flow) in every CTA, one
// cluster barrier per reduction.
struct GaussRed {
    double *slot;      // [2][4] this CTA's published partials (double-buffered)
    double *gath;      // [8][4] the CL CTAs' partials, gathered
    int CL, par;
};
__device__ __forceinline__ void gauss_cluster_sum(GaussRed &R, double *v, int n) {
    if (R.CL <= 1) return;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    double *my = R.slot + 4 * R.par;
    if (threadIdx.x < (unsigned)n) my[threadIdx.x] = threadIdx.x == 0 ? v[0] : threadIdx.x == 1 ? v[1] : v[2];
    cl.sync();
    if (threadIdx.x < (unsigned)(R.CL * n)) {
        const int q = threadIdx.x / n, i = threadIdx.x - q * n;
        R.gath[4 * q + i] = cl.map_shared_rank(my, q)[i];
    }
    __syncthreads();
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int q = 0; q < R.CL; ++q) acc += R.gath[4 * q + i];
        v[i] = acc;
    }
    R.par ^= 1;
}

// fp32 steering pass: mass(tau) and -d mass/d tau, fp32 terms and per-thread sums
template <int NT>
__device__ void gauss_mass32(const float *mu, const float *sg, const float *s2, int p0, int p1, int Lseq, float af,
                             int beta, float tf, double &mass, double &dmass, double *shd, GaussRed &R,
                             const double *gtab, double betaf) {
    float m = 0.f, dm = 0.f;
#pragma unroll 4
    for (int p = p0 + threadIdx.x; p < p1; p += NT) {
        const int i = p - p0;
        const float mp = mu[i], sp = sg ? sg[i] : sqrtf(s2[i]);
        const float num = af * mp - tf, den = af * sp;
        if (EKV_GAUSS_SKIP(num, den)) continue;
        const float cnt = (float)min(kP, Lseq - p * kP);
        float r, rm;
        if (beta == 0) {                          // non-integer beta: the table (fp64 terms)
            const GaussMoments g = trunc_moments_tab(gtab, betaf, (double)num, (double)den);
            r = (float)g.m; rm = (float)g.dm;
        } else if (!(den > 0.f)) {
            r = 1.f; rm = 1.f;
            for (int i2 = 0; i2 < beta; ++i2) { rm = r; r *= num; }
        } else {
            const float t = num / den;
            const float Ph = normcdff(t), ph = __expf(-0.5f * t * t) * 0.39894228f;
            const float m0 = Ph, m1 = num * Ph + den * ph;
            if (beta == 1) { r = m1; rm = m0; }
            else {
                float pr = m0, cu = m1;
                for (int k = 2; k <= beta; ++k) { const float nx = num * cu + (float)(k - 1) * den * den * pr; pr = cu; cu = nx; }
                r = cu; rm = pr;
            }
        }
        m = fmaf(cnt, r, m);
        dm = fmaf(cnt, rm, dm);
    }
    double a = m, b = beta == 0 ? (double)dm : (double)beta * dm;
    block_sum2_d<NT>(a, b, shd);
    double v[3] = {a, b, 0.0};
    gauss_cluster_sum(R, v, 2);
    mass = v[0]; dmass = v[1];
}

// fp64 pass: mass, -mass' and mass'' (the terms follow orc_gauss_mass: a, mu, sqrt(sigma2) in fp64)
template <int NT>
__device__ void gauss_mass64(const float *mu, const float *sg, const float *s2, int p0, int p1, int Lseq, float af,
                             int beta, double tau, double &mass, double &dmass, double &d2mass, double *shd,
                             GaussRed &R, const double *gtab, double betaf) {
    double m = 0.0, dm = 0.0, d2 = 0.0;
    const float tf = (float)tau;
    const double a = (double)af;
    for (int p = p0 + threadIdx.x; p < p1; p += NT) {
        const int i = p - p0;
        const float mp = mu[i], s2p = s2[i], sp = sg ? sg[i] : sqrtf(s2p);
        const float num = af * mp - tf, den = af * sp;
        if (EKV_GAUSS_SKIP(num, den)) continue;
        const double cnt = (double)min(kP, Lseq - p * kP);
        const GaussMoments g = beta == 0 ? trunc_moments_tab(gtab, betaf, a * (double)mp - tau, a * sqrt((double)s2p))
                                         : trunc_moments(beta, a * (double)mp - tau, a * sqrt((double)s2p));
        m = fma(cnt, g.m, m);
        dm = fma(cnt, g.dm, dm);
        d2 = fma(cnt, g.d2, d2);
    }
    if (beta > 0) {                               // (the table path returns them multiplied)
        dm *= (double)beta;
        d2 *= beta == 1 ? 1.0 : (double)(beta * (beta - 1));
    }
    block_sum3_d<NT>(m, dm, d2, shd);
    double v[3] = {m, dm, d2};
    gauss_cluster_sum(R, v, 3);
    mass = v[0]; dmass = v[1]; d2mass = v[2];
}

// One CTA per (b, q-head).  tau_hat solves  sum_p c_p E[(a S_p - tau)_+^beta] = 1
// (Eq. gaussian-threshold-main) with the App. D closed forms (beta integer,
// R15); the paper names Newton/Halley for it.  The row's mu, sigma2 and
// sqrt(sigma2) are staged in shared memory (rows up to cache_pages pages).
//  (1) fp32 steering: Newton on log mass (the terms are log-concave in tau: near-quadratic
//      in the Gaussian tails where the root usually lies), safeguarded by a bracket;
//  (2) fp64 Halley from the fp32 root (cubic: one pass, a second when the predicted error
//      (mass''/mass')^2 |step|^3 is not below 1e-15 relative); any large or non-finite step
//      falls back to a verified fp64 bracket + safeguarded Newton.
// Page rule (Eq. gaussian-selector-main, R14): keep p iff
// (double)a * fmaf(sqrtf(sigma2), zq[c], mu) > tau_hat - margin; empty -> argmax mu.
template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_gauss_select(const float *__restrict__ mu, const float *__restrict__ sigma2,
                                                     int Hq, int maxp, const int32_t *__restrict__ seq_lens,
                                                     float alpha, double margin, double q_page,
                                                     int32_t *__restrict__ page_idx, int32_t *__restrict__ n_sel,
                                                     int sel_stride, double *__restrict__ tau_hat_out, int cache_pages,
                                                     const double *__restrict__ gtab) {
    EKV_TRACE(8);
    pdl_enter();
    ph_stamp<8>(0);
    int n32 = 0, n64 = 0;
    extern __shared__ float gsm[];
    __shared__ double shd[3 * (NT / 32) + 3];
    __shared__ int shi[NT / 32 + 1];
    __shared__ float shf[NT / 32 + 1];
    __shared__ float zq[kP + 1];
    // zq[c] = Phi^{-1}(q_page^{1/c}), fp64 normcdfinv rounded to fp32 (R14)
    if (threadIdx.x >= 1 && threadIdx.x <= kP)
        zq[threadIdx.x] = (float)normcdfinv(pow(q_page, 1.0 / (double)threadIdx.x));
    // a row is split over the CL CTAs of a cluster (rows longer than the shared-memory stage):
    // CTA r owns pages [p0, p1) of the row
    namespace cg = cooperative_groups;
    const int CL = (int)cg::this_cluster().num_blocks(), rk = (int)cg::this_cluster().block_rank();
    __shared__ double red_slot[8], red_gath[32];
    GaussRed R{red_slot, red_gath, CL, 0};
    const int row = blockIdx.x / CL;
    const int b = row / Hq;
    const int Lseq = seq_lens[b];
    const int M = n_pages_of(Lseq);
    const int S = (maxp + CL - 1) / CL;
    const int p0 = min(M, rk * S), p1 = min(M, (rk + 1) * S);
    const float *mg = mu + (size_t)row * maxp + p0;
    const float *sgg = sigma2 + (size_t)row * maxp + p0;
    const bool cached = p1 - p0 <= cache_pages;
    float *c_mu = gsm, *c_s2 = gsm + cache_pages, *c_sg = gsm + 2 * cache_pages;
    const double a = (double)alpha - 1.0;
    const float af = (float)a;
    // integer beta in 1..4: App. D's closed forms (R15); any other beta: the table (N4, R28)
    const double betaf = 1.0 / a;
    const int beta = (fabs(betaf - rint(betaf)) < 1e-9 && rint(betaf) >= 1.0 && rint(betaf) <= 4.0) ? (int)rint(betaf) : 0;
    // stage the slice (and the bracket start a max_p (mu + 8 sigma))
    float tmax = -INFINITY;
    for (int i = threadIdx.x; i < p1 - p0; i += NT) {
        const float mp = __ldg(mg + i), s2p = __ldg(sgg + i), sp = sqrtf(s2p);
        if (cached) { c_mu[i] = mp; c_s2[i] = s2p; c_sg[i] = sp; }
        tmax = fmaxf(tmax, mp + 8.0f * sp);
    }
    tmax = block_max_f<NT>(tmax, shf);   // (its barriers publish the staged slice)
    if (CL > 1) {
        double v[3] = {(double)tmax, 0.0, 0.0};
        // (max via the sum machinery is wrong; exchange the CTA maxima explicitly)
        cg::cluster_group cl = cg::this_cluster();
        if (threadIdx.x == 0) red_slot[4] = (double)tmax;
        cl.sync();
        double mx = -INFINITY;
        for (int q = 0; q < CL; ++q) mx = fmax(mx, *cl.map_shared_rank(&red_slot[4], q));
        tmax = (float)mx;
        (void)v;
        cl.sync();                        // (red_slot[4] is reused by the first reduction)
    }
    const float *m_ = cached ? c_mu : mg, *s_ = cached ? c_s2 : sgg, *g_ = cached ? c_sg : nullptr;
    ph_stamp<8>(1);
    // (1) fp32 steering: Newton on log mass from the right end a max_p (mu + 8 sigma);
    // bisection once bracketed when a step leaves the bracket, doubling steps while a side
    // is still open
    double lo = -INFINITY, hi = INFINITY, tau = a * (double)tmax, w = 1.0, dxold = INFINITY, mass, dmass, d2mass;
    gauss_mass32<NT>(m_, g_, s_, p0, p1, Lseq, af, beta, (float)tau, mass, dmass, shd, R, gtab, betaf);
    ++n32;
    for (int it = 0; it < 80; ++it) {
        if (mass >= 1.0) lo = tau; else hi = tau;
        double nt = NAN;
        // Newton on log mass (log-concave terms: Gaussian tails and (c - tau)^beta alike are
        // near-quadratic / logarithmic there): tau + mass log(mass) / dmass
        if (dmass > 0.0 && mass > 0.0) nt = tau + mass * log(mass) / dmass;
        const bool closed = lo > -INFINITY && hi < INFINITY;
        // bisect when the step leaves the bracket or does not halve the previous one (a sum
        // of log-concave terms need not be log-concave: no cycling)
        bool newton = true;
        if (!(nt > lo && nt < hi) || (closed && fabs(nt - tau) > 0.5 * dxold)) {
            newton = false;
            if (closed) nt = 0.5 * (lo + hi);
            else { nt = lo > -INFINITY ? lo + w : hi - w; w *= 2.0; }
        }
        // (Newton from one side may converge without ever closing the bracket)
        const bool stop = (newton && fabs(nt - tau) <= 1e-5 * fmax(1.0, fabs(tau))) ||
                          (closed && hi - lo <= 1e-5 * fmax(1.0, fabs(hi)));
        dxold = fabs(nt - tau);
        tau = nt;
        if (stop) break;
        gauss_mass32<NT>(m_, g_, s_, p0, p1, Lseq, af, beta, (float)tau, mass, dmass, shd, R, gtab, betaf);
        ++n32;
    }
    ph_stamp<8>(2);
    // (2) fp64 Halley from the fp32 root
    bool done64 = false;
    {
        double t = tau;
        for (int it = 0; it < 4; ++it) {
            gauss_mass64<NT>(m_, g_, s_, p0, p1, Lseq, af, beta, t, mass, dmass, d2mass, shd, R, gtab, betaf);
            ++n64;
            if (!(dmass > 0.0)) break;
            const double f = mass - 1.0;
            const double den = 2.0 * dmass * dmass - f * d2mass;
            const double step = den > 0.0 ? 2.0 * f * dmass / den : f / dmass;
            if (!(fabs(step) <= 1e-3 * fmax(1.0, fabs(t)))) break;
            t += step;
            const double kq = d2mass / dmass;
            if (kq * kq * fabs(step) * step * step <= 1e-15 * fmax(1.0, fabs(t)) ||
                fabs(step) <= 1e-15 * fmax(1.0, fabs(t))) {
                done64 = true;
                break;
            }
        }
        if (done64) tau = t;
    }
    ph_stamp<8>(3);
    ph_count<8>(0, n32);
    ph_count<8>(1, n64 + (done64 ? 0 : 1000));
    double dl = 1e-4 * fmax(1.0, fabs(tau));
    if (!done64) {
    lo = tau - dl;
    for (int it = 0; it < 200; ++it) {
        gauss_mass64<NT>(m_, g_, s_, p0, p1, Lseq, af, beta, lo, mass, dmass, d2mass, shd, R, gtab, betaf);
        if (mass >= 1.0) break;
        dl *= 4.0; lo = tau - dl;
    }
    double dh = 1e-4 * fmax(1.0, fabs(tau));
    hi = tau + dh;
    for (int it = 0; it < 200; ++it) {
        gauss_mass64<NT>(m_, g_, s_, p0, p1, Lseq, af, beta, hi, mass, dmass, d2mass, shd, R, gtab, betaf);
        if (mass < 1.0) break;
        dh *= 4.0; hi = tau + dh;
    }
    tau = fmin(fmax(tau, lo), hi);
    for (int it = 0; it < 100; ++it) {
        gauss_mass64<NT>(m_, g_, s_, p0, p1, Lseq, af, beta, tau, mass, dmass, d2mass, shd, R, gtab, betaf);
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
    ph_stamp<8>(4);
    // page rule + ordered compaction (NT pages per round) over the slice; the slices' counts
    // are exchanged for the output offsets (rank order = page order)
    int32_t *out = page_idx + (size_t)row * sel_stride;
    __shared__ int x_cnt;
    __shared__ unsigned long long x_best;
    int cnt_local = 0;
    for (int r0 = p0; r0 < p1; r0 += NT) {
        const int p = r0 + threadIdx.x;
        int keep = 0;
        if (p < p1) {
            const int cnt = min(kP, Lseq - p * kP);
            const float sg = __fmaf_rn(g_ ? g_[p - p0] : sqrtf(s_[p - p0]), zq[cnt], m_[p - p0]);
            keep = (a * (double)sg > tau - margin) ? 1 : 0;
        }
        int tot;
        block_excl_scan<NT>(keep, shi, &tot);
        cnt_local += tot;
    }
    int off = 0, total = cnt_local;
    if (CL > 1) {
        cg::cluster_group cl = cg::this_cluster();
        if (threadIdx.x == 0) x_cnt = cnt_local;
        cl.sync();
        total = 0;
        for (int q = 0; q < CL; ++q) {
            const int c = *cl.map_shared_rank(&x_cnt, q);
            if (q < rk) off += c;
            total += c;
        }
    }
    int base = off;
    for (int r0 = p0; r0 < p1; r0 += NT) {
        const int p = r0 + threadIdx.x;
        int keep = 0;
        if (p < p1) {
            const int cnt = min(kP, Lseq - p * kP);
            const float sg = __fmaf_rn(g_ ? g_[p - p0] : sqrtf(s_[p - p0]), zq[cnt], m_[p - p0]);
            keep = (a * (double)sg > tau - margin) ? 1 : 0;
        }
        int tot;
        const int pos = block_excl_scan<NT>(keep, shi, &tot);
        if (keep) out[base + pos] = p;
        base += tot;
    }
    if (total == 0 && M > 0) {
        // argmax mu, lower index on ties (R6), over the whole row
        uint64_t best = 0;
        for (int p = p0 + threadIdx.x; p < p1; p += NT) {
            const uint64_t k = ((uint64_t)f2key(m_[p - p0]) << 32) | (uint32_t)(0xffffffffu - (uint32_t)p);
            best = best > k ? best : k;
        }
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
            x_best = r;
        }
        __syncthreads();
        uint64_t r = x_best;
        if (CL > 1) {
            cg::cluster_group cl = cg::this_cluster();
            cl.sync();
            for (int q = 0; q < CL; ++q) {
                const uint64_t y = *cl.map_shared_rank(&x_best, q);
                r = r > y ? r : y;
            }
        }
        if (rk == 0 && threadIdx.x == 0) out[0] = (int)(0xffffffffu - (uint32_t)(r & 0xffffffffu));
        total = 1;
    }
    if (rk == 0 && threadIdx.x == 0) {
        n_sel[row] = total;
        if (tau_hat_out) tau_hat_out[row] = tau;
    }
    if (CL > 1) cg::this_cluster().sync();   // keep shared memory alive for remote readers
    ph_stamp<8>(5);
}

}  // namespace ekv
