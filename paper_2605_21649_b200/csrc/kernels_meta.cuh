// kernels_meta.cuh -- a0 (append + page statistics) and a1 (page scoring).
#pragma once
#include "common.cuh"
#include <type_traits>

namespace ekv {

// zero a byte range (16-byte aligned, multiple of 16) -- replaces a memset node in the chain
static __global__ void __launch_bounds__(256) k_zero(uint4 *p, size_t n16) {
    pdl_enter();
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n16; i += (size_t)gridDim.x * 256) p[i] = make_uint4(0, 0, 0, 0);
}

// Stored page metadata (R5, R24): bounds in the KV dtype (exact) or e4m3 rounded outward
// (kmin down, kmax up: rd(min_t k_t) = min_t rd(k_t), so incremental and bulk builds agree
// bit for bit); kavg / kvar in fp32 or rounded to nearest-even bf16.
template <typename T>
__device__ __forceinline__ float load_kmin(const CacheView &c, size_t m) {
    return c.bound ? e4m3_to_f(reinterpret_cast<const uint8_t *>(c.kmin)[m]) : Elem<T>::to_f(reinterpret_cast<const T *>(c.kmin)[m]);
}
template <typename T>
__device__ __forceinline__ float load_kmax(const CacheView &c, size_t m) {
    return c.bound ? e4m3_to_f(reinterpret_cast<const uint8_t *>(c.kmax)[m]) : Elem<T>::to_f(reinterpret_cast<const T *>(c.kmax)[m]);
}
template <typename T>
__device__ __forceinline__ void store_meta(const CacheView &c, size_t m, float mn, float mx, float avg, float var) {
    if (c.bound) {
        reinterpret_cast<uint8_t *>(c.kmin)[m] = (uint8_t)e4m3_rd(mn);
        reinterpret_cast<uint8_t *>(c.kmax)[m] = (uint8_t)e4m3_ru(mx);
    } else {
        reinterpret_cast<T *>(c.kmin)[m] = Elem<T>::from_f(mn);
        reinterpret_cast<T *>(c.kmax)[m] = Elem<T>::from_f(mx);
    }
    if (c.stat) {
        reinterpret_cast<__nv_bfloat16 *>(c.kavg)[m] = __float2bfloat16_rn(avg);
        reinterpret_cast<__nv_bfloat16 *>(c.kvar)[m] = __float2bfloat16_rn(var);
    } else {
        reinterpret_cast<float *>(c.kavg)[m] = avg;
        reinterpret_cast<float *>(c.kvar)[m] = var;
    }
}

// ============================================================================ a0: append_kv
// One CTA per sequence; thread (h, i) owns dimension i of kv head h (loops when
// Hkv*D > blockDim).  Token t of the call goes to position L + t.  Statistics are
// updated in append order (R5): kmin/kmax by comparison, ksum += k, ksumsq =
// fma(k, k, ksumsq), kavg = ksum / c, kvar = max(0, ksumsq/c - kavg*kavg), all with
// explicit round-to-nearest intrinsics (no contraction).  seq_lens[b] is bumped after
// a CTA barrier.
template <typename T>
__global__ void __launch_bounds__(1024, 1) k_append(CacheView c, const T *__restrict__ k_new,
                                                 const T *__restrict__ v_new, int n_tokens) {
    EKV_TRACE(0);
    pdl_enter();
    pdl_trigger<0>();
    const int b = blockIdx.x;
    const int L = c.seq_lens[b];
    T *K = reinterpret_cast<T *>(c.Kw);
    T *V = reinterpret_cast<T *>(c.Vw);
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
                mn = load_kmin<T>(c, m); mx = load_kmax<T>(c, m);    // (e4m3: the rounded bound)
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
            store_meta<T>(c, m, mn, mx, avg, var);
            c.ksum[m] = s; c.ksumsq[m] = ss;
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
    EKV_TRACE(10);
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
    store_meta<T>(c, m, mn, mx, avg, var);
    c.ksum[m] = s; c.ksumsq[m] = ss;
}

// ============================================================================ a1: score_pages
// CTA = (chunk of PPC pages) x (sequence b), 256 threads = 16 half-warps.
//  - Thread 0 issues cp.async.bulk (TMA, 1-D) copies of each page's metadata blocks
//    (kmin and kmax: Hkv*d elements each, contiguous in HBM; kavg/kvar for the
//    Gaussian mode) into shared memory, one mbarrier per page, so the whole chunk is
//    in flight at once and no registers hold loads.
//  - Half-warp hw serves kv head hw / (16/Hkv) and pages sub, sub + 16/Hkv, ... of the
//    chunk; lane c owns dims [8c, 8c+8) and keeps q for the G query heads of the group
//    in registers (box: qpos/qneg per dim; Gaussian: q and q*q).  Reading one 256-byte
//    metadata row per half-warp from shared memory is conflict-free.
//  - dot16x8 (R1): per-lane fma chains (packed FFMA2 over head pairs, bit-identical to
//    scalar fmas) + the 16-lane reduce-scatter tree.  Box: max(q_i kmin_i, q_i kmax_i)
//    = q_i kext_i as two fmas with qneg = (q_i >= 0 ? 0 : q_i), qpos = (q_i >= 0 ? q_i
//    : 0): one of the two adds an exact zero, so the chain equals fma(q_i, kext_i, acc).
#ifndef EKV_SCORE_SP
#define EKV_SCORE_SP 8
#endif
#ifndef EKV_SCORE_NS
#define EKV_SCORE_NS 3
#endif
#ifndef EKV_SCORE_E4M3_CTAS
#define EKV_SCORE_E4M3_CTAS 2
#endif
#ifndef EKV_SCORE_E4M3_SP
#define EKV_SCORE_E4M3_SP 16
#endif
template <int MODES, int FMT = 0> struct ScoreCfg {
    // pages per stage: a stage carries about the same bytes whatever the stored form (the
    // ring's bytes in flight, not the page count, set the stream rate): e4m3 bounds = 2x pages
    static constexpr int SP = (MODES == 1) ? ((FMT & 1) ? EKV_SCORE_E4M3_SP : EKV_SCORE_SP)
                                           : ((FMT & 2) ? 8 : 4);
    static constexpr int NS = EKV_SCORE_NS;                      // ring stages
};

// Persistent, warp-specialised (288 threads = 8 consumer warps + 1 producer warp): the
// flattened (b, page) space is split into equal contiguous ranges, one per CTA; the
// producer streams the range's metadata through an NS-deep ring of SP-page stages
// (full/empty mbarriers, no CTA-wide barrier in the loop).
template <typename T, int G, int MODES, int FMT>
__global__ void __launch_bounds__(288, (MODES == 1 && (FMT & 1) && G <= 4 && sizeof(T) == 2) ? EKV_SCORE_E4M3_CTAS
                                       : (G <= 4 && MODES != 3) ? 2 : 1) k_score(CacheView c, const T *__restrict__ q, int Hq,
                                                   float *__restrict__ box, float *__restrict__ mu,
                                                   float *__restrict__ sigma2, uint4 *__restrict__ zero,
                                                   size_t zero_n16) {
    EKV_TRACE(1);
    // decode's per-step counters / union mask (read by the later kernels of the step) are
    // zeroed here, one slice per CTA -- no separate launch.  Their last readers ran two or more
    // launches back (pdl_enter invariant), so this runs before the wait.
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < zero_n16; i += (size_t)gridDim.x * blockDim.x)
        zero[i] = make_uint4(0, 0, 0, 0);
    pdl_enter();
    pdl_trigger<1>();
    constexpr int SP = ScoreCfg<MODES, FMT>::SP, NS = ScoreCfg<MODES, FMT>::NS;
    constexpr int NCW = 8;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t fullb[NS], emptyb[NS];
    __shared__ int d_b[NS], d_p0[NS], d_n[NS];
    __shared__ int l_phys[512];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long total = (long long)c.B * c.maxp;
    const long long r0 = total * blockIdx.x / gridDim.x, r1 = total * (blockIdx.x + 1) / gridDim.x;
    stamp_cta<2>(threadIdx.x == 0, 0);
    const int HD = c.Hkv * kD;
    constexpr bool BE = (FMT & 1) != 0;                       // e4m3 bounds (R24)
    constexpr bool SB = (FMT & 2) != 0;                       // bf16 kavg / kvar
    const uint32_t bmm = (uint32_t)(HD * (BE ? 1 : sizeof(T)));   // kmin / kmax block bytes
    const uint32_t bgs = (uint32_t)(HD * (SB ? 2 : 4));           // kavg / kvar block bytes
    const uint32_t per_page = ((MODES & 1) ? 2 * bmm : 0) + ((MODES & 2) ? 2 * bgs : 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&fullb[i], 1); mbar_init(&emptyb[i], NCW); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NCW) {
        // ------------------------------------------------ producer
        // The range is processed in chunks of 512 (b, page) slots: the warp first loads the
        // chunk's page-table entries into shared memory (16 independent loads per lane),
        // then lane 0 packs runs of valid pages (one sequence at a time) into ring stages.
        int si = 0;
        // (b, page) of the chunk start, advanced incrementally (no 64-bit divisions in the loop)
        int cb_b = (int)(r0 / c.maxp), cb_p = (int)(r0 % c.maxp);
        // the first chunk is short (64 slots: the first copies go out after one round trip);
        // page-table entry and sequence length are loaded together and masked afterwards
        for (long long cb = r0; cb < r1;) {
            const int nchk = (int)min((long long)(cb == r0 ? 64 : 512), r1 - cb);
#pragma unroll 4
            for (int i = lane; i < nchk; i += 32) {
                int bb = cb_b, p = cb_p + i;
                while (p >= c.maxp) { p -= c.maxp; ++bb; }
                const int ph = __ldg(c.page_table + (size_t)bb * c.maxp + p);
                l_phys[i] = (p < n_pages_of(__ldg(c.seq_lens + bb))) ? ph : -1;
            }
            __syncwarp();
            {
                // every lane walks the same runs (l_phys reads are broadcasts); lane 0 owns
                // the mbarrier protocol, and the stage's copies are issued one per lane
                constexpr int CPP = ((MODES & 1) ? 2 : 0) + ((MODES & 2) ? 2 : 0);   // copies per page
                int i = 0, bb = cb_b, p0 = cb_p;           // (bb, p0) tracks chunk slot i
                while (i < nchk) {
                    if (l_phys[i] < 0) {                   // past the sequence end
                        ++i;
                        if (++p0 == c.maxp) { p0 = 0; ++bb; }
                        continue;
                    }
                    // run length: leading valid slots of [i, i + SP) (one ballot, not a serial scan)
                    const bool vv = lane < SP && i + lane < nchk && l_phys[i + lane] >= 0 && p0 + lane < c.maxp;
                    const unsigned vb = __ballot_sync(0xffffffffu, vv);
                    const int n = min(SP, __ffs((int)~vb) - 1 < 0 ? 32 : __ffs((int)~vb) - 1);
                    const int slot = si % NS;
                    if (lane == 0) {
                        if (si >= NS) mbar_wait(&emptyb[slot], ((si / NS) - 1) & 1);
                        d_b[slot] = bb; d_p0[slot] = p0; d_n[slot] = n;
                        mbar_expect_tx(&fullb[slot], n * per_page);
                    }
                    __syncwarp();
                    for (int e = lane; e < n * CPP; e += 32) {
                        const int k = e / CPP, w = e - k * CPP;
                        const size_t phys = (size_t)l_phys[i + k];
                        unsigned char *dst = smem + ((size_t)slot * SP + k) * per_page;
                        if (MODES & 1) {
                            if (w == 0) bulk_g2s_stream(dst, reinterpret_cast<const unsigned char *>(c.kmin) + phys * bmm, bmm, &fullb[slot]);
                            if (w == 1) bulk_g2s_stream(dst + bmm, reinterpret_cast<const unsigned char *>(c.kmax) + phys * bmm, bmm, &fullb[slot]);
                            dst += 2 * bmm;
                        }
                        if (MODES & 2) {
                            const int w2 = w - ((MODES & 1) ? 2 : 0);
                            if (w2 == 0) bulk_g2s_stream(dst, reinterpret_cast<const unsigned char *>(c.kavg) + phys * bgs, bgs, &fullb[slot]);
                            if (w2 == 1) bulk_g2s_stream(dst + bgs, reinterpret_cast<const unsigned char *>(c.kvar) + phys * bgs, bgs, &fullb[slot]);
                        }
                    }
                    ++si;
                    i += n;
                    p0 += n;
                    if (p0 >= c.maxp) { p0 -= c.maxp; ++bb; }
                }
            }
            __syncwarp();
            cb += nchk;
            cb_p += nchk;
            while (cb_p >= c.maxp) { cb_p -= c.maxp; ++cb_b; }
        }
        if (lane == 0) {
            const int slot = si % NS;           // end marker
            if (si >= NS) mbar_wait(&emptyb[slot], ((si / NS) - 1) & 1);
            d_n[slot] = -1;
            mbar_arrive(&fullb[slot]);
        }
        return;
    }
    // ---------------------------------------------------- consumers
    const int l16 = threadIdx.x & 15;
    const int hw = threadIdx.x >> 4;
    const int hwpk = 16 / c.Hkv;
    const int kvh = hw / hwpk, sub = hw % hwpk;
    const int hq0 = kvh * G;
    if constexpr (MODES == 1 && sizeof(T) == 2 && !BE) {
        // Box, bf16: lane c keeps q's 4 bf16x2 words of its chunk per head and the PRMT
        // selectors picking kext_i = (q_i >= 0 ? kmax_i : kmin_i) bytewise from the packed
        // kmax/kmin words (R1's kext exactly, -0 counted as >= 0); the chain is FHFMA.BF16
        // on packed words (exact widening, fma_bf16lo).  IPR items per 16-lane reduce-scatter.
        constexpr int IPR = (16 / G) < 4 ? 16 / G : 4;
        constexpr int V = IPR * G;
        uint32_t qw[G][4], sel[G][4];
        int cur_b = -1;
        for (int si = 0;; ++si) {
            const int slot = si % NS;
            mbar_wait(&fullb[slot], (si / NS) & 1);
            const int n = d_n[slot];
            stamp_cta<2>(threadIdx.x == 0 && si == 0, 1);
            stamp_if(threadIdx.x == 0 && si < 16, 4, si);
            if (n < 0) { stamp_cta<2>(threadIdx.x == 0, 2); count_cta<2>(threadIdx.x == 0, si); break; }
            const int bb = d_b[slot], q0 = d_p0[slot];
            if (bb != cur_b) {
                cur_b = bb;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(q + ((size_t)bb * Hq + hq0 + g) * kD + 8 * l16));
                    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        qw[g][j] = ws[j];
                        const bool plo = __uint_as_float(ws[j] << 16) >= 0.0f;
                        const bool phi = __uint_as_float(ws[j] & 0xffff0000u) >= 0.0f;
                        sel[g][j] = (plo ? 0x10u : 0x54u) | ((phi ? 0x32u : 0x76u) << 8);
                    }
                }
            }
            bool released = false;
            for (int ib = 0; ib < n; ib += IPR * hwpk) {
                // all of the group's metadata words to registers first; the last group of
                // the stage then releases the ring slot before computing, so the producer
                // refills it while the FHFMA chains run
                uint32_t wn[IPR][4], wx[IPR][4];
#pragma unroll
                for (int j = 0; j < IPR; ++j) {
                    const int it = ib + sub + j * hwpk;
                    const unsigned char *pg = smem + ((size_t)slot * SP + (it < n ? it : 0)) * per_page;
                    const uint4 mn = *reinterpret_cast<const uint4 *>(pg + (size_t)(kvh * kD + 8 * l16) * 2);
                    const uint4 mx = *reinterpret_cast<const uint4 *>(pg + bmm + (size_t)(kvh * kD + 8 * l16) * 2);
                    wn[j][0] = mn.x; wn[j][1] = mn.y; wn[j][2] = mn.z; wn[j][3] = mn.w;
                    wx[j][0] = mx.x; wx[j][1] = mx.y; wx[j][2] = mx.z; wx[j][3] = mx.w;
                }
                if (ib + IPR * hwpk >= n) {                  // warp-uniform
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&emptyb[slot]);
                    released = true;
                }
                float acc[V];
#pragma unroll
                for (int j = 0; j < IPR; ++j) {
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        float a = 0.0f;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint32_t ke = prmt(wx[j][e], wn[j][e], sel[g][e]);
                            a = fma_bf16lo(qw[g][e], ke, a);
                            a = fma_bf16hi(qw[g][e], ke, a);
                        }
                        acc[j * G + g] = a;
                    }
                }
                const float r = __fmul_rn(rs_reduce16<V>(acc, lane), kCd);
                const int vv = rs_head<V>(lane);
                const int it = ib + sub + (vv / G) * hwpk, hh = vv % G;
                if (rs_writer<V>(lane) && it < n)
                    box[((size_t)bb * Hq + hq0 + hh) * c.maxp + q0 + it] = r;
            }
            if (!released) {                                 // no group (n <= sub): release now
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyb[slot]);
            }
            stamp_if(threadIdx.x == 0 && si < 16, 4, 16 + si);
        }
        return;
    }
    if constexpr (MODES == 1 && sizeof(T) == 2 && BE) {
        // Box, e4m3 bounds (R24), bf16 q: lane c unpacks its chunk's 8 kmin and 8 kmax bytes to
        // f16x2 (F2FP, exact) and runs R1's chain as FHFMA with f16 operands on the PRMT-selected
        // kext -- exact products, so bit-identical to fmaf(q_i, kext_i, acc).  q is converted to
        // f16 once per sequence; a lane whose q chunk is not exactly representable in f16
        // (|q_i| < 2^-17 or > 65504) runs the same chain in fp32 instead (same bits).
        constexpr int IPR = (16 / G) < 2 ? 16 / G : 2;
        constexpr int V = IPR * G;
        uint32_t qh[G][4], sel[G][4];
        bool qexact = true;
        int cur_b = -1;
        for (int si = 0;; ++si) {
            const int slot = si % NS;
            mbar_wait(&fullb[slot], (si / NS) & 1);
            const int n = d_n[slot];
            stamp_cta<2>(threadIdx.x == 0 && si == 0, 1);
            stamp_if(threadIdx.x == 0 && si < 16, 4, si);
            if (n < 0) { stamp_cta<2>(threadIdx.x == 0, 2); count_cta<2>(threadIdx.x == 0, si); break; }
            const int bb = d_b[slot], q0 = d_p0[slot];
            if (bb != cur_b) {
                cur_b = bb;
                qexact = true;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(q + ((size_t)bb * Hq + hq0 + g) * kD + 8 * l16));
                    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        qh[g][j] = bf2_to_h2(ws[j], qexact);
                        const bool plo = __uint_as_float(ws[j] << 16) >= 0.0f;
                        const bool phi = __uint_as_float(ws[j] & 0xffff0000u) >= 0.0f;
                        sel[g][j] = (plo ? 0x10u : 0x54u) | ((phi ? 0x32u : 0x76u) << 8);
                    }
                }
            }
            bool released = false;
            for (int ib = 0; ib < n; ib += IPR * hwpk) {
                uint32_t wn[IPR][4], wx[IPR][4];
#pragma unroll
                for (int j = 0; j < IPR; ++j) {
                    const int it = ib + sub + j * hwpk;
                    const unsigned char *pg = smem + ((size_t)slot * SP + (it < n ? it : 0)) * per_page;
                    const uint2 mn = *reinterpret_cast<const uint2 *>(pg + kvh * kD + 8 * l16);
                    const uint2 mx = *reinterpret_cast<const uint2 *>(pg + bmm + kvh * kD + 8 * l16);
                    wn[j][0] = mn.x; wn[j][1] = mn.y; wx[j][0] = mx.x; wx[j][1] = mx.y;
                }
                if (ib + IPR * hwpk >= n) {                  // warp-uniform
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&emptyb[slot]);
                    released = true;
                }
#pragma unroll
                for (int j = 0; j < IPR; ++j) {              // 8 bytes -> 4 f16x2 words per bound
                    const uint32_t a0 = wn[j][0], a1 = wn[j][1], b0 = wx[j][0], b1 = wx[j][1];
                    wn[j][0] = e4m3x2_to_h2(a0); wn[j][1] = e4m3x2_to_h2(a0 >> 16);
                    wn[j][2] = e4m3x2_to_h2(a1); wn[j][3] = e4m3x2_to_h2(a1 >> 16);
                    wx[j][0] = e4m3x2_to_h2(b0); wx[j][1] = e4m3x2_to_h2(b0 >> 16);
                    wx[j][2] = e4m3x2_to_h2(b1); wx[j][3] = e4m3x2_to_h2(b1 >> 16);
                }
                float acc[V];
                if (qexact) {
#pragma unroll
                    for (int j = 0; j < IPR; ++j) {
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            float a = 0.0f;
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const uint32_t ke = prmt(wx[j][e], wn[j][e], sel[g][e]);
                                a = fma_h_lo(qh[g][e], ke, a);
                                a = fma_h_hi(qh[g][e], ke, a);
                            }
                            acc[j * G + g] = a;
                        }
                    }
                } else {                                     // rare: the fp32 chain (q re-read from L1)
#pragma unroll
                    for (int j = 0; j < IPR; ++j) {
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const uint4 qq = __ldg(reinterpret_cast<const uint4 *>(q + ((size_t)bb * Hq + hq0 + g) * kD + 8 * l16));
                            const uint32_t qb[4] = {qq.x, qq.y, qq.z, qq.w};
                            float a = 0.0f;
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const uint32_t ke = prmt(wx[j][e], wn[j][e], sel[g][e]);
                                const float2 kf = __half22float2(*reinterpret_cast<const __half2 *>(&ke));
                                a = __fmaf_rn(__uint_as_float(qb[e] << 16), kf.x, a);
                                a = __fmaf_rn(__uint_as_float(qb[e] & 0xffff0000u), kf.y, a);
                            }
                            acc[j * G + g] = a;
                        }
                    }
                }
                const float r = __fmul_rn(rs_reduce16<V>(acc, lane), kCd);
                const int vv = rs_head<V>(lane);
                const int it = ib + sub + (vv / G) * hwpk, hh = vv % G;
                if (rs_writer<V>(lane) && it < n)
                    box[((size_t)bb * Hq + hq0 + hh) * c.maxp + q0 + it] = r;
            }
            if (!released) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyb[slot]);
            }
            stamp_if(threadIdx.x == 0 && si < 16, 4, 16 + si);
        }
        return;
    }
    constexpr int GP = (G + 1) / 2;          // head pairs
    float2 qp[GP][8], qn[GP][8], qa[GP][8], q2[GP][8];
    int cur_b = -1;
    for (int si = 0;; ++si) {
        const int slot = si % NS;
        mbar_wait(&fullb[slot], (si / NS) & 1);
        const int n = d_n[slot];
        stamp_if(threadIdx.x == 0 && si < 16, 4, si);
        if (n < 0) break;
        const int bb = d_b[slot], q0 = d_p0[slot];
        if (bb != cur_b) {
            cur_b = bb;
#pragma unroll
            for (int g = 0; g < GP; ++g) {
                float x0[8], x1[8];
                Elem<T>::load8(q + ((size_t)bb * Hq + hq0 + 2 * g) * kD + 8 * l16, x0);
                if (2 * g + 1 < G) Elem<T>::load8(q + ((size_t)bb * Hq + hq0 + 2 * g + 1) * kD + 8 * l16, x1);
                else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) x1[i] = 0.0f;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (MODES & 1) {
                        qp[g][i] = make_float2(x0[i] >= 0.0f ? x0[i] : 0.0f, x1[i] >= 0.0f ? x1[i] : 0.0f);
                        qn[g][i] = make_float2(x0[i] >= 0.0f ? 0.0f : x0[i], x1[i] >= 0.0f ? 0.0f : x1[i]);
                    }
                    if (MODES & 2) {
                        qa[g][i] = make_float2(x0[i], x1[i]);
                        q2[g][i] = make_float2(__fmul_rn(x0[i], x0[i]), __fmul_rn(x1[i], x1[i]));
                    }
                }
            }
        }
        // two items (pages) per iteration, interleaved; the 2G partials go through one
        // 16-lane reduce-scatter (same pairing tree per value: bit-identical to per-item)
        for (int ib = 0; ib < n; ib += 2 * hwpk) {
            const int i0 = ib + sub, i1 = ib + sub + hwpk;
            const bool v0 = i0 < n, v1 = i1 < n;
            const unsigned char *pg0 = smem + ((size_t)slot * SP + (v0 ? i0 : 0)) * per_page;
            const unsigned char *pg1 = smem + ((size_t)slot * SP + (v1 ? i1 : 0)) * per_page;
            if (MODES & 1) {
                float mn0[8], mx0[8], mn1[8], mx1[8];
                if constexpr (BE) {                           // e4m3 -> fp32 (exact; F2FP unpack)
                    load8_e4m3(pg0 + kvh * kD + 8 * l16, mn0);
                    load8_e4m3(pg0 + bmm + kvh * kD + 8 * l16, mx0);
                    load8_e4m3(pg1 + kvh * kD + 8 * l16, mn1);
                    load8_e4m3(pg1 + bmm + kvh * kD + 8 * l16, mx1);
                } else {
                    Elem<T>::load8(reinterpret_cast<const T *>(pg0) + kvh * kD + 8 * l16, mn0);
                    Elem<T>::load8(reinterpret_cast<const T *>(pg0 + bmm) + kvh * kD + 8 * l16, mx0);
                    Elem<T>::load8(reinterpret_cast<const T *>(pg1) + kvh * kD + 8 * l16, mn1);
                    Elem<T>::load8(reinterpret_cast<const T *>(pg1 + bmm) + kvh * kD + 8 * l16, mx1);
                }
                float acc[2 * G];
#pragma unroll
                for (int g = 0; g < GP; ++g) {
                    float2 a0 = make_float2(0.0f, 0.0f), a1 = make_float2(0.0f, 0.0f);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        a0 = ffma2(qn[g][e], mn0[e], a0);
                        a1 = ffma2(qn[g][e], mn1[e], a1);
                        a0 = ffma2(qp[g][e], mx0[e], a0);
                        a1 = ffma2(qp[g][e], mx1[e], a1);
                    }
                    acc[2 * g] = a0.x; acc[G + 2 * g] = a1.x;
                    if (2 * g + 1 < G) { acc[2 * g + 1] = a0.y; acc[G + 2 * g + 1] = a1.y; }
                }
                const float r = __fmul_rn(rs_reduce16<2 * G>(acc, lane), kCd);
                const int vv = rs_head<2 * G>(lane);
                const int it = vv / G, hh = vv % G;
                if (rs_writer<2 * G>(lane) && (it ? v1 : v0))
                    box[((size_t)bb * Hq + hq0 + hh) * c.maxp + q0 + (it ? i1 : i0)] = r;
            }
            if (MODES & 2) {
                const unsigned char *ps0 = pg0 + ((MODES & 1) ? 2 * bmm : 0);
                const unsigned char *ps1 = pg1 + ((MODES & 1) ? 2 * bmm : 0);
                float av0[8], vr0[8], av1[8], vr1[8];
                using ST = typename std::conditional<SB, __nv_bfloat16, float>::type;   // exact widening
                Elem<ST>::load8(reinterpret_cast<const ST *>(ps0) + kvh * kD + 8 * l16, av0);
                Elem<ST>::load8(reinterpret_cast<const ST *>(ps0 + bgs) + kvh * kD + 8 * l16, vr0);
                Elem<ST>::load8(reinterpret_cast<const ST *>(ps1) + kvh * kD + 8 * l16, av1);
                Elem<ST>::load8(reinterpret_cast<const ST *>(ps1 + bgs) + kvh * kD + 8 * l16, vr1);
                float am[2 * G], as[2 * G];
#pragma unroll
                for (int g = 0; g < GP; ++g) {
                    float2 m0 = make_float2(0.0f, 0.0f), s0 = make_float2(0.0f, 0.0f);
                    float2 m1 = make_float2(0.0f, 0.0f), s1 = make_float2(0.0f, 0.0f);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        m0 = ffma2(qa[g][e], av0[e], m0);
                        s0 = ffma2(q2[g][e], vr0[e], s0);
                        m1 = ffma2(qa[g][e], av1[e], m1);
                        s1 = ffma2(q2[g][e], vr1[e], s1);
                    }
                    am[2 * g] = m0.x; as[2 * g] = s0.x; am[G + 2 * g] = m1.x; as[G + 2 * g] = s1.x;
                    if (2 * g + 1 < G) {
                        am[2 * g + 1] = m0.y; as[2 * g + 1] = s0.y;
                        am[G + 2 * g + 1] = m1.y; as[G + 2 * g + 1] = s1.y;
                    }
                }
                const float rm = __fmul_rn(rs_reduce16<2 * G>(am, lane), kCd);
                const float rs = __fmul_rn(rs_reduce16<2 * G>(as, lane), 1.0f / (float)kD);
                const int vv = rs_head<2 * G>(lane);
                const int it = vv / G, hh = vv % G;
                if (rs_writer<2 * G>(lane) && (it ? v1 : v0)) {
                    const size_t o = ((size_t)bb * Hq + hq0 + hh) * c.maxp + q0 + (it ? i1 : i0);
                    mu[o] = rm;
                    sigma2[o] = rs;
                }
            }
        }
        __syncwarp();
        stamp_if(threadIdx.x == 0 && si < 16, 4, 16 + si);
        if (lane == 0) mbar_arrive(&emptyb[slot]);
    }
}

}  // namespace ekv
