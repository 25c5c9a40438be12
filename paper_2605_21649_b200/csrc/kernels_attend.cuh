// kernels_attend.cuh -- a3/a5/a6: token scores over the selected pages (TMA bulk
// copies of K tiles into shared memory), candidate extraction, exact alpha-entmax
// threshold + support, and the weighted V sum over the support.
#pragma once
#include "common.cuh"
#include <cooperative_groups.h>

namespace ekv {

// Score rows are indexed by token position: scores[b][h][j], j = page * P + t, over
// the whole sequence capacity (max_pages * P); only tokens of pages selected by head h
// are written.  rowmax[b][h] holds the ordered-int max score (atomicMax; 0 = empty).

// ============================================================================ K scores
// Persistent, warp-specialised: 288 threads = 8 consumer warps + 1 producer warp,
// 2 CTAs per SM (bf16).  The flattened work space (sparse: (row, i) over the page lists,
// each union page kept once -- from its lowest selecting head; full: (unit, page)) is
// split into equal contiguous ranges, one per CTA.
//  - Producer warp: collects the range's pages (page-table and union-mask lookups in
//    parallel), packs them into ring stages of SP = 8 pages and issues one
//    cp.async.bulk (TMA, 1-D) copy per page of the contiguous tile K[phys][kvh][0..P)[0..d)
//    completing on the stage's `full` mbarrier, after writing the stage's work items:
//    one (page, head) item per head of the unit whose union-mask bit is set (sparse:
//    ~1.1 items per page -- only heads that selected the page are scored; full: G).
//    It waits on the stage's `empty` mbarrier before reuse.  n = -1 ends.  (Per-row
//    copies into a padded layout were tried: 16 small copies per page are TMA-issue
//    bound, ~2x slower.)
//  - Consumers: a half-warp scores one item, lane = token t, computing dot16x8 (R1)
//    in registers: 16 independent chunk chains (bf16: FHFMA.BF16 straight from the
//    packed K and q words, no unpacking -- exact, see fma_bf16lo) and the pairwise tree
//    c+(c+8), c+(c+4), c+(c+2), c0+c1.  Bank conflicts: lane t handles chunk c ^ (t & 7)
//    in register slot c, so 8 consecutive lanes (rows 256 B apart) read 8 distinct 16-byte
//    bank groups; XOR-relabelling with s < 8 maps the butterfly's pairs (x, x+2^j) onto
//    themselves and fp add commutes, so slot 0 ends bit-identical to R1's tree.  q of the
//    item's unit (G heads) is cached per half-warp in shared memory.  s = fl32(dot * c_d)
//    (R2); -inf past seq_len; a half-warp stores 16 consecutive scores (64 B); one
//    atomicMax per item into rowmax.
#ifndef EKV_ATT_NCW
#define EKV_ATT_NCW 8
#endif
#ifndef EKV_ATT_NS
#define EKV_ATT_NS 3
#endif
#ifndef EKV_ATT_SP
#define EKV_ATT_SP 8
#endif
template <typename T> struct AttCfg {
    static constexpr int NCW = EKV_ATT_NCW;                // consumer warps (16 half-warps >= items per stage, usually)
    static constexpr int SP = EKV_ATT_SP;                  // pages per stage (item code: 3 bits)
    static constexpr int NS = sizeof(T) == 2 ? EKV_ATT_NS : 2;   // ring stages
    static constexpr int TILE = kP * kD * (int)sizeof(T);
    static constexpr int RING = NS * SP * TILE;
    template <int G> static constexpr int smem() { return RING + NCW * G * kD * (int)sizeof(T); }  // + q cache
};

template <typename T, int G>
__global__ void __launch_bounds__(32 * (AttCfg<T>::NCW + 1), sizeof(T) == 2 ? 2 : 1) k_attend_scores(
    CacheView c, const T *__restrict__ q, int Hq, const uint32_t *__restrict__ umask, int W,
    const int32_t *__restrict__ page_idx, const int32_t *__restrict__ n_sel, int stride,
    float *__restrict__ scores, uint32_t *__restrict__ rowmax, int full) {
    EKV_TRACE(4);
    pdl_enter();
    pdl_trigger<4>();
    ph_stamp<4>(0);
    constexpr int SP = AttCfg<T>::SP, NS = AttCfg<T>::NS, TILE = AttCfg<T>::TILE;
    constexpr int NCW = AttCfg<T>::NCW;
    constexpr int CHK = 256;                // work slots per producer chunk (8 per lane)
    extern __shared__ __align__(128) unsigned char smem[];   // [NS][SP][TILE]
    __shared__ uint64_t fullb[NS], emptyb[NS];
    __shared__ int d_page[NS][SP], d_unit[NS][SP], d_phys[NS][SP], d_n[NS], d_ni[NS];
    __shared__ uint8_t d_mask[NS][SP], d_items[NS][SP * G];
    __shared__ int l_unit[CHK], l_page[CHK], l_phys[CHK];
    __shared__ uint8_t l_mask[CHK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    stamp_cta<1>(threadIdx.x == 0, 0);
    const int ucap = full ? c.maxp : stride;
    // sparse rows: the work space is the concatenation of the rows' actual lists (prefix sums
    // of n_sel, computed by every producer), so CTAs get equal numbers of pages whatever the
    // list lengths (Gaussian selection: variable, often far below the capacity)
    constexpr int kMaxRowsBal = 1024;
    __shared__ int pref[kMaxRowsBal + 1];
    const int nrows = c.B * Hq;
    const bool bal = !full && nrows <= kMaxRowsBal;
    long long tot = full ? (long long)c.B * c.Hkv * c.maxp : (long long)c.B * Hq * stride;
    if (bal && warp == NCW) {
        // rows lane + 32 i: every n_sel load in flight at once, then a warp scan per 32 rows
        constexpr int MAXPER = kMaxRowsBal / 32;
        int v[MAXPER];
#pragma unroll
        for (int i = 0; i < MAXPER; ++i) {
            const int r = lane + 32 * i;
            v[i] = (r < nrows) ? __ldg(n_sel + r) : 0;
        }
        int carry = 0;
#pragma unroll
        for (int i = 0; i < MAXPER; ++i) {
            if (32 * i >= nrows) break;
            int incl = v[i];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += y; }
            const int r = lane + 32 * i;
            if (r < nrows) pref[r] = carry + incl - v[i];
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) pref[nrows] = carry;
        __syncwarp();
        tot = pref[nrows];
        ph_stamp_if<4>(lane == 0, 1);
    }
    // the CTA's range of the flattened work space (32-bit arithmetic when it fits: the 64-bit
    // division sequence sits on the producer's critical path)
    long long f0, f1;
    if (tot * ((long long)gridDim.x + 1) < (1ll << 32)) {
        const unsigned t32 = (unsigned)tot;
        f0 = (long long)(t32 * blockIdx.x / gridDim.x);
        f1 = (long long)(t32 * (blockIdx.x + 1) / gridDim.x);
    } else {
        f0 = tot * blockIdx.x / gridDim.x;
        f1 = tot * (blockIdx.x + 1) / gridDim.x;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&fullb[i], 1); mbar_init(&emptyb[i], NCW); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NCW) {
        // ------------------------------------------------ producer
        ph_stamp_if<4>(lane == 0, 7);
        const unsigned char *Kb = reinterpret_cast<const unsigned char *>(c.K);
        int si = 0, fill = 0;
        const int hkv = c.Hkv;
        const float inv_hq = 1.0f / (float)Hq, inv_hkv = 1.0f / (float)hkv;
        // The producer is one warp: its index arithmetic is latency, not throughput -- no integer
        // divisions by runtime values (27 of them, and a per-element row search, cost ~7500
        // cycles before the first copy) and every round of loads in flight at once.
        int cu = 0, cs = 0, urow = 0;        // unbalanced: (row or unit, slot) of the chunk start; balanced: lane's row
        if (bal) {                           // row of the range start: fixed-depth search (warp-uniform)
            int lo = 0;
#pragma unroll
            for (int stp = kMaxRowsBal / 2; stp > 0; stp >>= 1) {
                const int m = lo + stp;
                lo = (m < nrows && pref[m] <= f0) ? m : lo;
            }
            urow = lo;
        } else {
            cu = (int)(f0 / ucap);
            cs = (int)(f0 - (long long)cu * ucap);
        }
        for (long long cb = f0; cb < f1; cb += CHK) {
            const int nr = (int)min((long long)CHK, f1 - cb);      // elements of this chunk
            int un[CHK / 32], pg[CHK / 32], hg[CHK / 32], rw[CHK / 32], pb[CHK / 32];
            bool ok[CHK / 32];
#pragma unroll
            for (int r = 0; r < CHK / 32; ++r) {
                int u = 0, sl = 0;
                ok[r] = r * 32 + lane < nr;
                if (r * 32 < nr) {                                  // warp-uniform
                    if (bal) {
                        const int e = (int)cb + r * 32 + lane;
                        while (urow + 1 < nrows && pref[urow + 1] <= e) ++urow;   // (rows are long: ~never)
                        u = urow;
                        sl = e - pref[u];
                    } else {
                        u = cu;
                        sl = cs + r * 32 + lane;
                        while (sl >= ucap) { sl -= ucap; ++u; }
                    }
                }
                const int bb = qdiv_small(u, full ? hkv : Hq, full ? inv_hkv : inv_hq);   // u: full -> unit; sparse -> row
                const int hr = u - bb * Hq;
                rw[r] = u;
                pb[r] = bb;
                un[r] = full ? u : bb * hkv + hr / G;
                hg[r] = full ? 0 : hr % G;
                pg[r] = sl;
            }
            if (!bal) {
                cs += CHK;
                while (cs >= ucap) { cs -= ucap; ++cu; }
                int lim[CHK / 32];                       // unbalanced rows / full: the row bound first
#pragma unroll
                for (int r = 0; r < CHK / 32; ++r)
                    lim[r] = ok[r] ? __ldg(full ? c.seq_lens + pb[r] : n_sel + rw[r]) : 0;
#pragma unroll
                for (int r = 0; r < CHK / 32; ++r) ok[r] = ok[r] && pg[r] < (full ? n_pages_of(lim[r]) : lim[r]);
            }
            if (!full) {
#pragma unroll
                for (int r = 0; r < CHK / 32; ++r) pg[r] = ok[r] ? __ldg(page_idx + (size_t)rw[r] * stride + pg[r]) : 0;
            }
            ph_stamp_if<4>(lane == 0 && cb == f0 && pg[0] >= 0, 2);
            int ph[CHK / 32];
            uint8_t mk[CHK / 32];
#pragma unroll
            for (int r = 0; r < CHK / 32; ++r) {
                ph[r] = ok[r] ? __ldg(c.page_table + (size_t)pb[r] * c.maxp + pg[r]) : 0;
                mk[r] = full ? (uint8_t)((1u << G) - 1u)
                             : ok[r] ? (uint8_t)((__ldg(umask + (size_t)un[r] * W + (pg[r] >> 2)) >> ((pg[r] & 3) * 8)) & 0xffu)
                                     : (uint8_t)0;
            }
            ph_stamp_if<4>(lane == 0 && cb == f0 && ph[0] >= 0 && mk[0] < 255, 3);
#pragma unroll
            for (int r = 0; r < CHK / 32; ++r)      // keep each union page once: lowest selecting head
                if (ok[r] && !full && (__ffs((int)mk[r]) - 1) != hg[r]) ok[r] = false;
            int nl = 0;
#pragma unroll
            for (int r = 0; r < CHK / 32; ++r) {
                const unsigned bal = __ballot_sync(0xffffffffu, ok[r]);
                if (ok[r]) {
                    const int pos = nl + __popc(bal & ((1u << lane) - 1u));
                    l_unit[pos] = un[r]; l_page[pos] = pg[r]; l_phys[pos] = ph[r]; l_mask[pos] = mk[r];
                }
                nl += __popc(bal);
            }
            __syncwarp();
            for (int i = 0; i < nl;) {              // warp-uniform; up to SP pages per iteration
                const int slot = si % NS;
                if (fill == 0) {
                    if (lane == 0 && si >= NS) mbar_wait(&emptyb[slot], ((si / NS) - 1) & 1);
                    __syncwarp();
                }
                const int cnt = min(SP - fill, nl - i);
                if (lane < cnt) {                       // lane-parallel stage entries
                    d_unit[slot][fill + lane] = l_unit[i + lane]; d_page[slot][fill + lane] = l_page[i + lane];
                    d_mask[slot][fill + lane] = l_mask[i + lane]; d_phys[slot][fill + lane] = l_phys[i + lane];
                }
                i += cnt;
                fill += cnt;
                if (fill == SP) {
                    __syncwarp();
                    // items (page k, head g) in page order: lane k writes its page's heads at
                    // the prefix of the head counts (full: every (page, head), codes computed
                    // by the consumers)
                    int ni = SP * G;
                    if (!full) {
                        const unsigned m = lane < SP ? (unsigned)d_mask[slot][lane] : 0u;
                        int incl = __popc(m);
#pragma unroll
                        for (int o = 1; o < 8; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += y; }
                        int off = incl - __popc(m);
                        for (unsigned mm = m; mm; mm &= mm - 1u) d_items[slot][off++] = (uint8_t)(lane * 8 + __ffs((int)mm) - 1);
                        ni = __shfl_sync(0xffffffffu, incl, SP - 1);
                        __syncwarp();                  // the lanes' d_items stores before lane 0's release
                    }
                    if (lane == 0) {
                        d_n[slot] = SP;
                        d_ni[slot] = ni;
                        mbar_expect_tx(&fullb[slot], (uint32_t)(SP * TILE));
                    }
                    __syncwarp();
                    if (lane < SP)
                        bulk_g2s_stream(smem + ((size_t)slot * SP + lane) * TILE,
                                 Kb + ((size_t)d_phys[slot][lane] * hkv + (d_unit[slot][lane] - qdiv_small(d_unit[slot][lane], hkv, inv_hkv) * hkv)) * TILE,
                                 TILE, &fullb[slot]);
                    ph_stamp_if<4>(lane == 0 && si == 0, 4);
                    ++si;
                    fill = 0;
                }
            }
            __syncwarp();
        }
        if (fill > 0) {
            const int slot = si % NS;
            __syncwarp();
            if (lane == 0) {
                d_n[slot] = fill;
                int ni = fill * G;
                if (!full) {
                    ni = 0;
                    for (int kk = 0; kk < fill; ++kk)
                        for (unsigned m = d_mask[slot][kk]; m; m &= m - 1u) d_items[slot][ni++] = (uint8_t)(kk * 8 + __ffs((int)m) - 1);
                }
                d_ni[slot] = ni;
                mbar_expect_tx(&fullb[slot], (uint32_t)(fill * TILE));
            }
            __syncwarp();
            if (lane < fill)
                bulk_g2s_stream(smem + ((size_t)slot * SP + lane) * TILE,
                         Kb + ((size_t)d_phys[slot][lane] * hkv + (d_unit[slot][lane] - qdiv_small(d_unit[slot][lane], hkv, inv_hkv) * hkv)) * TILE,
                         TILE, &fullb[slot]);
            ++si;
        }
        if (lane == 0) {
            const int slot = si % NS;           // end marker
            if (si >= NS) mbar_wait(&emptyb[slot], ((si / NS) - 1) & 1);
            d_n[slot] = -1;
            mbar_arrive(&fullb[slot]);
        }
        return;
    }
    // ---------------------------------------------------- consumers (half-warp = item, lane = token)
    const size_t ntok = (size_t)c.maxp * kP;
    const int half = lane >> 4, t = lane & 15, sw = t & 7;
    const unsigned hm = 0xffffu << (16 * half);
    T *qsh = reinterpret_cast<T *>(smem + AttCfg<T>::RING) + warp * G * kD;   // q cache of the warp
    int cu = -1, L = 0;                           // unit whose q is in qsh
    // running row maxima of the current unit (lanes 0 and 16: their half-warp's items),
    // flushed with one atomicMax per (head, half-warp) when the unit changes and at the end
    // (one atomic per item would serialise on the few rowmax words in full mode)
    float hmax[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) hmax[gg] = -INFINITY;
    auto flush = [&](int u) {
        if (u >= 0 && t == 0) {
            const int row0 = (u / c.Hkv) * Hq + (u % c.Hkv) * G;
#pragma unroll
            for (int gg = 0; gg < G; ++gg)
                if (hmax[gg] > -INFINITY) atomicMax(rowmax + row0 + gg, f2key(hmax[gg]));
        }
#pragma unroll
        for (int gg = 0; gg < G; ++gg) hmax[gg] = -INFINITY;
    };
    for (int si = 0;; ++si) {
        const int slot = si % NS;
        mbar_wait(&fullb[slot], (si / NS) & 1);
        const int n = d_n[slot];
        stamp_cta<1>(threadIdx.x == 0 && si == 0, 1);
        stamp_if(threadIdx.x == 0 && si < 16, 3, si);
        ph_stamp_if<4>(threadIdx.x == 0 && si == 0, 5);
        if (n < 0) {
            flush(cu);
            ph_stamp_if<4>(threadIdx.x == 0, 6);
            stamp_cta<1>(threadIdx.x == 0, 2); count_cta<1>(threadIdx.x == 0, si);
            break;
        }
        const int ni = d_ni[slot];
        for (int base = 2 * warp; base < ni; base += 2 * NCW) {            // warp-uniform
            const int it = base + half;
            const bool act = it < ni;
            const int itc = act ? it : base;
            const int code = full ? ((itc / G) * 8 + itc % G) : d_items[slot][itc];
            const int k = code >> 3, g = code & 7;
            const int unit = d_unit[slot][k];
            const int unitA = __shfl_sync(0xffffffffu, unit, 0), unitB = __shfl_sync(0xffffffffu, unit, 16);
            for (int pass = 0; pass < (unitA != unitB ? 2 : 1); ++pass) {  // warp-uniform
                const int u = pass ? unitB : unitA;
                if (u != cu) {                                             // warp-uniform
                    flush(cu);
                    const int bb = u / c.Hkv, kh = u % c.Hkv;
                    __syncwarp();
                    const uint4 *src = reinterpret_cast<const uint4 *>(q + ((size_t)bb * Hq + kh * G) * kD);
                    uint4 *dst = reinterpret_cast<uint4 *>(qsh);
                    for (int e = lane; e < G * kD * (int)sizeof(T) / 16; e += 32) dst[e] = __ldg(src + e);
                    __syncwarp();
                    cu = u;
                    L = __ldg(c.seq_lens + bb);
                }
                if (!act || unit != u) continue;                            // half-warp-uniform
            const unsigned char *tile = smem + ((size_t)slot * SP + k) * TILE;
            float acc[16];
            if constexpr (sizeof(T) == 2) {
                const uint4 *krow = reinterpret_cast<const uint4 *>(tile) + t * (kD / 8);
                const uint4 *qrow = reinterpret_cast<const uint4 *>(qsh) + g * (kD / 8);
#pragma unroll
                for (int cc = 0; cc < 16; ++cc) {
                    const int ch = cc ^ sw;
                    const uint4 kv = krow[ch], qv = qrow[ch];
                    float a = 0.0f;
                    a = fma_bf16lo(qv.x, kv.x, a); a = fma_bf16hi(qv.x, kv.x, a);
                    a = fma_bf16lo(qv.y, kv.y, a); a = fma_bf16hi(qv.y, kv.y, a);
                    a = fma_bf16lo(qv.z, kv.z, a); a = fma_bf16hi(qv.z, kv.z, a);
                    a = fma_bf16lo(qv.w, kv.w, a); a = fma_bf16hi(qv.w, kv.w, a);
                    acc[cc] = a;
                }
            } else {
                const float4 *krow = reinterpret_cast<const float4 *>(tile) + t * (kD / 4);
                const float4 *qrow = reinterpret_cast<const float4 *>(qsh) + g * (kD / 4);
#pragma unroll
                for (int cc = 0; cc < 16; ++cc) {
                    const int ch = cc ^ sw;
                    const float4 k0 = krow[2 * ch], k1 = krow[2 * ch + 1], q0 = qrow[2 * ch], q1 = qrow[2 * ch + 1];
                    float a = 0.0f;
                    a = fmaf(q0.x, k0.x, a); a = fmaf(q0.y, k0.y, a); a = fmaf(q0.z, k0.z, a); a = fmaf(q0.w, k0.w, a);
                    a = fmaf(q1.x, k1.x, a); a = fmaf(q1.y, k1.y, a); a = fmaf(q1.z, k1.z, a); a = fmaf(q1.w, k1.w, a);
                    acc[cc] = a;
                }
            }
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) acc[cc] = __fadd_rn(acc[cc], acc[cc + 8]);
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) acc[cc] = __fadd_rn(acc[cc], acc[cc + 4]);
            acc[0] = __fadd_rn(acc[0], acc[2]);
            acc[1] = __fadd_rn(acc[1], acc[3]);
            const float sv = __fmul_rn(__fadd_rn(acc[0], acc[1]), kCd);
            const int page = d_page[slot][k];
            const int tok = page * kP + t;
            const int bb = unit / c.Hkv, row = bb * Hq + (unit % c.Hkv) * G + g;
            const float v = tok < L ? sv : -INFINITY;
            scores[(size_t)row * ntok + tok] = v;
            float m = v;
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(hm, m, o));
            (void)row;
#pragma unroll
            for (int gg = 0; gg < G; ++gg) if (gg == g) hmax[gg] = fmaxf(hmax[gg], m);
            }
        }
        __syncwarp();
        stamp_if(threadIdx.x == 0 && si < 16, 3, 16 + si);
        if (lane == 0) mbar_arrive(&emptyb[slot]);
    }
}

// ============================================================================ candidates
// Full rows (a5): grid (chunk of 256 pages = 4096 tokens, b * Hq + h), 128 threads.  A token
// is a candidate iff z = (double)a * s > tau_lo = a * s_max - 1 (tau >= z_max - 1 since
// F(z_max - 1) >= 1, R9).  Each chunk writes its candidates in token order into its own
// region cand[row][chunk][0..kCpc) and its count into ccount[row][chunk]; the tau kernel
// concatenates the chunks in order, so the candidate order is deterministic.  The chunk's
// 16 KiB of scores arrive by one TMA bulk copy into shared memory (8 CTAs per SM keep
// 128 KiB in flight per SM; registers no longer bound the bytes in flight); thread t
// takes float4 t + 128 v (v < 8), and the token order is recovered from two block scans
// of four packed 16-bit counts.  The chunk-local tightening (many candidates: small
// alpha) runs out of line.  (max_pages <= 65536 -> at most 256 chunks per row.)
constexpr int kCandNT = 128;
static __device__ __noinline__ double chunk_tighten(const float *__restrict__ s4k, int nt, double a, double tau_lo) {
    // Local tightening: the chunk's own entmax threshold tau_c is a lower bound of tau
    // (F_all >= F_chunk), so tokens with z <= tau_c can never be in the support.  Newton on
    // ||(z - t)_+||_beta - 1 from the chunk's z_max - 1 (monotone from the left),
    // deterministic block reductions over the staged chunk (shared memory).
    __shared__ double shd[18];
    __shared__ float shf[9];
    const double beta = 1.0 / a;
    const int ib = (fabs(beta - rint(beta)) < 1e-12 && beta <= 4.5) ? (int)rint(beta) : 0;
    float lm = -INFINITY;
    for (int t = threadIdx.x; t < nt; t += kCandNT) lm = fmaxf(lm, s4k[t]);
    lm = block_max_f<kCandNT>(lm, shf);
    double tc = a * (double)lm - 1.0;
    for (int it = 0; it < 100; ++it) {
        double F = 0.0, Fd = 0.0;
        for (int t = threadIdx.x; t < nt; t += kCandNT) {
            const float sv = s4k[t];
            if (sv == -INFINITY) continue;
            const double d = a * (double)sv - tc;
            if (d > 0.0) { F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
        }
        block_sum2_d<kCandNT>(F, Fd, shd);
        if (!(Fd > 0.0)) break;
        const float Ff = (float)F, rootf = (ib == 1) ? Ff : (ib == 2) ? sqrtf(Ff) : (ib == 4) ? sqrtf(sqrtf(Ff)) : powf(Ff, (float)(1.0 / beta));
        const double step = (double)((rootf - 1.0f) * Ff / (rootf * (float)Fd));
        tc += step;
        if (!(fabs(step) > 1e-9 * fmax(1.0, fabs(tc)))) break;
    }
    tc -= 1e-7 * fmax(1.0, fabs(tc));      // margin: stay below the chunk threshold
    return tc > tau_lo ? tc : tau_lo;
}

static __global__ void __launch_bounds__(kCandNT, 8) k_candidates(const float *__restrict__ scores, size_t ntok,
                                                                  const uint32_t *__restrict__ rowmax,
                                                                  const int32_t *__restrict__ seq_lens, int Hq,
                                                                  float alpha, int nch, int *__restrict__ ccount,
                                                                  float *__restrict__ cand_s,
                                                                  int32_t *__restrict__ cand_j) {
    EKV_TRACE(5);
    __shared__ __align__(128) float st[256 * kP];
    __shared__ uint64_t bar;
    __shared__ unsigned long long sh[2][5];
    const int row = blockIdx.y;
    const int t0 = blockIdx.x * 256 * kP;        // first token of the chunk
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    pdl_enter();
    const int L = seq_lens[row / Hq];
    if (t0 >= L) return;
    const uint32_t mk = rowmax[row];
    if (mk == 0u) return;
    const int nt = min(256 * kP, L - t0);
    const float *s4k = scores + (size_t)row * ntok + t0;
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)min((size_t)256 * kP, ntok - (size_t)t0) * 4u;
        mbar_expect_tx(&bar, bytes);
        bulk_g2s(st, s4k, bytes, &bar);
    }
    const double a = (double)alpha - 1.0;
    const double zmax = a * (double)key2f(mk);
    const double tau_lo = zmax - 1.0 - 1e-12 * fmax(1.0, fabs(zmax));
    mbar_wait(&bar, 0);
    const float4 *p4 = reinterpret_cast<const float4 *>(st);
    auto packed = [&](double cut, int h) {       // counts of float4 t + 128 (4 h + v), v < 4
        unsigned long long c = 0ull;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int f = threadIdx.x + kCandNT * (4 * h + v);
            const float4 x = p4[f];
            const float sv[4] = {x.x, x.y, x.z, x.w};
            unsigned int n = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) n += (4 * f + e < nt && sv[e] != -INFINITY && a * (double)sv[e] > cut) ? 1u : 0u;
            c |= (unsigned long long)n << (16 * v);
        }
        return c;
    };
    auto fsum = [](unsigned long long t) {
        return (int)((t & 0xffff) + ((t >> 16) & 0xffff) + ((t >> 32) & 0xffff) + (t >> 48));
    };
    double tcut = tau_lo;
    unsigned long long cnt0 = packed(tcut, 0), cnt1 = packed(tcut, 1), tot0, tot1;
    unsigned long long pos0 = block_excl_scan_u64<kCandNT>(cnt0, sh[0], &tot0);
    unsigned long long pos1 = block_excl_scan_u64<kCandNT>(cnt1, sh[1], &tot1);
    if (fsum(tot0) + fsum(tot1) > 256) {           // block-uniform
        tcut = chunk_tighten(st, nt, a, tau_lo);
        if (tcut > tau_lo) {
            cnt0 = packed(tcut, 0);
            cnt1 = packed(tcut, 1);
            pos0 = block_excl_scan_u64<kCandNT>(cnt0, sh[0], &tot0);
            pos1 = block_excl_scan_u64<kCandNT>(cnt1, sh[1], &tot1);
        }
    }
    const size_t reg = ((size_t)row * nch + blockIdx.x) * kCpc;
    if (threadIdx.x == 0) ccount[(size_t)row * nch + blockIdx.x] = fsum(tot0) + fsum(tot1);
    if (!(cnt0 | cnt1)) return;
    int base = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const unsigned long long pos = w < 4 ? pos0 : pos1, tot = w < 4 ? tot0 : tot1;
        const int sh16 = 16 * (w & 3);
        int p = base + (int)((pos >> sh16) & 0xffff);
        const int f = threadIdx.x + kCandNT * w;
        const float4 x = p4[f];
        const float sv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (4 * f + e < nt && sv[e] != -INFINITY && a * (double)sv[e] > tcut) {
                if (p < kCpc) { cand_s[reg + p] = sv[e]; cand_j[reg + p] = t0 + 4 * f + e; }
                ++p;
            }
        }
        base += (int)((tot >> sh16) & 0xffff);
    }
}

// ============================================================================ exact tau + PV
// The tau / support / PV kernel is k_tau_sparse (kernels_tau.cuh); the shared pieces live here.
template <typename T>
__device__ __forceinline__ void ldv4(const T *vr, float (&vx)[4]) {
    if constexpr (sizeof(T) == 2) {
        const uint2 w = *reinterpret_cast<const uint2 *>(vr);
        vx[0] = bf_lo(w.x); vx[1] = bf_hi(w.x); vx[2] = bf_lo(w.y); vx[3] = bf_hi(w.y);
    } else {
        const float4 w = *reinterpret_cast<const float4 *>(vr);
        vx[0] = w.x; vx[1] = w.y; vx[2] = w.z; vx[3] = w.w;
    }
}
__device__ __forceinline__ double lbeta_step(double F, double Fd, double beta, int ib) {
    // Newton step on g(tau) = ||(z - tau)_+||_beta - 1:  (F^{1/b} - 1) / (F^{1/b - 1} Fd).
    // F and Fd are fp64 sums; the step itself only steers the iteration (its fixed point is
    // F(tau) = 1 whatever the step's rounding), so it is evaluated in fp32, with F^{1/b} - 1
    // formed from the accurate F - 1 to keep full relative precision near convergence.
    const float dF = (float)(F - 1.0), Ff = (float)F, Fdf = (float)Fd;
    float root, rm1;
    if (ib == 1) { root = Ff; rm1 = dF; }
    else if (ib == 2) { root = sqrtf(Ff); rm1 = dF / (root + 1.0f); }
    else if (ib == 4) { root = sqrtf(sqrtf(Ff)); rm1 = dF / ((1.0f + root) * (1.0f + root * root)); }
    else { rm1 = expm1f(log1pf(dF) / (float)beta); root = 1.0f + rm1; }
    return (double)(rm1 * Ff / (root * Fdf));
}

// ============================================================================ a4: certified delta_bar
// delta_bar = sum_{p not in C_page} c_p [a * box_p - tau~]_+^beta  (R16; Prop. B.1 gives
// z_j <= a * box_p, and tau >= tau~).  Grid (chunk of 2048 pages, b * Hq + h): each CTA
// marks its row's selected pages of the chunk in a shared bitmap, sums its chunk
// (deterministic block tree) into partial[row][chunk]; the last CTA of a row (ticket
// counter) adds the partials in chunk order, so the result is deterministic.
// delta_bar (R16, P:409-420 certificate): per (b, q-head) row, sum over the UNSELECTED
// valid pages p of n_p * ((alpha-1) * box_p - tau)_+^beta.  Grid (chunks, rows), the
// chunks of a row form one thread-block cluster (<= 8).  Every thread issues its 8 float4
// box loads, 8 union-mask words (bit (page, g) = page selected by head g of the unit), the
// row's tau and sequence length together, then the fp64 terms (integer beta IB is a
// template constant: no pow); the CTA partials are summed in fixed order by rank 0 through
// distributed shared memory (deterministic, no global ticket).
template <int IB>
__global__ void __launch_bounds__(256) k_delta_bar(const float *__restrict__ box, int maxp,
                                                   const int32_t *__restrict__ seq_lens, int Hq, int G,
                                                   const uint32_t *__restrict__ umask, int W,
                                                   const double *__restrict__ tau, DbConst k,
                                                   double *__restrict__ out) {
    EKV_TRACE(7);
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int R = kDbChunk / 1024;
    __shared__ double rbuf[2 * 2 * 8];
    __shared__ double part;
    BlockRed2<256> Rd{rbuf, 0};
    const int row = blockIdx.y, b = row / Hq, h = row - b * Hq;
    const int unit = b * (Hq / G) + h / G, g = h - (h / G) * G;
    const int p0 = blockIdx.x * kDbChunk;
    const float *bx = box + (size_t)row * maxp;
    const uint32_t *um = umask + (size_t)unit * W;
    const bool vec = (maxp & 3) == 0;
    const int L = __ldg(seq_lens + b);
    float bv[4 * R];
    uint32_t mw[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int p = p0 + 4 * (threadIdx.x + 256 * r);
        if (vec && p + 3 < maxp) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(bx + p));
            bv[4 * r] = v.x; bv[4 * r + 1] = v.y; bv[4 * r + 2] = v.z; bv[4 * r + 3] = v.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) bv[4 * r + e] = (p + e < maxp) ? __ldg(bx + p + e) : -INFINITY;
        }
        mw[r] = (p < maxp) ? __ldg(um + (p >> 2)) : 0u;
    }
    // box (page scoring), the union marks (top-k) and seq_lens (append) are two or more launches
    // back: loaded above, before the wait; tau comes from the immediately preceding kernel
    pdl_enter();
    const double t = tau[row];
    const int M = n_pages_of(L);
    double db = 0.0, dz = 0.0;
    if (t == t) {   // tau is NaN for an empty row
        // fp32 pre-test: a*box - tau > 0 needs box > tau/a; thr is rounded well below it
        const float tf = (float)(t * k.inv_a);
        const float thr = tf - 1e-3f * fmaxf(1.0f, fabsf(tf));
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int p = p0 + 4 * (threadIdx.x + 256 * r) + e;
                const bool sel = (mw[r] >> (8 * e + g)) & 1u;      // page selected by head h
                if (p >= M || sel || !(bv[4 * r + e] > thr)) continue;
                const double d = k.a * (double)bv[4 * r + e] - t;
                if (d > 0.0) {
                    double w;
                    if constexpr (IB == 1) w = d;
                    else if constexpr (IB == 2) w = d * d;
                    else if constexpr (IB == 3) w = d * d * d;
                    else if constexpr (IB == 4) { const double d2 = d * d; w = d2 * d2; }
                    else w = pow(d, k.beta);
                    db += (p == M - 1) ? (double)(L - p * kP) * w : (double)kP * w;
                }
            }
    }
    Rd.sum(db, dz);
    if (threadIdx.x == 0) part = db;
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        double sum = 0.0;
        for (int q = 0; q < (int)cl.num_blocks(); ++q) sum += *cl.map_shared_rank(&part, q);
        out[row] = (t == t) ? sum : NAN;
    }
    cl.sync();                               // keep shared memory alive for rank 0's reads
}

// ============================================================================ eval: exact delta / rho
// One CTA per (b, q-head): the full pass's support list (token positions j, p_j)
// against the sparse selection (ascending page list of head h): delta = sum of p_j
// whose page is not selected (Eq. delta), recovered = |S cap C_tok|,
// full_supp = |S| (Eq. rho).
static __global__ void __launch_bounds__(256) k_eval_metrics(const int32_t *__restrict__ tok_list, const double *__restrict__ p_list,
                                                      const int32_t *__restrict__ n_list, int list_cap,
                                                      const int32_t *__restrict__ page_idx, const int32_t *__restrict__ n_sel,
                                                      int sel_stride, double *delta, int32_t *recovered, int32_t *full_supp) {
    EKV_TRACE(9);
    __shared__ double shd[2 * 8 + 2];
    __shared__ int shi[9];
    const int row = blockIdx.x;
    const int n = min(n_list[row], list_cap);
    const int32_t *pl = page_idx + (size_t)row * sel_stride;
    const int ns = n_sel[row];
    double dl = 0.0, dz = 0.0;
    int rec = 0;
    for (int i = threadIdx.x; i < n; i += 256) {
        const int j = tok_list[(size_t)row * list_cap + i];
        const int p = j / kP;
        int lo = 0, hi = ns;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (pl[mid] < p) lo = mid + 1; else hi = mid; }
        if (lo < ns && pl[lo] == p) ++rec;
        else dl += p_list[(size_t)row * list_cap + i];
    }
    block_sum2_d<256>(dl, dz, shd);
    rec = block_sum_i<256>(rec, shi);
    if (threadIdx.x == 0) {
        if (delta) delta[row] = dl;
        if (recovered) recovered[row] = rec;
        if (full_supp) full_supp[row] = n_list[row];
    }
}

}  // namespace ekv
