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
template <typename T> struct AttCfg {
    static constexpr int NCW = EKV_ATT_NCW;                // consumer warps (16 half-warps >= items per stage, usually)
    static constexpr int SP = 8;                           // pages per stage (item code: 3 bits)
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
        const int per = (nrows + 31) / 32;
        int run = 0;
        for (int i = 0; i < per; ++i) { const int r = lane * per + i; run += r < nrows ? __ldg(n_sel + r) : 0; }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += y; }
        int acc = incl - run;
        for (int i = 0; i < per; ++i) {
            const int r = lane * per + i;
            if (r < nrows) { pref[r] = acc; acc += __ldg(n_sel + r); }
        }
        if (lane == 31) pref[nrows] = incl;
        __syncwarp();
        tot = pref[nrows];
    }
    const long long f0 = tot * blockIdx.x / gridDim.x, f1 = tot * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&fullb[i], 1); mbar_init(&emptyb[i], NCW); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NCW) {
        // ------------------------------------------------ producer
        const unsigned char *Kb = reinterpret_cast<const unsigned char *>(c.K);
        int si = 0, fill = 0;
        int cu = (int)(f0 / ucap), cs = (int)(f0 % ucap);   // (row or unit, slot) of the chunk start
        int brow = 0;                                        // balanced: row of the chunk start
        if (bal) { while (brow + 1 < nrows && pref[brow + 1] <= f0) ++brow; }
        for (long long cb = f0; cb < f1; cb += CHK) {
            int un[CHK / 32], pg[CHK / 32], hg[CHK / 32];
            bool ok[CHK / 32];
            if (bal) { while (brow + 1 < nrows && pref[brow + 1] <= cb) ++brow; }
#pragma unroll
            for (int r = 0; r < CHK / 32; ++r) {
                int u = cu, sl = cs + r * 32 + lane;
                if (bal) {
                    const int e = (int)(cb + r * 32 + lane);
                    u = brow;
                    while (u + 1 < nrows && pref[u + 1] <= e) ++u;
                    sl = e - pref[u];
                } else {
                    while (sl >= ucap) { sl -= ucap; ++u; }
                }
                const int bb = full ? u / c.Hkv : u / Hq;      // u: full -> unit; sparse -> row
                un[r] = full ? u : bb * c.Hkv + (u % Hq) / G;
                hg[r] = full ? 0 : (u % Hq) % G;
                ok[r] = false;
                pg[r] = 0;
                if (cb + r * 32 + lane < f1) {
                    if (full) { pg[r] = sl; ok[r] = sl < n_pages_of(__ldg(c.seq_lens + bb)); }
                    else if (sl < __ldg(n_sel + u)) { pg[r] = __ldg(page_idx + (size_t)u * stride + sl); ok[r] = true; }
                }
            }
            cs += CHK;
            while (cs >= ucap) { cs -= ucap; ++cu; }
            int ph[CHK / 32];
            uint8_t mk[CHK / 32];
#pragma unroll
            for (int r = 0; r < CHK / 32; ++r) {
                ph[r] = 0; mk[r] = 0;
                if (ok[r]) {
                    ph[r] = __ldg(c.page_table + (size_t)(un[r] / c.Hkv) * c.maxp + pg[r]);
                    mk[r] = full ? (uint8_t)((1u << G) - 1u)
                                 : (uint8_t)((__ldg(umask + (size_t)un[r] * W + (pg[r] >> 2)) >> ((pg[r] & 3) * 8)) & 0xffu);
                }
            }
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
            for (int i = 0; i < nl; ++i) {          // warp-uniform
                const int slot = si % NS;
                if (fill == 0) {
                    if (lane == 0 && si >= NS) mbar_wait(&emptyb[slot], ((si / NS) - 1) & 1);
                    __syncwarp();
                }
                if (lane == 0) {
                    d_unit[slot][fill] = l_unit[i]; d_page[slot][fill] = l_page[i];
                    d_mask[slot][fill] = l_mask[i]; d_phys[slot][fill] = l_phys[i];
                }
                if (++fill == SP) {
                    __syncwarp();
                    if (lane == 0) {
                        d_n[slot] = SP;
                        int ni = 0;
                        for (int kk = 0; kk < SP; ++kk)
                            for (unsigned m = d_mask[slot][kk]; m; m &= m - 1u) d_items[slot][ni++] = (uint8_t)(kk * 8 + __ffs((int)m) - 1);
                        d_ni[slot] = ni;
                        mbar_expect_tx(&fullb[slot], (uint32_t)(SP * TILE));
                    }
                    __syncwarp();
                    if (lane < SP)
                        bulk_g2s(smem + ((size_t)slot * SP + lane) * TILE,
                                 Kb + ((size_t)d_phys[slot][lane] * c.Hkv + d_unit[slot][lane] % c.Hkv) * TILE,
                                 TILE, &fullb[slot]);
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
                int ni = 0;
                for (int kk = 0; kk < fill; ++kk)
                    for (unsigned m = d_mask[slot][kk]; m; m &= m - 1u) d_items[slot][ni++] = (uint8_t)(kk * 8 + __ffs((int)m) - 1);
                d_ni[slot] = ni;
                mbar_expect_tx(&fullb[slot], (uint32_t)(fill * TILE));
            }
            __syncwarp();
            if (lane < fill)
                bulk_g2s(smem + ((size_t)slot * SP + lane) * TILE,
                         Kb + ((size_t)d_phys[slot][lane] * c.Hkv + d_unit[slot][lane] % c.Hkv) * TILE,
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
    for (int si = 0;; ++si) {
        const int slot = si % NS;
        mbar_wait(&fullb[slot], (si / NS) & 1);
        const int n = d_n[slot];
        stamp_cta<1>(threadIdx.x == 0 && si == 0, 1);
        stamp_if(threadIdx.x == 0 && si < 16, 3, si);
        if (n < 0) { stamp_cta<1>(threadIdx.x == 0, 2); count_cta<1>(threadIdx.x == 0, si); break; }
        const int ni = d_ni[slot];
        for (int base = 2 * warp; base < ni; base += 2 * NCW) {            // warp-uniform
            const int it = base + half;
            const bool act = it < ni;
            const int code = d_items[slot][act ? it : base];
            const int k = code >> 3, g = code & 7;
            const int unit = d_unit[slot][k];
            const int unitA = __shfl_sync(0xffffffffu, unit, 0), unitB = __shfl_sync(0xffffffffu, unit, 16);
            for (int pass = 0; pass < (unitA != unitB ? 2 : 1); ++pass) {  // warp-uniform
                const int u = pass ? unitB : unitA;
                if (u != cu) {                                             // warp-uniform
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
            if (t == 0 && m > -INFINITY) atomicMax(rowmax + row, f2key(m));
            }
        }
        __syncwarp();
        stamp_if(threadIdx.x == 0 && si < 16, 3, 16 + si);
        if (lane == 0) mbar_arrive(&emptyb[slot]);
    }
}

// ============================================================================ candidates
// Grid (chunk of 256 page-list entries, b * Hq + h); thread = one selected page of the
// row (sparse: page_idx[row][i]; full: page i).  A token is a candidate iff
// z = (double)a * s > tau_lo = a * s_max - 1 (tau >= z_max - 1 since F(z_max - 1) >= 1,
// R9).  Each chunk writes its candidates, in page-list order (block scan), into its own
// region cand[row][chunk][0..kCpc) and its count into ccount[row][chunk]; the tau
// kernel concatenates the chunks in order, so the candidate order is deterministic.
// (max_pages <= 65536 -> at most 256 chunks per row.)
constexpr int kCpc = 1024;          // candidates per chunk region
__global__ void __launch_bounds__(256) k_candidates(const float *__restrict__ scores, size_t ntok,
                                                    const uint32_t *__restrict__ rowmax,
                                                    const int32_t *__restrict__ page_idx,
                                                    const int32_t *__restrict__ n_sel, int sel_stride,
                                                    const int32_t *__restrict__ seq_lens, int Hq, int full,
                                                    float alpha, int transform, int nch,
                                                    int *__restrict__ ccount, float *__restrict__ cand_s,
                                                    int32_t *__restrict__ cand_j) {
    EKV_TRACE(5);
    __shared__ int sh[9];
    const int row = blockIdx.y;
    const int b = row / Hq;
    const int L = seq_lens[b];
    const int nlist = full ? n_pages_of(L) : n_sel[row];
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (blockIdx.x * 256 >= nlist) return;
    const uint32_t mk = rowmax[row];
    if (mk == 0u || transform == 1) return;     // softmax rows stream the row in k_tau_pv
    const double a = (double)alpha - 1.0;
    const double zmax = a * (double)key2f(mk);
    const double tau_lo = zmax - 1.0 - 1e-12 * fmax(1.0, fabs(zmax));
    float sv[kP];
    int page = 0, cnt = 0;
    const float *srow = scores + (size_t)row * ntok;
    if (i < nlist) {
        page = full ? i : page_idx[(size_t)row * sel_stride + i];
        const float4 *p4 = reinterpret_cast<const float4 *>(srow + (size_t)page * kP);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const float4 x = p4[v];
            sv[4 * v] = x.x; sv[4 * v + 1] = x.y; sv[4 * v + 2] = x.z; sv[4 * v + 3] = x.w;
        }
#pragma unroll
        for (int t = 0; t < kP; ++t)
            cnt += ((page * kP + t < L) && sv[t] != -INFINITY && a * (double)sv[t] > tau_lo) ? 1 : 0;
    }
    // Local tightening: the chunk's own entmax threshold tau_c is a lower bound of tau
    // (F_all >= F_chunk), so tokens with z <= tau_c can never be in the support.  Used when
    // the chunk has many candidates (small alpha); Newton on ||(z - t)_+||_beta - 1 from the
    // chunk's z_max - 1 (monotone from the left), deterministic block reductions.
    __shared__ double shd[18];
    __shared__ float shf[9];
    double tcut = tau_lo;
    int ctot = block_sum_i<256>(cnt, sh);
    if (ctot > 256) {
        const double beta = 1.0 / a;
        const int ib = (fabs(beta - rint(beta)) < 1e-12 && beta <= 4.5) ? (int)rint(beta) : 0;
        float lm = -INFINITY;
        if (i < nlist) {
#pragma unroll
            for (int t = 0; t < kP; ++t) if (page * kP + t < L) lm = fmaxf(lm, sv[t]);
        }
        lm = block_max_f<256>(lm, shf);
        double tc = a * (double)lm - 1.0;
        for (int it = 0; it < 100; ++it) {
            double F = 0.0, Fd = 0.0;
            if (i < nlist) {
#pragma unroll
                for (int t = 0; t < kP; ++t) {
                    if (page * kP + t >= L || sv[t] == -INFINITY) continue;
                    const double d = a * (double)sv[t] - tc;
                    if (d > 0.0) { F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
                }
            }
            block_sum2_d<256>(F, Fd, shd);
            if (!(Fd > 0.0)) break;
            const float Ff = (float)F, rootf = (ib == 1) ? Ff : (ib == 2) ? sqrtf(Ff) : (ib == 4) ? sqrtf(sqrtf(Ff)) : powf(Ff, (float)(1.0 / beta));
            const double step = (double)((rootf - 1.0f) * Ff / (rootf * (float)Fd));
            tc += step;
            if (!(fabs(step) > 1e-9 * fmax(1.0, fabs(tc)))) break;
        }
        tc -= 1e-7 * fmax(1.0, fabs(tc));      // margin: stay below the chunk threshold
        if (tc > tcut) {
            tcut = tc;
            cnt = 0;
            if (i < nlist) {
#pragma unroll
                for (int t = 0; t < kP; ++t)
                    cnt += ((page * kP + t < L) && sv[t] != -INFINITY && a * (double)sv[t] > tcut) ? 1 : 0;
            }
        }
    }
    int tot;
    int pos = block_excl_scan<256>(cnt, sh, &tot);
    const size_t reg = ((size_t)row * nch + blockIdx.x) * kCpc;
    if (threadIdx.x == 0) ccount[(size_t)row * nch + blockIdx.x] = tot;
    if (i < nlist && cnt) {
#pragma unroll
        for (int t = 0; t < kP; ++t) {
            if ((page * kP + t < L) && sv[t] != -INFINITY && a * (double)sv[t] > tcut) {
                if (pos < kCpc) { cand_s[reg + pos] = sv[t]; cand_j[reg + pos] = page * kP + t; }
                ++pos;
            }
        }
    }
}

// ============================================================================ exact tau + PV
// One CTA (256 threads) per (b, q-head):
//  1. candidates {z > tau_lo = z_max - 1} in a FIXED order (fp64 sums below are then
//     deterministic): sparse rows are read directly from the score row over the head's
//     page list (block scan per round of 4 pages per thread); full rows come from the
//     k_candidates chunk regions concatenated in chunk order.  Overflow -> Newton
//     streamed over the source moves tau_lo just below tau, then an ordered re-extraction.
//  2. Newton on g(tau) = ||(z - tau)_+||_beta - 1 from tau_lo (convex, decreasing:
//     monotone from the left, exact in one step for one active token);
//  3. support by R9: z > tau_N + band -> in, z < tau_N - band -> out, else F(z_j) < 1;
//  4. tau from the support: beta = 1: (S1 - 1)/k; beta = 2: m - sqrt((1 - ss)/k);
//     otherwise one Newton polish on sum_S (z - tau)^beta = 1;
//  5. p_j = (z_j - tau)^beta; out = sum p_j v_j / sum p_j (R12): support tokens are
//     compacted NT at a time, their page-table entries fetched in parallel, then warps
//     gather the V rows (4 in flight per warp; lane = 4 dims);
// Softmax rows (a6): p = exp(s - s_max) over every valid token (dense V).
constexpr int kTauNT = 256;
constexpr int kCap = 12288;         // shared-memory candidate capacity
constexpr int kPr = 2048;           // pruned-list capacity (tau solver)
constexpr int kTauSmem = (8 + 1 + 4) * kCap + (8 + 4) * kPr;

struct TauArgs {
    const float *scores; size_t ntok;
    const uint32_t *rowmax; const int *ccount; const float *cand_s; const int32_t *cand_j; int nch;
    const int32_t *page_idx; const int32_t *n_sel; int sel_stride; int full;
    int Hq, G; float alpha; int transform;
    float *out; double *tau_out; int32_t *supp_out;
    int32_t *tok_list; double *p_list; int32_t *n_list; int list_cap;     // eval list
};

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

template <typename T>
__global__ void __launch_bounds__(kTauNT, 1) k_tau_pv(CacheView c, TauArgs A) {
    EKV_TRACE(6);
    constexpr int NT = kTauNT;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long *ck = reinterpret_cast<unsigned long long *>(smem);   // [kCap] (j << 32 | s bits)
    uint8_t *cin = reinterpret_cast<uint8_t *>(smem + sizeof(unsigned long long) * kCap);   // [kCap]
    int *cphys = reinterpret_cast<int *>(smem + (sizeof(unsigned long long) + 1) * kCap);    // [kCap] (direct path)
    __shared__ double rbuf[2 * 2 * NW];
    __shared__ double shd[2 * NW + 2];
    __shared__ int shi[NW + 1];
    __shared__ float red[NW][kD];
    constexpr int kSup = 2048;
    __shared__ int sup_j[kSup], sup_phys[kSup];
    __shared__ float sup_p[kSup];
    BlockRed2<NT> R{rbuf, 0};

    stamp(0, 0);
    const int row = blockIdx.x;
    const int b = row / A.Hq, h = row % A.Hq, kvh = h / A.G;
    const int L = c.seq_lens[b];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t mk = A.rowmax[row];
    if (mk == 0u) {   // empty C_tok
        if (threadIdx.x < kD) A.out[(size_t)row * kD + threadIdx.x] = 0.0f;
        if (threadIdx.x == 0) {
            if (A.tau_out) A.tau_out[row] = NAN;
            if (A.supp_out) A.supp_out[row] = 0;
            if (A.n_list) A.n_list[row] = 0;
        }
        return;
    }
    const float smax = key2f(mk);
    const int nlist = A.full ? n_pages_of(L) : A.n_sel[row];
    const int32_t *plist = A.page_idx + (size_t)row * A.sel_stride;
    const float *srow = A.scores + (size_t)row * A.ntok;
    const T *Vb = reinterpret_cast<const T *>(c.V);

    if (A.transform == 1) {
        // ---------------- softmax over C_tok: every valid token of the page list (dense V)
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        double zs = 0.0, dz = 0.0;
        int cnt = 0;
        for (int e = warp; e < nlist * kP; e += NW) {
            const int pg = A.full ? e / kP : plist[e / kP];
            const int j = pg * kP + e % kP;
            if (j >= L) continue;
            const float p = expf(srow[j] - smax);
            if (lane == 0) { zs += (double)p; ++cnt; }
            const int phys = c.page_table[(size_t)b * c.maxp + pg];
            float vx[4];
            ldv4<T>(Vb + (((size_t)phys * c.Hkv + kvh) * kP + (j % kP)) * kD + 4 * lane, vx);
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) acc[e2] = __fmaf_rn(p, vx[e2], acc[e2]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) red[warp][4 * lane + e] = acc[e];
        R.sum(zs, dz);
        cnt = block_sum_i<NT>(cnt, shi);
        if (threadIdx.x < kD) {
            float o = 0.f;
            for (int w = 0; w < NW; ++w) o = __fadd_rn(o, red[w][threadIdx.x]);
            A.out[(size_t)row * kD + threadIdx.x] = (float)((double)o / zs);
        }
        if (threadIdx.x == 0) {
            if (A.tau_out) A.tau_out[row] = (double)smax + log(zs);
            if (A.supp_out) A.supp_out[row] = cnt;
        }
        return;
    }

    // ---------------- exact alpha-entmax
    const double a = (double)A.alpha - 1.0;
    const double beta = 1.0 / a;
    const int ib = (fabs(beta - rint(beta)) < 1e-12 && beta <= 4.5) ? (int)rint(beta) : 0;
    const double zmax = a * (double)smax;
    double tau_lo = zmax - 1.0 - 1e-12 * fmax(1.0, fabs(zmax));
    int ncand = 0;
    bool overflow = false;
    bool have_phys = false;                 // cphys[] valid (direct extraction without overflow)

    if (!A.full) {
        // (direct) rounds of up to 4 list pages per thread: loads in flight, count, scan, write
        // fp32 pre-test (conservative: a * s > tau_lo needs s > tau_lo / a; -inf never passes)
        const float thr_c = (float)(tau_lo / a);
        const float thr_f = thr_c - 1e-6f * fmaxf(1.0f, fabsf(thr_c));
        for (int r0 = 0; r0 < nlist; r0 += 4 * NT) {
            float sv[4][kP];
            int pgs[4], phs[4];
            int cnt = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int li = r0 + threadIdx.x + u * NT;
                pgs[u] = li < nlist ? plist[li] : -1;
                phs[u] = 0;
                if (pgs[u] >= 0) {
                    phs[u] = __ldg(c.page_table + (size_t)b * c.maxp + pgs[u]);
                    const float4 *p4 = reinterpret_cast<const float4 *>(srow + (size_t)pgs[u] * kP);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const float4 x = p4[v];
                        sv[u][4 * v] = x.x; sv[u][4 * v + 1] = x.y; sv[u][4 * v + 2] = x.z; sv[u][4 * v + 3] = x.w;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (pgs[u] >= 0) {
#pragma unroll
                    for (int t = 0; t < kP; ++t)
                        cnt += (pgs[u] * kP + t < L && sv[u][t] >= thr_f && a * (double)sv[u][t] > tau_lo);
                }
            int tot;
            int pos = ncand + block_excl_scan<NT>(cnt, shi, &tot);
            if (ncand + tot > kCap) { overflow = true; break; }   // uniform
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (pgs[u] >= 0) {
#pragma unroll
                    for (int t = 0; t < kP; ++t)
                        if (pgs[u] * kP + t < L && sv[u][t] >= thr_f && a * (double)sv[u][t] > tau_lo) {
                            cphys[pos] = phs[u];
                            ck[pos++] = ((unsigned long long)(uint32_t)(pgs[u] * kP + t) << 32) | __float_as_uint(sv[u][t]);
                        }
                }
            ncand += tot;
        }
        have_phys = !overflow;
        __syncthreads();
    } else {
        // (full) chunk regions from k_candidates, concatenated in chunk order (nch <= NT)
        int ccnt = 0, tot = 0;
        bool chunk_ovf = false;
        if (threadIdx.x < A.nch) {
            ccnt = A.ccount[(size_t)row * A.nch + threadIdx.x];
            chunk_ovf = ccnt > kCpc;
        }
        const int coff = block_excl_scan<NT>(ccnt, shi, &tot);
        chunk_ovf = __syncthreads_or(chunk_ovf);
        const float *gs = A.cand_s + (size_t)row * A.nch * kCpc;
        const int32_t *gj = A.cand_j + (size_t)row * A.nch * kCpc;
        if (!chunk_ovf && tot <= kCap) {
            int *s_off = reinterpret_cast<int *>(cin);       // cin is free until the support pass
            if (threadIdx.x < A.nch) s_off[threadIdx.x] = coff;
            __syncthreads();
#pragma unroll 4
            for (int e = threadIdx.x; e < tot; e += NT) {
                int lo = 0, hi = A.nch - 1;               // last chunk with offset <= e
                while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_off[mid] <= e) lo = mid; else hi = mid - 1; }
                const size_t g = (size_t)lo * kCpc + (e - s_off[lo]);
                ck[e] = ((unsigned long long)(uint32_t)__ldg(gj + g) << 32) | __float_as_uint(__ldg(gs + g));
            }
            ncand = tot;
            __syncthreads();
        } else if (!chunk_ovf) {
            // too many for shared memory: Newton over the chunk regions (thread t <-> chunk t)
            double tau = tau_lo;
            for (int it = 0; it < 200; ++it) {
                double F = 0.0, Fd = 0.0;
                if (threadIdx.x < A.nch) {
                    const size_t g0 = (size_t)threadIdx.x * kCpc;
                    for (int k = 0; k < ccnt; ++k) {
                        const double d = a * (double)__ldg(gs + g0 + k) - tau;
                        if (d > 0.0) { F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
                    }
                }
                R.sum(F, Fd);
                if (!(Fd > 0.0)) break;
                const double step = lbeta_step(F, Fd, beta, ib);
                tau += step;
                if (!(fabs(step) > 1e-12 * fmax(1.0, fabs(tau)))) break;
            }
            tau_lo = fmax(tau_lo, tau - 1e-7 * fmax(1.0, fabs(tau)));
            int mine = 0;
            if (threadIdx.x < A.nch) {
                const size_t g0 = (size_t)threadIdx.x * kCpc;
                for (int k = 0; k < ccnt; ++k) mine += a * (double)__ldg(gs + g0 + k) > tau_lo;
            }
            int tt;
            int pos = block_excl_scan<NT>(mine, shi, &tt);
            if (tt > kCap) overflow = true;
            else {
                if (threadIdx.x < A.nch) {
                    const size_t g0 = (size_t)threadIdx.x * kCpc;
                    for (int k = 0; k < ccnt; ++k) {
                        const float sj = __ldg(gs + g0 + k);
                        if (a * (double)sj > tau_lo)
                            ck[pos++] = ((unsigned long long)(uint32_t)__ldg(gj + g0 + k) << 32) | __float_as_uint(sj);
                    }
                }
                ncand = tt;
            }
            __syncthreads();
        } else {
            overflow = true;
        }
    }
    if (overflow) {
        // Newton streamed over the whole score row (coalesced, fixed thread mapping), then
        // an ordered re-extraction by contiguous per-thread segments of the page list.
        const int ntk = nlist * kP;
        double tau = tau_lo;
        for (int it = 0; it < 200; ++it) {
            double F = 0.0, Fd = 0.0;
            for (int e = threadIdx.x; e < ntk; e += NT) {
                const int pg = A.full ? e / kP : plist[e / kP];
                const int j = pg * kP + e % kP;
                if (j >= L) continue;
                const float sj = srow[j];
                if (sj == -INFINITY) continue;
                const double d = a * (double)sj - tau;
                if (d > 0.0) { F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
            }
            R.sum(F, Fd);
            if (!(Fd > 0.0)) break;
            const double step = lbeta_step(F, Fd, beta, ib);
            tau += step;
            if (!(fabs(step) > 1e-12 * fmax(1.0, fabs(tau)))) break;
        }
        tau_lo = fmax(tau_lo, tau - 1e-7 * fmax(1.0, fabs(tau)));
        const int seg = (nlist + NT - 1) / NT;            // pages per thread, contiguous in list order
        int mine = 0;
        for (int li = threadIdx.x * seg; li < min(nlist, (threadIdx.x + 1) * seg); ++li) {
            const int pg = A.full ? li : plist[li];
            for (int t = 0; t < kP; ++t) {
                const int j = pg * kP + t;
                if (j < L && srow[j] != -INFINITY && a * (double)srow[j] > tau_lo) ++mine;
            }
        }
        int tt;
        int pos = block_excl_scan<NT>(mine, shi, &tt);
        if (tt > kCap) {             // support larger than the shared-memory capacity
            if (threadIdx.x < kD) A.out[(size_t)row * kD + threadIdx.x] = NAN;
            if (threadIdx.x == 0) {
                if (A.tau_out) A.tau_out[row] = NAN;
                if (A.supp_out) A.supp_out[row] = -tt;
            }
            return;
        }
        for (int li = threadIdx.x * seg; li < min(nlist, (threadIdx.x + 1) * seg); ++li) {
            const int pg = A.full ? li : plist[li];
            for (int t = 0; t < kP; ++t) {
                const int j = pg * kP + t;
                if (j < L && srow[j] != -INFINITY && a * (double)srow[j] > tau_lo)
                    ck[pos++] = ((unsigned long long)(uint32_t)j << 32) | __float_as_uint(srow[j]);
            }
        }
        ncand = tt;
        __syncthreads();
    }
    stamp(0, 2);
#ifdef EKV_STAMPS
    if (blockIdx.x == 0 && threadIdx.x == 0) ekv_stamps[0][14] = (unsigned long long)ncand;
#endif
#define ZOF(k) (a * (double)__uint_as_float((uint32_t)(ck[k] & 0xffffffffu)))
    // ---- tau and support by warp 0 alone (warp-shuffle sums, no block barriers; the xor
    // butterfly leaves the same value on every lane, so every result is deterministic):
    //  (a) fp32 Newton on the candidates (cheap; only steers),
    //  (b) certified lower bound lo2 = tau32 - 1e-3 max(1, |tau32|) if F(lo2) >= 1 in fp64
    //      (F decreasing -> tau >= lo2; else lo2 = tau_lo), and the list {z > lo2} in fp64
    //      compacted into shared memory (every token outside it has F(z) >= 1: not in S),
    //  (c) fp64 Newton on the list from lo2, R9 support, tau from the support (closed forms),
    //  (d) the support's p_j and V addresses for the PV gather.
    double *zp = reinterpret_cast<double *>(smem + (sizeof(unsigned long long) + 1 + 4) * kCap);   // [kPr]
    int *ip = reinterpret_cast<int *>(smem + (sizeof(unsigned long long) + 1 + 4) * kCap + 8 * kPr); // [kPr]
    __shared__ double s_tau, s_kk, s_psum;
    __shared__ int s_nsup, s_mode;
    if (warp == 0) {
        const float af = (float)a;
        const float betaf = (float)beta;
        float tf = (float)tau_lo;
        // a few fp32 Newton steps from the left: only a pruning point, not a result
        for (int it = 0; it < 6; ++it) {
            float F0 = 0.f, F1 = 0.f, D0 = 0.f, D1 = 0.f;
            for (int k = lane; k < ncand; k += 64) {
                const float d0 = af * __uint_as_float((uint32_t)ck[k]) - tf;
                if (d0 > 0.f) { F0 += powbf(d0, betaf, ib); D0 += powbm1f(d0, betaf, ib); }
                if (k + 32 < ncand) {
                    const float d1 = af * __uint_as_float((uint32_t)ck[k + 32]) - tf;
                    if (d1 > 0.f) { F1 += powbf(d1, betaf, ib); D1 += powbm1f(d1, betaf, ib); }
                }
            }
            float F = F0 + F1, D = D0 + D1;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                F += __shfl_xor_sync(0xffffffffu, F, o);
                D += __shfl_xor_sync(0xffffffffu, D, o);
            }
            if (!(D > 0.f)) break;
            const float step = (float)lbeta_step((double)F, (double)D, beta, ib);
            tf += step;
            if (!(fabsf(step) > 1e-4f * fmaxf(1.0f, fabsf(tf)))) break;
        }
        stamp(6, 1);
        auto wsum2 = [&](double &x, double &y) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                x += __shfl_xor_sync(0xffffffffu, x, o);
                y += __shfl_xor_sync(0xffffffffu, y, o);
            }
        };
        // (b) list {z > base} with the fp64 mass F(base); an fp32 pre-test skips the
        // fp64 work of tokens far below base (conservative margin)
        auto build = [&](double base, double &F) -> int {
            int np = 0;
            double f = 0.0, dz = 0.0;
            const float bf = (float)base;
            const float bpre = bf - 1e-3f * fmaxf(1.0f, fabsf(bf));
            for (int k0 = 0; k0 < ncand; k0 += 32) {
                const int k = k0 + lane;
                const bool pre = k < ncand && af * __uint_as_float((uint32_t)ck[k]) > bpre;
                if (!__any_sync(0xffffffffu, pre)) continue;
                double z = 0.0;
                bool in = false;
                if (pre) {
                    z = ZOF(k);
                    const double d = z - base;
                    if (d > 0.0) { f += powb(d, beta, ib); in = true; }
                }
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                const int pos = np + __popc(bal & ((1u << lane) - 1u));
                if (in && pos < kPr) { zp[pos] = z; ip[pos] = k; }
                np += __popc(bal);
            }
            wsum2(f, dz);
            F = f;
            return np;
        };
        double base = (double)tf - 1e-4 * fmax(1.0, fabs((double)tf));
        double Fb = 0.0;
        int np = -1;
        if (base > tau_lo && tf == tf) {
            np = build(base, Fb);
            if (!(Fb >= 1.0)) np = -1;
        }
        if (np < 0) { base = tau_lo; np = build(base, Fb); }
        stamp(6, 2);
        const bool listed = np <= kPr;      // else: work on the whole candidate array
        const int nl = listed ? np : ncand;
#define ZL(i) (listed ? zp[i] : ZOF(i))
        for (int k = lane; k < ncand; k += 32) cin[k] = 0;
        __syncwarp();
        double tauN = base;
        int n_it = 0, amb = 0;
        if (listed && np <= 64) {
            // (c1) short list: the R9 criterion itself, F(z_j) = sum_i (z_i - z_j)_+^beta < 1,
            // for every entry (all pairs; z_i broadcast from shared memory)
            for (int i = lane; i < nl; i += 32) {
                const double zj = zp[i];
                double F = 0.0;
                for (int i2 = 0; i2 < nl; ++i2) {
                    const double d = zp[i2] - zj;
                    if (d > 0.0) F += powb(d, beta, ib);
                }
                cin[ip[i]] = (F < 1.0) ? 1 : 0;
            }
            __syncwarp();
            if (ib != 1 && ib != 2) {
                // Newton polish start for the general-beta tau below: the largest listed z
                // outside the support (or base) has F >= 1, i.e. lies left of tau
                double t0 = base, dz = 0.0;
                for (int i = lane; i < nl; i += 32)
                    if (!cin[ip[i]]) t0 = fmax(t0, zp[i]);
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) t0 = fmax(t0, __shfl_xor_sync(0xffffffffu, t0, o));
                tauN = t0;
                for (int it = 0; it < 60; ++it) {
                    double F = 0.0, Fd = 0.0;
                    for (int i = lane; i < nl; i += 32)
                        if (cin[ip[i]]) { const double d = zp[i] - tauN; F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
                    wsum2(F, Fd);
                    if (!(Fd > 0.0)) break;
                    const double step = lbeta_step(F, Fd, beta, ib);
                    tauN += step;
                    if (!(fabs(step) > 1e-15 * fmax(1.0, fabs(tauN)))) break;
                }
                (void)dz;
            }
        } else {
            // (c2) fp64 Newton from base (monotone from the left), then R9 with a band
            for (int it = 0; it < 200; ++it) {
                n_it = it + 1;
                double F = 0.0, Fd = 0.0;
                for (int i = lane; i < nl; i += 32) {
                    const double d = ZL(i) - tauN;
                    if (d > 0.0) { F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
                }
                wsum2(F, Fd);
                if (!(Fd > 0.0)) break;
                const double step = lbeta_step(F, Fd, beta, ib);
                tauN += step;
                // 1e-14 relative is far inside the support band (R9) and the final tau is
                // recomputed from the support; a tighter test can oscillate at the ulp level
                if (!(fabs(step) > 1e-14 * fmax(1.0, fabs(tauN))) || it >= 63) break;
            }
            stamp(6, 3);
            // support (R9): z > tau_N + band -> in, z < tau_N - band -> out, else F(z_j) < 1
            // (list entries only: every other candidate has z <= base <= tau)
            const double band = 1e-9 * fmax(1.0, fabs(tauN));
            for (int i = lane; i < nl; i += 32) {
                const double z = ZL(i);
                const uint8_t f = (z > tauN + band) ? 1 : (z < tauN - band) ? 0 : 2;
                cin[listed ? ip[i] : i] = f;
                amb += (f == 2);
            }
            amb = __reduce_add_sync(0xffffffffu, amb);
            __syncwarp();
            if (amb > 0) {
                for (int i0 = 0; i0 < nl; ++i0) {
                    const int k0 = listed ? ip[i0] : i0;
                    if (cin[k0] != 2) continue;
                    const double zk = ZL(i0);
                    double F = 0.0, dz = 0.0;
                    for (int i = lane; i < nl; i += 32) {
                        const double d = ZL(i) - zk;
                        if (d > 0.0) F += powb(d, beta, ib);
                    }
                    wsum2(F, dz);
                    __syncwarp();
                    if (lane == 0) cin[k0] = (F < 1.0) ? 1 : 0;
                    __syncwarp();
                }
            }
        }
#ifdef EKV_STAMPS
        if (blockIdx.x == 0 && lane == 0) {
            ekv_stamps[0][13] = (unsigned long long)n_it; ekv_stamps[0][12] = (unsigned long long)amb;
            ekv_stamps[0][11] = (unsigned long long)np;
        }
#endif
        stamp(6, 4);
        // tau from the support
        double S1 = 0.0, kk = 0.0;
        for (int i = lane; i < nl; i += 32)
            if (cin[listed ? ip[i] : i]) { S1 += ZL(i); kk += 1.0; }
        wsum2(S1, kk);
        double tau;
        if (ib == 1) {
            tau = (S1 - 1.0) / kk;
        } else if (ib == 2) {
            const double m = S1 / kk;
            double ss = 0.0, dz = 0.0;
            for (int i = lane; i < nl; i += 32)
                if (cin[listed ? ip[i] : i]) { const double d = ZL(i) - m; ss += d * d; }
            wsum2(ss, dz);
            tau = m - sqrt(fmax(0.0, 1.0 - ss) / kk);
        } else {
            double F = 0.0, Fd = 0.0;
            for (int i = lane; i < nl; i += 32)
                if (cin[listed ? ip[i] : i]) { const double d = ZL(i) - tauN; F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
            wsum2(F, Fd);
            tau = tauN + (F - 1.0) / (beta * Fd);
        }
        stamp(6, 5);
        // (d) support entries (list order) with p_j, if they fit the shared support arrays
        int nsup = 0;
        double psum = 0.0, dz = 0.0;
        if (listed && kk <= (double)kSup) {
            for (int i0 = 0; i0 < nl; i0 += 32) {
                const int i = i0 + lane;
                const int k = i < nl ? ip[i] : 0;
                const bool in = i < nl && cin[k];
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                const int pos = nsup + __popc(bal & ((1u << lane) - 1u));
                if (in) {
                    const int j = (int)(ck[k] >> 32);
                    const double d = zp[i] - tau;
                    const double pd = d > 0.0 ? powb(d, beta, ib) : 0.0;
                    sup_j[pos] = j;
                    sup_p[pos] = (float)pd;
                    sup_phys[pos] = have_phys ? cphys[k] : __ldg(c.page_table + (size_t)b * c.maxp + j / kP);
                    psum += pd;
                }
                nsup += __popc(bal);
            }
            wsum2(psum, dz);
        }
#undef ZL
        stamp(6, 6);
        if (lane == 0) {
            s_tau = tau; s_kk = kk; s_psum = psum; s_nsup = nsup;
            s_mode = (listed && kk <= (double)kSup) ? 1 : 0;
        }
    }
    stamp(0, 3);
    __syncthreads();
    const double tau = s_tau, kk = s_kk;
    stamp(0, 4);
    // ---- PV: warp w gathers support entries w, w + NW, ... (4 V rows in flight per warp)
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    double psum = 0.0;
    auto gather = [&](int nsup) {
        for (int e0 = warp; e0 < nsup; e0 += 4 * NW) {
            float vx[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * NW;
                if (e < nsup) {
                    const int j = sup_j[e];
                    ldv4<T>(Vb + (((size_t)sup_phys[e] * c.Hkv + kvh) * kP + (j % kP)) * kD + 4 * lane, vx[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * NW;
                if (e < nsup) {
                    const float p = sup_p[e];
#pragma unroll
                    for (int q2 = 0; q2 < 4; ++q2) acc[q2] = __fmaf_rn(p, vx[u][q2], acc[q2]);
                }
            }
        }
    };
    if (s_mode == 1) {
        gather(s_nsup);
        if (threadIdx.x == 0) psum = s_psum;
    } else {
        // large support: compacted in candidate order, rounds of kSup entries
        for (int r0 = 0; r0 < ncand;) {
            int nsup = 0, r1 = r0;
            while (r1 < ncand) {
                const int k = r1 + threadIdx.x;
                const bool in = k < ncand && cin[k];
                int tot;
                const int pos = nsup + block_excl_scan<NT>(in ? 1 : 0, shi, &tot);
                if (nsup + tot > kSup) break;             // uniform
                if (in) {
                    const int j = (int)(ck[k] >> 32);
                    const double d = ZOF(k) - tau;
                    const double pd = d > 0.0 ? powb(d, beta, ib) : 0.0;
                    sup_j[pos] = j;
                    sup_p[pos] = (float)pd;
                    sup_phys[pos] = have_phys ? cphys[k] : __ldg(c.page_table + (size_t)b * c.maxp + j / kP);
                    psum += pd;
                }
                nsup += tot;
                r1 += NT;
            }
            __syncthreads();
            gather(nsup);
            __syncthreads();
            r0 = r1;
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) red[warp][4 * lane + e] = acc[e];
    double pz = 0.0;
    R.sum(psum, pz);
    if (threadIdx.x < kD) {
        float o = 0.f;
        for (int w = 0; w < NW; ++w) o = __fadd_rn(o, red[w][threadIdx.x]);
        A.out[(size_t)row * kD + threadIdx.x] = (float)((double)o / psum);
    }
    if (threadIdx.x == 0) {
        if (A.tau_out) A.tau_out[row] = tau;
        if (A.supp_out) A.supp_out[row] = (int)kk;
    }
    stamp(0, 5);
    // ---- eval list: support token positions and p (for exact delta / rho)
    if (A.tok_list) {
        int base = 0;
        for (int r0 = 0; r0 < ncand; r0 += NT) {
            const int k = r0 + threadIdx.x;
            const int keep = (k < ncand && cin[k]) ? 1 : 0;
            int tot;
            const int pos = block_excl_scan<NT>(keep, shi, &tot);
            if (keep && base + pos < A.list_cap) {
                const double d = ZOF(k) - tau;
                A.tok_list[(size_t)row * A.list_cap + base + pos] = (int32_t)(ck[k] >> 32);
                A.p_list[(size_t)row * A.list_cap + base + pos] = d > 0.0 ? powb(d, beta, ib) : 0.0;
            }
            base += tot;
        }
        if (threadIdx.x == 0) A.n_list[row] = base;
    }
#undef ZOF
    stamp(0, 6);
}

// ============================================================================ a4: certified delta_bar
// delta_bar = sum_{p not in C_page} c_p [a * box_p - tau~]_+^beta  (R16; Prop. B.1 gives
// z_j <= a * box_p, and tau >= tau~).  Grid (chunk of 2048 pages, b * Hq + h): each CTA
// marks its row's selected pages of the chunk in a shared bitmap, sums its chunk
// (deterministic block tree) into partial[row][chunk]; the last CTA of a row (ticket
// counter) adds the partials in chunk order, so the result is deterministic.
constexpr int kDbChunk = 8192;   // pages per CTA: 256 threads x 8 groups of 4 pages
struct DbConst {                 // per-call constants of alpha (host-computed)
    double a, beta, inv_a;       // a = alpha - 1, beta = 1/a
    int ib;                      // integer beta in 1..4, else 0
};
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
    const double t = __ldg(tau + row);
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
__global__ void __launch_bounds__(256) k_eval_metrics(const int32_t *__restrict__ tok_list, const double *__restrict__ p_list,
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
