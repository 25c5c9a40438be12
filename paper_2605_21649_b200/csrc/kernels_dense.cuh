// kernels_dense.cuh -- a6 (softmax over the same kernels) and the dense-V pass of the a5
// full-cache baseline: split flash-decoding style partials + an ordered combine.
#pragma once
#include <type_traits>
#include "kernels_attend.cuh"

namespace ekv {
// ============================================================================ a6: softmax rows
// Softmax over C_tok (the Quest-style baseline on the same kernels): dense
// V over every valid token of the page list, split flash-decoding style.  The row maximum is
// already known (the K-score pass's rowmax), so the chunk partials need no rescaling:
// p_j = exp(s_j - s_max); chunk c of kSmxPages list pages -> acc[c][dv] = sum p_j v_j (fp32),
// l[c] = sum p_j (fp64); k_softmax_combine adds the chunks in order (deterministic).
// The same split dense-V pass serves the dense-V full-cache entmax baseline (the
// reference reads all scores and V): weights p_j = ((alpha-1) s_j - tau)_+^beta in fp64 from
// the row's exact tau (ent_tau != NULL), every V row streamed whether p_j is zero or not.
template <typename T>
__global__ void __launch_bounds__(256) k_softmax_partial(CacheView c, const float *__restrict__ scores, size_t ntok,
                                                         const uint32_t *__restrict__ rowmax,
                                                         const int32_t *__restrict__ page_idx,
                                                         const int32_t *__restrict__ n_sel, int stride, int full,
                                                         int Hq, int G, int nch, float *__restrict__ pacc,
                                                         double *__restrict__ pl, int32_t *__restrict__ pcnt,
                                                         const double *__restrict__ ent_tau, float alpha) {
    pdl_enter();
    __shared__ float red[8][kD];
    __shared__ double wl[8];
    __shared__ int wc[8];
    const int row = blockIdx.y, ch = blockIdx.x;
    const int b = row / Hq, kvh = (row % Hq) / G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int L = __ldg(c.seq_lens + b);
    const int nlist = full ? n_pages_of(L) : __ldg(n_sel + row);
    const uint32_t mk = __ldg(rowmax + row);
    const float smax = mk ? key2f(mk) : 0.f;
    const float *srow = scores + (size_t)row * ntok;
    const T *Vb = reinterpret_cast<const T *>(c.V);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    double l = 0.0;
    int cnt = 0;
    const int i0 = ch * kSmxPages;
    if (mk && i0 < nlist) {
        // warp w: list pages i0 + w, i0 + w + 8, ...; per page the 16 tokens' weights are
        // computed once (lane t: token t) and broadcast, and all 16 V rows are in flight at once
        for (int ii = i0 + warp; ii < min(nlist, i0 + kSmxPages); ii += 8) {
            const int pg = full ? ii : __ldg(page_idx + (size_t)row * stride + ii);
            const int phys = __ldg(c.page_table + (size_t)b * c.maxp + pg);
            const int tl = lane & (kP - 1);
            const float sv = srow[(size_t)pg * kP + tl];
            const bool tv = lane < kP && pg * kP + tl < L && sv != -INFINITY;
            float pw = 0.f;
            if (tv) {
                if (ent_tau) {
                    const double a = (double)alpha - 1.0, d = a * (double)sv - ent_tau[row];
                    pw = d > 0.0 ? (float)pow(d, 1.0 / a) : 0.0f;
                } else {
                    pw = expf(sv - smax);
                }
                l += (double)pw;
                ++cnt;
            }
            const T *vp = Vb + ((size_t)phys * c.Hkv + kvh) * kP * kD + 4 * lane;
            const int nt = min(kP, L - pg * kP);
            using W = typename std::conditional<sizeof(T) == 2, uint2, float4>::type;
            W raw[kP];
#pragma unroll
            for (int t = 0; t < kP; ++t)
                if (t < nt) raw[t] = *reinterpret_cast<const W *>(vp + (size_t)t * kD);
#pragma unroll
            for (int t = 0; t < kP; ++t) {
                const float p = __shfl_sync(0xffffffffu, pw, t);
                if (t < nt && p != 0.f) {
                    float vx[4];
                    if constexpr (sizeof(T) == 2) {
                        vx[0] = bf_lo(raw[t].x); vx[1] = bf_hi(raw[t].x); vx[2] = bf_lo(raw[t].y); vx[3] = bf_hi(raw[t].y);
                    } else {
                        vx[0] = raw[t].x; vx[1] = raw[t].y; vx[2] = raw[t].z; vx[3] = raw[t].w;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[q] = __fmaf_rn(p, vx[q], acc[q]);
                }
            }
        }
    }
    // per-token weights and counts were taken by lanes 0..15
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) { l += __shfl_xor_sync(0xffffffffu, l, o); cnt += __shfl_xor_sync(0xffffffffu, cnt, o); }
#pragma unroll
    for (int q = 0; q < 4; ++q) red[warp][4 * lane + q] = acc[q];
    if (lane == 0) { wl[warp] = l; wc[warp] = cnt; }
    __syncthreads();
    const size_t o = (size_t)row * nch + ch;
    if (threadIdx.x < kD) {
        float s = 0.f;
        for (int w = 0; w < 8; ++w) s = __fadd_rn(s, red[w][threadIdx.x]);
        pacc[o * kD + threadIdx.x] = s;
    }
    if (threadIdx.x == 0) {
        double sl = 0.0;
        int sc = 0;
        for (int w = 0; w < 8; ++w) { sl += wl[w]; sc += wc[w]; }
        pl[o] = sl;
        pcnt[o] = sc;
    }
}

// Ordered combine of the chunk partials: kCombSeg segments of the chunk range per row, one
// thread per (segment, dim); the segment sums are added in segment order (deterministic).
constexpr int kCombSeg = 8;
static __global__ void __launch_bounds__(128 * kCombSeg) k_softmax_combine(const float *__restrict__ pacc, const double *__restrict__ pl,
                                                         const int32_t *__restrict__ pcnt, const uint32_t *__restrict__ rowmax,
                                                         int nch, float *__restrict__ out, double *__restrict__ tau,
                                                         int32_t *__restrict__ supp) {
    pdl_enter();
    __shared__ float so[kCombSeg][kD];
    __shared__ double sl[kCombSeg];
    __shared__ int sc[kCombSeg];
    const int row = blockIdx.x;
    const int d = threadIdx.x % kD, seg = threadIdx.x / kD;
    const int c0 = nch * seg / kCombSeg, c1 = nch * (seg + 1) / kCombSeg;
    float o = 0.f;
    double l = 0.0;
    int cnt = 0;
#pragma unroll 8
    for (int ch = c0; ch < c1; ++ch) {
        const size_t i = (size_t)row * nch + ch;
        o = __fadd_rn(o, pacc[i * kD + d]);
        if (d == 0) { l += pl[i]; cnt += pcnt[i]; }
    }
    so[seg][d] = o;
    if (d == 0) { sl[seg] = l; sc[seg] = cnt; }
    __syncthreads();
    if (seg == 0) {
        const uint32_t mk = rowmax[row];
        float ot = 0.f;
        double lt = 0.0;
        int ct = 0;
        for (int q = 0; q < kCombSeg; ++q) { ot = __fadd_rn(ot, so[q][d]); lt += sl[q]; ct += sc[q]; }
        out[(size_t)row * kD + d] = (mk && lt > 0.0) ? (float)((double)ot / lt) : 0.0f;
        if (d == 0) {                     // (entmax dense-V: tau / supp come from the tau kernel)
            if (tau) tau[row] = mk ? (double)key2f(mk) + log(lt) : NAN;
            if (supp) supp[row] = ct;
        }
    }
}
}  // namespace ekv

namespace ekv {
// 8 dims of one V row (lane chunk c) -> fp32
template <typename T> __device__ __forceinline__ void ldv8(const T *p, float (&x)[8]) { Elem<T>::load8(p, x); }

// Full rows (every page, every head of the group): one CTA per (chunk, KV unit) streams each
// V row ONCE for the G heads of the group (weights from the G score rows): softmax p =
// exp(s - s_max), entmax p = ((alpha-1) s - tau)_+^beta with integer beta by products.
// Layout for memory-level parallelism: a warp takes a page; lane = (token parity h, 8-dim
// chunk c): its 8 loads of 16 bytes (tokens 2 i + h) go out together, then the weights.
// Writes the same per-(row, chunk) partials as k_softmax_partial.
#ifndef EKV_DG_CTAS
#define EKV_DG_CTAS 2
#endif
template <typename T, int G>
__global__ void __launch_bounds__(256, EKV_DG_CTAS) k_dense_group_partial(CacheView c, const float *__restrict__ scores, size_t ntok,
                                                             const uint32_t *__restrict__ rowmax, int Hq, int nch,
                                                             float *__restrict__ pacc, double *__restrict__ pl,
                                                             int32_t *__restrict__ pcnt,
                                                             const double *__restrict__ ent_tau, float alpha, int ib) {
    pdl_enter();
    __shared__ float red[8][kD];
    __shared__ double wl[8][G];
    __shared__ int wc[8];
    const int unit = blockIdx.y, ch = blockIdx.x;
    const int b = unit / c.Hkv, kvh = unit % c.Hkv;
    const int row0 = b * Hq + kvh * G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int hpar = lane >> 4, cdim = lane & 15;
    const int L = __ldg(c.seq_lens + b);
    const int nlist = n_pages_of(L);
    const double a = (double)alpha - 1.0;
    float smax[G];
    double tau[G];
    bool live[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const uint32_t mk = __ldg(rowmax + row0 + g);
        live[g] = mk != 0u;
        smax[g] = mk ? key2f(mk) : 0.f;
        tau[g] = ent_tau ? ent_tau[row0 + g] : 0.0;
    }
    const T *Vb = reinterpret_cast<const T *>(c.V);
    float acc[G][8];
    double l[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        l[g] = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[g][i] = 0.f;
    }
    int cnt = 0;
    const int i0 = ch * kSmxPages;
    for (int pg = i0 + warp; pg < min(nlist, i0 + kSmxPages); pg += 8) {
        const int phys = __ldg(c.page_table + (size_t)b * c.maxp + pg);
        const int nt = min(kP, L - pg * kP);
        // the page's weights once per (token, head): lane l computes token l % 16 for every head
        // (both lane halves: no shuffle to fill the upper half), the token loop broadcasts them
        const int tw = lane & (kP - 1);
        float pw[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float s = scores[(size_t)(row0 + g) * ntok + (size_t)pg * kP + tw];
            float p = 0.f;
            if (live[g] && tw < nt && s != -INFINITY) {
                if (ent_tau) {
                    const double d = a * (double)s - tau[g];
                    double w = 0.0;
                    if (d > 0.0) {
                        if (ib == 1) w = d;
                        else if (ib == 2) w = d * d;
                        else if (ib == 3) w = d * d * d;
                        else if (ib == 4) { const double d2 = d * d; w = d2 * d2; }
                        else w = pow(d, 1.0 / a);
                    }
                    p = (float)w;
                    if (lane < kP) l[g] += w;
                } else {
                    p = expf(s - smax[g]);
                    if (lane < kP) l[g] += (double)p;
                }
            }
            pw[g] = p;
        }
        const T *vp = Vb + ((size_t)phys * c.Hkv + kvh) * kP * kD + 8 * cdim;
        // raw 16-byte words in flight (bf16: 8 dims; fp32: 4 dims, two words per row)
        constexpr int WPR = sizeof(T) == 2 ? 1 : 2;
        uint4 raw[kP / 2][WPR];
#pragma unroll
        for (int i = 0; i < kP / 2; ++i) {                                  // every V row is read
            const int t = 2 * i + hpar;
#pragma unroll
            for (int w = 0; w < WPR; ++w)
                raw[i][w] = (t < nt) ? __ldg(reinterpret_cast<const uint4 *>(vp + (size_t)t * kD) + w) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < kP / 2; ++i) {
            const int t = 2 * i + hpar;
            float vx[1][8];
            if constexpr (sizeof(T) == 2) {
                vx[0][0] = bf_lo(raw[i][0].x); vx[0][1] = bf_hi(raw[i][0].x); vx[0][2] = bf_lo(raw[i][0].y);
                vx[0][3] = bf_hi(raw[i][0].y); vx[0][4] = bf_lo(raw[i][0].z); vx[0][5] = bf_hi(raw[i][0].z);
                vx[0][6] = bf_lo(raw[i][0].w); vx[0][7] = bf_hi(raw[i][0].w);
            } else {
                const uint4 r0 = raw[i][0], r1 = raw[i][WPR - 1];
                vx[0][0] = __uint_as_float(r0.x); vx[0][1] = __uint_as_float(r0.y); vx[0][2] = __uint_as_float(r0.z);
                vx[0][3] = __uint_as_float(r0.w); vx[0][4] = __uint_as_float(r1.x); vx[0][5] = __uint_as_float(r1.y);
                vx[0][6] = __uint_as_float(r1.z); vx[0][7] = __uint_as_float(r1.w);
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float p = __shfl_sync(0xffffffffu, pw[g], t);
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[g][e] = __fmaf_rn(p, vx[0][e], acc[g][e]);
            }
        }
        if (lane == 0) cnt += nt;
    }
    // fold the two token parities (lanes c and c + 16), then the warps in fixed order
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[g][e] = __fadd_rn(acc[g][e], __shfl_xor_sync(0xffffffffu, acc[g][e], 16));
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) l[g] += __shfl_xor_sync(0xffffffffu, l[g], o);   // lanes 0..15: a token each
    }
    for (int g = 0; g < G; ++g) {
        if (lane < 16) {
#pragma unroll
            for (int e = 0; e < 8; ++e) red[warp][8 * cdim + e] = acc[g][e];
        }
        if (lane == 0) wl[warp][g] = l[g];
        __syncthreads();
        const size_t o = (size_t)(row0 + g) * nch + ch;
        if (threadIdx.x < kD) {
            float sacc = 0.f;
            for (int w = 0; w < 8; ++w) sacc = __fadd_rn(sacc, red[w][threadIdx.x]);
            pacc[o * kD + threadIdx.x] = sacc;
        }
        if (threadIdx.x == 0) {
            double sl = 0.0;
            for (int w = 0; w < 8; ++w) sl += wl[w][g];
            pl[o] = sl;
        }
        __syncthreads();
    }
    if (lane == 0) wc[warp] = cnt;
    __syncthreads();
    if (threadIdx.x < G) {
        int sc = 0;
        for (int w = 0; w < 8; ++w) sc += wc[w];
        pcnt[(size_t)(row0 + threadIdx.x) * nch + ch] = sc;
    }
}
}  // namespace ekv

namespace ekv {
// ============================================================================ a5 dense-V: the V stream
// The dense-V full-cache baseline reads every V row, as the paper's reference does (it
// "reads all scores and V").  Its output equals the support-V variant's (p_j = 0 off the
// support), so the tau kernel's exact PV over the support gives out, and this kernel streams
// the whole V of every valid page once: a warp takes one (b, page) -- the page's Hkv tiles are
// contiguous (Hkv * P * dv elements) -- with 8 x 16-byte loads per lane in flight, folding the
// words into an xor checksum (one atomic per warp into `sink`) so the reads are real work.
template <typename T>
__global__ void __launch_bounds__(256) k_vstream(CacheView c, uint32_t *__restrict__ sink) {
    pdl_enter();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long total = (long long)c.B * c.maxp;
    const long long wtot = (long long)gridDim.x * 8;
    const int n16 = c.Hkv * kP * kD * (int)sizeof(T) / 16;
    const uint4 *V = reinterpret_cast<const uint4 *>(c.V);
    uint32_t x = 0u;
    for (long long sl = (long long)blockIdx.x * 8 + warp; sl < total; sl += wtot) {
        const int b = (int)(sl / c.maxp), p = (int)(sl % c.maxp);
        if (p >= n_pages_of(__ldg(c.seq_lens + b))) continue;               // warp-uniform
        const uint4 *src = V + (size_t)__ldg(c.page_table + (size_t)b * c.maxp + p) * n16;
        for (int i0 = 0; i0 < n16; i0 += 32 * 8) {
            uint4 r[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + 32 * u + lane;
                r[u] = i < n16 ? __ldcs(src + i) : make_uint4(0, 0, 0, 0);    // streaming (evict-first)
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) x ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
        }
    }
    x = __reduce_xor_sync(0xffffffffu, x);
    if (lane == 0) atomicXor(sink, x);
}
}  // namespace ekv


namespace ekv {
// ============================================================================ a5: full-cache K scores on tensor cores
// The full-cache baseline's score pass (every token of every page, G heads of a KV group) as a
// dense bf16 contraction: per 16-token page tile, S[16 tok][8 heads] = K[16][128] q^T[128][8]
// with mma.sync m16n8k16 (bf16 x bf16 -> fp32; heads >= G are zero columns).  Products are
// exact; the accumulation is the tensor core's own (not R1's order), so these scores are the
// baseline's, not bit-identical to the oracle's -- DESIGN R26 (the sparse path keeps R1).
// A warp owns a contiguous range of (unit, page) slots; tiles arrive by cp.async (16-byte
// chunks, chunk index XOR (row & 7): ldmatrix reads conflict-free), double-buffered per warp.
__device__ __forceinline__ void cpa16(void *s, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
template <int G>
__global__ void __launch_bounds__(256, 3) k_full_scores_mma(CacheView c, const __nv_bfloat16 *__restrict__ q, int Hq,
                                                            float *__restrict__ scores, uint32_t *__restrict__ rowmax) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char fsm[];       // [8 warps][2][4096]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    unsigned char *buf = fsm + (size_t)warp * 2 * 4096;
    const long long total = (long long)c.B * c.Hkv * c.maxp;
    const long long wtot = (long long)gridDim.x * 8, wid = (long long)blockIdx.x * 8 + warp;
    const long long s0 = total * wid / wtot, s1 = total * (wid + 1) / wtot;
    const size_t ntok = (size_t)c.maxp * kP;
    const unsigned char *Kb = reinterpret_cast<const unsigned char *>(c.K);
    // slot -> (unit, page); valid pages only (others skipped)
    auto valid = [&](long long sl, int &unit, int &pg, int &L) -> bool {
        unit = (int)(sl / c.maxp); pg = (int)(sl % c.maxp);
        L = __ldg(c.seq_lens + unit / c.Hkv);
        return pg < n_pages_of(L);
    };
    auto issue = [&](long long sl, int slot) {
        int unit, pg, L;
        if (sl >= s1 || !valid(sl, unit, pg, L)) return;
        const int b = unit / c.Hkv, kvh = unit % c.Hkv;
        const size_t phys = (size_t)__ldg(c.page_table + (size_t)b * c.maxp + pg);
        const unsigned char *src = Kb + (phys * c.Hkv + kvh) * 4096;
        unsigned char *dst = buf + slot * 4096;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int ch = lane + 32 * u;                  // 16-byte chunk: row r = ch / 16, col chunk cc = ch % 16
            const int r = ch >> 4, cc = ch & 15;
            cpa16(dst + r * 256 + ((cc ^ (r & 7)) << 4), src + ch * 16);
        }
    };
    int cur_unit = -1;
    uint32_t bq[8][2];                                    // B fragments of q (8 k-steps)
    float hmax0 = -INFINITY, hmax1 = -INFINITY;          // running maxima of heads 2 tig, 2 tig + 1
    auto flush = [&](int unit) {
        if (unit < 0) return;
        float m0 = hmax0, m1 = hmax1;
#pragma unroll
        for (int o = 4; o <= 16; o <<= 1) {
            m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
            m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
        }
        const int row0 = (unit / c.Hkv) * Hq + (unit % c.Hkv) * G;
        if (gid == 0) {
            if (2 * tig < G && m0 > -INFINITY) atomicMax(rowmax + row0 + 2 * tig, f2key(m0));
            if (2 * tig + 1 < G && m1 > -INFINITY) atomicMax(rowmax + row0 + 2 * tig + 1, f2key(m1));
        }
        hmax0 = hmax1 = -INFINITY;
    };
    issue(s0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    int slot = 0;
    for (long long sl = s0; sl < s1; ++sl, slot ^= 1) {
        issue(sl + 1, slot ^ 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        int unit, pg, L;
        if (valid(sl, unit, pg, L)) {                      // warp-uniform
            if (unit != cur_unit) {
                flush(cur_unit);
                cur_unit = unit;
                const int qrow = (unit / c.Hkv) * Hq + (unit % c.Hkv) * G + gid;   // head n = gid
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if (gid < G) {
                        const uint32_t *qp = reinterpret_cast<const uint32_t *>(q + (size_t)qrow * kD + kk * 16 + 2 * tig);
                        bq[kk][0] = __ldg(qp);
                        bq[kk][1] = __ldg(qp + 4);
                    } else {
                        bq[kk][0] = bq[kk][1] = 0u;
                    }
                }
            }
            const unsigned char *tile = buf + slot * 4096;
            float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                // ldmatrix.x4: matrix m = lane / 8 -> rows (lane % 8) + 8 (m & 1), chunk 2 kk + (m >> 1)
                const int m = lane >> 3, r = (lane & 7) + 8 * (m & 1), cc = 2 * kk + (m >> 1);
                const uint32_t addr = smem_u32(tile + r * 256 + ((cc ^ (r & 7)) << 4));
                uint32_t a0, a1, a2, a3;
                asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                             : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(addr));
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                             "{%0,%1,%2,%3};"
                             : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bq[kk][0]), "r"(bq[kk][1]));
            }
            // d0, d1: token gid, heads 2 tig, 2 tig + 1; d2, d3: token gid + 8
            const int row0 = (unit / c.Hkv) * Hq + (unit % c.Hkv) * G;
            const int t0 = pg * kP + gid, t1 = t0 + 8;
            const float s00 = t0 < L ? __fmul_rn(d0, kCd) : -INFINITY, s01 = t0 < L ? __fmul_rn(d1, kCd) : -INFINITY;
            const float s10 = t1 < L ? __fmul_rn(d2, kCd) : -INFINITY, s11 = t1 < L ? __fmul_rn(d3, kCd) : -INFINITY;
            if (2 * tig < G) {
                float *sr = scores + (size_t)(row0 + 2 * tig) * ntok;
                sr[t0] = s00; sr[t1] = s10;
                hmax0 = fmaxf(hmax0, fmaxf(s00, s10));
            }
            if (2 * tig + 1 < G) {
                float *sr = scores + (size_t)(row0 + 2 * tig + 1) * ntok;
                sr[t0] = s01; sr[t1] = s11;
                hmax1 = fmaxf(hmax1, fmaxf(s01, s11));
            }
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    flush(cur_unit);
}
}  // namespace ekv
