// kernels_dense.cuh -- a6 (softmax over the same kernels) and the dense-V pass of the a5
// full-cache baseline: split flash-decoding style partials + an ordered combine.
#pragma once
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
        // warp w: list pages i0 + w, i0 + w + 8, ...; the 16 tokens of a page, 4 V rows in flight
        for (int ii = i0 + warp; ii < min(nlist, i0 + kSmxPages); ii += 8) {
            const int pg = full ? ii : __ldg(page_idx + (size_t)row * stride + ii);
            const int phys = __ldg(c.page_table + (size_t)b * c.maxp + pg);
            const float sv = (lane < kP) ? srow[(size_t)pg * kP + lane] : -INFINITY;
            const T *vp = Vb + ((size_t)phys * c.Hkv + kvh) * kP * kD + 4 * lane;
#pragma unroll 4
            for (int t = 0; t < kP; ++t) {
                const float s = __shfl_sync(0xffffffffu, sv, t);
                if (pg * kP + t >= L || s == -INFINITY) continue;        // warp-uniform
                float p;
                if (ent_tau) {
                    const double a = (double)alpha - 1.0, d = a * (double)s - ent_tau[row];
                    p = d > 0.0 ? (float)pow(d, 1.0 / a) : 0.0f;
                } else {
                    p = expf(s - smax);
                }
                float vx[4];
                ldv4<T>(vp + (size_t)t * kD, vx);
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = __fmaf_rn(p, vx[q], acc[q]);
                if (lane == 0) { l += (double)p; ++cnt; }
            }
        }
    }
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

static __global__ void __launch_bounds__(128) k_softmax_combine(const float *__restrict__ pacc, const double *__restrict__ pl,
                                                         const int32_t *__restrict__ pcnt, const uint32_t *__restrict__ rowmax,
                                                         int nch, float *__restrict__ out, double *__restrict__ tau,
                                                         int32_t *__restrict__ supp) {
    pdl_enter();
    const int row = blockIdx.x;
    const uint32_t mk = rowmax[row];
    float o = 0.f;
    double l = 0.0;
    int cnt = 0;
    for (int ch = 0; ch < nch; ++ch) {
        const size_t i = (size_t)row * nch + ch;
        o = __fadd_rn(o, pacc[i * kD + threadIdx.x]);
        l += pl[i];
        cnt += pcnt[i];
    }
    out[(size_t)row * kD + threadIdx.x] = (mk && l > 0.0) ? (float)((double)o / l) : 0.0f;
    if (threadIdx.x == 0) {             // (entmax dense-V: tau / supp come from the tau kernel)
        if (tau) tau[row] = mk ? (double)key2f(mk) + log(l) : NAN;
        if (supp) supp[row] = cnt;
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
template <typename T, int G>
__global__ void __launch_bounds__(256, 2) k_dense_group_partial(CacheView c, const float *__restrict__ scores, size_t ntok,
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
        float sv[G];
#pragma unroll
        for (int g = 0; g < G; ++g) sv[g] = (lane < kP) ? scores[(size_t)(row0 + g) * ntok + (size_t)pg * kP + lane] : -INFINITY;
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
                const float s = __shfl_sync(0xffffffffu, sv[g], t);
                float p = 0.f;
                double w = 0.0;
                if (live[g] && t < nt && s != -INFINITY) {
                    if (ent_tau) {
                        const double d = a * (double)s - tau[g];
                        if (d > 0.0) {
                            if (ib == 1) w = d;
                            else if (ib == 2) w = d * d;
                            else if (ib == 3) w = d * d * d;
                            else if (ib == 4) { const double d2 = d * d; w = d2 * d2; }
                            else w = pow(d, 1.0 / a);
                        }
                        p = (float)w;
                    } else {
                        p = expf(s - smax[g]);
                        w = (double)p;
                    }
                }
                if (cdim == 0) l[g] += w;
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
        l[g] += __shfl_xor_sync(0xffffffffu, l[g], 16);
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
