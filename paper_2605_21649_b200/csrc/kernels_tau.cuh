// kernels_tau.cuh -- a3 hot path: exact alpha-entmax threshold, support and weighted V
// sum of one (b, q-head) row over its selected pages (sparse decode, R8-R12).
// The general kernel k_tau_pv (kernels_attend.cuh) serves full rows, softmax rows and the
// eval lists; this lean kernel serves the decode step's sparse entmax rows, with the
// integer beta = 1/(alpha-1) a compile-time constant (IB in 1..4; 0 = any other alpha).
//
// One CTA (256 threads) per row.  Work is shaped around latency (one CTA per row, few
// rows): every pass over the candidates is block-parallel, and only the short exact phase
// runs on one warp.
// Global-memory round trips dominate (~1 us each), so the kernel issues every independent
// load up front: row max, list length and the page list of the first round (12 items of
// 4 scores per thread: 768 pages) go out together, then the scores and page-table entries.
//  1. Candidates {j in C_tok : z_j > tau_lo = z_max - 1} (tau >= z_max - 1 since
//     F(z_max - 1) >= 1): fp32 pre-test then the fp64 test, block-scan compaction (fixed
//     order: deterministic sums below).
//  2. fp32 Newton steps on ||(z - t)_+||_beta - 1 from tau_lo (block sums): a pruning
//     point t32 only -- nothing is decided in fp32.
//  3. base = t32 - 1e-4 max(1, |t32|) is kept iff F(base) >= 1 in fp64 (then tau >= base
//     because F decreases); else base = tau_lo.  The list {z > base} (z in fp64) is
//     compacted in candidate order.  Every candidate outside it has z <= base <= tau,
//     i.e. F(z) >= 1: not in the support (R9).
//     The V rows of a short list (<= 64 entries) are copied to shared memory now
//     (cp.async), overlapping step 4.
//  4. Support by R9 itself: short lists (<= 32, beta = 1 or 2): F(z_j) = sum_i (z_i -
//     z_j)_+^beta < 1 for every entry, all pairs over the whole block (8 threads per entry),
//     tau from the support's closed form by block sums.  Otherwise warp 0: all pairs (<= 64)
//     or fp64 Newton from base, then z > tau_N + band in, z < tau_N - band out, F(z_j) < 1
//     in between; tau by the closed forms (beta = 1, 2) or Newton on the support.
//  5. PV: p_j = (z_j - tau)^beta; warps accumulate p_j v_j (V from shared memory for short
//     lists, else gathered, 4 rows in flight per warp; lane = 4 dims);
//     out = sum p_j v_j / sum p_j (R12).
// Overflow (more candidates than shared memory): fp64 Newton streamed over the score row
// raises tau_lo to just below tau, then the extraction is repeated.
#pragma once
#include <cooperative_groups.h>
#include "kernels_attend.cuh"

namespace ekv {

template <int IB> __device__ __forceinline__ double powB(double x, double beta) {
    if constexpr (IB == 1) return x;
    else if constexpr (IB == 2) return x * x;
    else if constexpr (IB == 3) return (x * x) * x;
    else if constexpr (IB == 4) { const double x2 = x * x; return x2 * x2; }
    else return pow(x, beta);
}
template <int IB> __device__ __forceinline__ double powBm1(double x, double beta) {
    if constexpr (IB == 1) return 1.0;
    else if constexpr (IB == 2) return x;
    else if constexpr (IB == 3) return x * x;
    else if constexpr (IB == 4) return (x * x) * x;
    else return pow(x, beta - 1.0);
}
template <int IB> __device__ __forceinline__ float powBf(float x, float beta) {
    if constexpr (IB == 1) return x;
    else if constexpr (IB == 2) return x * x;
    else if constexpr (IB == 3) return (x * x) * x;
    else if constexpr (IB == 4) { const float x2 = x * x; return x2 * x2; }
    else return __powf(x, beta);
}
template <int IB> __device__ __forceinline__ float powBm1f(float x, float beta) {
    if constexpr (IB == 1) return 1.0f;
    else if constexpr (IB == 2) return x;
    else if constexpr (IB == 3) return x * x;
    else if constexpr (IB == 4) return (x * x) * x;
    else return __powf(x, beta - 1.0f);
}

// deterministic block sum of two floats (fixed order; alternating buffers: one barrier)
template <int NT> struct BlockRed2f {
    float *buf;   // [2][2 * NT/32]
    int ph;
    __device__ __forceinline__ void sum(float &a, float &b) {
        constexpr int NW = NT / 32;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        float *s = buf + ph * 2 * NW;
        ph ^= 1;
        if ((threadIdx.x & 31) == 0) { s[2 * (threadIdx.x >> 5)] = a; s[2 * (threadIdx.x >> 5) + 1] = b; }
        __syncthreads();
        float x = 0.f, y = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) { x += s[2 * w]; y += s[2 * w + 1]; }
        a = x; b = y;
    }
};

__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// FULL: full-cache rows (candidates from k_candidates' chunk regions, eval lists); the decode
// path instantiates FULL = false, which keeps only the sparse code (less instruction fetch:
// the kernel runs once per step on cold instruction caches)
// Overflow path of k_tau_sparse: fp64 Newton on ||(z - t)_+||_beta - 1 streamed over the
// whole list
template <int NT, int IB>
__device__ __noinline__ double streamed_newton(const float *srow, const int32_t *plist, bool full, int nlist, int L,
                                               double a, double beta, double t0, BlockRed2<NT> &Rd) {
    // (items of 4 scores, 8 in flight per thread: the row is read from L2 once per pass)
    const int nit = nlist * 4;
    double t = t0;
    for (int it = 0; it < 200; ++it) {
        double F = 0.0, Fd = 0.0;
        for (int r0 = 0; r0 < nit; r0 += 8 * NT) {
            int pv[8];
            float4 v4[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = r0 + threadIdx.x + NT * u;
                pv[u] = e < nit ? (full ? (e >> 2) : __ldg(plist + (e >> 2))) : -1;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = r0 + threadIdx.x + NT * u;
                if (pv[u] >= 0) v4[u] = *reinterpret_cast<const float4 *>(srow + (size_t)pv[u] * kP + 4 * (e & 3));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (pv[u] < 0) continue;
                const int e = r0 + threadIdx.x + NT * u;
                const int j0 = pv[u] * kP + 4 * (e & 3);
                const float sv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double d = a * (double)sv[q] - t;
                    if (j0 + q < L && d > 0.0) { F += powB<IB>(d, beta); Fd += powBm1<IB>(d, beta); }
                }
            }
        }
        Rd.sum(F, Fd);
        if (!(Fd > 0.0)) break;
        const double step = lbeta_step(F, Fd, beta, IB);
        t += step;
        if (!(fabs(step) > 1e-12 * fmax(1.0, fabs(t)))) break;
    }
    return t;
}

template <typename T, int IB, bool FULL>
__global__ void __launch_bounds__(kTsNT, 2) k_tau_sparse(CacheView c, TauArgs A) {
    EKV_TRACE(6);
    pdl_enter();
    pdl_trigger<6>();
    constexpr int NT = kTsNT, NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    // capacities: cap candidates (<= kTsCap; sparse rows: the list's token count, so short
    // lists take little shared memory and several CTAs fit an SM), pr list entries
    const int cap = A.cap, pr = A.pr;
    float *zs = reinterpret_cast<float *>(smem);                           // raw scores s
    int *cj = reinterpret_cast<int *>(smem + 4 * cap);                     // token positions
    int *cph = reinterpret_cast<int *>(smem + 8 * cap);                    // physical pages
    double *zp = reinterpret_cast<double *>(smem + 12 * cap);              // list z (fp64)
    int *ip = reinterpret_cast<int *>(smem + 12 * cap + 8 * pr);           // list -> candidate slot
    T *vpre = reinterpret_cast<T *>(smem + 12 * cap + 12 * pr);            // [kTsVpre][kD] staged V rows
    uint8_t *cin = reinterpret_cast<uint8_t *>(smem + 12 * cap + 12 * pr + kTsVpre * kD * sizeof(T));
    __shared__ float red[NW][kD];
    __shared__ int sup_j[kTsSup], sup_phys[kTsSup];   // (staged path: sup_j = list index)
    __shared__ float sup_p[kTsSup];
    __shared__ double rbuf[2 * 2 * NW];
    __shared__ float rbuff[2 * 2 * NW];
    __shared__ int shi[NW + 1];
    __shared__ double s_tau, s_kk, s_psum;
    __shared__ int s_nsup, s_mode;
    BlockRed2<NT> Rd{rbuf, 0};
    BlockRed2f<NT> Rf{rbuff, 0};

    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int CL = (int)cl.num_blocks(), rk = (int)cl.block_rank();
    const int row = blockIdx.x / CL;
    if (A.retry_pass && A.retry[row] == 0) return;           // (uniform over the cluster)
    const int b = row / A.Hq, h = row % A.Hq, kvh = h / A.G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t *plist = A.page_idx + (size_t)row * A.sel_stride;
    // independent loads first (one round trip): row max, list length, sequence length and
    // this rank's first-round page list
    const uint32_t mk = __ldg(A.rowmax + row);
    const int L = __ldg(c.seq_lens + b);
    const int nlist = FULL ? n_pages_of(L) : __ldg(A.n_sel + row);
    // logical page of list entry i (full rows: every page, in order)
    auto page_of = [&](int i) -> int { return FULL ? i : __ldg(plist + i); };
    // rank rk extracts the items [rk S, (rk + 1) S) (item = 4 scores), S from the list capacity
    // (variable-length lists, e.g. the Gaussian selector: from the list length -- one round
    // trip more, but every rank gets work)
    const int S = (((A.var ? nlist : A.sel_stride) * 4 + CL - 1) / CL + 3) & ~3;
    // thread t owns list page (item r0 / 4 + t) of each round: its kTsU = 4 items are that
    // page's 4 quads, so the block scan compacts candidates in list order = token order
    static_assert(kTsU == 4, "one page (4 quads of 4 scores) per thread and round");
    int pg;
    {
        const int i = (rk * S >> 2) + threadIdx.x;
        pg = (!FULL && 4 * i < (rk + 1) * S && i < A.sel_stride) ? __ldg(plist + i) : -1;
    }
    ph_stamp<6>(0);
    if (mk == 0u) {   // empty C_tok (uniform over the cluster)
        if (rk == 0 && threadIdx.x < kD) A.out[(size_t)row * kD + threadIdx.x] = 0.0f;
        if (rk == 0 && threadIdx.x == 0) {
            if (A.tau_out) A.tau_out[row] = NAN;
            if (A.supp_out) A.supp_out[row] = 0;
        }
        return;
    }
    const float smax = key2f(mk);
    const float *srow = A.scores + (size_t)row * A.ntok;
    const int32_t *ptab = c.page_table + (size_t)b * c.maxp;
    const T *Vb = reinterpret_cast<const T *>(c.V);
    const double a = (double)A.alpha - 1.0;
    const double beta = 1.0 / a;
    const float af = (float)a, betaf = (float)beta;
    const double zmax = a * (double)smax;
    double tau_lo = zmax - 1.0 - 1e-12 * fmax(1.0, fabs(zmax));

    // ---- 1. candidates {z > tau_lo} (returns -1 on overflow; uniform)
    // items [lo, min(hi, 4 nlist)) in rounds of U * NT; candidates compacted in item order
    __shared__ int s_xw[2][NW];              // extraction scans: warp totals, alternating rounds
    int xr = 0;
    auto extract = [&](double tlo, bool have_pg, int lo, int hi) -> int {
        const float thr_c = (float)(tlo / a);
        const float thr_f = thr_c - 1e-6f * fmaxf(1.0f, fabsf(thr_c));   // conservative fp32 pre-test
        const int nitems = min(nlist * 4, hi);
        int n = 0;
        for (int r0 = lo; r0 < nitems; r0 += kTsU * NT) {       // lo, r0, nitems: multiples of 4
            const int e0 = r0 + 4 * threadIdx.x;                     // this thread's page's first item
            if (r0 > lo || !have_pg) pg = e0 < nitems ? page_of(e0 >> 2) : -1;
            if (e0 >= nitems) pg = -1;
            float4 v[kTsU];
            int ph = 0;
            if (pg >= 0) {
#pragma unroll
                for (int u = 0; u < kTsU; ++u) v[u] = *reinterpret_cast<const float4 *>(srow + (size_t)pg * kP + 4 * u);
                ph = __ldg(ptab + pg);
            }
            uint32_t bits = 0u;
            if (pg >= 0) {
                const int j0 = pg * kP;
#pragma unroll
                for (int u = 0; u < kTsU; ++u) {
                    const float sv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (j0 + 4 * u + q < L && sv[q] >= thr_f && a * (double)sv[q] > tlo) bits |= 1u << (4 * u + q);
                }
            }
            int tot;
            int pos = n + block_excl_scan1<NT>(__popc(bits), s_xw[xr & 1], &tot);   // (alternating buffers)
            ++xr;
            if (n + tot > cap) return -1;
            if (bits) {
#pragma unroll
                for (int u = 0; u < kTsU; ++u) {
                    if (!((bits >> (4 * u)) & 15u)) continue;
                    const float sv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if ((bits >> (4 * u + q)) & 1u) {
                            zs[pos] = sv[q];
                            cj[pos] = pg * kP + 4 * u + q;
                            cph[pos] = ph;
                            ++pos;
                        }
                }
            }
            n += tot;
        }
        return n;
    };
    // One extraction call site (the kernel runs on cold instruction caches: code size is
    // latency).  Attempt 0: FULL rows from the chunk regions, sparse rows from this rank's
    // slice (merged into rank 0); later attempts (rank 0 alone): the whole list, after a
    // cluster overflow, or after the streamed Newton raised tau_lo past an overflow.
    int ncand = -1;
    int xlo = rk * S, xhi = (rk + 1) * S;
    bool have_pg = true, first = true, newton_done = false;
    for (;;) {
        if (FULL && first) {
            // full rows: k_candidates' chunk regions concatenated in chunk order (nch <= NT)
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
            if (!chunk_ovf && tot > cap) {
                // too many for shared memory: fp64 Newton over the chunk regions (thread t <->
                // chunk t) moves tau_lo just below tau, then an ordered re-extraction {z > tau_lo}
                double t = tau_lo;
                for (int it = 0; it < 200; ++it) {
                    double F = 0.0, Fd = 0.0;
                    if (threadIdx.x < A.nch) {
                        const size_t g0 = (size_t)threadIdx.x * kCpc;
                        for (int k = 0; k < ccnt; ++k) {
                            const double d = a * (double)__ldg(gs + g0 + k) - t;
                            if (d > 0.0) { F += powB<IB>(d, beta); Fd += powBm1<IB>(d, beta); }
                        }
                    }
                    Rd.sum(F, Fd);
                    if (!(Fd > 0.0)) break;
                    const double step = lbeta_step(F, Fd, beta, IB);
                    t += step;
                    if (!(fabs(step) > 1e-12 * fmax(1.0, fabs(t)))) break;
                }
                tau_lo = fmax(tau_lo, t - 1e-7 * fmax(1.0, fabs(t)));
                int mine = 0;
                if (threadIdx.x < A.nch) {
                    const size_t g0 = (size_t)threadIdx.x * kCpc;
                    for (int k = 0; k < ccnt; ++k) mine += a * (double)__ldg(gs + g0 + k) > tau_lo;
                }
                int tt;
                int pos = block_excl_scan<NT>(mine, shi, &tt);
                if (tt <= cap) {
                    if (threadIdx.x < A.nch) {
                        const size_t g0 = (size_t)threadIdx.x * kCpc;
                        for (int k = 0; k < ccnt; ++k) {
                            const float sj = __ldg(gs + g0 + k);
                            if (a * (double)sj > tau_lo) {
                                const int j = __ldg(gj + g0 + k);
                                zs[pos] = sj; cj[pos] = j; cph[pos] = __ldg(ptab + j / kP);
                                ++pos;
                            }
                        }
                    }
                    ncand = tt;
                } else {
                    ncand = -1;
                }
            } else if (!chunk_ovf) {
                __shared__ int s_off[256];
                if (threadIdx.x < A.nch) s_off[threadIdx.x] = coff;
                __syncthreads();
                for (int e = threadIdx.x; e < tot; e += NT) {
                    int lo = 0, hi = A.nch - 1;                // last chunk with offset <= e
                    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_off[mid] <= e) lo = mid; else hi = mid - 1; }
                    const size_t g = (size_t)lo * kCpc + (e - s_off[lo]);
                    const int j = __ldg(gj + g);
                    zs[e] = __ldg(gs + g);
                    cj[e] = j;
                    cph[e] = __ldg(ptab + j / kP);
                }
                ncand = tot;
            } else {
                ncand = -1;
            }
        } else {
            ncand = extract(tau_lo, have_pg, xlo, xhi);
        }
        if (first && CL > 1) {
            // merge: ranks publish their counts; if everything fits, ranks >= 1 store their
            // candidates into rank 0's arrays (rank order: deterministic) and leave
            __shared__ int s_cnt;
            if (threadIdx.x == 0) s_cnt = ncand;
            cl.sync();
            // the ranks' counts: lane q reads rank q (one round of remote loads, not CL in a row)
            const int nq = lane < CL ? *cl.map_shared_rank(&s_cnt, lane) : 0;
            const int tot = __reduce_add_sync(0xffffffffu, nq);
            const int off = __reduce_add_sync(0xffffffffu, lane < rk ? nq : 0);
            bool ovf = __any_sync(0xffffffffu, nq < 0);
            if (tot > cap) ovf = true;
            if (!ovf && rk > 0 && ncand > 0) {
                float *zs0 = cl.map_shared_rank(zs, 0);
                int *cj0 = cl.map_shared_rank(cj, 0), *cph0 = cl.map_shared_rank(cph, 0);
                for (int i = threadIdx.x; i < ncand; i += NT) {
                    zs0[off + i] = zs[i]; cj0[off + i] = cj[i]; cph0[off + i] = cph[i];
                }
            }
            cl.sync();
            if (rk > 0) return;
            if (!ovf) { ncand = tot; break; }
            ncand = -1;
        }
        first = false;
        if (ncand >= 0) break;
        xlo = 0; xhi = 1 << 30; have_pg = false;
        if (newton_done) {             // support larger than the shared-memory capacity
            if (A.retry && !A.retry_pass && cap < kTsCap) {  // reduced capacity: re-run at kTsCap
                if (threadIdx.x == 0) A.retry[row] = 1;
                return;
            }
            if (threadIdx.x < kD) A.out[(size_t)row * kD + threadIdx.x] = NAN;
            if (threadIdx.x == 0) {
                if (A.tau_out) A.tau_out[row] = NAN;
                if (A.supp_out) A.supp_out[row] = -1;
                if (A.status) atomicOr(A.status, kStatusCapacity);    // EKV_ERR_CAPACITY on request
            }
            return;
        }
            // overflow: fp64 Newton streamed over the whole row moves tau_lo just below tau
            // (out of line: the hot path's code stays contiguous -- cold instruction fetch)
            const double t = streamed_newton<NT, IB>(srow, plist, FULL, nlist, L, a, beta, tau_lo, Rd);
            tau_lo = fmax(tau_lo, t - 1e-7 * fmax(1.0, fabs(t)));
        newton_done = true;
    }
    __syncthreads();
    ph_stamp<6>(1);
    ph_count<6>(0, ncand);

    // ---- approximate tau (attn flag: the paper's kernel recipe; DESIGN R23): histogram
    // initialisation over (z_max - 1, z_max] with the certified lower bound of F at the bin
    // edges, then A.approx_h Halley steps; support {z > tau}; PV below (candidate rounds)
    bool staged = false;
    if (A.approx_h > 0) {
        __shared__ unsigned hcnt[64];
        __shared__ double s_t0;
        if (A.tau_init) {
            // the Gaussian variant: start at the selector's tau_hat; outside
            // [z_max - 1, z_max) (where the exact tau lies) the start is z_max - 1 (R25)
            const double t0 = A.tau_init[row];
            if (threadIdx.x == 0) s_t0 = (t0 >= zmax - 1.0 && t0 < zmax) ? t0 : zmax - 1.0;
        } else {
        if (threadIdx.x < 64) hcnt[threadIdx.x] = 0u;
        __syncthreads();
        for (int k = threadIdx.x; k < ncand; k += NT) {
            const double z = a * (double)zs[k];
            if (!(z > zmax - 1.0)) continue;
            const double fb = floor((zmax - z) * 64.0);
            atomicAdd(&hcnt[fb > 63.0 ? 63 : (int)fb], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            // lane l: edges k = l + 1 and l + 33; the same b-ascending sums as the oracle
            double lb0 = 0.0, lb1 = 0.0;
            const int k0 = lane + 1, k1 = lane + 33;
            for (int bb = 0; bb < k1; ++bb) {
                const double term1 = __dmul_rn((double)hcnt[bb], powB<IB>((double)(k1 - 1 - bb) / 64.0, beta));
                lb1 = __dadd_rn(lb1, term1);
                if (bb < k0) {
                    const double term0 = __dmul_rn((double)hcnt[bb], powB<IB>((double)(k0 - 1 - bb) / 64.0, beta));
                    lb0 = __dadd_rn(lb0, term0);
                }
            }
            const unsigned m0 = __ballot_sync(0xffffffffu, lb0 >= 1.0), m1 = __ballot_sync(0xffffffffu, lb1 >= 1.0);
            int kst = 0;
            if (m0) kst = __ffs(m0);             // smallest k with LB_k >= 1
            else if (m1) kst = 32 + __ffs(m1);
            if (lane == 0) s_t0 = kst ? zmax - (double)kst / 64.0 : zmax - 1.0;
        }
        }
        __syncthreads();
        double t = s_t0;
        for (int it = 0; it < A.approx_h; ++it) {
            double S0 = 0.0, S1 = 0.0, S2 = 0.0, dz = 0.0;
            for (int k = threadIdx.x; k < ncand; k += NT) {
                const double w = a * (double)zs[k] - t;
                if (w > 0.0) {
                    S0 += powB<IB>(w, beta);
                    S1 += powBm1<IB>(w, beta);
                    S2 += (IB == 1) ? 0.0 : (IB == 2 ? 1.0 : (IB == 3 ? w : (IB == 4 ? w * w : pow(w, beta - 2.0))));
                }
            }
            Rd.sum(S0, S1);
            Rd.sum(S2, dz);
            const double f = S0 - 1.0, fp = -beta * S1, fpp = beta * (beta - 1.0) * S2;
            const double den = 2.0 * fp * fp - f * fpp;
            if (!(den != 0.0)) break;
            t -= 2.0 * f * fp / den;
            t = fmax(t, zmax - 1.0);       // R25: never below the exact tau's lower bound
        }
        int mine = 0;
        for (int k = threadIdx.x; k < ncand; k += NT) {
            const bool in = a * (double)zs[k] > t;
            cin[k] = in ? 1 : 0;
            mine += in;
        }
        mine = block_sum_i<NT>(mine, shi);
        if (threadIdx.x == 0) { s_tau = t; s_kk = (double)mine; s_mode = 0; s_nsup = 0; s_psum = 0.0; }
        __syncthreads();
    } else {

    // ---- small candidate sets (<= 32, the usual top-k decode row: z_max - 1 prunes to a few
    // tokens): one warp does R9 by all pairs, tau and the support list with shuffles -- no
    // block barrier until PV (each barrier step of the general path below costs ~1000 cycles);
    // the candidates' V rows are staged in shared memory meanwhile
    if (ncand >= 1 && ncand <= 32) {
        if (warp == 0) {
            const bool have = lane < ncand;
            const double zl = have ? a * (double)zs[lane] : -INFINITY;
            if (have) {
                constexpr int CH = kD * (int)sizeof(T) / 16;          // 16-byte chunks per row
                const int j = cj[lane];
                const T *src = Vb + (((size_t)cph[lane] * c.Hkv + kvh) * kP + (j % kP)) * kD;
                for (int ch = 0; ch < CH; ++ch)
                    cp_async16(reinterpret_cast<char *>(vpre + (size_t)lane * kD) + 16 * ch,
                               reinterpret_cast<const char *>(src) + 16 * ch);
            }
            cp_async_commit();
            auto wsum = [&](double x) {
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                return x;
            };
            double F = 0.0;                          // R9: F(z_j) = sum_i (z_i - z_j)_+^beta
            for (int i = 0; i < ncand; ++i) {
                const double d = __shfl_sync(0xffffffffu, zl, i) - zl;
                if (d > 0.0) F += powB<IB>(d, beta);
            }
            const bool in = have && F < 1.0;
            const double S1 = wsum(in ? zl : 0.0), kk = wsum(in ? 1.0 : 0.0);
            double tau;
            if constexpr (IB == 1) {
                tau = (S1 - 1.0) / kk;
            } else if constexpr (IB == 2) {
                const double m = S1 / kk;
                const double ss = wsum(in ? (zl - m) * (zl - m) : 0.0);
                tau = m - sqrt(fmax(0.0, 1.0 - ss) / kk);
            } else {
                // Newton on sum_S (z - t)^beta = 1 from the largest z outside S (or tau_lo): F >= 1
                // there, so the iteration is monotone from the left
                double t0 = (have && !in) ? zl : tau_lo;
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) t0 = fmax(t0, __shfl_xor_sync(0xffffffffu, t0, o));
                tau = t0;
                for (int it = 0; it < 60; ++it) {
                    const double dd = zl - tau;
                    const double Fs = wsum(in ? powB<IB>(dd, beta) : 0.0), Fd = wsum(in ? powBm1<IB>(dd, beta) : 0.0);
                    if (!(Fd > 0.0)) break;
                    const double step = lbeta_step(Fs, Fd, beta, IB);
                    tau += step;
                    if (!(fabs(step) > 1e-15 * fmax(1.0, fabs(tau)))) break;
                }
                const double dd = zl - tau;
                const double Fs = wsum(in ? powB<IB>(dd, beta) : 0.0), Fd = wsum(in ? powBm1<IB>(dd, beta) : 0.0);
                if (Fd > 0.0) tau += (Fs - 1.0) / (beta * Fd);
            }
            // support entries in candidate order (= token order), V rows staged (mode 2)
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            const int pos = __popc(bal & ((1u << lane) - 1u));
            double pd = 0.0;
            if (in) {
                const double d = zl - tau;
                pd = d > 0.0 ? powB<IB>(d, beta) : 0.0;
                sup_j[pos] = lane;
                sup_phys[pos] = cph[lane];
                sup_p[pos] = (float)pd;
            }
            if (have) cin[lane] = in ? 1 : 0;
            const double psum = wsum(pd);
            if (lane == 0) { s_tau = tau; s_kk = kk; s_nsup = __popc(bal); s_mode = 2; s_psum = psum; }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
    } else {
    // ---- 2. fp32 Newton steps (pruning point only)
    float tf = (float)tau_lo;
    for (int it = 0; it < 3; ++it) {      // Newton from the left: every iterate is below tau
        float F = 0.f, D = 0.f;
        for (int k = threadIdx.x; k < ncand; k += NT) {
            const float d = af * zs[k] - tf;
            if (d > 0.f) { F += powBf<IB>(d, betaf); D += powBm1f<IB>(d, betaf); }
        }
        Rf.sum(F, D);
        if (!(D > 0.f)) break;
        const float step = (float)lbeta_step((double)F, (double)D, beta, IB);
        tf += step;
        if (!(fabsf(step) > 1e-3f * fmaxf(1.0f, fabsf(tf)))) break;
    }
    ph_stamp<6>(2);

    // ---- 3. certified base and the list {z > base}
    auto build = [&](double base, double &Fb) -> int {
        const float bf = (float)base;
        const float bpre = bf - 1e-3f * fmaxf(1.0f, fabsf(bf));
        // thread t owns the contiguous candidate slots [t L, (t + 1) L): one block scan in total
        const int per = (ncand + NT - 1) / NT;
        const int k0 = threadIdx.x * per, k1 = min(ncand, k0 + per);
        double f = 0.0, dz = 0.0;
        int mine = 0;
        for (int k = k0; k < k1; ++k)
            if (af * zs[k] > bpre) {
                const double z = a * (double)zs[k];
                if (z > base) { ++mine; f += powB<IB>(z - base, beta); }
            }
        int np;
        int pos = block_excl_scan<NT>(mine, shi, &np);
        if (mine)
            for (int k = k0; k < k1; ++k)
                if (af * zs[k] > bpre) {
                    const double z = a * (double)zs[k];
                    if (z > base) { if (pos < pr) { zp[pos] = z; ip[pos] = k; } ++pos; }
                }
        Rd.sum(f, dz);
        Fb = f;
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
    const bool listed = np <= pr;
    staged = np <= kTsVpre;
    if (staged) {
        // V rows of the list entries -> shared memory, in flight during step 4
        constexpr int CH = kD * (int)sizeof(T) / 16;          // 16-byte chunks per row
        for (int e = threadIdx.x; e < np * CH; e += NT) {
            const int i = e / CH, ch = e - i * CH;
            const int k = ip[i];
            const int j = cj[k];
            const T *src = Vb + (((size_t)cph[k] * c.Hkv + kvh) * kP + (j % kP)) * kD;
            cp_async16(reinterpret_cast<char *>(vpre + (size_t)i * kD) + 16 * ch,
                       reinterpret_cast<const char *>(src) + 16 * ch);
        }
        cp_async_commit();
    }
    for (int k = threadIdx.x; k < ncand; k += NT) cin[k] = 0;
    ph_stamp<6>(3);
    ph_count<6>(1, np);

    // ---- 4. support and tau
    const bool block_path = listed && np <= NT;
    if (block_path) {
        // R9 on every list entry: TPE threads per entry (npad = np rounded up to a power of
        // two >= 8), partial sums over i = lane-in-group (mod TPE), xor-shuffle combine
        int npad = 8;
        while (npad < np) npad <<= 1;
        const int TPE = NT / npad;                // 1..32
        const int jj = threadIdx.x / TPE, cc = threadIdx.x % TPE;
        double F = 0.0, zj = 0.0;
        if (jj < np) {
            zj = zp[jj];
            for (int i2 = cc; i2 < np; i2 += TPE) {
                const double d = zp[i2] - zj;
                if (d > 0.0) F += powB<IB>(d, beta);
            }
        }
        for (int o = 1; o < TPE; o <<= 1) F += __shfl_xor_sync(0xffffffffu, F, o);
        const bool own = jj < np && cc == 0;
        const bool in = own && F < 1.0;
        double S1 = in ? zj : 0.0, kk = in ? 1.0 : 0.0;
        Rd.sum(S1, kk);
        double tau;
        if constexpr (IB == 1) {
            tau = (S1 - 1.0) / kk;
        } else if constexpr (IB == 2) {
            const double m = S1 / kk;
            double ss = in ? (zj - m) * (zj - m) : 0.0, dz = 0.0;
            Rd.sum(ss, dz);
            tau = m - sqrt(fmax(0.0, 1.0 - ss) / kk);
        } else {
            // Newton on sum_S (z - t)^beta = 1 from the largest listed z outside S (or base):
            // F >= 1 there, so the iteration is monotone from the left
            double t0 = (own && !in) ? zj : base, dz = 0.0;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) t0 = fmax(t0, __shfl_xor_sync(0xffffffffu, t0, o));
            __shared__ double s_mx[NW];
            if (lane == 0) s_mx[warp] = t0;
            __syncthreads();
            t0 = base;
            for (int w = 0; w < NW; ++w) t0 = fmax(t0, s_mx[w]);
            tau = t0;
            for (int it = 0; it < 60; ++it) {
                double Fs = 0.0, Fd = 0.0;
                if (in) { const double d = zj - tau; Fs = powB<IB>(d, beta); Fd = powBm1<IB>(d, beta); }
                Rd.sum(Fs, Fd);
                if (!(Fd > 0.0)) break;
                const double step = lbeta_step(Fs, Fd, beta, IB);
                tau += step;
                if (!(fabs(step) > 1e-15 * fmax(1.0, fabs(tau)))) break;
            }
            // final polish on the support sum itself (as the warp path)
            double Fs = 0.0, Fd = 0.0;
            if (in) { const double d = zj - tau; Fs = powB<IB>(d, beta); Fd = powBm1<IB>(d, beta); }
            Rd.sum(Fs, Fd);
            if (Fd > 0.0) tau += (Fs - 1.0) / (beta * Fd);
            (void)dz;
        }
        // support entries in list order (block scan over the entry owners)
        int tot;
        const int pos = block_excl_scan<NT>(in ? 1 : 0, shi, &tot);
        double pd = 0.0;
        const bool fits = tot <= kTsSup;
        if (in && fits) {
            const double d = zj - tau;
            pd = d > 0.0 ? powB<IB>(d, beta) : 0.0;
            const int k = ip[jj];
            sup_j[pos] = staged ? jj : cj[k];     // list index (V staged) or token position
            sup_phys[pos] = cph[k];
            sup_p[pos] = (float)pd;
        }
        if (own) cin[ip[jj]] = in ? 1 : 0;       // (large-support fallback reads the flags)
        if (threadIdx.x == 0) { s_tau = tau; s_kk = kk; s_nsup = tot; s_mode = fits ? (staged ? 2 : 1) : 0; }
        double psum = pd, dz2 = 0.0;
        Rd.sum(psum, dz2);                         // (barrier: sup_*, cin and s_* visible)
        if (threadIdx.x == 0) s_psum = psum;
    } else if (warp == 0) {
        auto wsum2 = [&](double &x, double &y) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                x += __shfl_xor_sync(0xffffffffu, x, o);
                y += __shfl_xor_sync(0xffffffffu, y, o);
            }
        };
        const int nl = listed ? np : ncand;
#define ZL(i) (listed ? zp[i] : a * (double)zs[i])
#define SL(i) (listed ? ip[i] : (i))
        double tauN = base;
        if (listed && np <= 64) {
            // short list: R9 itself, F(z_j) = sum_i (z_i - z_j)_+^beta < 1, all pairs
            for (int i = lane; i < nl; i += 32) {
                const double zj = zp[i];
                double F0 = 0.0, F1 = 0.0;
                int i2 = 0;
                for (; i2 + 1 < nl; i2 += 2) {
                    const double d0 = zp[i2] - zj, d1 = zp[i2 + 1] - zj;
                    if (d0 > 0.0) F0 += powB<IB>(d0, beta);
                    if (d1 > 0.0) F1 += powB<IB>(d1, beta);
                }
                if (i2 < nl) { const double d0 = zp[i2] - zj; if (d0 > 0.0) F0 += powB<IB>(d0, beta); }
                cin[ip[i]] = (F0 + F1 < 1.0) ? 1 : 0;
            }
            __syncwarp();
            if constexpr (IB != 1 && IB != 2) {
                // Newton start for the tau polish: the largest listed z outside the support
                // (or base) has F >= 1, i.e. lies left of tau
                double t0 = base;
                for (int i = lane; i < nl; i += 32)
                    if (!cin[ip[i]]) t0 = fmax(t0, zp[i]);
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) t0 = fmax(t0, __shfl_xor_sync(0xffffffffu, t0, o));
                tauN = t0;
                for (int it = 0; it < 60; ++it) {
                    double F = 0.0, Fd = 0.0;
                    for (int i = lane; i < nl; i += 32)
                        if (cin[ip[i]]) { const double d = zp[i] - tauN; F += powB<IB>(d, beta); Fd += powBm1<IB>(d, beta); }
                    wsum2(F, Fd);
                    if (!(Fd > 0.0)) break;
                    const double step = lbeta_step(F, Fd, beta, IB);
                    tauN += step;
                    if (!(fabs(step) > 1e-15 * fmax(1.0, fabs(tauN)))) break;
                }
            }
        } else {
            for (int it = 0; it < 64; ++it) {
                double F = 0.0, Fd = 0.0;
                for (int i = lane; i < nl; i += 32) {
                    const double d = ZL(i) - tauN;
                    if (d > 0.0) { F += powB<IB>(d, beta); Fd += powBm1<IB>(d, beta); }
                }
                wsum2(F, Fd);
                if (!(Fd > 0.0)) break;
                const double step = lbeta_step(F, Fd, beta, IB);
                tauN += step;
                // 1e-14 relative is far inside the support band (R9) and the final tau is
                // recomputed from the support; a tighter test can oscillate at the ulp level
                if (!(fabs(step) > 1e-14 * fmax(1.0, fabs(tauN)))) break;
            }
            const double band = 1e-9 * fmax(1.0, fabs(tauN));
            int amb = 0;
            for (int i = lane; i < nl; i += 32) {
                const double z = ZL(i);
                const uint8_t f = (z > tauN + band) ? 1 : (z < tauN - band) ? 0 : 2;
                cin[SL(i)] = f;
                amb += (f == 2);
            }
            amb = __reduce_add_sync(0xffffffffu, amb);
            __syncwarp();
            if (amb > 0) {
                for (int i0 = 0; i0 < nl; ++i0) {
                    const int k0 = SL(i0);
                    if (cin[k0] != 2) continue;
                    const double zk = ZL(i0);
                    double F = 0.0, dz = 0.0;
                    for (int i = lane; i < nl; i += 32) {
                        const double d = ZL(i) - zk;
                        if (d > 0.0) F += powB<IB>(d, beta);
                    }
                    wsum2(F, dz);
                    __syncwarp();
                    if (lane == 0) cin[k0] = (F < 1.0) ? 1 : 0;
                    __syncwarp();
                }
            }
        }
        // tau from the support
        double S1 = 0.0, kk = 0.0;
        for (int i = lane; i < nl; i += 32)
            if (cin[SL(i)]) { S1 += ZL(i); kk += 1.0; }
        wsum2(S1, kk);
        double tau;
        if constexpr (IB == 1) {
            tau = (S1 - 1.0) / kk;
        } else if constexpr (IB == 2) {
            const double m = S1 / kk;
            double ss = 0.0, dz = 0.0;
            for (int i = lane; i < nl; i += 32)
                if (cin[SL(i)]) { const double d = ZL(i) - m; ss += d * d; }
            wsum2(ss, dz);
            tau = m - sqrt(fmax(0.0, 1.0 - ss) / kk);
        } else {
            double F = 0.0, Fd = 0.0;
            for (int i = lane; i < nl; i += 32)
                if (cin[SL(i)]) { const double d = ZL(i) - tauN; F += powB<IB>(d, beta); Fd += powBm1<IB>(d, beta); }
            wsum2(F, Fd);
            tau = tauN + (F - 1.0) / (beta * Fd);
        }
        // support entries (list order) with p_j, if they fit one gather round
        int nsup = 0;
        double psum = 0.0, dz = 0.0;
        const bool one_round = listed && kk <= (double)kTsSup;
        if (one_round) {
            for (int i0 = 0; i0 < nl; i0 += 32) {
                const int i = i0 + lane;
                const int k = i < nl ? ip[i] : 0;
                const bool in = i < nl && cin[k];
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                const int pos = nsup + __popc(bal & ((1u << lane) - 1u));
                if (in) {
                    const double d = zp[i] - tau;
                    const double pd = d > 0.0 ? powB<IB>(d, beta) : 0.0;
                    sup_j[pos] = staged ? i : cj[k];
                    sup_p[pos] = (float)pd;
                    sup_phys[pos] = cph[k];
                    psum += pd;
                }
                nsup += __popc(bal);
            }
            wsum2(psum, dz);
        }
#undef ZL
#undef SL
        if (lane == 0) {
            s_tau = tau; s_kk = kk; s_psum = psum; s_nsup = nsup;
            s_mode = one_round ? (staged ? 2 : 1) : 0;
        }
    }
    }   // general path
    }   // exact tau
    if (staged) cp_async_commit_wait_all();
    __syncthreads();
    ph_stamp<6>(4);
    const double tau = s_tau, kk = s_kk;

    if (A.no_pv) {                       // dense-V baseline: V is streamed by k_softmax_partial
        if (threadIdx.x == 0) {
            if (A.tau_out) A.tau_out[row] = tau;
            if (A.supp_out) A.supp_out[row] = (int)kk;
        }
        return;
    }
    // ---- 5. PV
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
    if (s_mode == 2) {
        // staged V rows: warp w takes entries w, w + NW, ...
        const int nsup = s_nsup;
        for (int e = warp; e < nsup; e += NW) {
            float vx[4];
            ldv4<T>(vpre + (size_t)sup_j[e] * kD + 4 * lane, vx);
            const float p = sup_p[e];
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) acc[q2] = __fmaf_rn(p, vx[q2], acc[q2]);
        }
        if (threadIdx.x == 0) psum = s_psum;
    } else if (s_mode == 1) {
        gather(s_nsup);
        if (threadIdx.x == 0) psum = s_psum;
    } else {
        // large support: compacted in candidate order, rounds of kTsSup entries
        for (int r0 = 0; r0 < ncand;) {
            int nsup = 0, r1 = r0;
            while (r1 < ncand) {
                const int k = r1 + threadIdx.x;
                const bool in = k < ncand && cin[k];
                int tot;
                const int pos = nsup + block_excl_scan<NT>(in ? 1 : 0, shi, &tot);
                if (nsup + tot > kTsSup) break;             // uniform
                if (in) {
                    const double d = a * (double)zs[k] - tau;
                    const double pd = d > 0.0 ? powB<IB>(d, beta) : 0.0;
                    sup_j[pos] = cj[k];
                    sup_p[pos] = (float)pd;
                    sup_phys[pos] = cph[k];
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
    Rd.sum(psum, pz);
    if (threadIdx.x < kD) {
        float o = 0.f;
        for (int w = 0; w < NW; ++w) o = __fadd_rn(o, red[w][threadIdx.x]);
        A.out[(size_t)row * kD + threadIdx.x] = (float)((double)o / psum);
    }
    if (threadIdx.x == 0) {
        if (A.tau_out) A.tau_out[row] = tau;
        if (A.supp_out) A.supp_out[row] = (int)kk;
    }
    // support token positions, ascending (candidates are extracted in list order = token order)
    if (!FULL && A.supp_tok) {
        int base = 0;
        for (int r0 = 0; r0 < ncand; r0 += NT) {
            const int k = r0 + threadIdx.x;
            const bool keep = k < ncand && cin[k];
            int tot;
            const int pos = base + block_excl_scan<NT>(keep ? 1 : 0, shi, &tot);
            if (keep && pos < A.supp_cap) A.supp_tok[(size_t)row * A.supp_cap + pos] = cj[k];
            base += tot;
        }
    }
    // eval list: support token positions and p_j in candidate order (exact delta / rho)
    if (FULL && A.tok_list) {
        int base = 0;
        for (int r0 = 0; r0 < ncand; r0 += NT) {
            const int k = r0 + threadIdx.x;
            const bool keep = k < ncand && cin[k];
            int tot;
            const int pos = base + block_excl_scan<NT>(keep ? 1 : 0, shi, &tot);
            if (keep && pos < A.list_cap) {
                const double d = a * (double)zs[k] - tau;
                A.tok_list[(size_t)row * A.list_cap + pos] = cj[k];
                A.p_list[(size_t)row * A.list_cap + pos] = d > 0.0 ? powB<IB>(d, beta) : 0.0;
            }
            base += tot;
        }
        if (threadIdx.x == 0) A.n_list[row] = base;
    }
    ph_stamp<6>(5);
}

}  // namespace ekv

