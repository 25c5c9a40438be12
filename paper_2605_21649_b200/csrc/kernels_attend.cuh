// kernels_attend.cuh -- a3/a5/a6: token scores over the selected pages (TMA bulk
// copies of K tiles into shared memory), exact alpha-entmax threshold + support,
// and the weighted V sum over the support.
#pragma once
#include "common.cuh"

namespace ekv {

// ============================================================================ K scores
// Grid (union-slot chunk of PPC pages, b * Hkv + kvh); 128 threads = 8 half-warps.
// Thread 0 issues one cp.async.bulk (TMA, 1-D) per page tile K[phys][kvh][0..P)[0..d)
// (4 KiB bf16 / 8 KiB fp32, contiguous in HBM) into its own shared-memory slot, each
// with its own mbarrier, so all PPC tiles are in flight at once.  Half-warp hw then
// scores tokens of pages hw, hw+8, ...: lane c reads the 16-byte chunk c of the token's
// row (a contiguous 256-byte row per half-warp: conflict-free), runs the 8-element fma
// chains for the G query heads of the group and the reduce-scatter tree (R1);
// s = fl32(dot * c_d) (R2).  Tokens of pages that query head h did not select, and
// tokens beyond seq_len, get -inf.  Output scores[b][h][slot * P + t] fp32.
// full != 0: the union is every page of the sequence (a5).
template <typename T, int G, int PPC>
__global__ void __launch_bounds__(128) k_attend_scores(CacheView c, const T *__restrict__ q, int Hq,
                                                       const int32_t *__restrict__ union_pages,
                                                       const uint8_t *__restrict__ union_mask,
                                                       const int32_t *__restrict__ union_len, int ucap,
                                                       float *__restrict__ scores, int full) {
    constexpr int TILE = kP * kD * (int)sizeof(T);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[PPC];
    __shared__ int s_page[PPC];
    __shared__ uint8_t s_mask[PPC];
    const int unit = blockIdx.y;
    const int b = unit / c.Hkv, kvh = unit % c.Hkv;
    const int L = c.seq_lens[b];
    const int ulen = full ? n_pages_of(L) : union_len[unit];
    const int u0 = blockIdx.x * PPC;
    if (u0 >= ulen) return;
    const int nu = min(PPC, ulen - u0);
    if (threadIdx.x < nu) {
        const int u = u0 + threadIdx.x;
        s_page[threadIdx.x] = full ? u : union_pages[(size_t)unit * ucap + u];
        s_mask[threadIdx.x] = full ? (uint8_t)0xff : union_mask[(size_t)unit * ucap + u];
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < nu; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned char *Kb = reinterpret_cast<const unsigned char *>(c.K);
        for (int i = 0; i < nu; ++i) {
            const int phys = c.page_table[(size_t)b * c.maxp + s_page[i]];
            mbar_expect_tx(&bars[i], TILE);
            bulk_g2s(smem + (size_t)i * TILE, Kb + ((size_t)phys * c.Hkv + kvh) * TILE, TILE, &bars[i]);
        }
    }
    const int lane = threadIdx.x & 31;
    const int l16 = threadIdx.x & 15;
    const int hw = threadIdx.x >> 4;
    float qr[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g)
        Elem<T>::load8(q + ((size_t)b * Hq + kvh * G + g) * kD + 8 * l16, qr[g]);
    const int hsel = rs_head<G>(lane);
    const bool writer = rs_writer<G>(lane);
    const size_t ntok = (size_t)ucap * kP;
    float *srow = scores + ((size_t)b * Hq + kvh * G + hsel) * ntok;
    // warp-uniform loop: both half-warps of a warp iterate over the same i range
    for (int ib = (hw & ~1); ib < nu + 1; ib += 8) {
        const int i = ib + (hw & 1);
        const bool active = i < nu;
        if (ib >= nu) break;
        if (active) mbar_wait(&bars[i], 0);
        const int page = active ? s_page[i] : 0;
        const bool hsel_ok = active && ((s_mask[active ? i : 0] >> hsel) & 1);
        const T *tile = reinterpret_cast<const T *>(smem + (size_t)(active ? i : 0) * TILE);
#pragma unroll 4
        for (int t = 0; t < kP; ++t) {
            float kx[8];
            if (active) Elem<T>::load8(tile + t * kD + 8 * l16, kx);
            else {
#pragma unroll
                for (int e = 0; e < 8; ++e) kx[e] = 0.0f;
            }
            float acc[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float a = 0.0f;
#pragma unroll
                for (int e = 0; e < 8; ++e) a = __fmaf_rn(qr[g][e], kx[e], a);
                acc[g] = a;
            }
            const float s = __fmul_rn(rs_reduce16<G>(acc, lane), kCd);
            const int tok = page * kP + t;
            if (writer && active) srow[(size_t)(u0 + i) * kP + t] = (hsel_ok && tok < L) ? s : -INFINITY;
        }
    }
}

// ============================================================================ exact tau + PV
// One CTA (NT = 256) per (b, q-head).  On the row of fp32 scores over the group's
// union slots (-inf = not in C_tok(b,h)):
//  1. s_max (block max);  z = (double)a * (double)s  (R9).
//  2. tau_lo = z_max - 1 (F(z_max - 1) >= 1, so tau >= tau_lo).  Candidates
//     {z > tau_lo} are compacted IN SLOT ORDER into shared memory (deterministic).  If
//     more than CAP, the threshold of the first CAP candidates (a subset, so a lower
//     bound of tau: F_subset <= F) raises tau_lo and the compaction repeats.
//  3. Newton on g(tau) = ||(z - tau)_+||_beta - 1 (convex, decreasing -> monotone from
//     the left, exact in one step for a single active token).
//  4. Support by R9: z > tau_N + band -> in, z < tau_N - band -> out, otherwise decide
//     by F(z_j) < 1 evaluated over all candidates (fp64).
//  5. tau from the support: beta = 1: (S1 - 1)/k; beta = 2: m - sqrt((1 - ss)/k);
//     otherwise one Newton polish of sum_S (z - tau)^beta = 1.
//  6. p_j = (z_j - tau)^beta; out = sum p_j v_j / sum p_j (R12), V rows gathered only
//     for support tokens (warp per token, lane = 4 dims).
// Softmax (a6): p = exp(s - s_max) over every valid token, dense V.
constexpr int kTauNT = 256;
constexpr int kCap = 6144;

struct TauArgs {
    const float *scores; size_t ntok_stride;
    const int32_t *union_pages; const int32_t *union_len; int ucap; int full;
    int Hq, G; float alpha; int transform;
    float *out; double *tau_out; int32_t *supp_out;
    // optional statistics
    const float *box; const int32_t *page_idx; const int32_t *n_sel; int sel_stride;
    double *delta_bar;
    // eval: membership of each token in C_tok of the sparse selection (for full pass)
    int32_t *tok_list; double *p_list; int32_t *n_list; int list_cap;
};

__device__ __forceinline__ double zsafe_sub(double z, double t) { return z - t; }

template <typename T>
__global__ void __launch_bounds__(kTauNT) k_tau_pv(CacheView c, TauArgs A) {
    constexpr int NT = kTauNT;
    extern __shared__ __align__(16) unsigned char smem[];
    float *cs = reinterpret_cast<float *>(smem);                 // candidate scores [kCap]
    int *cj = reinterpret_cast<int *>(smem + sizeof(float) * kCap);   // candidate slots [kCap]
    uint8_t *cin = reinterpret_cast<uint8_t *>(smem + (sizeof(float) + sizeof(int)) * kCap);
    __shared__ double shd[2 * (NT / 32) + 2];
    __shared__ float shf[NT / 32 + 1];
    __shared__ int shi[NT / 32 + 1];
    __shared__ float red[NT / 32][kD];

    const int row = blockIdx.x;
    const int b = row / A.Hq, h = row % A.Hq, kvh = h / A.G;
    const int unit = b * c.Hkv + kvh;
    const int L = c.seq_lens[b];
    const int ulen = A.full ? n_pages_of(L) : A.union_len[unit];
    const int n = ulen * kP;
    const float *s = A.scores + (size_t)row * A.ntok_stride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    float smax = -INFINITY;
    for (int j = threadIdx.x; j < n; j += NT) smax = fmaxf(smax, s[j]);
    smax = block_max_f<NT>(smax, shf);
    if (smax == -INFINITY) {   // empty C_tok
        if (threadIdx.x < kD) A.out[(size_t)row * kD + threadIdx.x] = 0.0f;
        if (threadIdx.x == 0) {
            if (A.tau_out) A.tau_out[row] = NAN;
            if (A.supp_out) A.supp_out[row] = 0;
        }
        return;
    }
    auto v_row = [&](int j) -> const T * {
        const int u = j / kP, t = j % kP;
        const int page = A.full ? u : A.union_pages[(size_t)unit * A.ucap + u];
        const int phys = c.page_table[(size_t)b * c.maxp + page];
        return reinterpret_cast<const T *>(c.V) + (((size_t)phys * c.Hkv + kvh) * kP + t) * kD;
    };

    if (A.transform == 1) {
        // ---------------- softmax over C_tok (dense V)
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        double zs = 0.0;
        for (int j = warp; j < n; j += NT / 32) {
            const float sj = s[j];
            if (sj == -INFINITY) continue;
            const float p = expf(sj - smax);
            if (lane == 0) zs += (double)p;
            const T *vr = v_row(j) + 4 * lane;
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] = __fmaf_rn(p, Elem<T>::to_f(vr[e]), acc[e]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) red[warp][4 * lane + e] = acc[e];
        double zt = block_sum_d<NT>(zs, shd);
        int cnt = 0;
        for (int j = threadIdx.x; j < n; j += NT) cnt += (s[j] != -INFINITY);
        cnt = block_sum_i<NT>(cnt, shi);
        if (threadIdx.x < kD) {
            float o = 0.f;
            for (int w = 0; w < NT / 32; ++w) o = __fadd_rn(o, red[w][threadIdx.x]);
            A.out[(size_t)row * kD + threadIdx.x] = (float)((double)o / zt);
        }
        if (threadIdx.x == 0) {
            if (A.tau_out) A.tau_out[row] = (double)smax + log(zt);
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

    auto newton = [&](int nc, double tau0) -> double {
        double tau = tau0;
        for (int it = 0; it < 200; ++it) {
            double F = 0.0, Fd = 0.0;
            for (int k = threadIdx.x; k < nc; k += NT) {
                const double d = a * (double)cs[k] - tau;
                if (d > 0.0) { F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
            }
            block_sum2_d<NT>(F, Fd, shd);
            if (!(Fd > 0.0)) break;
            double root = (ib == 1) ? F : (ib == 2) ? sqrt(F) : (ib == 4) ? sqrt(sqrt(F)) : pow(F, 1.0 / beta);
            // step = (F^{1/b} - 1) / (F^{1/b - 1} * Fd)
            const double step = (root - 1.0) * F / (root * Fd);
            const double nt = tau + step;
            if (!(fabs(step) > 2e-16 * fmax(1.0, fabs(tau)))) { tau = nt; break; }
            tau = nt;
        }
        return tau;
    };

    auto compact = [&](double tlo) -> int {
        int base = 0;
        for (int r0 = 0; r0 < n; r0 += NT) {
            const int j = r0 + threadIdx.x;
            const int keep = (j < n && s[j] != -INFINITY && a * (double)s[j] > tlo) ? 1 : 0;
            int tot;
            const int pos = block_excl_scan<NT>(keep, shi, &tot);
            if (keep && base + pos < kCap) { cs[base + pos] = s[j]; cj[base + pos] = j; }
            base += tot;
        }
        __syncthreads();
        return base;
    };
    ncand = compact(tau_lo);
    if (ncand > kCap) {
        // overflow: Newton streamed over the whole row (global/L2) to approach tau from
        // below, then re-compact just below it.
        double tau = tau_lo;
        for (int it = 0; it < 200; ++it) {
            double F = 0.0, Fd = 0.0;
            for (int j = threadIdx.x; j < n; j += NT) {
                const float sj = s[j];
                if (sj == -INFINITY) continue;
                const double d = a * (double)sj - tau;
                if (d > 0.0) { F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
            }
            block_sum2_d<NT>(F, Fd, shd);
            if (!(Fd > 0.0)) break;
            const double root = (ib == 1) ? F : (ib == 2) ? sqrt(F) : (ib == 4) ? sqrt(sqrt(F)) : pow(F, 1.0 / beta);
            const double step = (root - 1.0) * F / (root * Fd);
            tau += step;
            if (!(fabs(step) > 1e-12 * fmax(1.0, fabs(tau)))) break;
        }
        tau_lo = fmax(tau_lo, tau - 1e-7 * fmax(1.0, fabs(tau)));
        ncand = compact(tau_lo);
        if (ncand > kCap) {          // support larger than the shared-memory capacity
            if (threadIdx.x < kD) A.out[(size_t)row * kD + threadIdx.x] = NAN;
            if (threadIdx.x == 0) {
                if (A.tau_out) A.tau_out[row] = NAN;
                if (A.supp_out) A.supp_out[row] = -ncand;
            }
            return;
        }
    }
    const double tauN = newton(ncand, tau_lo);
    // ---- support (R9)
    const double band = 1e-9 * fmax(1.0, fabs(tauN));
    int amb = 0;
    for (int k = threadIdx.x; k < ncand; k += NT) {
        const double z = a * (double)cs[k];
        uint8_t f = (z > tauN + band) ? 1 : (z < tauN - band) ? 0 : 2;
        cin[k] = f;
        amb += (f == 2);
    }
    amb = block_sum_i<NT>(amb, shi);
    if (amb > 0) {
        for (int k0 = 0; k0 < ncand; ++k0) {
            if (cin[k0] != 2) continue;           // uniform: cin is shared memory
            const double zk = a * (double)cs[k0];
            double F = 0.0, dummy = 0.0;
            for (int k = threadIdx.x; k < ncand; k += NT) {
                const double d = a * (double)cs[k] - zk;
                if (d > 0.0) F += powb(d, beta, ib);
            }
            block_sum2_d<NT>(F, dummy, shd);
            if (threadIdx.x == 0) cin[k0] = (F < 1.0) ? 1 : 0;
            __syncthreads();
        }
    }
    // ---- tau from the support
    double S1 = 0.0, kk = 0.0;
    for (int k = threadIdx.x; k < ncand; k += NT)
        if (cin[k]) { S1 += a * (double)cs[k]; kk += 1.0; }
    block_sum2_d<NT>(S1, kk, shd);
    double tau;
    if (ib == 1) {
        tau = (S1 - 1.0) / kk;
    } else if (ib == 2) {
        const double m = S1 / kk;
        double ss = 0.0, dz = 0.0;
        for (int k = threadIdx.x; k < ncand; k += NT)
            if (cin[k]) { const double d = a * (double)cs[k] - m; ss += d * d; }
        block_sum2_d<NT>(ss, dz, shd);
        tau = m - sqrt(fmax(0.0, 1.0 - ss) / kk);
    } else {
        double F = 0.0, Fd = 0.0;
        for (int k = threadIdx.x; k < ncand; k += NT)
            if (cin[k]) { const double d = a * (double)cs[k] - tauN; F += powb(d, beta, ib); Fd += powbm1(d, beta, ib); }
        block_sum2_d<NT>(F, Fd, shd);
        tau = tauN + (F - 1.0) / (beta * Fd);
    }
    // ---- p and PV (warp per support token, lane = 4 dims)
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    double psum = 0.0;
    for (int k = warp; k < ncand; k += NT / 32) {
        if (!cin[k]) continue;
        const double d = a * (double)cs[k] - tau;
        const double pd = d > 0.0 ? powb(d, beta, ib) : 0.0;
        if (lane == 0) psum += pd;
        const float p = (float)pd;
        const T *vr = v_row(cj[k]) + 4 * lane;
        float vx[4];
        if constexpr (sizeof(T) == 2) {
            const uint2 w = *reinterpret_cast<const uint2 *>(vr);
            vx[0] = bf_lo(w.x); vx[1] = bf_hi(w.x); vx[2] = bf_lo(w.y); vx[3] = bf_hi(w.y);
        } else {
            const float4 w = *reinterpret_cast<const float4 *>(vr);
            vx[0] = w.x; vx[1] = w.y; vx[2] = w.z; vx[3] = w.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = __fmaf_rn(p, vx[e], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) red[warp][4 * lane + e] = acc[e];
    const double pt = block_sum_d<NT>(psum, shd);
    if (threadIdx.x < kD) {
        float o = 0.f;
        for (int w = 0; w < NT / 32; ++w) o = __fadd_rn(o, red[w][threadIdx.x]);
        A.out[(size_t)row * kD + threadIdx.x] = (float)((double)o / pt);
    }
    if (threadIdx.x == 0) {
        if (A.tau_out) A.tau_out[row] = tau;
        if (A.supp_out) A.supp_out[row] = (int)kk;
    }
    // ---- eval list: support tokens (slot index) and p, for exact delta / rho
    if (A.tok_list) {
        int base = 0;
        for (int r0 = 0; r0 < ncand; r0 += NT) {
            const int k = r0 + threadIdx.x;
            const int keep = (k < ncand && cin[k]) ? 1 : 0;
            int tot;
            const int pos = block_excl_scan<NT>(keep, shi, &tot);
            if (keep && base + pos < A.list_cap) {
                const double d = a * (double)cs[k] - tau;
                A.tok_list[(size_t)row * A.list_cap + base + pos] = cj[k];
                A.p_list[(size_t)row * A.list_cap + base + pos] = d > 0.0 ? powb(d, beta, ib) : 0.0;
            }
            base += tot;
        }
        if (threadIdx.x == 0) A.n_list[row] = base;
    }
    // ---- certified dropped-mass bound (R16): sum over unselected pages
    if (A.delta_bar) {
        const int M = n_pages_of(L);
        const int32_t *pl = A.page_idx + (size_t)row * A.sel_stride;
        const int ns = A.n_sel[row];
        const float *bx = A.box + (size_t)row * c.maxp;
        double db = 0.0, dz = 0.0;
        for (int p = threadIdx.x; p < M; p += NT) {
            // membership by binary search in the ascending page list
            int lo = 0, hi = ns;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (pl[mid] < p) lo = mid + 1; else hi = mid; }
            if (lo < ns && pl[lo] == p) continue;
            const double d = a * (double)bx[p] - tau;
            if (d > 0.0) db += (double)min(kP, L - p * kP) * powb(d, beta, ib);
        }
        block_sum2_d<NT>(db, dz, shd);
        if (threadIdx.x == 0) A.delta_bar[row] = db;
    }
}

// ============================================================================ eval: exact delta / rho
// One CTA per (b, q-head): the full pass's support list (token positions j and p_j)
// against the sparse selection (page list of head h): delta = sum of p_j over tokens
// whose page is not selected (Eq. delta), recovered = |S cap C_tok|,
// full_supp = |S| (Eq. rho).
__global__ void __launch_bounds__(256) k_eval_metrics(const int32_t *__restrict__ tok_list, const double *__restrict__ p_list,
                                                      const int32_t *__restrict__ n_list, int list_cap,
                                                      const int32_t *__restrict__ page_idx, const int32_t *__restrict__ n_sel,
                                                      int sel_stride, double *delta, int32_t *recovered, int32_t *full_supp) {
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
        const int p = j / kP;        // full pass: slot == token position
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
