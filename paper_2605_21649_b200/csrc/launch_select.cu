// launch_select.cu -- launches of the a2 (top-k), a2' (Gaussian selector) and union-mark kernels.
#include <algorithm>
#include <cmath>
#include "host.h"
#include "kernels_select.cuh"

namespace ekvh {

// top-k: one cluster of CL CTAs per row, CL = pages / 8192 rounded up to a power of two
ekv_status launch_topk(const float *box, int B, int Hq, int maxp, const int32_t *sl, int k, int32_t *pi, int32_t *ns,
                       int stride, int G, const UnionOut &u, cudaStream_t st) {
    // short rows: 256-thread CTAs (more CTAs per SM when there are many rows)
    const int NT = maxp <= 4096 ? 256 : 512;
    const int per = NT * kTkKPT;
    int CL = 1;
    while (CL * per < maxp) CL *= 2;
    if (CL > 8) return fail(EKV_ERR_UNSUPPORTED, "top-k supports at most %d pages", 8 * per);
    const int smem = 2 * kTkCap * 8;      // sample-pivot candidate lists
    set_smem(k_topk<256>, smem);
    set_smem(k_topk<512>, smem);
    cudaError_t e = NT == 256
        ? launch_ex(k_topk<256>, dim3((unsigned)(B * Hq * CL)), dim3(256), smem, st, (unsigned)CL, box, Hq, maxp, sl, k,
                    pi, ns, stride, G, u.umask, u.W)
        : launch_ex(k_topk<512>, dim3((unsigned)(B * Hq * CL)), dim3(512), smem, st, (unsigned)CL, box, Hq, maxp, sl, k,
                    pi, ns, stride, G, u.umask, u.W);
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "k_topk: %s", cudaGetErrorString(e));
    return check_launch("k_topk");
}

ekv_status launch_mark(int B, int Hq, int G, const int32_t *pi, const int32_t *ns, int stride, uint32_t *um, int W,
                       cudaStream_t st) {
    launch_ex(k_mark, dim3(B * Hq), dim3(256), 0, st, 0, Hq, G, pi, ns, stride, um, W);
    return check_launch("k_mark");
}

ekv_status launch_box_certified(const float *box, int B, int Hq, int G, int maxp, const int32_t *seq_lens,
                                const double *tau_hat, float alpha, int32_t *pi, int32_t *ns, int stride,
                                uint32_t *um, int W, cudaStream_t st) {
    launch_ex(k_box_certified, dim3(B * Hq), dim3(512), 0, st, 0, box, Hq, G, maxp, seq_lens, tau_hat, alpha, pi, ns,
              stride, um, W);
    return check_launch("k_box_certified");
}

// a2': one CTA per (b, q-head); rows of up to 8192 pages staged in shared memory.  Many rows
// (>= 2 per SM): 512-thread CTAs, two per SM, so one row's reductions overlap the other's
// passes (C3: 244 -> 212 us); few rows: 1024 threads per row.
template <int NT>
static ekv_status launch_gauss_nt(const ekv_cache *cache, int Hq, const float *mu, const float *s2, float alpha,
                                  const ekv_select_params *sel, int32_t *pi, int32_t *ns, int stride, double *th,
                                  const double *gtab, int CL, cudaStream_t st) {
    const int maxp = cache->max_pages_per_seq;
    const int cache_pages = std::min((maxp + CL - 1) / CL, 8192);
    const int smem = 12 * cache_pages;
    set_smem(k_gauss_select<NT>, 12 * 8192);
    cudaError_t e = launch_ex(k_gauss_select<NT>, dim3((unsigned)(cache->batch * Hq * CL)), dim3(NT), smem, st,
                              (unsigned)(CL > 1 ? CL : 0), mu, s2, Hq, maxp, (const int32_t *)cache->seq_lens, alpha,
                              sel->margin, sel->q_page, pi, ns, stride, th, cache_pages, gtab);
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "k_gauss_select: %s", cudaGetErrorString(e));
    return check_launch("k_gauss_select");
}
ekv_status launch_gauss(const ekv_cache *cache, int Hq, const float *mu, const float *s2, float alpha,
                        const ekv_select_params *sel, int32_t *pi, int32_t *ns, int stride, double *th, double *gtab,
                        cudaStream_t st) {
    // non-integer beta (or beta > 4): the per-call moment table first (N4, R28)
    const double bf = 1.0 / ((double)alpha - 1.0);
    const bool closed = std::fabs(bf - std::rint(bf)) < 1e-9 && std::rint(bf) >= 1.0 && std::rint(bf) <= 4.0;
    if (!closed) {
        if (!gtab) return fail(EKV_ERR_INVALID_ARG, "non-integer beta: the Gaussian selector needs the workspace");
        launch_ex(k_gauss_table, dim3(kGtI), dim3(kGtN), 0, st, 0u, bf, gtab);
        EKV_TRY(check_launch("k_gauss_table"));
    }
    // rows longer than the 8192-page shared-memory stage are split over a cluster of CL CTAs
    // (C4: 65536 pages -> 8 CTAs per row, each row's slices staged in shared memory).  The
    // block size and CL (and so the fp64 reduction order of tau_hat) depend on the shape:
    // tau_hat is reproducible per configuration, and within 1e-10 relative of the oracle (R14)
    int CL = 1;
    while (CL < 8 && (cache->max_pages_per_seq + CL - 1) / CL > 8192) CL *= 2;
    const long long ctas = (long long)cache->batch * Hq * CL;
    if (ctas > num_sms())
        return launch_gauss_nt<512>(cache, Hq, mu, s2, alpha, sel, pi, ns, stride, th, gtab, CL, st);
    return launch_gauss_nt<1024>(cache, Hq, mu, s2, alpha, sel, pi, ns, stride, th, gtab, CL, st);
}

}  // namespace ekvh
