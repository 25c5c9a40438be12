// launch_attend.cu -- launches of the K-score, candidate, delta_bar, eval-metric and split
// dense-V / softmax kernels (a3-a6).
#include <algorithm>
#include <cmath>
#include "host.h"
#include "kernels_dense.cuh"

namespace ekvh {

namespace {
template <typename T, int G>
void scores_t(const CacheView &v, const void *q, int Hq, const uint32_t *um, int W, const int32_t *pi,
              const int32_t *ns, int stride, float *scores, uint32_t *rowmax, int full, cudaStream_t st) {
    constexpr int smem = AttCfg<T>::template smem<G>();
    constexpr int NT = 32 * (AttCfg<T>::NCW + 1);
    set_smem(k_attend_scores<T, G>, smem);
    const int per_sm = resident_per_sm(k_attend_scores<T, G>, NT, smem);
    const long long slots = full ? (long long)v.B * v.Hkv * v.maxp : (long long)v.B * Hq * stride;
    long long gx = (slots + 31) / 32;                                // >= 32 work slots per CTA
    if (gx > (long long)per_sm * num_sms()) gx = (long long)per_sm * num_sms();
    if (gx < 1) gx = 1;
    launch_ex(k_attend_scores<T, G>, dim3((unsigned)gx), dim3(NT), smem, st, 0, v, static_cast<const T *>(q), Hq, um, W,
              pi, ns, stride, scores, rowmax, full);
}
template <typename T>
void scores_dt(const CacheView &v, const void *q, int Hq, const uint32_t *um, int W, const int32_t *pi,
               const int32_t *ns, int stride, float *scores, uint32_t *rowmax, int full, cudaStream_t st) {
    switch (Hq / v.Hkv) {
    case 1: scores_t<T, 1>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st); break;
    case 2: scores_t<T, 2>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st); break;
    case 4: scores_t<T, 4>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st); break;
    default: scores_t<T, 8>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st); break;
    }
}
}  // namespace

ekv_status launch_scores(const CacheView &v, const void *q, int Hq, const uint32_t *um, int W, const int32_t *pi,
                         const int32_t *ns, int stride, float *scores, uint32_t *rowmax, int full, cudaStream_t st) {
    if (v.dtype == EKV_BF16) scores_dt<__nv_bfloat16>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st);
    else scores_dt<float>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st);
    return check_launch("k_attend_scores");
}

ekv_status launch_candidates(const float *scores, size_t ntok, const uint32_t *rowmax, const int32_t *seq_lens,
                             int Hq, float alpha, int nch, int rows, int *ccount, float *cs, int32_t *cj,
                             cudaStream_t st) {
    dim3 cg(nch, rows);
    k_candidates<<<cg, kCandNT, 0, st>>>(scores, ntok, rowmax, seq_lens, Hq, alpha, nch, ccount, cs, cj);
    return check_launch("k_candidates");
}

ekv_status launch_delta_bar(const float *box, int maxp, const int32_t *seq_lens, int rows, int Hq, int G,
                            const uint32_t *umask, int W, const double *tau, float alpha, double *out, cudaStream_t st) {
    const int nch = (maxp + kDbChunk - 1) / kDbChunk;   // <= 8 (max_pages <= 65536)
    DbConst kc;
    kc.a = (double)alpha - 1.0;
    kc.beta = 1.0 / kc.a;
    kc.inv_a = kc.beta;
    kc.ib = int_beta(alpha);
    const dim3 dg((unsigned)nch, (unsigned)rows), db(256);
    cudaError_t ce;
    switch (kc.ib) {
    case 1: ce = launch_ex(k_delta_bar<1>, dg, db, 0, st, (unsigned)nch, box, maxp, seq_lens, Hq, G, umask, W, tau, kc, out); break;
    case 2: ce = launch_ex(k_delta_bar<2>, dg, db, 0, st, (unsigned)nch, box, maxp, seq_lens, Hq, G, umask, W, tau, kc, out); break;
    case 3: ce = launch_ex(k_delta_bar<3>, dg, db, 0, st, (unsigned)nch, box, maxp, seq_lens, Hq, G, umask, W, tau, kc, out); break;
    case 4: ce = launch_ex(k_delta_bar<4>, dg, db, 0, st, (unsigned)nch, box, maxp, seq_lens, Hq, G, umask, W, tau, kc, out); break;
    default: ce = launch_ex(k_delta_bar<0>, dg, db, 0, st, (unsigned)nch, box, maxp, seq_lens, Hq, G, umask, W, tau, kc, out); break;
    }
    if (ce != cudaSuccess) return fail(EKV_ERR_CUDA, "k_delta_bar: %s", cudaGetErrorString(ce));
    return check_launch("k_delta_bar");
}

ekv_status launch_eval_metrics(int rows, const int32_t *tok_list, const double *p_list, const int32_t *n_list,
                               int list_cap, const int32_t *pi, const int32_t *ns, int stride, double *delta,
                               int32_t *recovered, int32_t *full_supp, cudaStream_t st) {
    k_eval_metrics<<<rows, 256, 0, st>>>(tok_list, p_list, n_list, list_cap, pi, ns, stride, delta, recovered, full_supp);
    return check_launch("k_eval_metrics");
}

ekv_status launch_softmax_partial(const CacheView &v, const float *scores, size_t ntok, const uint32_t *rowmax,
                                  const int32_t *pi, const int32_t *ns, int stride, int full, int Hq, int nch,
                                  int rows, float *pacc, double *pl, int32_t *pc, cudaStream_t st) {
    dim3 g(nch, rows);
    if (v.dtype == EKV_BF16)
        k_softmax_partial<__nv_bfloat16><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, pi, ns, stride, full, Hq,
                                                             Hq / v.Hkv, nch, pacc, pl, pc, nullptr, 0.f);
    else
        k_softmax_partial<float><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, pi, ns, stride, full, Hq, Hq / v.Hkv, nch,
                                                    pacc, pl, pc, nullptr, 0.f);
    return check_launch("k_softmax_partial");
}

namespace {
template <typename T>
void dense_group_t(const CacheView &v, const float *scores, size_t ntok, const uint32_t *rowmax, int Hq, int nch,
                   float *pacc, double *pl, int32_t *pc, const double *ent_tau, float alpha, int ib, cudaStream_t st) {
    dim3 g(nch, v.B * v.Hkv);
    switch (Hq / v.Hkv) {
    case 1: k_dense_group_partial<T, 1><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    case 2: k_dense_group_partial<T, 2><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    case 4: k_dense_group_partial<T, 4><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    default: k_dense_group_partial<T, 8><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    }
}
}  // namespace

ekv_status launch_dense_group(const CacheView &v, const float *scores, size_t ntok, const uint32_t *rowmax, int Hq,
                              int nch, float *pacc, double *pl, int32_t *pc, const double *ent_tau, float alpha,
                              cudaStream_t st) {
    const int ib = ent_tau ? int_beta(alpha) : 0;
    if (v.dtype == EKV_BF16) dense_group_t<__nv_bfloat16>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib, st);
    else dense_group_t<float>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib, st);
    return check_launch("k_dense_group_partial");
}

ekv_status launch_full_scores_mma(const CacheView &v, const void *q, int Hq, float *scores, uint32_t *rowmax,
                                  cudaStream_t st) {
    const int G = Hq / v.Hkv;
    const int smem = 8 * 2 * 4096;
    const long long slots = (long long)v.B * v.Hkv * v.maxp;
    long long g = (slots + 63) / 64;                              // >= 8 slots per warp
    const long long cap = (long long)num_sms() * 3;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    const __nv_bfloat16 *qq = static_cast<const __nv_bfloat16 *>(q);
    cudaError_t e;
    switch (G) {
    case 1: set_smem(k_full_scores_mma<1>, smem); e = launch_ex(k_full_scores_mma<1>, dim3((unsigned)g), dim3(256), smem, st, 0, v, qq, Hq, scores, rowmax); break;
    case 2: set_smem(k_full_scores_mma<2>, smem); e = launch_ex(k_full_scores_mma<2>, dim3((unsigned)g), dim3(256), smem, st, 0, v, qq, Hq, scores, rowmax); break;
    case 4: set_smem(k_full_scores_mma<4>, smem); e = launch_ex(k_full_scores_mma<4>, dim3((unsigned)g), dim3(256), smem, st, 0, v, qq, Hq, scores, rowmax); break;
    default: set_smem(k_full_scores_mma<8>, smem); e = launch_ex(k_full_scores_mma<8>, dim3((unsigned)g), dim3(256), smem, st, 0, v, qq, Hq, scores, rowmax); break;
    }
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "k_full_scores_mma: %s", cudaGetErrorString(e));
    return check_launch("k_full_scores_mma");
}

ekv_status launch_vstream(const CacheView &v, uint32_t *sink, cudaStream_t st) {
    const long long slots = (long long)v.B * v.maxp;
    long long g = (slots + 7) / 8;
    const long long cap = (long long)num_sms() * 8;          // 8 CTAs (64 warps) per SM
    if (g > cap) g = cap;
    if (v.dtype == EKV_BF16) launch_ex(k_vstream<__nv_bfloat16>, dim3((unsigned)g), dim3(256), 0, st, 0, v, sink);
    else launch_ex(k_vstream<float>, dim3((unsigned)g), dim3(256), 0, st, 0, v, sink);
    return check_launch("k_vstream");
}

ekv_status launch_softmax_combine(int rows, const float *pacc, const double *pl, const int32_t *pc,
                                  const uint32_t *rowmax, int nch, float *out, double *tau, int32_t *supp,
                                  cudaStream_t st) {
    k_softmax_combine<<<rows, 128 * kCombSeg, 0, st>>>(pacc, pl, pc, rowmax, nch, out, tau, supp);
    return check_launch("k_softmax_combine");
}

}  // namespace ekvh
