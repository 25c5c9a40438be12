// launch_meta.cu -- launches of the a0 (append, rebuild) and a1 (page scoring) kernels.
#include "host.h"
#include "kernels_meta.cuh"

namespace ekvh {

ekv_status launch_append(const CacheView &v, const void *k_new, const void *v_new, int n_tokens, cudaStream_t st) {
    int nt = v.Hkv * kD;
    if (nt > 1024) nt = 1024;
    if (v.dtype == EKV_BF16)
        launch_ex(k_append<__nv_bfloat16>, dim3(v.B), dim3(nt), 0, st, 0, v, static_cast<const __nv_bfloat16 *>(k_new),
                  static_cast<const __nv_bfloat16 *>(v_new), n_tokens);
    else
        launch_ex(k_append<float>, dim3(v.B), dim3(nt), 0, st, 0, v, static_cast<const float *>(k_new),
                  static_cast<const float *>(v_new), n_tokens);
    return check_launch("k_append");
}

ekv_status launch_rebuild(const CacheView &v, cudaStream_t st) {
    const size_t per_seq = (size_t)v.maxp * v.Hkv * kD;
    dim3 grid((unsigned)((per_seq + 255) / 256), v.B);
    if (v.dtype == EKV_BF16) k_rebuild<__nv_bfloat16><<<grid, 256, 0, st>>>(v);
    else k_rebuild<float><<<grid, 256, 0, st>>>(v);
    return check_launch("k_rebuild");
}

ekv_status launch_zero(uint4 *p, size_t n16, cudaStream_t st) {
    launch_ex(k_zero, dim3((unsigned)std::min<size_t>(148, (n16 + 255) / 256 + 1)), dim3(256), 0, st, 0, p, n16);
    return check_launch("k_zero");
}

namespace {
template <typename T, int G, int MODES, int FMT>
void score_go(const CacheView &v, const T *q, int Hq, float *box, float *mu, float *s2, uint4 *zero, size_t zero_n16,
              cudaStream_t st) {
    constexpr int SP = ScoreCfg<MODES, FMT>::SP, NS = ScoreCfg<MODES, FMT>::NS;
    const int HD = v.Hkv * kD;
    const int per_page = ((MODES & 1) ? 2 * HD * ((FMT & 1) ? 1 : (int)sizeof(T)) : 0) +
                         ((MODES & 2) ? 2 * HD * ((FMT & 2) ? 2 : 4) : 0);
    const int smem = NS * SP * per_page;
    set_smem(k_score<T, G, MODES, FMT>, smem);
    const int per_sm = resident_per_sm(k_score<T, G, MODES, FMT>, 288, smem);
    // persistent: one wave of resident CTAs over the flattened (b, page) space, >= 8 pages per CTA
    long long gx = ((long long)v.B * v.maxp + 7) / 8;
    if (gx > (long long)per_sm * num_sms()) gx = (long long)per_sm * num_sms();
    if (gx < 1) gx = 1;
    launch_ex(k_score<T, G, MODES, FMT>, dim3((unsigned)gx), dim3(288), smem, st, 0, v, q, Hq, box, mu, s2, zero, zero_n16);
}
template <typename T, int G>
void score_t(const CacheView &v, const void *q, int Hq, int modes, float *box, float *mu, float *s2, uint4 *zero,
             size_t zero_n16, cudaStream_t st) {
    const T *qq = static_cast<const T *>(q);
    // FMT: bit 0 = e4m3 bounds (box), bit 1 = bf16 kavg / kvar (Gaussian)
    const int be = v.bound ? 1 : 0, sb = v.stat ? 2 : 0;
    if (modes == 1) {
        if (be) score_go<T, G, 1, 1>(v, qq, Hq, box, mu, s2, zero, zero_n16, st);
        else score_go<T, G, 1, 0>(v, qq, Hq, box, mu, s2, zero, zero_n16, st);
    } else if (modes == 2) {
        if (sb) score_go<T, G, 2, 2>(v, qq, Hq, box, mu, s2, zero, zero_n16, st);
        else score_go<T, G, 2, 0>(v, qq, Hq, box, mu, s2, zero, zero_n16, st);
    } else {
        switch (be | sb) {
        case 0: score_go<T, G, 3, 0>(v, qq, Hq, box, mu, s2, zero, zero_n16, st); break;
        case 1: score_go<T, G, 3, 1>(v, qq, Hq, box, mu, s2, zero, zero_n16, st); break;
        case 2: score_go<T, G, 3, 2>(v, qq, Hq, box, mu, s2, zero, zero_n16, st); break;
        default: score_go<T, G, 3, 3>(v, qq, Hq, box, mu, s2, zero, zero_n16, st); break;
        }
    }
}
template <typename T>
void score_dt(const CacheView &v, const void *q, int Hq, int modes, float *box, float *mu, float *s2, uint4 *zero,
              size_t zero_n16, cudaStream_t st) {
    switch (Hq / v.Hkv) {
    case 1: score_t<T, 1>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st); break;
    case 2: score_t<T, 2>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st); break;
    case 4: score_t<T, 4>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st); break;
    default: score_t<T, 8>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st); break;
    }
}
}  // namespace

ekv_status launch_score(const CacheView &v, const void *q, int Hq, int modes, float *box, float *mu, float *s2,
                        uint4 *zero, size_t zero_n16, cudaStream_t st) {
    if (v.dtype == EKV_BF16) score_dt<__nv_bfloat16>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st);
    else score_dt<float>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st);
    return check_launch("k_score");
}

}  // namespace ekvh
