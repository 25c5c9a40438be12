// launch_tau.cu -- launches of the exact-tau / support / PV kernel (a3).  Compiled once per
// KV dtype (EKV_TAU_T = __nv_bfloat16 or float) so the two heavy instantiation sets build in
// parallel.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include "host.h"
#include "kernels_tau.cuh"

#ifndef EKV_TAU_T
#define EKV_TAU_T __nv_bfloat16
#endif

namespace ekvh {

namespace {
template <typename T, int IB, bool FULL>
ekv_status tau_ibf(const CacheView &v, const TauArgs &A0, int rows, cudaStream_t st) {
    TauArgs A = A0;
    A.cap = A.full ? kTsCap : std::min(kTsCap, (A.sel_stride * kP + 255) & ~255);
    if (A.retry_pass) A.cap = kTsCap;
    // variable-length (Gaussian) lists run many rows of up to max_pages entries: a smaller
    // candidate capacity keeps two CTAs per SM (measured C3: 126 -> 71 us); an overflowing
    // row falls back to the streamed path.  EKV_TS_CAP overrides.
    static const int cap_env = getenv("EKV_TS_CAP") ? atoi(getenv("EKV_TS_CAP")) : 0;
    const int cap_lim = cap_env > 0 ? cap_env : A.var ? 4096 : 0;
    if (cap_lim > 0 && !A.full && !A.retry_pass) A.cap = std::min(A.cap, (cap_lim + 255) & ~255);
    A.pr = std::min(kPr, A.cap);
    const int smem = (4 + 4 + 4 + 1) * A.cap + (8 + 4) * A.pr + kTsVpre * kD * (int)sizeof(T);
    set_smem(k_tau_sparse<T, IB, FULL>, ts_smem<T>(), /*nonportable_cluster=*/true);
    // a cluster of up to 4 CTAs per row splits the candidate extraction (page-list reads are
    // latency bound per SM); rank 0 then finishes the row
    const int CL = A.full ? 1 : A.sel_stride > 384 ? 4 : A.sel_stride > 128 ? 2 : 1;
    cudaError_t e = launch_ex(k_tau_sparse<T, IB, FULL>, dim3((unsigned)(rows * CL)), dim3(kTsNT), smem, st, (unsigned)CL, v, A);
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "k_tau_sparse: %s", cudaGetErrorString(e));
    return check_launch("k_tau_sparse");
}
template <typename T, int IB>
ekv_status tau_ib(const CacheView &v, const TauArgs &A0, int rows, cudaStream_t st) {
    if (A0.full) return tau_ibf<T, IB, true>(v, A0, rows, st);
    return tau_ibf<T, IB, false>(v, A0, rows, st);
}
}  // namespace

// integer beta = 1/(alpha-1) in 1..4 is a template constant; any other alpha -> IB = 0
template <typename T>
ekv_status tau_dispatch(const CacheView &v, const TauArgs &A, int rows, cudaStream_t st) {
    switch (int_beta(A.alpha)) {
    case 1: return tau_ib<T, 1>(v, A, rows, st);
    case 2: return tau_ib<T, 2>(v, A, rows, st);
    case 3: return tau_ib<T, 3>(v, A, rows, st);
    case 4: return tau_ib<T, 4>(v, A, rows, st);
    default: return tau_ib<T, 0>(v, A, rows, st);
    }
}
template <typename T>
ekv_status launch_tau_sparse(const CacheView &v, const TauArgs &A, int rows, cudaStream_t st) {
    EKV_TRY(tau_dispatch<T>(v, A, rows, st));
    // variable-length lists run at a reduced candidate capacity: rows whose support did not fit
    // are re-run at the full capacity (CTAs of the other rows exit at once)
    const bool reduced = !A.full && A.var && A.retry;
    if (!reduced) return EKV_OK;
    TauArgs B = A;
    B.retry_pass = 1;
    return tau_dispatch<T>(v, B, rows, st);
}
template ekv_status launch_tau_sparse<EKV_TAU_T>(const CacheView &, const TauArgs &, int, cudaStream_t);

}  // namespace ekvh
