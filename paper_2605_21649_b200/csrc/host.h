// host.h -- host-side internals of libentmaxkv shared by its translation units:
// status/error helpers, the launch wrapper (PDL + clusters), per-device attribute caches,
// the workspace layout and the per-kernel-family launch functions (each defined in the
// launch_*.cu file that includes that family's kernels).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string.h>
#include <utility>

#include "entmaxkv.h"
#include "types.cuh"

namespace ekvh {
using namespace ekv;

ekv_status fail(ekv_status st, const char *fmt, ...);
ekv_status check_launch(const char *what);          // cudaGetLastError + launch count
ekv_status check_err(cudaError_t e, const char *what);

#define EKV_TRY(x)                       \
    do {                                 \
        ekv_status _s = (x);             \
        if (_s != EKV_OK) return _s;     \
    } while (0)

bool pdl_enabled();
// Launch with programmatic stream serialisation (PDL; EKV_NO_PDL=1 disables it) and an
// optional thread-block cluster.  Every kernel of the decode chain starts with
// griddepcontrol.wait, so the next launch overlaps this one's tail.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, unsigned cluster,
                      Args &&...args) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// current device's SM count (cached per device)
int num_sms();
// kernel attributes are per device context: cached per (kernel, device)
void set_smem_raw(const void *kernel, int bytes, bool nonportable_cluster = false);
int resident_per_sm_raw(const void *kernel, int threads, int smem);
template <typename K> void set_smem(K kernel, int bytes, bool nonportable_cluster = false) {
    set_smem_raw(reinterpret_cast<const void *>(kernel), bytes, nonportable_cluster);
}
template <typename K> int resident_per_sm(K kernel, int threads, int smem) {
    return resident_per_sm_raw(reinterpret_cast<const void *>(kernel), threads, smem);
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
template <typename P> P *at(void *ws, size_t off) { return reinterpret_cast<P *>(static_cast<char *>(ws) + off); }

int sel_cap(const ekv_cache *c, const ekv_select_params *s);
void begin_call();                                  // clears the thread's error and launch count
// NVTX range per C-ABI call (nvtx3, header-only: no cost unless a tool such as nsys / ncu
// --nvtx is attached); EKV_CALL(name) = begin_call() + a range scoped to the entry point
struct NvtxRange {
    explicit NvtxRange(const char *name);
    ~NvtxRange();
};
#define EKV_CALL(name) ::ekvh::NvtxRange ekv_nvtx_range_(name); ::ekvh::begin_call()
ekv_status check_cache(const ekv_cache *c, int Hq);
ekv_status check_q(const void *q);
ekv_status check_attn(const ekv_attn_params *a);
ekv_status check_sel(const ekv_select_params *s, float alpha);
CacheView view(const ekv_cache *c);

// ---------------------------------------------------------------- workspace layout
// One layout serves decode (incl. eval_exact), select, sparse_attend and full_attend.
struct Layout {
    size_t box, mu, sigma2, page_idx, n_sel, tau_hat, gtab;
    size_t zero, status, retry, rowmax, ccount, umask, zero_bytes;   // zeroed per step / attention pass
    size_t tau_int, smx_acc, smx_l, smx_cnt, sink;
    int smx_nch;
    size_t scores, cand_s, cand_j, tok_list, p_list, n_list, full_out, total;
    int cap, W, list_cap;
};
Layout layout(const ekv_cache *c, int Hq, const ekv_select_params *sel);

// ---------------------------------------------------------------- launch_meta.cu
ekv_status launch_append(const CacheView &v, const void *k_new, const void *v_new, int n_tokens, cudaStream_t st);
ekv_status launch_rebuild(const CacheView &v, cudaStream_t st);
ekv_status launch_score(const CacheView &v, const void *q, int Hq, int modes, float *box, float *mu, float *s2,
                        uint4 *zero, size_t zero_n16, cudaStream_t st);
ekv_status launch_zero(uint4 *p, size_t n16, cudaStream_t st);

// ---------------------------------------------------------------- launch_select.cu
struct UnionOut {            // optional union marks done by the selection kernel
    uint32_t *umask; int W;
};
ekv_status launch_topk(const float *box, int B, int Hq, int maxp, const int32_t *sl, int k, int32_t *pi, int32_t *ns,
                       int stride, int G, const UnionOut &u, cudaStream_t st);
ekv_status launch_box_certified(const float *box, int B, int Hq, int G, int maxp, const int32_t *seq_lens,
                                const double *tau_hat, float alpha, int32_t *pi, int32_t *ns, int stride,
                                uint32_t *um, int W, cudaStream_t st);
ekv_status launch_mark(int B, int Hq, int G, const int32_t *pi, const int32_t *ns, int stride, uint32_t *um, int W,
                       cudaStream_t st);
ekv_status launch_gauss(const ekv_cache *cache, int Hq, const float *mu, const float *s2, float alpha,
                        const ekv_select_params *sel, int32_t *pi, int32_t *ns, int stride, double *th, double *gtab,
                        cudaStream_t st);

// ---------------------------------------------------------------- launch_attend.cu
ekv_status launch_scores(const CacheView &v, const void *q, int Hq, const uint32_t *um, int W, const int32_t *pi,
                         const int32_t *ns, int stride, float *scores, uint32_t *rowmax, int full, cudaStream_t st);
ekv_status launch_candidates(const float *scores, size_t ntok, const uint32_t *rowmax, const int32_t *seq_lens,
                             int Hq, float alpha, int nch, int rows, int *ccount, float *cs, int32_t *cj,
                             cudaStream_t st);
ekv_status launch_delta_bar(const float *box, int maxp, const int32_t *seq_lens, int rows, int Hq, int G,
                            const uint32_t *umask, int W, const double *tau, float alpha, double *out, cudaStream_t st);
ekv_status launch_eval_metrics(int rows, const int32_t *tok_list, const double *p_list, const int32_t *n_list,
                               int list_cap, const int32_t *pi, const int32_t *ns, int stride, double *delta,
                               int32_t *recovered, int32_t *full_supp, cudaStream_t st);
// split dense-V / softmax passes (kernels_dense.cuh)
ekv_status launch_softmax_partial(const CacheView &v, const float *scores, size_t ntok, const uint32_t *rowmax,
                                  const int32_t *pi, const int32_t *ns, int stride, int full, int Hq, int nch,
                                  int rows, float *pacc, double *pl, int32_t *pc, cudaStream_t st);
ekv_status launch_dense_group(const CacheView &v, const float *scores, size_t ntok, const uint32_t *rowmax, int Hq,
                              int nch, float *pacc, double *pl, int32_t *pc, const double *ent_tau, float alpha,
                              cudaStream_t st);
ekv_status launch_vstream(const CacheView &v, uint32_t *sink, cudaStream_t st);   // dense-V: every V row read
ekv_status launch_full_scores_mma(const CacheView &v, const void *q, int Hq, float *scores, uint32_t *rowmax,
                                  cudaStream_t st);                                // a5 scores on tensor cores (R26)
ekv_status launch_softmax_combine(int rows, const float *pacc, const double *pl, const int32_t *pc,
                                  const uint32_t *rowmax, int nch, float *out, double *tau, int32_t *supp,
                                  cudaStream_t st);

// ---------------------------------------------------------------- launch_tau.cu (one object per dtype)
template <typename T> ekv_status launch_tau_sparse(const CacheView &v, const TauArgs &A, int rows, cudaStream_t st);
inline ekv_status launch_tau(const CacheView &v, const TauArgs &A, int rows, cudaStream_t st) {
    return v.dtype == EKV_BF16 ? launch_tau_sparse<__nv_bfloat16>(v, A, rows, st) : launch_tau_sparse<float>(v, A, rows, st);
}

// integer beta = 1/(alpha-1) in 1..4, else 0
int int_beta(float alpha);

const char *last_error();
int last_launches();
}  // namespace ekvh
#include <vector>
namespace ekvh {
std::vector<ekv::DebugReader> &debug_readers();   // per-TU stamp readers (-DEKV_STAMPS builds)

}  // namespace ekvh
