// entmaxkv.cu -- host side of libentmaxkv.so: argument validation, workspace
// carve-out and kernel launches behind the C ABI of include/entmaxkv.h.
// Everything runs on the caller's stream; no allocation, no synchronisation.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
#include <utility>

#include "entmaxkv.h"
#include "common.cuh"
#include "kernels_meta.cuh"
#include "kernels_select.cuh"
#include "kernels_attend.cuh"
#include "kernels_tau.cuh"
#include "kernels_shard.cuh"

using namespace ekv;

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

ekv_status fail(ekv_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

ekv_status check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    ++g_launches;
    return EKV_OK;
}

// Launch with programmatic stream serialisation (PDL; EKV_NO_PDL=1 disables it) and an
// optional thread-block cluster.  Every kernel of the decode chain starts with
// griddepcontrol.launch_dependents / wait, so the next launch overlaps this one's tail.
bool pdl_enabled() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("EKV_NO_PDL"); v = (e && e[0] == '1') ? 0 : 1; }
    return v == 1;
}
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

#define EKV_TRY(x)                       \
    do {                                 \
        ekv_status _s = (x);             \
        if (_s != EKV_OK) return _s;     \
    } while (0)

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

ekv_status check_cache(const ekv_cache *c, int Hq) {
    if (!c) return fail(EKV_ERR_INVALID_ARG, "cache is NULL");
    if (c->dtype != EKV_BF16 && c->dtype != EKV_F32) return fail(EKV_ERR_INVALID_ARG, "bad dtype %d", c->dtype);
    if (c->head_dim != kD || c->value_dim != kD)
        return fail(EKV_ERR_UNSUPPORTED, "head_dim/value_dim must be %d (got %d/%d)", kD, c->head_dim, c->value_dim);
    if (c->page_size != kP) return fail(EKV_ERR_UNSUPPORTED, "page_size must be %d (got %d)", kP, c->page_size);
    const int hk = c->n_kv_heads;
    if (!(hk == 1 || hk == 2 || hk == 4 || hk == 8 || hk == 16))
        return fail(EKV_ERR_UNSUPPORTED, "n_kv_heads must be 1,2,4,8,16 (got %d)", hk);
    if (c->batch < 1 || c->max_pages_per_seq < 1 || c->n_phys_pages < 1)
        return fail(EKV_ERR_INVALID_ARG, "batch/max_pages/n_phys must be >= 1");
    if (c->max_pages_per_seq > 65536) return fail(EKV_ERR_UNSUPPORTED, "max_pages_per_seq > 65536");
    if (Hq > 0) {
        if (Hq % hk) return fail(EKV_ERR_INVALID_ARG, "n_q_heads %d not a multiple of n_kv_heads %d", Hq, hk);
        const int G = Hq / hk;
        if (!(G == 1 || G == 2 || G == 4 || G == 8)) return fail(EKV_ERR_UNSUPPORTED, "group size G=%d not in {1,2,4,8}", G);
    }
    if (!c->k_pages || !c->v_pages || !c->page_table || !c->seq_lens)
        return fail(EKV_ERR_INVALID_ARG, "NULL cache buffer");
    if (((uintptr_t)c->k_pages | (uintptr_t)c->v_pages) & 15)
        return fail(EKV_ERR_INVALID_ARG, "k_pages/v_pages must be 16-byte aligned");
    return EKV_OK;
}

ekv_status check_q(const void *q) {
    if (!q) return fail(EKV_ERR_INVALID_ARG, "q is NULL");
    if ((uintptr_t)q & 15) return fail(EKV_ERR_INVALID_ARG, "q must be 16-byte aligned");
    return EKV_OK;
}

CacheView view(const ekv_cache *c) {
    CacheView v;
    v.dtype = c->dtype; v.B = c->batch; v.Hkv = c->n_kv_heads; v.maxp = c->max_pages_per_seq;
    v.nphys = c->n_phys_pages;
    v.K = c->k_pages; v.V = c->v_pages; v.Kw = c->k_pages; v.Vw = c->v_pages;
    v.kmin = c->kmin; v.kmax = c->kmax;
    v.ksum = c->ksum; v.ksumsq = c->ksumsq; v.kavg = c->kavg; v.kvar = c->kvar;
    v.page_table = c->page_table; v.seq_lens = c->seq_lens;
    return v;
}

int c_max(const ekv_cache *c) { return c->max_pages_per_seq; }

int sel_cap(const ekv_cache *c, const ekv_select_params *s) {
    if (!s || s->policy != EKV_TOPK) return c->max_pages_per_seq;
    return s->k_pages < c->max_pages_per_seq ? s->k_pages : c->max_pages_per_seq;
}

// ---------------------------------------------------------------- workspace layout
// One layout serves decode (incl. eval_exact), select, sparse_attend and full_attend.
struct Layout {
    size_t box, mu, sigma2, page_idx, n_sel, tau_hat;
    size_t zero, rowmax, ccount, umask, zero_bytes;   // zeroed per step / attention pass
    size_t tau_int, smx_acc, smx_l, smx_cnt;
    int smx_nch;
    size_t scores, cand_s, cand_j, tok_list, p_list, n_list, full_out, total;
    int cap, W, list_cap;
};

Layout layout(const ekv_cache *c, int Hq, const ekv_select_params *sel) {
    Layout L;
    const size_t B = c->batch, Hkv = c->n_kv_heads, maxp = c->max_pages_per_seq;
    L.cap = sel_cap(c, sel);
    L.W = (int)((maxp + 3) / 4);
    L.list_cap = kCap;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += align256(bytes); return r; };
    L.box = take(B * Hq * maxp * 4);
    L.mu = take(B * Hq * maxp * 4);
    L.sigma2 = take(B * Hq * maxp * 4);
    L.page_idx = take(B * Hq * maxp * 4);          // capacity max_pages: also serves the eval pass
    L.n_sel = take(B * Hq * 4);
    L.tau_hat = take(B * Hq * 8);
    L.zero = o;
    L.rowmax = take(B * Hq * 4);
    L.ccount = take(B * Hq * (size_t)((maxp + 255) / 256) * 4);
    L.umask = take(B * Hkv * (size_t)L.W * 4);
    L.zero_bytes = o - L.zero;
    L.scores = take(B * Hq * maxp * kP * 4);
    L.cand_s = take(B * Hq * (size_t)((maxp + 255) / 256) * kCpc * 4);
    L.cand_j = take(B * Hq * (size_t)((maxp + 255) / 256) * kCpc * 4);
    L.tok_list = take(B * Hq * (size_t)L.list_cap * 4);
    L.p_list = take(B * Hq * (size_t)L.list_cap * 8);
    L.n_list = take(B * Hq * 4);
    L.full_out = take(B * Hq * kD * 4);
    L.tau_int = take(B * Hq * 8);
    L.smx_nch = (int)((maxp + kSmxPages - 1) / kSmxPages);
    L.smx_acc = take(B * Hq * (size_t)L.smx_nch * kD * 4);
    L.smx_l = take(B * Hq * (size_t)L.smx_nch * 8);
    L.smx_cnt = take(B * Hq * (size_t)L.smx_nch * 4);
    L.total = o;
    return L;
}

template <typename P> P *at(void *ws, size_t off) { return reinterpret_cast<P *>(static_cast<char *>(ws) + off); }

template <typename K> void set_smem(K kernel, int bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
// resident CTAs per SM of a persistent kernel (>= 1): grids are sized to one wave
template <typename K> int resident_per_sm(K kernel, int threads, int smem) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess || n < 1) n = 1;
    return n;
}

// ---------------------------------------------------------------- launch helpers
int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <typename T, int G, int MODES>
void score_go(const CacheView &v, const T *q, int Hq, float *box, float *mu, float *s2, uint4 *zero, size_t zero_n16,
              cudaStream_t st) {
    constexpr int SP = ScoreCfg<MODES>::SP, NS = ScoreCfg<MODES>::NS;
    const int HD = v.Hkv * kD;
    const int per_page = ((MODES & 1) ? 2 * HD * (int)sizeof(T) : 0) + ((MODES & 2) ? 2 * HD * 4 : 0);
    const int smem = NS * SP * per_page;
    static int init = 0, per_sm = 1;
    if (smem > init) {
        set_smem(k_score<T, G, MODES>, smem);
        init = smem;
    }
    static int occ_for = -1;
    if (occ_for != smem) { per_sm = resident_per_sm(k_score<T, G, MODES>, 288, smem); occ_for = smem; }
    // persistent: one wave of resident CTAs over the flattened (b, page) space, >= 8 pages per CTA
    long long gx = ((long long)v.B * v.maxp + 7) / 8;
    if (gx > per_sm * num_sms()) gx = per_sm * num_sms();
    if (gx < 1) gx = 1;
    launch_ex(k_score<T, G, MODES>, dim3((unsigned)gx), dim3(288), smem, st, 0, v, q, Hq, box, mu, s2, zero, zero_n16);
}
template <typename T, int G>
ekv_status launch_score_t(const CacheView &v, const void *q, int Hq, int modes, float *box, float *mu, float *s2,
                          uint4 *zero, size_t zero_n16,
                          cudaStream_t st) {
    const T *qq = static_cast<const T *>(q);
    if (modes == 1) score_go<T, G, 1>(v, qq, Hq, box, mu, s2, zero, zero_n16, st);
    else if (modes == 2) score_go<T, G, 2>(v, qq, Hq, box, mu, s2, zero, zero_n16, st);
    else score_go<T, G, 3>(v, qq, Hq, box, mu, s2, zero, zero_n16, st);
    return check_launch("k_score");
}
template <typename T>
ekv_status launch_score(const CacheView &v, const void *q, int Hq, int modes, float *box, float *mu, float *s2,
                        uint4 *zero, size_t zero_n16,
                        cudaStream_t st) {
    switch (Hq / v.Hkv) {
    case 1: return launch_score_t<T, 1>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st);
    case 2: return launch_score_t<T, 2>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st);
    case 4: return launch_score_t<T, 4>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st);
    default: return launch_score_t<T, 8>(v, q, Hq, modes, box, mu, s2, zero, zero_n16, st);
    }
}

struct UnionOut {            // optional union marks done by the selection kernel
    uint32_t *umask; int W;
};

// top-k: one cluster of CL CTAs per row, CL = pages / 8192 rounded up to a power of two
ekv_status launch_topk(const float *box, int B, int Hq, int maxp, const int32_t *sl, int k, int32_t *pi, int32_t *ns,
                       int stride, int G, const UnionOut &u, cudaStream_t st) {
    // short rows: 256-thread CTAs (more CTAs per SM when there are many rows)
    const int NT = maxp <= 4096 ? 256 : 512;
    const int per = NT * kTkKPT;
    int CL = 1;
    while (CL * per < maxp) CL *= 2;
    if (CL > 8) return fail(EKV_ERR_UNSUPPORTED, "top-k supports at most %d pages", 8 * per);
    cudaError_t e = NT == 256
        ? launch_ex(k_topk<256>, dim3((unsigned)(B * Hq * CL)), dim3(256), 0, st, (unsigned)CL, box, Hq, maxp, sl, k,
                    pi, ns, stride, G, u.umask, u.W)
        : launch_ex(k_topk<512>, dim3((unsigned)(B * Hq * CL)), dim3(512), 0, st, (unsigned)CL, box, Hq, maxp, sl, k,
                    pi, ns, stride, G, u.umask, u.W);
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "k_topk: %s", cudaGetErrorString(e));
    return check_launch("k_topk");
}

ekv_status launch_mark(const ekv_cache *c, int Hq, const int32_t *pi, const int32_t *ns, int stride, uint32_t *um,
                       int W, cudaStream_t st) {
    launch_ex(k_mark, dim3(c->batch * Hq), dim3(256), 0, st, 0, Hq, Hq / c->n_kv_heads, pi, ns, stride, um, W);
    return check_launch("k_mark");
}

template <typename T, int G>
ekv_status launch_scores_t(const CacheView &v, const void *q, int Hq, const uint32_t *um, int W, const int32_t *pi,
                           const int32_t *ns, int stride, float *scores, uint32_t *rowmax, int full, cudaStream_t st) {
    constexpr int smem = AttCfg<T>::template smem<G>();
    static int per_sm = 0;
    if (!per_sm) {
        set_smem(k_attend_scores<T, G>, smem);
        per_sm = resident_per_sm(k_attend_scores<T, G>, 32 * (AttCfg<T>::NCW + 1), smem);
    }
    const long long slots = full ? (long long)v.B * v.Hkv * v.maxp : (long long)v.B * Hq * stride;
    long long gx = (slots + 31) / 32;                                // >= 32 work slots per CTA
    if (gx > per_sm * num_sms()) gx = per_sm * num_sms();
    if (gx < 1) gx = 1;
    launch_ex(k_attend_scores<T, G>, dim3((unsigned)gx), dim3(32 * (AttCfg<T>::NCW + 1)), smem, st, 0, v,
              static_cast<const T *>(q), Hq, um, W, pi, ns, stride, scores, rowmax, full);
    return check_launch("k_attend_scores");
}
template <typename T>
ekv_status launch_scores(const CacheView &v, const void *q, int Hq, const uint32_t *um, int W, const int32_t *pi,
                         const int32_t *ns, int stride, float *scores, uint32_t *rowmax, int full, cudaStream_t st) {
    switch (Hq / v.Hkv) {
    case 1: return launch_scores_t<T, 1>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st);
    case 2: return launch_scores_t<T, 2>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st);
    case 4: return launch_scores_t<T, 4>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st);
    default: return launch_scores_t<T, 8>(v, q, Hq, um, W, pi, ns, stride, scores, rowmax, full, st);
    }
}

template <typename T, int IB, bool FULL>
ekv_status launch_tau_sparse_ibf(const CacheView &v, const TauArgs &A0, int rows, cudaStream_t st) {
    static bool init = false;
    TauArgs A = A0;
    A.cap = A.full ? kTsCap : std::min(kTsCap, (A.sel_stride * kP + 255) & ~255);
    // variable-length (Gaussian) lists run many rows of up to max_pages entries: a smaller
    // candidate capacity keeps two CTAs per SM (measured C3: 126 -> 71 us); an overflowing
    // row falls back to the streamed path (correct, slower).  EKV_TS_CAP overrides.
    static const int cap_env = getenv("EKV_TS_CAP") ? atoi(getenv("EKV_TS_CAP")) : 0;
    const int cap_lim = cap_env > 0 ? cap_env : A.var ? 4096 : 0;
    if (cap_lim > 0 && !A.full) A.cap = std::min(A.cap, (cap_lim + 255) & ~255);
    A.pr = std::min(kPr, A.cap);
    const int smem = (4 + 4 + 4 + 1) * A.cap + (8 + 4) * A.pr + kTsVpre * kD * (int)sizeof(T);
    if (!init) {
        set_smem(k_tau_sparse<T, IB, FULL>, ts_smem<T>());
        cudaFuncSetAttribute(k_tau_sparse<T, IB, FULL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        init = true;
    }
    // a cluster of up to 4 CTAs per row splits the candidate extraction (page-list reads are
    // latency bound per SM); rank 0 then finishes the row
    const int CL = A.full ? 1 : A.sel_stride > 384 ? 4 : A.sel_stride > 128 ? 2 : 1;
    cudaError_t e = launch_ex(k_tau_sparse<T, IB, FULL>, dim3((unsigned)(rows * CL)), dim3(kTsNT), smem, st, (unsigned)CL, v, A);
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "k_tau_sparse: %s", cudaGetErrorString(e));
    return check_launch("k_tau_sparse");
}
template <typename T, int IB>
ekv_status launch_tau_sparse_ib(const CacheView &v, const TauArgs &A0, int rows, cudaStream_t st) {
    if (A0.full) return launch_tau_sparse_ibf<T, IB, true>(v, A0, rows, st);
    return launch_tau_sparse_ibf<T, IB, false>(v, A0, rows, st);
}
// integer beta = 1/(alpha-1) in 1..4 is a template constant; any other alpha -> IB = 0
template <typename T>
ekv_status launch_tau_sparse(const CacheView &v, const TauArgs &A, int rows, cudaStream_t st) {
    const double beta = 1.0 / ((double)A.alpha - 1.0);
    const int ib = (std::fabs(beta - std::rint(beta)) < 1e-12 && beta <= 4.5) ? (int)std::rint(beta) : 0;
    switch (ib) {
    case 1: return launch_tau_sparse_ib<T, 1>(v, A, rows, st);
    case 2: return launch_tau_sparse_ib<T, 2>(v, A, rows, st);
    case 3: return launch_tau_sparse_ib<T, 3>(v, A, rows, st);
    case 4: return launch_tau_sparse_ib<T, 4>(v, A, rows, st);
    default: return launch_tau_sparse_ib<T, 0>(v, A, rows, st);
    }
}

template <typename T>
ekv_status launch_dense_group(const CacheView &v, const float *scores, size_t ntok, const uint32_t *rowmax, int Hq,
                              int nch, float *pacc, double *pl, int32_t *pc, const double *ent_tau, float alpha,
                              cudaStream_t st) {
    const int G = Hq / v.Hkv;
    int ib = 0;
    if (ent_tau) {
        const double beta = 1.0 / ((double)alpha - 1.0);
        ib = (std::fabs(beta - std::rint(beta)) < 1e-12 && beta <= 4.5) ? (int)std::rint(beta) : 0;
    }
    dim3 g(nch, v.B * v.Hkv);
    switch (G) {
    case 1: k_dense_group_partial<T, 1><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    case 2: k_dense_group_partial<T, 2><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    case 4: k_dense_group_partial<T, 4><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    default: k_dense_group_partial<T, 8><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, ent_tau, alpha, ib); break;
    }
    return check_launch("k_dense_group_partial");
}

// a2': one CTA per (b, q-head); rows of up to 8192 pages staged in shared memory.  Many rows
// (>= 2 per SM): 512-thread CTAs, two per SM, so one row's reductions overlap the other's
// passes (C3: 244 -> 212 us); few rows: 1024 threads per row.
template <int NT>
ekv_status launch_gauss_nt(const ekv_cache *cache, int Hq, const float *mu, const float *s2, float alpha,
                           const ekv_select_params *sel, int32_t *pi, int32_t *ns, int stride, double *th,
                           cudaStream_t st) {
    static bool init = false;
    const int cache_pages = std::min(cache->max_pages_per_seq, 8192);
    const int smem = 12 * cache_pages;
    if (!init) {
        set_smem(k_gauss_select<NT>, 12 * 8192);
        init = true;
    }
    cudaError_t e = launch_ex(k_gauss_select<NT>, dim3((unsigned)(cache->batch * Hq)), dim3(NT), smem, st, 0u, mu, s2, Hq,
                              (int)cache->max_pages_per_seq, (const int32_t *)cache->seq_lens, alpha, sel->margin,
                              sel->q_page, pi, ns, stride, th, cache_pages);
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "k_gauss_select: %s", cudaGetErrorString(e));
    return check_launch("k_gauss_select");
}
ekv_status launch_gauss(const ekv_cache *cache, int Hq, const float *mu, const float *s2, float alpha,
                        const ekv_select_params *sel, int32_t *pi, int32_t *ns, int stride, double *th, cudaStream_t st) {
    if (cache->batch * Hq >= 2 * 148)
        return launch_gauss_nt<512>(cache, Hq, mu, s2, alpha, sel, pi, ns, stride, th, st);
    return launch_gauss_nt<1024>(cache, Hq, mu, s2, alpha, sel, pi, ns, stride, th, st);
}

ekv_status check_attn(const ekv_attn_params *a) {
    if (!a) return fail(EKV_ERR_INVALID_ARG, "attn params NULL");
    if (a->transform != EKV_ENTMAX && a->transform != EKV_SOFTMAX) return fail(EKV_ERR_INVALID_ARG, "bad transform");
    if (a->transform == EKV_ENTMAX && !(a->alpha > 1.0f)) return fail(EKV_ERR_INVALID_ARG, "alpha must be > 1");
    if (a->tau_halley < 0 || a->tau_halley > 32) return fail(EKV_ERR_INVALID_ARG, "tau_halley must be in 0..32");
    return EKV_OK;
}

ekv_status check_sel(const ekv_select_params *s, float alpha) {
    if (!s) return fail(EKV_ERR_INVALID_ARG, "select params NULL");
    if (s->policy == EKV_TOPK) {
        if (s->k_pages < 1) return fail(EKV_ERR_INVALID_ARG, "k_pages must be >= 1");
    } else if (s->policy == EKV_GAUSS) {
        if (!(s->q_page > 0.0 && s->q_page < 1.0)) return fail(EKV_ERR_INVALID_ARG, "q_page must be in (0,1)");
        if (!(s->margin >= 0.0)) return fail(EKV_ERR_INVALID_ARG, "margin must be >= 0");
        const double beta = 1.0 / ((double)alpha - 1.0);
        const double rb = (double)(long long)(beta + 0.5);
        if (!(alpha > 1.0f) || fabs(beta - rb) > 1e-9 || rb < 1 || rb > 4)
            return fail(EKV_ERR_UNSUPPORTED, "Gaussian selector needs integer beta=1/(alpha-1) in {1,2,3,4} (alpha=%g)",
                        (double)alpha);
    } else if (s->policy != EKV_ALL) {
        return fail(EKV_ERR_INVALID_ARG, "bad policy %d", s->policy);
    }
    return EKV_OK;
}

// attention of every (b, q-head) over its page list (full: every page):
// memset(rowmax, ccount, umask) -> [mark] -> K scores -> candidates -> tau/PV
ekv_status attend_impl(const ekv_cache *c, const void *q, int Hq, const int32_t *pi, const int32_t *ns, int stride,
                       int full, const ekv_attn_params *attn, float *out, double *tau, int32_t *supp, void *ws,
                       const Layout &L, cudaStream_t st, const TauArgs *extra, bool marked = false) {
    const CacheView v = view(c);
    uint32_t *rowmax = at<uint32_t>(ws, L.rowmax);
    int *ccount = at<int>(ws, L.ccount);
    uint32_t *um = at<uint32_t>(ws, L.umask);
    float *scores = at<float>(ws, L.scores);
    if (!marked && cudaMemsetAsync(at<char>(ws, L.zero), 0, L.zero_bytes, st) != cudaSuccess)
        return fail(EKV_ERR_CUDA, "memset: %s", cudaGetErrorString(cudaGetLastError()));
    if (!full && !marked) EKV_TRY(launch_mark(c, Hq, pi, ns, stride, um, L.W, st));
    if (c->dtype == EKV_BF16)
        EKV_TRY(launch_scores<__nv_bfloat16>(v, q, Hq, um, L.W, pi, ns, stride, scores, rowmax, full, st));
    else EKV_TRY(launch_scores<float>(v, q, Hq, um, L.W, pi, ns, stride, scores, rowmax, full, st));
#ifdef EKV_STAMPS
    if (getenv("EKV_ATT_TWICE")) {                 // debug: warm instruction cache experiment
        if (c->dtype == EKV_BF16)
            EKV_TRY(launch_scores<__nv_bfloat16>(v, q, Hq, um, L.W, pi, ns, stride, scores, rowmax, full, st));
        else EKV_TRY(launch_scores<float>(v, q, Hq, um, L.W, pi, ns, stride, scores, rowmax, full, st));
    }
#endif
    const int rows = c->batch * Hq;
    const size_t ntok = (size_t)c->max_pages_per_seq * kP;
    float *cs = at<float>(ws, L.cand_s);
    int32_t *cj = at<int32_t>(ws, L.cand_j);
    // full rows are long: candidates extracted by a wide kernel; sparse rows are read by
    // the tau kernel directly from the score row (one launch less)
    const int nch = full ? (c->max_pages_per_seq + 255) / 256 : 0;
    if (full && attn->transform == EKV_ENTMAX) {
        dim3 cg(nch, rows);
        k_candidates<<<cg, 256, 0, st>>>(scores, ntok, rowmax, pi, ns, stride, c->seq_lens, Hq, full, attn->alpha,
                                         attn->transform, nch, ccount, cs, cj);
        EKV_TRY(check_launch("k_candidates"));
    }
    TauArgs A;
    memset(&A, 0, sizeof(A));
    if (extra) A = *extra;
    A.scores = scores; A.ntok = ntok; A.rowmax = rowmax; A.ccount = ccount; A.cand_s = cs; A.cand_j = cj;
    A.nch = nch; A.page_idx = pi; A.n_sel = ns; A.sel_stride = stride; A.full = full;
    A.Hq = Hq; A.G = Hq / c->n_kv_heads; A.alpha = attn->alpha; A.transform = attn->transform;
    A.out = out; A.tau_out = tau; A.supp_out = supp;
    A.approx_h = attn->tau_halley > 0 ? attn->tau_halley : 0;
    if (attn->transform == EKV_SOFTMAX) {
        // a6: split dense-V softmax (flash-decoding chunks) + ordered combine
        const int nch = full ? (c->max_pages_per_seq + kSmxPages - 1) / kSmxPages : (stride + kSmxPages - 1) / kSmxPages;
        dim3 g(nch, rows);
        float *pacc = at<float>(ws, L.smx_acc);
        double *pl = at<double>(ws, L.smx_l);
        int32_t *pc = at<int32_t>(ws, L.smx_cnt);
        if (full) {
            if (c->dtype == EKV_BF16)
                EKV_TRY(launch_dense_group<__nv_bfloat16>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, nullptr, 0.f, st));
            else EKV_TRY(launch_dense_group<float>(v, scores, ntok, rowmax, Hq, nch, pacc, pl, pc, nullptr, 0.f, st));
        } else {
            if (c->dtype == EKV_BF16)
                k_softmax_partial<__nv_bfloat16><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, pi, ns, stride, full, Hq,
                                                                     Hq / c->n_kv_heads, nch, pacc, pl, pc, nullptr, 0.f);
            else
                k_softmax_partial<float><<<g, 256, 0, st>>>(v, scores, ntok, rowmax, pi, ns, stride, full, Hq,
                                                            Hq / c->n_kv_heads, nch, pacc, pl, pc, nullptr, 0.f);
            EKV_TRY(check_launch("k_softmax_partial"));
        }
        k_softmax_combine<<<rows, 128, 0, st>>>(pacc, pl, pc, rowmax, nch, out, tau, supp);
        return check_launch("k_softmax_combine");
    }
    const bool dense = full && (attn->flags & EKV_ATTN_DENSE_V) && !A.tok_list;
    if (dense) {
        // dense-V baseline: exact tau first (no PV), then every V row streamed with p_j
        A.no_pv = 1;
        if (!tau) A.tau_out = at<double>(ws, L.tau_int);
    }
    if (c->dtype == EKV_BF16) EKV_TRY(launch_tau_sparse<__nv_bfloat16>(v, A, rows, st));
    else EKV_TRY(launch_tau_sparse<float>(v, A, rows, st));
#ifdef EKV_STAMPS
    if (getenv("EKV_TAU_TWICE")) {                 // debug: warm instruction cache experiment
        if (c->dtype == EKV_BF16) EKV_TRY(launch_tau_sparse<__nv_bfloat16>(v, A, rows, st));
        else EKV_TRY(launch_tau_sparse<float>(v, A, rows, st));
    }
#endif
    if (!dense) return EKV_OK;
    const int dch = (c->max_pages_per_seq + kSmxPages - 1) / kSmxPages;
    dim3 g(dch, rows);
    float *pacc = at<float>(ws, L.smx_acc);
    double *pl = at<double>(ws, L.smx_l);
    int32_t *pc = at<int32_t>(ws, L.smx_cnt);
    (void)g;
    if (c->dtype == EKV_BF16)
        EKV_TRY(launch_dense_group<__nv_bfloat16>(v, scores, ntok, rowmax, Hq, dch, pacc, pl, pc, A.tau_out, attn->alpha, st));
    else EKV_TRY(launch_dense_group<float>(v, scores, ntok, rowmax, Hq, dch, pacc, pl, pc, A.tau_out, attn->alpha, st));
    k_softmax_combine<<<rows, 128, 0, st>>>(pacc, pl, pc, rowmax, dch, out, nullptr, nullptr);
    return check_launch("k_softmax_combine");
}


// ---------------------------------------------------------------- sequence sharding (P2)
struct ShardLayout {
    size_t pack_s, pack_g, recv_s, recv_g, zmax, cz, cj, cph, ncand, rowst, part, sums, tau, num, den, open, total;
    int kc;
};
ShardLayout shard_layout(const ekv_cache *c, int Hq, const ekv_select_params *sel, int world, size_t base) {
    ShardLayout S;
    const size_t rows = (size_t)c->batch * Hq;
    S.kc = sel_cap(c, sel);
    size_t o = base;
    auto take = [&](size_t bytes) { size_t r = o; o += align256(bytes); return r; };
    S.pack_s = take(rows * S.kc * 4);
    S.pack_g = take(rows * S.kc * 4);
    S.recv_s = take((size_t)world * rows * S.kc * 4);
    S.recv_g = take((size_t)world * rows * S.kc * 4);
    S.zmax = take(rows * 4);
    S.cz = take(rows * kShCap * 8);
    S.cj = take(rows * kShCap * 4);
    S.cph = take(rows * kShCap * 4);
    S.ncand = take(rows * 4);
    S.rowst = take(rows * sizeof(ShardRow));
    S.part = take(rows * kShP * 3 * 8);
    S.sums = take(rows * kShSums * 8);
    S.tau = take(rows * 8);
    S.num = take(rows * kD * 4);
    S.den = take(rows * 8);
    S.open = take(4);
    S.total = o;
    return S;
}

ekv_status comm_allreduce(const ekv_comm *cm, void *buf, size_t count, int dtype, int op, cudaStream_t st) {
    if (cm->world <= 1) return EKV_OK;
    if (cm->allreduce(buf, count, dtype, op, cm->user, st) != 0) return fail(EKV_ERR_COMM, "allreduce callback failed");
    return EKV_OK;
}
}  // namespace

// =============================================================================== C ABI
extern "C" {

const char *entmaxkv_last_error(void) { return g_err; }
const char *entmaxkv_version(void) { return "entmaxkv-b200 0.1 (sm_100a)"; }
int32_t entmaxkv_last_launch_count(void) { return g_launches; }

/* Debug (not in the public header): copy in-kernel phase stamps (ns) and the last top-k
 * candidate count; returns 0 when the library was built without -DEKV_STAMPS. */
int entmaxkv_debug_cta(unsigned long long *out /*[4*1024]*/) {
#ifdef EKV_STAMPS
    cudaMemcpyFromSymbol(out, ekv::ekv_cta, sizeof(unsigned long long) * 4 * 1024);
    return 1;
#else
    (void)out;
    return 0;
#endif
}
/* Debug: whole-kernel trace [16][2] (first CTA start, last CTA end; ns of %globaltimer);
 * reset != 0 re-arms it.  Returns 0 without -DEKV_STAMPS. */
int entmaxkv_debug_trace(unsigned long long *out, int reset) {
#ifdef EKV_STAMPS
    if (reset) {
        unsigned long long init[16][2];
        for (int i = 0; i < 16; ++i) { init[i][0] = ~0ull; init[i][1] = 0ull; }
        cudaMemcpyToSymbol(ekv::ekv_trace, init, sizeof(init));
    } else {
        cudaMemcpyFromSymbol(out, ekv::ekv_trace, sizeof(unsigned long long) * 32);
    }
    return 1;
#else
    (void)out; (void)reset;
    return 0;
#endif
}
/* Debug: per-CTA phase stamps [8][1024] ns and counters [2][1024]. */
int entmaxkv_debug_phases(unsigned long long *ph, long long *cnt) {
#ifdef EKV_STAMPS
    cudaMemcpyFromSymbol(ph, ekv::ekv_ph, sizeof(unsigned long long) * 8 * 1024);
    cudaMemcpyFromSymbol(cnt, ekv::ekv_phc, sizeof(long long) * 2 * 1024);
    return 1;
#else
    (void)ph; (void)cnt;
    return 0;
#endif
}
int entmaxkv_debug_stamps(unsigned long long *out /*[8*32]*/, int *nc) {
#ifdef EKV_STAMPS
    cudaMemcpyFromSymbol(out, ekv_stamps, sizeof(unsigned long long) * 8 * 32);
    *nc = 0;
    return 1;
#else
    (void)out; (void)nc;
    return 0;
#endif
}

size_t entmaxkv_workspace_size(const ekv_cache *cache, int32_t n_q_heads, const ekv_select_params *sel) {
    if (check_cache(cache, n_q_heads) != EKV_OK) return 0;
    return layout(cache, n_q_heads, sel).total;
}

int32_t entmaxkv_select_capacity(const ekv_cache *cache, const ekv_select_params *sel) {
    if (!cache) return 0;
    return sel_cap(cache, sel);
}

ekv_status entmaxkv_append_kv(const ekv_cache *cache, const void *k_new, const void *v_new, int32_t n_tokens,
                              void *stream) {
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, 0));
    if (!k_new || !v_new || n_tokens < 1) return fail(EKV_ERR_INVALID_ARG, "append: bad k/v or n_tokens");
    if (!cache->kmin || !cache->kmax || !cache->ksum || !cache->ksumsq || !cache->kavg || !cache->kvar)
        return fail(EKV_ERR_INVALID_ARG, "append: metadata buffers NULL");
    g_launches = 0;
    CacheView v = view(cache);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int nt = cache->n_kv_heads * kD;
    if (nt > 1024) nt = 1024;
    if (cache->dtype == EKV_BF16)
        launch_ex(k_append<__nv_bfloat16>, dim3(cache->batch), dim3(nt), 0, st, 0, v,
                  static_cast<const __nv_bfloat16 *>(k_new), static_cast<const __nv_bfloat16 *>(v_new), n_tokens);
    else
        launch_ex(k_append<float>, dim3(cache->batch), dim3(nt), 0, st, 0, v, static_cast<const float *>(k_new),
                  static_cast<const float *>(v_new), n_tokens);
    return check_launch("k_append");
}

ekv_status entmaxkv_rebuild_page_stats(const ekv_cache *cache, void *stream) {
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, 0));
    if (!cache->kmin || !cache->kmax || !cache->ksum || !cache->ksumsq || !cache->kavg || !cache->kvar)
        return fail(EKV_ERR_INVALID_ARG, "rebuild: metadata buffers NULL");
    g_launches = 0;
    CacheView v = view(cache);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t per_seq = (size_t)cache->max_pages_per_seq * cache->n_kv_heads * kD;
    dim3 grid((unsigned)((per_seq + 255) / 256), cache->batch);
    if (cache->dtype == EKV_BF16) k_rebuild<__nv_bfloat16><<<grid, 256, 0, st>>>(v);
    else k_rebuild<float><<<grid, 256, 0, st>>>(v);
    return check_launch("k_rebuild");
}

ekv_status entmaxkv_score_pages(const ekv_cache *cache, const void *q, int32_t n_q_heads, int32_t modes, float *box,
                                float *mu, float *sigma2, void *workspace, void *stream) {
    (void)workspace;
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_q(q));
    if (modes < 1 || modes > 3) return fail(EKV_ERR_INVALID_ARG, "modes must be 1..3");
    if ((modes & 1) && (!box || !cache->kmin || !cache->kmax)) return fail(EKV_ERR_INVALID_ARG, "box mode needs box/kmin/kmax");
    if ((modes & 2) && (!mu || !sigma2 || !cache->kavg || !cache->kvar))
        return fail(EKV_ERR_INVALID_ARG, "gauss mode needs mu/sigma2/kavg/kvar");
    g_launches = 0;
    CacheView v = view(cache);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cache->dtype == EKV_BF16) return launch_score<__nv_bfloat16>(v, q, n_q_heads, modes, box, mu, sigma2, nullptr, 0, st);
    return launch_score<float>(v, q, n_q_heads, modes, box, mu, sigma2, nullptr, 0, st);
}

ekv_status entmaxkv_select(const ekv_cache *cache, int32_t n_q_heads, const float *box, const float *mu,
                           const float *sigma2, const ekv_select_params *sel, float alpha, int32_t *page_idx,
                           int32_t *n_sel, int32_t sel_stride, double *tau_hat, void *workspace, void *stream) {
    (void)workspace;
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_sel(sel, alpha));
    if (!page_idx || !n_sel) return fail(EKV_ERR_INVALID_ARG, "page_idx/n_sel NULL");
    if (sel_stride < sel_cap(cache, sel)) return fail(EKV_ERR_CAPACITY, "sel_stride %d < capacity %d", sel_stride, sel_cap(cache, sel));
    g_launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int maxp = cache->max_pages_per_seq;
    if (sel->policy == EKV_TOPK) {
        if (!box) return fail(EKV_ERR_INVALID_ARG, "top-k needs box scores");
        return launch_topk(box, cache->batch, n_q_heads, maxp, cache->seq_lens, sel->k_pages, page_idx, n_sel, sel_stride,
                           n_q_heads / cache->n_kv_heads, UnionOut{nullptr, 0}, st);
    }
    if (sel->policy == EKV_ALL) {
        return launch_topk(box ? box : nullptr, cache->batch, n_q_heads, maxp, cache->seq_lens, maxp, page_idx, n_sel,
                           sel_stride, n_q_heads / cache->n_kv_heads, UnionOut{nullptr, 0}, st);
    }
    if (!mu || !sigma2) return fail(EKV_ERR_INVALID_ARG, "Gaussian selector needs mu/sigma2");
    return launch_gauss(cache, n_q_heads, mu, sigma2, alpha, sel, page_idx, n_sel, sel_stride, tau_hat, st);
}

ekv_status entmaxkv_sparse_attend(const ekv_cache *cache, const void *q, int32_t n_q_heads, const int32_t *page_idx,
                                  const int32_t *n_sel, int32_t sel_stride, const ekv_attn_params *attn, float *out,
                                  double *tau, int32_t *supp, void *workspace, void *stream) {
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    if (!q || !page_idx || !n_sel || !out || !workspace) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    if (sel_stride < 1) return fail(EKV_ERR_INVALID_ARG, "sel_stride < 1");
    g_launches = 0;
    Layout L = layout(cache, n_q_heads, nullptr);
    return attend_impl(cache, q, n_q_heads, page_idx, n_sel, sel_stride, 0, attn, out, tau, supp, workspace, L,
                       static_cast<cudaStream_t>(stream), nullptr);
}

ekv_status entmaxkv_full_attend(const ekv_cache *cache, const void *q, int32_t n_q_heads, const ekv_attn_params *attn,
                                float *out, double *tau, int32_t *supp, void *workspace, void *stream) {
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    if (!q || !out || !workspace) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    g_launches = 0;
    Layout L = layout(cache, n_q_heads, nullptr);
    return attend_impl(cache, q, n_q_heads, at<int32_t>(workspace, L.page_idx), at<int32_t>(workspace, L.n_sel),
                       c_max(cache), 1, attn, out, tau, supp, workspace, L, static_cast<cudaStream_t>(stream), nullptr);
}

ekv_status entmaxkv_decode(const ekv_cache *cache, const void *q, int32_t n_q_heads, const ekv_select_params *sel,
                           const ekv_attn_params *attn, float *out, ekv_decode_stats *stats, void *workspace,
                           void *stream) {
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    EKV_TRY(check_sel(sel, attn->alpha));
    if (!q || !out || !workspace) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    if (sel->policy == EKV_GAUSS && attn->transform != EKV_ENTMAX)
        return fail(EKV_ERR_INVALID_ARG, "Gaussian selector is entmax-specific");
    g_launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const CacheView v = view(cache);
    Layout L = layout(cache, n_q_heads, sel);
    float *box = at<float>(workspace, L.box);
    float *mu = at<float>(workspace, L.mu);
    float *s2 = at<float>(workspace, L.sigma2);
    int32_t *pi = at<int32_t>(workspace, L.page_idx);
    int32_t *ns = at<int32_t>(workspace, L.n_sel);
    double *th = at<double>(workspace, L.tau_hat);
    const bool want_db = stats && stats->delta_bar && attn->transform == EKV_ENTMAX;
    const int Gq = n_q_heads / cache->n_kv_heads;
    const UnionOut uo{at<uint32_t>(workspace, L.umask), L.W};
    // a1: page scores (box for top-k and for the certificate; mu/sigma2 for Gaussian); the
    // per-step counters / union mask are zeroed by the scoring kernel (or a k_zero launch
    // when nothing is scored) -- kernels only, so the PDL chain is unbroken
    int modes = 0;
    if (sel->policy == EKV_TOPK || want_db) modes |= EKV_SCORE_BOX;
    if (sel->policy == EKV_GAUSS) modes |= EKV_SCORE_GAUSS;
    uint4 *zp = at<uint4>(workspace, L.zero);
    const size_t zn16 = L.zero_bytes / 16;
    if (modes) {
        if (cache->dtype == EKV_BF16) EKV_TRY(launch_score<__nv_bfloat16>(v, q, n_q_heads, modes, box, mu, s2, zp, zn16, st));
        else EKV_TRY(launch_score<float>(v, q, n_q_heads, modes, box, mu, s2, zp, zn16, st));
    } else {
        launch_ex(k_zero, dim3((unsigned)std::min<size_t>(148, (zn16 + 255) / 256)), dim3(256), 0, st, 0, zp, zn16);
        EKV_TRY(check_launch("k_zero"));
    }
    // a2 / a2'
    const int maxp = cache->max_pages_per_seq;
    if (sel->policy == EKV_TOPK || sel->policy == EKV_ALL) {
        const int k = sel->policy == EKV_TOPK ? sel->k_pages : maxp;
        EKV_TRY(launch_topk(box, cache->batch, n_q_heads, maxp, cache->seq_lens, k, pi, ns, L.cap, Gq, uo, st));
    } else {
        EKV_TRY(launch_gauss(cache, n_q_heads, mu, s2, attn->alpha, sel, pi, ns, L.cap, th, st));
        EKV_TRY(launch_mark(cache, n_q_heads, pi, ns, L.cap, uo.umask, L.W, st));
    }
    // a3
    double *tau_p = (stats && stats->tau) ? stats->tau : at<double>(workspace, L.tau_int);
    TauArgs xa;
    memset(&xa, 0, sizeof(xa));
    xa.var = sel->policy == EKV_GAUSS;
    EKV_TRY(attend_impl(cache, q, n_q_heads, pi, ns, L.cap, 0, attn, out, tau_p,
                        stats ? stats->supp_count : nullptr, workspace, L, st, &xa, /*marked=*/true));
    const int rows = cache->batch * n_q_heads;
    // a4: certified dropped-mass bound (wide kernel; deterministic ticketed final sum)
    if (want_db) {
        const int nch = (maxp + kDbChunk - 1) / kDbChunk;   // <= 8 (max_pages <= 65536)
        DbConst kc;
        kc.a = (double)attn->alpha - 1.0;
        kc.beta = 1.0 / kc.a;
        kc.inv_a = kc.beta;
        kc.ib = (std::fabs(kc.beta - std::rint(kc.beta)) < 1e-12 && kc.beta <= 4.5) ? (int)std::rint(kc.beta) : 0;
        const dim3 dg((unsigned)nch, (unsigned)rows), db(256);
        cudaError_t ce;
        switch (kc.ib) {
        case 1: ce = launch_ex(k_delta_bar<1>, dg, db, 0, st, (unsigned)nch, (const float *)box, maxp, (const int32_t *)cache->seq_lens, n_q_heads, Gq, (const uint32_t *)uo.umask, L.W, (const double *)tau_p, kc, stats->delta_bar); break;
        case 2: ce = launch_ex(k_delta_bar<2>, dg, db, 0, st, (unsigned)nch, (const float *)box, maxp, (const int32_t *)cache->seq_lens, n_q_heads, Gq, (const uint32_t *)uo.umask, L.W, (const double *)tau_p, kc, stats->delta_bar); break;
        case 3: ce = launch_ex(k_delta_bar<3>, dg, db, 0, st, (unsigned)nch, (const float *)box, maxp, (const int32_t *)cache->seq_lens, n_q_heads, Gq, (const uint32_t *)uo.umask, L.W, (const double *)tau_p, kc, stats->delta_bar); break;
        case 4: ce = launch_ex(k_delta_bar<4>, dg, db, 0, st, (unsigned)nch, (const float *)box, maxp, (const int32_t *)cache->seq_lens, n_q_heads, Gq, (const uint32_t *)uo.umask, L.W, (const double *)tau_p, kc, stats->delta_bar); break;
        default: ce = launch_ex(k_delta_bar<0>, dg, db, 0, st, (unsigned)nch, (const float *)box, maxp, (const int32_t *)cache->seq_lens, n_q_heads, Gq, (const uint32_t *)uo.umask, L.W, (const double *)tau_p, kc, stats->delta_bar); break;
        }
        if (ce != cudaSuccess) return fail(EKV_ERR_CUDA, "k_delta_bar: %s", cudaGetErrorString(ce));
        EKV_TRY(check_launch("k_delta_bar"));
    }

    if (stats) {
        if (stats->n_sel) {
            if (cudaMemcpyAsync(stats->n_sel, ns, rows * sizeof(int32_t), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return fail(EKV_ERR_CUDA, "n_sel copy");
        }
        if (stats->tau_hat && sel->policy == EKV_GAUSS) {
            if (cudaMemcpyAsync(stats->tau_hat, th, rows * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return fail(EKV_ERR_CUDA, "tau_hat copy");
        }
        if (stats->eval_exact && attn->transform == EKV_ENTMAX) {
            // a4 eval: full-cache pass keeping the support list, then delta / rho counts (R16);
            // the sparse page lists (pi, ns) stay untouched by the full pass.
            TauArgs ex;
            memset(&ex, 0, sizeof(ex));
            ex.tok_list = at<int32_t>(workspace, L.tok_list);
            ex.p_list = at<double>(workspace, L.p_list);
            ex.n_list = at<int32_t>(workspace, L.n_list);
            ex.list_cap = L.list_cap;
            EKV_TRY(attend_impl(cache, q, n_q_heads, pi, ns, L.cap, 1, attn, at<float>(workspace, L.full_out),
                                stats->tau_full, nullptr, workspace, L, st, &ex));
            k_eval_metrics<<<rows, 256, 0, st>>>(ex.tok_list, ex.p_list, ex.n_list, ex.list_cap, pi, ns, L.cap,
                                                 stats->delta, stats->recovered, stats->full_supp);
            EKV_TRY(check_launch("k_eval_metrics"));
        }
    }
    return EKV_OK;
}


size_t entmaxkv_shard_workspace_size(const ekv_cache *local, int32_t n_q_heads, const ekv_select_params *sel,
                                     int32_t world) {
    if (check_cache(local, n_q_heads) != EKV_OK || world < 1) return 0;
    const size_t base = layout(local, n_q_heads, sel).total;
    return shard_layout(local, n_q_heads, sel, world, base).total;
}

ekv_status entmaxkv_decode_sharded(const ekv_cache *cache, const int32_t *global_seq_lens, const void *q,
                                   int32_t n_q_heads, const ekv_select_params *sel, const ekv_attn_params *attn,
                                   const ekv_comm *comm, float *out, ekv_decode_stats *stats, void *workspace,
                                   void *stream) {
    g_err[0] = 0;
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    EKV_TRY(check_sel(sel, attn->alpha));
    if (!q || !out || !workspace || !comm || !global_seq_lens) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world || (comm->world > 1 && (!comm->allreduce || !comm->allgather)))
        return fail(EKV_ERR_INVALID_ARG, "bad communicator (rank %d, world %d)", comm->rank, comm->world);
    if (sel->policy != EKV_TOPK || attn->transform != EKV_ENTMAX)
        return fail(EKV_ERR_UNSUPPORTED, "sharded decode supports top-k selection with entmax");
    const double beta = 1.0 / ((double)attn->alpha - 1.0);
    const int ib = (std::fabs(beta - std::rint(beta)) < 1e-9 && beta <= 4.5 && beta >= 0.5) ? (int)std::rint(beta) : 0;
    if (ib < 1 || ib > 4)
        return fail(EKV_ERR_UNSUPPORTED, "sharded decode needs integer beta = 1/(alpha-1) in {1,2,3,4} (alpha=%g)",
                    (double)attn->alpha);
    const int W = comm->world, rk = comm->rank;
    g_launches = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const CacheView v = view(cache);
    Layout L = layout(cache, n_q_heads, sel);
    ShardLayout S = shard_layout(cache, n_q_heads, sel, W, L.total);
    if ((long long)W * S.kc > (long long)kShMergeNT * kShMergeKPT)
        return fail(EKV_ERR_UNSUPPORTED, "world * k = %lld exceeds %d", (long long)W * S.kc, kShMergeNT * kShMergeKPT);
    const int rows = cache->batch * n_q_heads, Gq = n_q_heads / cache->n_kv_heads;
    const int maxp = cache->max_pages_per_seq;
    float *box = at<float>(workspace, L.box);
    int32_t *pi = at<int32_t>(workspace, L.page_idx);
    int32_t *ns = at<int32_t>(workspace, L.n_sel);
    uint32_t *um = at<uint32_t>(workspace, L.umask);
    if (cudaMemsetAsync(at<char>(workspace, L.zero), 0, L.zero_bytes, st) != cudaSuccess)
        return fail(EKV_ERR_CUDA, "memset: %s", cudaGetErrorString(cudaGetLastError()));
    // 1. local scores + local top-k, then the global merge
    if (cache->dtype == EKV_BF16) EKV_TRY(launch_score<__nv_bfloat16>(v, q, n_q_heads, EKV_SCORE_BOX, box, nullptr, nullptr, nullptr, 0, st));
    else EKV_TRY(launch_score<float>(v, q, n_q_heads, EKV_SCORE_BOX, box, nullptr, nullptr, nullptr, 0, st));
    EKV_TRY(launch_topk(box, cache->batch, n_q_heads, maxp, cache->seq_lens, sel->k_pages, pi, ns, L.cap, Gq,
                        UnionOut{nullptr, 0}, st));
    float *ps = at<float>(workspace, S.pack_s), *rs = at<float>(workspace, S.recv_s);
    int32_t *pg = at<int32_t>(workspace, S.pack_g), *rg = at<int32_t>(workspace, S.recv_g);
    k_shard_pack<<<rows, 256, 0, st>>>(box, maxp, pi, ns, L.cap, S.kc, rk, W, ps, pg);
    EKV_TRY(check_launch("k_shard_pack"));
    const size_t pbytes = (size_t)rows * S.kc * 4;
    if (W > 1) {
        if (comm->allgather(ps, rs, pbytes, comm->user, st) != 0 || comm->allgather(pg, rg, pbytes, comm->user, st) != 0)
            return fail(EKV_ERR_COMM, "allgather callback failed");
    } else {
        cudaMemcpyAsync(rs, ps, pbytes, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(rg, pg, pbytes, cudaMemcpyDeviceToDevice, st);
    }
    k_shard_merge<<<rows, kShMergeNT, 0, st>>>(rs, rg, rows, S.kc, sel->k_pages, rk, W, global_seq_lens, pi, ns, L.cap,
                                               n_q_heads, Gq, um, L.W);
    EKV_TRY(check_launch("k_shard_merge"));
    // 2. K scores of the local share, global z_max
    float *scores = at<float>(workspace, L.scores);
    uint32_t *rowmax = at<uint32_t>(workspace, L.rowmax);
    if (cache->dtype == EKV_BF16)
        EKV_TRY(launch_scores<__nv_bfloat16>(v, q, n_q_heads, um, L.W, pi, ns, L.cap, scores, rowmax, 0, st));
    else EKV_TRY(launch_scores<float>(v, q, n_q_heads, um, L.W, pi, ns, L.cap, scores, rowmax, 0, st));
    float *zmax = at<float>(workspace, S.zmax);
    k_shard_zmax<<<(rows + 255) / 256, 256, 0, st>>>(rowmax, rows, zmax);
    EKV_TRY(check_launch("k_shard_zmax"));
    EKV_TRY(comm_allreduce(comm, zmax, rows, 0, 1, st));
    // 3. local candidates
    double *cz = at<double>(workspace, S.cz);
    int32_t *cj = at<int32_t>(workspace, S.cj), *cph = at<int32_t>(workspace, S.cph), *nc = at<int32_t>(workspace, S.ncand);
    ShardRow *rst = at<ShardRow>(workspace, S.rowst);
    k_shard_cand<<<rows, 256, 0, st>>>(scores, (size_t)maxp * kP, pi, ns, L.cap, cache->seq_lens, cache->page_table, maxp,
                                       n_q_heads, zmax, attn->alpha, cz, cj, cph, nc, rst);
    EKV_TRY(check_launch("k_shard_cand"));
    // 4. multisection rounds (host loop; one small device->host read per round)
    double *part = at<double>(workspace, S.part);
    int *openp = at<int>(workspace, S.open);
    auto probe = [&](const double *red) -> ekv_status {
        switch (ib) {
        case 1: k_shard_probe<1><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part); break;
        case 2: k_shard_probe<2><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part); break;
        case 3: k_shard_probe<3><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part); break;
        default: k_shard_probe<4><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part); break;
        }
        return check_launch("k_shard_probe");
    };
    EKV_TRY(probe(nullptr));
    for (int round = 0; round < 13; ++round) {
        EKV_TRY(comm_allreduce(comm, part, (size_t)rows * kShP * 3, 1, 0, st));
        EKV_TRY(probe(part));
        if (round < 1) continue;              // two rounds (12 bits) before the first check
        k_shard_open<<<1, 256, 0, st>>>(rst, rows, openp);
        EKV_TRY(check_launch("k_shard_open"));
        int open = 0;
        if (cudaMemcpyAsync(&open, openp, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(EKV_ERR_CUDA, "round sync: %s", cudaGetErrorString(cudaGetLastError()));
        if (open == 0) break;
    }
    // 5. power sums -> tau
    double *sums = at<double>(workspace, S.sums);
    k_shard_sums<<<rows, 256, 0, st>>>(cz, nc, rst, sums);
    EKV_TRY(check_launch("k_shard_sums"));
    EKV_TRY(comm_allreduce(comm, sums, (size_t)rows * kShSums, 1, 0, st));
    double *tau = (stats && stats->tau) ? stats->tau : at<double>(workspace, S.tau);
    k_shard_tau<<<(rows + 127) / 128, 128, 0, st>>>(sums, ib, rst, rows, tau, stats ? stats->supp_count : nullptr);
    EKV_TRY(check_launch("k_shard_tau"));
    // 6. numerator / denominator
    float *num = at<float>(workspace, S.num);
    double *den = at<double>(workspace, S.den);
    auto pv = [&](auto tag) -> ekv_status {
        using T = decltype(tag);
        switch (ib) {
        case 1: k_shard_pv<T, 1><<<rows, 256, 0, st>>>(v, cz, cj, cph, nc, rst, tau, beta, n_q_heads, Gq, num, den); break;
        case 2: k_shard_pv<T, 2><<<rows, 256, 0, st>>>(v, cz, cj, cph, nc, rst, tau, beta, n_q_heads, Gq, num, den); break;
        case 3: k_shard_pv<T, 3><<<rows, 256, 0, st>>>(v, cz, cj, cph, nc, rst, tau, beta, n_q_heads, Gq, num, den); break;
        default: k_shard_pv<T, 4><<<rows, 256, 0, st>>>(v, cz, cj, cph, nc, rst, tau, beta, n_q_heads, Gq, num, den); break;
        }
        return check_launch("k_shard_pv");
    };
    if (cache->dtype == EKV_BF16) EKV_TRY(pv(__nv_bfloat16()));
    else EKV_TRY(pv(0.0f));
    EKV_TRY(comm_allreduce(comm, num, (size_t)rows * kD, 0, 0, st));
    EKV_TRY(comm_allreduce(comm, den, (size_t)rows, 1, 0, st));
    k_shard_out<<<(rows * kD + 255) / 256, 256, 0, st>>>(num, den, tau, rows, out);
    EKV_TRY(check_launch("k_shard_out"));
    if (stats && stats->n_sel) {
        // global selection size: min(k, global pages) per row
        k_shard_nsel<<<(rows + 127) / 128, 128, 0, st>>>(global_seq_lens, n_q_heads, rows, sel->k_pages, stats->n_sel);
        EKV_TRY(check_launch("k_shard_nsel"));
    }
    return EKV_OK;
}

}  // extern "C"
