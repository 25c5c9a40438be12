// entmaxkv.cu -- the C ABI of libentmaxkv.so (include/entmaxkv.h): argument validation,
// workspace carve-out and the orchestration of the kernel launches (launch_*.cu) on the
// caller's stream; no allocation, no synchronisation.
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
#include <cmath>
#include <mutex>
#include <map>
#include <vector>
#include <utility>
#include <algorithm>

#include "host.h"

using namespace ekv;

namespace ekvh {

namespace {
thread_local char g_err[512] = "";
thread_local int g_launches = 0;
}  // namespace

NvtxRange::NvtxRange(const char *name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

void begin_call() {
    g_err[0] = 0;
    g_launches = 0;
}

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

ekv_status check_err(cudaError_t e, const char *what) {
    if (e != cudaSuccess) return fail(EKV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return EKV_OK;
}

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("EKV_NO_PDL"); v = (e && e[0] == '1') ? 0 : 1; }
    return v == 1;
}

// ---------------------------------------------------------------- per-device caches
namespace {
std::mutex g_mu;
std::map<int, int> g_sms;                                          // device -> SM count
std::map<std::pair<const void *, int>, int> g_smem;                // (kernel, device) -> smem set
std::map<std::pair<std::pair<const void *, int>, std::pair<int, int>>, int> g_occ;   // ((k, dev), (thr, smem))
int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
}  // namespace

int num_sms() {
    const int d = cur_dev();
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_sms.find(d);
    if (it != g_sms.end()) return it->second;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n <= 0) n = 148;
    g_sms[d] = n;
    return n;
}

void set_smem_raw(const void *kernel, int bytes, bool nonportable_cluster) {
    const int d = cur_dev();
    std::lock_guard<std::mutex> lk(g_mu);
    int &have = g_smem[{kernel, d}];
    if (have >= bytes && have > 0) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (nonportable_cluster) cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    have = bytes > 0 ? bytes : 1;
}

int resident_per_sm_raw(const void *kernel, int threads, int smem) {
    const int d = cur_dev();
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(std::make_pair(kernel, d), std::make_pair(threads, smem));
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess || n < 1) n = 1;
    g_occ[key] = n;
    return n;
}

int int_beta(float alpha) {
    const double beta = 1.0 / ((double)alpha - 1.0);
    return (std::fabs(beta - std::rint(beta)) < 1e-12 && beta <= 4.5 && beta >= 0.5) ? (int)std::rint(beta) : 0;
}

// ---------------------------------------------------------------- validation
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
    if (c->bound_dtype != EKV_BOUND_KV && c->bound_dtype != EKV_BOUND_E4M3)
        return fail(EKV_ERR_INVALID_ARG, "bad bound_dtype %d", c->bound_dtype);
    if (c->stat_dtype != EKV_STAT_F32 && c->stat_dtype != EKV_STAT_BF16)
        return fail(EKV_ERR_INVALID_ARG, "bad stat_dtype %d", c->stat_dtype);
    if (((uintptr_t)c->k_pages | (uintptr_t)c->v_pages) & 15)
        return fail(EKV_ERR_INVALID_ARG, "k_pages/v_pages must be 16-byte aligned");
    return EKV_OK;
}

ekv_status check_q(const void *q) {
    if (!q) return fail(EKV_ERR_INVALID_ARG, "q is NULL");
    if ((uintptr_t)q & 15) return fail(EKV_ERR_INVALID_ARG, "q must be 16-byte aligned");
    return EKV_OK;
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
        // integer beta in 1..4: App. D's closed forms; any other beta <= 32: the numerical
        // expectation (N4)
        const double beta = 1.0 / ((double)alpha - 1.0);
        if (!(alpha > 1.0f) || !(beta <= 32.0))
            return fail(EKV_ERR_UNSUPPORTED, "Gaussian selector needs alpha > 1 + 1/32 (alpha=%g)", (double)alpha);
    } else if (s->policy == EKV_CERTIFIED) {
        if (s->k_pages < 1) return fail(EKV_ERR_INVALID_ARG, "k_pages (first pass) must be >= 1");
    } else if (s->policy != EKV_ALL) {
        return fail(EKV_ERR_INVALID_ARG, "bad policy %d", s->policy);
    }
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
    v.bound = c->bound_dtype; v.stat = c->stat_dtype;
    return v;
}

int sel_cap(const ekv_cache *c, const ekv_select_params *s) {
    if (!s || s->policy != EKV_TOPK) return c->max_pages_per_seq;
    return s->k_pages < c->max_pages_per_seq ? s->k_pages : c->max_pages_per_seq;
}

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
    L.gtab = take(64 * 48 * 8);           // non-integer-beta moment table (N4)
    L.zero = o;
    L.status = take(16);
    L.retry = take(B * Hq * 4);
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
    L.sink = take(16);
    L.smx_nch = (int)((maxp + kSmxPages - 1) / kSmxPages);
    L.smx_acc = take(B * Hq * (size_t)L.smx_nch * kD * 4);
    L.smx_l = take(B * Hq * (size_t)L.smx_nch * 8);
    L.smx_cnt = take(B * Hq * (size_t)L.smx_nch * 4);
    L.total = o;
    return L;
}

const char *last_error() { return g_err; }
int last_launches() { return g_launches; }

std::vector<DebugReader> &debug_readers() {
    static std::vector<DebugReader> r;
    return r;
}

}  // namespace ekvh

void ekv::debug_register(DebugReader r) { ekvh::debug_readers().push_back(r); }

using namespace ekvh;

namespace {

// attention of every (b, q-head) over its page list (full: every page):
// zero(rowmax, ccount, umask) -> [mark] -> K scores -> candidates -> tau/PV
ekv_status attend_impl(const ekv_cache *c, const void *q, int Hq, const int32_t *pi, const int32_t *ns, int stride,
                       int full, const ekv_attn_params *attn, float *out, double *tau, int32_t *supp, void *ws,
                       const Layout &L, cudaStream_t st, const TauArgs *extra, bool marked = false) {
    const CacheView v = view(c);
    uint32_t *rowmax = at<uint32_t>(ws, L.rowmax);
    int *ccount = at<int>(ws, L.ccount);
    uint32_t *um = at<uint32_t>(ws, L.umask);
    float *scores = at<float>(ws, L.scores);
    if (!marked) {   // (the eval pass keeps the sparse pass's status word)
        const size_t z0 = (extra && extra->tok_list) ? L.rowmax : L.zero;
        EKV_TRY(launch_zero(at<uint4>(ws, z0), (L.zero_bytes - (z0 - L.zero)) / 16, st));
    }
    if (!full && !marked) EKV_TRY(launch_mark(c->batch, Hq, Hq / c->n_kv_heads, pi, ns, stride, um, L.W, st));
    // full rows (a5/a6 baseline) of a bf16 cache: the score pass is a dense contraction, run on
    // tensor cores (R26); the eval pass and EKV_ATTN_CANONICAL keep the canonical order (R1)
    const int G = Hq / c->n_kv_heads;
    const bool tc = full && c->dtype == EKV_BF16 && !(extra && extra->tok_list) &&
                    !(attn->flags & EKV_ATTN_CANONICAL) && (G == 1 || G == 2 || G == 4 || G == 8);
    if (tc) EKV_TRY(launch_full_scores_mma(v, q, Hq, scores, rowmax, st));
    else EKV_TRY(launch_scores(v, q, Hq, um, L.W, pi, ns, stride, scores, rowmax, full, st));
    const int rows = c->batch * Hq;
    const size_t ntok = (size_t)c->max_pages_per_seq * kP;
    float *cs = at<float>(ws, L.cand_s);
    int32_t *cj = at<int32_t>(ws, L.cand_j);
    // full rows are long: candidates extracted by a wide kernel; sparse rows are read by
    // the tau kernel directly from the score row (one launch less)
    const int nch = full ? (c->max_pages_per_seq + 255) / 256 : 0;
    if (full && attn->transform == EKV_ENTMAX)
        EKV_TRY(launch_candidates(scores, ntok, rowmax, c->seq_lens, Hq, attn->alpha, nch, rows, ccount, cs, cj, st));
    TauArgs A;
    memset(&A, 0, sizeof(A));
    if (extra) A = *extra;
    A.scores = scores; A.ntok = ntok; A.rowmax = rowmax; A.ccount = ccount; A.cand_s = cs; A.cand_j = cj;
    A.nch = nch; A.page_idx = pi; A.n_sel = ns; A.sel_stride = stride; A.full = full;
    A.Hq = Hq; A.G = Hq / c->n_kv_heads; A.alpha = attn->alpha; A.transform = attn->transform;
    A.out = out; A.tau_out = tau; A.supp_out = supp;
    A.approx_h = attn->tau_halley > 0 ? attn->tau_halley : 0;
    A.status = at<uint32_t>(ws, L.status);
    A.retry = at<int32_t>(ws, L.retry);
    float *pacc = at<float>(ws, L.smx_acc);
    double *pl = at<double>(ws, L.smx_l);
    int32_t *pc = at<int32_t>(ws, L.smx_cnt);
    if (attn->transform == EKV_SOFTMAX) {
        // a6: split dense-V softmax (flash-decoding chunks) + ordered combine
        const int snch = full ? (c->max_pages_per_seq + kSmxPages - 1) / kSmxPages : (stride + kSmxPages - 1) / kSmxPages;
        if (full) EKV_TRY(launch_dense_group(v, scores, ntok, rowmax, Hq, snch, pacc, pl, pc, nullptr, 0.f, st));
        else EKV_TRY(launch_softmax_partial(v, scores, ntok, rowmax, pi, ns, stride, full, Hq, snch, rows, pacc, pl, pc, st));
        return launch_softmax_combine(rows, pacc, pl, pc, rowmax, snch, out, tau, supp, st);
    }
    const bool dense = full && (attn->flags & EKV_ATTN_DENSE_V) && !A.tok_list;
    // exact tau, support and PV over the support
    EKV_TRY(launch_tau(v, A, rows, st));
    if (!dense) return EKV_OK;
    // dense-V baseline (R22): every V row streamed once as well (p_j = 0 off the support, so the
    // output is the PV above; the stream is the paper's reference's V traffic)
    return launch_vstream(v, at<uint32_t>(ws, L.sink), st);
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

const char *entmaxkv_last_error(void) { return last_error(); }
const char *entmaxkv_version(void) { return "entmaxkv-b200 0.2 (sm_100a)"; }
int32_t entmaxkv_last_launch_count(void) { return last_launches(); }

/* Debug (not in the public header): in-kernel phase stamps, merged over the library's
 * translation units; each returns 0 when the library was built without -DEKV_STAMPS. */
int entmaxkv_debug_cta(unsigned long long *out /*[4*1024]*/) {
#ifdef EKV_STAMPS
    std::vector<unsigned long long> buf(4 * 1024);
    memset(out, 0, sizeof(unsigned long long) * 4 * 1024);
    for (auto r : debug_readers()) {
        r(1, buf.data(), 0);
        for (int i = 0; i < 4 * 1024; ++i) out[i] = std::max(out[i], buf[i]);
    }
    return 1;
#else
    (void)out;
    return 0;
#endif
}
/* Debug: whole-kernel trace [16][2] (first CTA start, last CTA end; ns of %globaltimer);
 * reset != 0 re-arms it. */
int entmaxkv_debug_trace(unsigned long long *out, int reset) {
#ifdef EKV_STAMPS
    if (reset) {
        for (auto r : debug_readers()) r(0, nullptr, 1);
        return 1;
    }
    unsigned long long buf[32];
    for (int i = 0; i < 16; ++i) { out[2 * i] = ~0ull; out[2 * i + 1] = 0ull; }
    for (auto r : debug_readers()) {
        r(0, buf, 0);
        for (int i = 0; i < 16; ++i) {
            out[2 * i] = std::min(out[2 * i], buf[2 * i]);
            out[2 * i + 1] = std::max(out[2 * i + 1], buf[2 * i + 1]);
        }
    }
    return 1;
#else
    (void)out; (void)reset;
    return 0;
#endif
}
/* Debug: per-CTA phase stamps [8][1024] ns and counters [8][1024]. */
int entmaxkv_debug_phases(unsigned long long *ph, long long *cnt) {
#ifdef EKV_STAMPS
    std::vector<unsigned long long> b1(8 * 1024);
    std::vector<long long> b2(8 * 1024);
    memset(ph, 0, sizeof(unsigned long long) * 8 * 1024);
    memset(cnt, 0, sizeof(long long) * 8 * 1024);
    for (auto r : debug_readers()) {
        r(2, b1.data(), 0);
        r(3, b2.data(), 0);
        for (int i = 0; i < 8 * 1024; ++i) ph[i] = std::max(ph[i], b1[i]);
        for (int i = 0; i < 8 * 1024; ++i) cnt[i] = std::max(cnt[i], b2[i]);
    }
    return 1;
#else
    (void)ph; (void)cnt;
    return 0;
#endif
}
int entmaxkv_debug_stamps(unsigned long long *out /*[8*32]*/, int *nc) {
#ifdef EKV_STAMPS
    unsigned long long buf[8 * 32];
    memset(out, 0, sizeof(buf));
    for (auto r : debug_readers()) {
        r(4, buf, 0);
        for (int i = 0; i < 8 * 32; ++i) out[i] = std::max(out[i], buf[i]);
    }
    *nc = 0;
    return 1;
#else
    (void)out; (void)nc;
    return 0;
#endif
}

ekv_status entmaxkv_workspace_status(const ekv_cache *cache, int32_t n_q_heads, const ekv_select_params *sel,
                                     const void *workspace, int32_t *flags, void *stream) {
    EKV_CALL("entmaxkv_workspace_status");
    EKV_TRY(check_cache(cache, n_q_heads));
    if (!workspace || !flags) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    const Layout L = layout(cache, n_q_heads, sel);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t f = 0u;
    EKV_TRY(check_err(cudaMemcpyAsync(&f, static_cast<const char *>(workspace) + L.status, sizeof(f),
                                      cudaMemcpyDeviceToHost, st), "status read"));
    EKV_TRY(check_err(cudaStreamSynchronize(st), "status sync"));
    *flags = (int32_t)f;
    if (f & kStatusTimeout)
        return fail(EKV_ERR_COMM, "in-kernel collectives: a peer's exchange did not arrive (rows NaN; re-zero the exchange buffers)");
    if (f & kStatusCapacity)
        return fail(EKV_ERR_CAPACITY, "a row's candidate set exceeded the kernel capacity (its out/tau are NaN, supp -1)");
    return EKV_OK;
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
    EKV_CALL("entmaxkv_append_kv");
    EKV_TRY(check_cache(cache, 0));
    if (!k_new || !v_new || n_tokens < 1) return fail(EKV_ERR_INVALID_ARG, "append: bad k/v or n_tokens");
    if (!cache->kmin || !cache->kmax || !cache->ksum || !cache->ksumsq || !cache->kavg || !cache->kvar)
        return fail(EKV_ERR_INVALID_ARG, "append: metadata buffers NULL");
    return launch_append(view(cache), k_new, v_new, n_tokens, static_cast<cudaStream_t>(stream));
}

ekv_status entmaxkv_rebuild_page_stats(const ekv_cache *cache, void *stream) {
    EKV_CALL("entmaxkv_rebuild_page_stats");
    EKV_TRY(check_cache(cache, 0));
    if (!cache->kmin || !cache->kmax || !cache->ksum || !cache->ksumsq || !cache->kavg || !cache->kvar)
        return fail(EKV_ERR_INVALID_ARG, "rebuild: metadata buffers NULL");
    return launch_rebuild(view(cache), static_cast<cudaStream_t>(stream));
}

ekv_status entmaxkv_score_pages(const ekv_cache *cache, const void *q, int32_t n_q_heads, int32_t modes, float *box,
                                float *mu, float *sigma2, void *workspace, void *stream) {
    (void)workspace;
    EKV_CALL("entmaxkv_score_pages");
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_q(q));
    if (modes < 1 || modes > 3) return fail(EKV_ERR_INVALID_ARG, "modes must be 1..3");
    if ((modes & 1) && (!box || !cache->kmin || !cache->kmax)) return fail(EKV_ERR_INVALID_ARG, "box mode needs box/kmin/kmax");
    if ((modes & 2) && (!mu || !sigma2 || !cache->kavg || !cache->kvar))
        return fail(EKV_ERR_INVALID_ARG, "gauss mode needs mu/sigma2/kavg/kvar");
    return launch_score(view(cache), q, n_q_heads, modes, box, mu, sigma2, nullptr, 0, static_cast<cudaStream_t>(stream));
}

ekv_status entmaxkv_select(const ekv_cache *cache, int32_t n_q_heads, const float *box, const float *mu,
                           const float *sigma2, const ekv_select_params *sel, float alpha, int32_t *page_idx,
                           int32_t *n_sel, int32_t sel_stride, double *tau_hat, void *workspace, void *stream) {
    (void)workspace;
    EKV_CALL("entmaxkv_select");
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_sel(sel, alpha));
    if (!page_idx || !n_sel) return fail(EKV_ERR_INVALID_ARG, "page_idx/n_sel NULL");
    if (sel_stride < sel_cap(cache, sel)) return fail(EKV_ERR_CAPACITY, "sel_stride %d < capacity %d", sel_stride, sel_cap(cache, sel));
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
    double *gtab = workspace ? at<double>(workspace, layout(cache, n_q_heads, sel).gtab) : nullptr;
    return launch_gauss(cache, n_q_heads, mu, sigma2, alpha, sel, page_idx, n_sel, sel_stride, tau_hat, gtab, st);
}

ekv_status entmaxkv_sparse_attend(const ekv_cache *cache, const void *q, int32_t n_q_heads, const int32_t *page_idx,
                                  const int32_t *n_sel, int32_t sel_stride, const double *tau_init,
                                  const ekv_attn_params *attn, float *out, double *tau, int32_t *supp, void *workspace,
                                  void *stream) {
    EKV_CALL("entmaxkv_sparse_attend");
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    if (!q || !page_idx || !n_sel || !out || !workspace) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    if (sel_stride < 1) return fail(EKV_ERR_INVALID_ARG, "sel_stride < 1");
    Layout L = layout(cache, n_q_heads, nullptr);
    TauArgs xa;
    memset(&xa, 0, sizeof(xa));
    xa.tau_init = tau_init;
    return attend_impl(cache, q, n_q_heads, page_idx, n_sel, sel_stride, 0, attn, out, tau, supp, workspace, L,
                       static_cast<cudaStream_t>(stream), &xa);
}

ekv_status entmaxkv_full_attend(const ekv_cache *cache, const void *q, int32_t n_q_heads, const ekv_attn_params *attn,
                                float *out, double *tau, int32_t *supp, void *workspace, void *stream) {
    EKV_CALL("entmaxkv_full_attend");
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    if (!q || !out || !workspace) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    Layout L = layout(cache, n_q_heads, nullptr);
    return attend_impl(cache, q, n_q_heads, at<int32_t>(workspace, L.page_idx), at<int32_t>(workspace, L.n_sel),
                       cache->max_pages_per_seq, 1, attn, out, tau, supp, workspace, L,
                       static_cast<cudaStream_t>(stream), nullptr);
}

ekv_status entmaxkv_decode(const ekv_cache *cache, const void *q, int32_t n_q_heads, const ekv_select_params *sel,
                           const ekv_attn_params *attn, float *out, ekv_decode_stats *stats, void *workspace,
                           void *stream) {
    EKV_CALL("entmaxkv_decode");
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    EKV_TRY(check_sel(sel, attn->alpha));
    if (!q || !out || !workspace) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    if ((sel->policy == EKV_GAUSS || sel->policy == EKV_CERTIFIED) && attn->transform != EKV_ENTMAX)
        return fail(EKV_ERR_INVALID_ARG, "Gaussian / certified selection is entmax-specific");
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
    const bool cert = sel->policy == EKV_CERTIFIED;
    if (sel->policy == EKV_TOPK || cert || want_db) modes |= EKV_SCORE_BOX;
    if (sel->policy == EKV_GAUSS) modes |= EKV_SCORE_GAUSS;
    uint4 *zp = at<uint4>(workspace, L.zero);
    const size_t zn16 = L.zero_bytes / 16;
    if (modes) EKV_TRY(launch_score(v, q, n_q_heads, modes, box, mu, s2, zp, zn16, st));
    else EKV_TRY(launch_zero(zp, zn16, st));
    // a2 / a2'
    const int maxp = cache->max_pages_per_seq;
    if (sel->policy == EKV_TOPK || sel->policy == EKV_ALL || cert) {
        const int k = sel->policy == EKV_ALL ? maxp : sel->k_pages;
        EKV_TRY(launch_topk(box, cache->batch, n_q_heads, maxp, cache->seq_lens, k, pi, ns, L.cap, Gq, uo, st));
    } else {
        EKV_TRY(launch_gauss(cache, n_q_heads, mu, s2, attn->alpha, sel, pi, ns, L.cap, th, at<double>(workspace, L.gtab), st));
        EKV_TRY(launch_mark(cache->batch, n_q_heads, Gq, pi, ns, L.cap, uo.umask, L.W, st));
    }
    // a3
    double *tau_p = (stats && stats->tau) ? stats->tau : at<double>(workspace, L.tau_int);
    TauArgs xa;
    memset(&xa, 0, sizeof(xa));
    xa.var = sel->policy == EKV_GAUSS;
    if (sel->policy == EKV_GAUSS && attn->tau_halley > 0) xa.tau_init = th;   // tau_hat + Halley
    if (stats && stats->supp_tok && stats->supp_cap > 0 && attn->transform == EKV_ENTMAX) {
        xa.supp_tok = stats->supp_tok;
        xa.supp_cap = stats->supp_cap;
    }
    const int rows = cache->batch * n_q_heads;
    if (cert) {
        // N4 (Prop. B.2): the top-k pass's exact tau~ <= tau certifies {p : a box(p) > tau~};
        // the second pass attends that superset of the support's pages (exact, Prop. 2)
        TauArgs x1;
        memset(&x1, 0, sizeof(x1));
        EKV_TRY(attend_impl(cache, q, n_q_heads, pi, ns, L.cap, 0, attn, out, th, nullptr, workspace, L, st, &x1,
                            /*marked=*/true));
        EKV_TRY(launch_zero(at<uint4>(workspace, L.retry), (L.zero_bytes - (L.retry - L.zero)) / 16, st));
        EKV_TRY(launch_box_certified(box, cache->batch, n_q_heads, Gq, maxp, cache->seq_lens, th, attn->alpha, pi, ns,
                                     L.cap, uo.umask, L.W, st));
        xa.var = 1;
    }
    EKV_TRY(attend_impl(cache, q, n_q_heads, pi, ns, L.cap, 0, attn, out, tau_p,
                        stats ? stats->supp_count : nullptr, workspace, L, st, &xa, /*marked=*/true));
    // a4: certified dropped-mass bound
    if (want_db)
        EKV_TRY(launch_delta_bar(box, maxp, cache->seq_lens, rows, n_q_heads, Gq, uo.umask, L.W, tau_p, attn->alpha,
                                 stats->delta_bar, st));
    if (stats) {
        if (stats->n_sel)
            EKV_TRY(check_err(cudaMemcpyAsync(stats->n_sel, ns, rows * sizeof(int32_t), cudaMemcpyDeviceToDevice, st),
                              "n_sel copy"));
        if (stats->tau_hat && (sel->policy == EKV_GAUSS || cert))
            EKV_TRY(check_err(cudaMemcpyAsync(stats->tau_hat, th, rows * sizeof(double), cudaMemcpyDeviceToDevice, st),
                              "tau_hat copy"));
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
            EKV_TRY(launch_eval_metrics(rows, ex.tok_list, ex.p_list, ex.n_list, ex.list_cap, pi, ns, L.cap,
                                        stats->delta, stats->recovered, stats->full_supp, st));
        }
    }
    return EKV_OK;
}

}  // extern "C"
