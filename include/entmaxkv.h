/*
 * entmaxkv.h -- C ABI of libentmaxkv.so, the B200 (sm_100a) EntmaxKV sparse
 * alpha-entmax decode step (arxiv 2605.21649).
 *
 * Citations: "P:L" = PAPER.md line L; "S:L" = SPEC.md line L; R<n> = reading n
 * in DESIGN.md section 2.
 *
 * Conventions (every entry point):
 *  - Returns ekv_status; EKV_OK = 0.  Never throws, never synchronises the
 *    stream, never allocates device memory.  entmaxkv_last_error() returns a
 *    thread-local message for the last non-OK status of the calling thread.
 *  - All tensor arguments are DEVICE pointers owned by the caller; they must
 *    stay valid until the work enqueued on `stream` completes.  Scratch comes
 *    from a caller-owned device workspace of entmaxkv_workspace_size() bytes
 *    (256-byte aligned); distinct concurrent calls need distinct workspaces.
 *  - Work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = the
 *    legacy default stream).  Calls are CUDA-graph capturable.
 *  - Layouts are row-major, innermost dimension last; q, k_pages and v_pages must be
 *    16-byte aligned (else EKV_ERR_INVALID_ARG).  Supported shapes:
 *    head_dim = value_dim = 128 (R1), page_size = 16, n_kv_heads in {1,2,4,8,16},
 *    G = n_q_heads / n_kv_heads in {1,2,4,8}, max_pages_per_seq <= 65536.
 *    Anything else -> EKV_ERR_UNSUPPORTED.
 *  - Precondition (not checked): inputs are finite.
 */
#ifndef ENTMAXKV_H
#define ENTMAXKV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    EKV_OK = 0,
    EKV_ERR_INVALID_ARG = 1,  /* bad sizes, alpha <= 1, k < 1, q_page outside (0,1), NULL pointers */
    EKV_ERR_UNSUPPORTED = 2,  /* shape outside the supported set; Gaussian with non-integer beta */
    EKV_ERR_CAPACITY = 3,     /* a caller buffer is too small */
    EKV_ERR_EMPTY = 4,        /* empty cache */
    EKV_ERR_CUDA = 5,         /* a CUDA launch failed (message has cudaGetErrorString) */
    EKV_ERR_COMM = 6          /* a communicator callback returned non-zero (sharded decode) */
} ekv_status;

typedef enum { EKV_BF16 = 0, EKV_F32 = 1 } ekv_dtype;
typedef enum { EKV_ENTMAX = 0, EKV_SOFTMAX = 1 } ekv_transform;     /* P:128-136 / P:121-124 */
typedef enum { EKV_TOPK = 0, EKV_GAUSS = 1, EKV_ALL = 2, EKV_CERTIFIED = 3 } ekv_policy;
enum { EKV_SCORE_BOX = 1, EKV_SCORE_GAUSS = 2 };

/*
 * Paged KV cache (PagedAttention layout).  Caller-owned device buffers.
 *   k_pages  [n_phys_pages][n_kv_heads][page_size][head_dim]   dtype
 *   v_pages  [n_phys_pages][n_kv_heads][page_size][value_dim]  dtype
 *   kmin,kmax[n_phys_pages][n_kv_heads][head_dim]   bound_dtype:
 *       EKV_BOUND_KV   -- the KV dtype, exact copies of the coordinate-wise min / max;
 *       EKV_BOUND_E4M3 -- one byte each, fp8 e4m3 (OCP FN: bias 7, no infinities, max 448),
 *                         kmin rounded DOWN and kmax rounded UP to the e4m3 grid (outward
 *                         rounding: kmin8 <= kmin, kmax8 >= kmax, so the box bound of
 *                         Prop. B.1 stays an upper bound of every token score;
 *                         DESIGN R24).  Precondition: |k| <= 448 (beyond it the bound
 *                         saturates to +-448 and is no longer certified).
 *   ksum, ksumsq [n_phys_pages][n_kv_heads][head_dim]  fp32 append accumulators (R5)
 *   kavg, kvar   [n_phys_pages][n_kv_heads][head_dim]  stat_dtype:
 *       EKV_STAT_F32 -- fp32 (R5);  EKV_STAT_BF16 -- the fp32 values rounded to nearest-even
 *       bf16 (half the bytes the Gaussian scorer reads; R24).
 *   page_table [batch][max_pages_per_seq] int32: logical page -> physical page
 *   seq_lens   [batch] int32 (device; append_kv increments it)
 * Token j of sequence b lives in physical page page_table[b][j / P], slot j % P.
 * A zero-initialised bound_dtype / stat_dtype is the exact layout (KV dtype bounds, fp32 stats).
 */
enum { EKV_BOUND_KV = 0, EKV_BOUND_E4M3 = 1 };
enum { EKV_STAT_F32 = 0, EKV_STAT_BF16 = 1 };
typedef struct {
    int32_t dtype;             /* ekv_dtype of K, V, kmin, kmax */
    int32_t batch;
    int32_t n_kv_heads;
    int32_t head_dim;
    int32_t value_dim;
    int32_t page_size;
    int32_t max_pages_per_seq;
    int32_t n_phys_pages;
    void *k_pages, *v_pages;
    void *kmin, *kmax;         /* bound_dtype */
    float *ksum, *ksumsq;
    void *kavg, *kvar;         /* stat_dtype */
    const int32_t *page_table;
    int32_t *seq_lens;
    int32_t bound_dtype;       /* EKV_BOUND_KV | EKV_BOUND_E4M3 */
    int32_t stat_dtype;        /* EKV_STAT_F32 | EKV_STAT_BF16 */
} ekv_cache;

/* alpha > 1; transform = ekv_transform (softmax ignores alpha).
 * flags: EKV_ATTN_DENSE_V -- entmaxkv_full_attend streams EVERY V row (weights p_j, zero
 * outside the support), the paper's full-cache reference that reads all scores and V
 * (P:1343); without it the full path reads V of the support only.  Ignored elsewhere.
 * EKV_ATTN_CANONICAL -- the full path of a bf16 cache scores every token on tensor cores by
 *   default (mma bf16 -> fp32; the products are exact, the accumulation order is the tensor
 *   core's, DESIGN R26), so its scores may differ from the canonical order of R1 in the last
 *   bits; this flag keeps R1 (bit-identical to the sparse path's scores). */
enum { EKV_ATTN_DENSE_V = 1, EKV_ATTN_CANONICAL = 2 };
/* tau_halley > 0 (entmax): the paper's approximate threshold instead of the exact one
 * ("a histogram-based initialization followed by Halley iterations"; DESIGN R23):
 * tau_0 from a 64-bin histogram of z over (z_max - 1, z_max] (the largest bin edge whose
 * certified lower bound of F reaches 1), then tau_halley Halley steps on
 * sum_{z > t} (z - t)^beta = 1; p_j = (z_j - tau)_+^beta renormalised (R12).  0 = exact. */
typedef struct {
    float alpha;
    int32_t transform;
    int32_t flags;
    int32_t tau_halley;
} ekv_attn_params;

/*
 * policy TOPK: k_pages >= 1 pages per query head (R3 tie-break).
 * policy GAUSS: q_page in (0,1) page-max confidence, margin = Delta >= 0
 *   (Eq. gaussian-selector-main).  beta = 1/(alpha-1) in {1,2,3,4}: App. D's closed
 *   forms (R15); any other beta <= 32 (alpha > 1 + 1/32): the expectation evaluated numerically
 *   (DESIGN R28) -- a per-call table of log E[(m + Z)_+^beta]
 *   (Chebyshev series from tanh-sinh quadrature, one extra launch) in the workspace, so
 *   entmaxkv_select then needs a workspace.  Rows longer than 8192 pages run on a cluster of
 *   CTAs.  Else EKV_ERR_UNSUPPORTED.
 * policy ALL: every page (the full cache).
 * policy CERTIFIED (Prop. B.2 "no false negatives from deterministic page
 *   bounds"): entmaxkv_decode only.  A first top-k pass (k_pages) gives the exact
 *   sparse threshold tau~, a lower bound of the full-cache tau (DESIGN R13); then every page
 *   with (alpha-1) * box(p) > tau~ (fp64 decision) is selected and attended.  That selection
 *   contains every support token's page, so the output IS full-cache entmax (Prop. 2,
 *   P:213-216) and delta_bar = 0.  stats->tau_hat receives tau~, n_sel the final |C_page|;
 *   the workspace holds full-length page lists.  With loose box bounds the selection can
 *   cover most pages (App. C) -- an exactness mode, not a fast one.  Entmax only.
 */
typedef struct {
    int32_t policy;
    int32_t k_pages;
    double q_page;
    double margin;
} ekv_select_params;

/*
 * Per-(b, q-head) decode statistics, all [batch][n_q_heads], any may be NULL.
 *   tau        f64  exact alpha-entmax threshold over C_tok (R9)
 *   supp_count i32  |S~| support size within C_tok (softmax: |C_tok|)
 *   n_sel      i32  |C_page|
 *   delta_bar  f64  certified dropped-mass bound (R16; top-k and Gaussian)
 *   tau_hat    f64  Gaussian threshold estimate (GAUSS only)
 * eval_exact != 0 additionally runs a full-cache pass (all K; R16) and fills
 *   delta f64 exact dropped mass (Eq. delta),
 *   recovered i32 |S cap C_tok|, full_supp i32 |S| (Eq. rho),
 *   tau_full f64.
 * supp_tok (may be NULL): [batch][n_q_heads][supp_cap] i32, the token positions of S~ (the
 *   support within C_tok, R9) in ascending order; a row with more than supp_cap support tokens
 *   gets its first supp_cap (supp_count holds the total).  Entmax only.
 */
typedef struct {
    double *tau;
    int32_t *supp_count;
    int32_t *n_sel;
    double *delta_bar;
    double *tau_hat;
    int32_t eval_exact;
    double *delta;
    int32_t *recovered;
    int32_t *full_supp;
    double *tau_full;
    int32_t *supp_tok;
    int32_t supp_cap;
} ekv_decode_stats;

/* Last error message of the calling thread ("" if none). */
const char *entmaxkv_last_error(void);

/* Library version string. */
const char *entmaxkv_version(void);

/*
 * Workspace bytes needed by score/select/sparse_attend/full_attend/decode for
 * this cache shape, n_q_heads and selection policy (sel may be NULL = ALL).
 */
size_t entmaxkv_workspace_size(const ekv_cache *cache, int32_t n_q_heads,
                               const ekv_select_params *sel);

/*
 * Selection capacity (pages per query head) that page_idx buffers must hold:
 * min(k_pages, max_pages) for TOPK, max_pages for GAUSS/ALL.
 */
int32_t entmaxkv_select_capacity(const ekv_cache *cache, const ekv_select_params *sel);

/*
 * a0: append n_tokens tokens per sequence.  k_new [batch][n_tokens][n_kv_heads][head_dim],
 * v_new [batch][n_tokens][n_kv_heads][value_dim] (cache dtype).  Token t of
 * sequence b goes to position seq_lens[b] + t; page_table[b][(seq_lens[b]+t)/P]
 * must already map a physical page (precondition).  Updates kmin/kmax/ksum/ksumsq
 * incrementally and rewrites kavg/kvar of the touched page (R5), then
 * seq_lens[b] += n_tokens.
 */
ekv_status entmaxkv_append_kv(const ekv_cache *cache, const void *k_new, const void *v_new,
                              int32_t n_tokens, void *stream);

/*
 * a0 (bulk): recompute kmin/kmax/ksum/ksumsq/kavg/kvar of every valid page of
 * every sequence from the stored keys (identical bits to incremental appends).
 */
ekv_status entmaxkv_rebuild_page_stats(const ekv_cache *cache, void *stream);

/*
 * a1: page scores for every query head.  q [batch][n_q_heads][head_dim] (cache dtype).
 * modes = EKV_SCORE_BOX and/or EKV_SCORE_GAUSS.  Outputs (NULL if not requested)
 * [batch][n_q_heads][max_pages_per_seq] fp32; entries for pages >= ceil(seq_len/P)
 * are left untouched.
 *   box    = fl32(dot16x8(q, kext) * c_d), kext_i = q_i >= 0 ? kmax_i : kmin_i
 *            (Eq. box-page-bound, R1, R2)
 *   mu     = fl32(dot16x8(q, kavg) * c_d)
 *   sigma2 = fl32(dot16x8(q*q, kvar) * (1/d))
 */
ekv_status entmaxkv_score_pages(const ekv_cache *cache, const void *q, int32_t n_q_heads,
                                int32_t modes, float *box, float *mu, float *sigma2,
                                void *workspace, void *stream);

/*
 * a2 / a2': page selection per (b, q-head).  Inputs are score_pages outputs
 * (box for TOPK; mu, sigma2 for GAUSS).  Outputs:
 *   page_idx [batch][n_q_heads][sel_stride] int32, ascending logical page ids;
 *   n_sel    [batch][n_q_heads] int32;
 *   tau_hat  [batch][n_q_heads] f64 (GAUSS; may be NULL).
 * sel_stride >= entmaxkv_select_capacity(), else EKV_ERR_CAPACITY.
 */
ekv_status entmaxkv_select(const ekv_cache *cache, int32_t n_q_heads, const float *box,
                           const float *mu, const float *sigma2, const ekv_select_params *sel,
                           float alpha, int32_t *page_idx, int32_t *n_sel, int32_t sel_stride,
                           double *tau_hat, void *workspace, void *stream);

/*
 * a3 (+a6): attention of every (b, q-head) over its own page list:
 * C_tok = tokens of page_idx[b][h][0..n_sel) below seq_len; p~ = alpha-entmax (exact
 * tau, R8/R9) or softmax of {s_j : j in C_tok}; out = sum p~_j v_j / sum p~_j (R12).
 * K of the KV-group union is read once (R17); V only for support tokens.
 * tau_init (nullable, device [batch][n_q_heads] f64): with attn->tau_halley > 0, the start of
 *   the Halley refinement instead of the histogram initialisation -- the paper's Gaussian variant,
 *   "the selected page indices and estimated threshold are then passed to the decode kernel.
 *   Inside the kernel, we perform one additional Halley refinement using the actual selected
 *   scores"; a start outside [z_max - 1, z_max) is replaced by z_max - 1 (DESIGN R25).
 *   Ignored for the exact threshold (tau_halley = 0).  entmaxkv_decode passes the Gaussian
 *   selector's tau_hat itself when policy = GAUSS and tau_halley > 0.
 *   out  [batch][n_q_heads][value_dim] fp32
 *   tau  [batch][n_q_heads] f64 (softmax: log-normaliser)   (may be NULL)
 *   supp [batch][n_q_heads] int32                            (may be NULL)
 * page lists must be ascending and unique.
 */
ekv_status entmaxkv_sparse_attend(const ekv_cache *cache, const void *q, int32_t n_q_heads,
                                  const int32_t *page_idx, const int32_t *n_sel,
                                  int32_t sel_stride, const double *tau_init,
                                  const ekv_attn_params *attn,
                                  float *out, double *tau, int32_t *supp,
                                  void *workspace, void *stream);

/* a5 (+a6): the dense baseline: the same attention over every page (all K read). */
ekv_status entmaxkv_full_attend(const ekv_cache *cache, const void *q, int32_t n_q_heads,
                                const ekv_attn_params *attn, float *out, double *tau,
                                int32_t *supp, void *workspace, void *stream);

/*
 * Fused decode step: score_pages -> select -> sparse_attend (+ statistics a4),
 * all enqueued on `stream` with no host synchronisation.
 * out [batch][n_q_heads][value_dim] fp32.  stats may be NULL.
 */
ekv_status entmaxkv_decode(const ekv_cache *cache, const void *q, int32_t n_q_heads,
                           const ekv_select_params *sel, const ekv_attn_params *attn,
                           float *out, ekv_decode_stats *stats, void *workspace, void *stream);

/*
 * Sequence sharding (north star: "sequence sharding of the page cache across
 * 2/4/8 GPUs over NVLink with NCCL allreduce of per-head partial sum (z - tau)_+^beta during
 * tau bisection and of partial numerator/denominator outputs").
 *
 * Striping: rank r of `world` holds the global pages p = r + i * world as its local pages
 * i = 0, 1, ... (its own ekv_cache: local page table, local seq_lens = the number of tokens
 * in those pages; only the global last page can be partial and it is the owner's last local
 * page).  Every rank calls entmaxkv_decode_sharded with the same q and parameters; each gets
 * the full output (replicated).
 *
 * The library never talks to a network itself: collectives go through the caller's
 * callbacks (e.g. NCCL via torch.distributed), enqueued on `stream`, in the same order on
 * every rank.  Both callbacks return 0 on success.  Buffers passed to them lie inside the
 * caller's workspace.
 *   allreduce(buf, count, dtype, op): in place; dtype 0 = f32, 1 = f64; op 0 = sum, 1 = max.
 *   allgather(send, recv, bytes): rank r's `bytes` bytes from send land at recv + r * bytes.
 */
typedef struct {
    int32_t rank, world;
    int32_t (*allreduce)(void *buf, size_t count, int32_t dtype, int32_t op, void *user, void *stream);
    int32_t (*allgather)(const void *send, void *recv, size_t bytes, void *user, void *stream);
    void *user;
    /* 0: adaptive multisection (stops when every row converged; one small synchronous device->host
     * read per round).  R > 0: exactly R rounds with no host read -- the step is then CUDA-graph
     * capturable if the callbacks are (NCCL on the same stream is); R >= 12 always converges (R20). */
    int32_t fixed_rounds;
    /* In-kernel collectives: when peers[0] != NULL the step exchanges its data
     * inside its own kernels over peer memory and the callbacks / fixed_rounds are ignored.
     * peers[q] (q < world <= 8) = rank q's exchange buffer as mapped in this process: device
     * memory of entmaxkv_peer_buffer_size() bytes per rank, ZEROED once before the first step,
     * reachable from this device (CUDA IPC with peer access over NVLink / NVSwitch across GPUs;
     * plain device pointers for virtual ranks sharing one GPU).  Each exchange: every rank stores
     * its payload into every rank's buffer and raises a flag there (release, system scope); a
     * rank waits on its own buffer's flags (acquire) and reduces the W payloads in rank order, so
     * every rank computes identical bits and the multisection rounds stop on every rank at the
     * same round with no host read.  The top-k lists, z_max, the round partials, the power sums
     * and numerator / denominator all go this way (2 + rounds + 2 exchanges per row and step).
     * The step is then CUDA-graph capturable (the exchange counters live in the buffers).  All
     * ranks' steps must run concurrently; a flag missing for ~2 s marks the row failed
     * (EKV_STATUS_TIMEOUT: NaN out/tau, supp -1) instead of hanging, after which the buffers
     * must be re-zeroed on every rank.  The buffer memory stays owned by the caller. */
    void *peers[8];
} ekv_comm;

/* Bytes of one rank's exchange buffer for the in-kernel collective mode (ekv_comm.peers);
 * 0 on invalid arguments (world must be 1..8). */
size_t entmaxkv_peer_buffer_size(const ekv_cache *local, int32_t n_q_heads, const ekv_select_params *sel,
                                 int32_t world);

/* Workspace bytes for entmaxkv_decode_sharded on this local cache shape. */
size_t entmaxkv_shard_workspace_size(const ekv_cache *local, int32_t n_q_heads, const ekv_select_params *sel,
                                     int32_t world);

/*
 * One sequence-sharded decode step (top-k selection, exact entmax):
 *   1. local box scores + local top-k; (score, global page) lists all-gathered; the global
 *      top-k (R3 tie-break on the global page index, i.e. identical to the 1-GPU selection)
 *      is merged on every rank, which keeps its own pages;
 *   2. K scores of the local share; all-reduce(max) of the row maxima;
 *   3. local candidates z > z_max - 1;
 *   4. multisection rounds on F(x) = sum (z - x)_+^beta: per round an all-reduce(sum) of
 *      F, #{z > x}, #{z >= x} at 64 probes per row, until no z lies strictly inside the
 *      bracket (the support is then exact, R9); one device->host read per round from the
 *      second round on;
 *   5. all-reduce(sum) of the support's power sums -> tau (closed form / polynomial Newton);
 *   6. all-reduce(sum) of the numerator sum p_j v_j and denominator sum p_j -> out.
 * global_seq_lens: device [batch] int32, the unsharded sequence lengths.
 * Supported: policy TOPK, transform ENTMAX, integer beta = 1/(alpha-1) in {1,2,3,4}, world * k
 * <= 16384.  A row with more than 8192 candidates on some rank is marked on every rank in the same
 * round (NaN out / tau, supp_count -1, EKV_STATUS_CAPACITY in the workspace status word); the
 * adaptive mode also returns EKV_ERR_CAPACITY after the step's collectives complete.
 * stats may be NULL; fills tau, supp_count (global |S~|) and n_sel (global |C_page|).
 * Graph-capturable with comm->fixed_rounds > 0 (see ekv_comm).
 */
ekv_status entmaxkv_decode_sharded(const ekv_cache *local, const int32_t *global_seq_lens, const void *q,
                                   int32_t n_q_heads, const ekv_select_params *sel, const ekv_attn_params *attn,
                                   const ekv_comm *comm, float *out, ekv_decode_stats *stats, void *workspace,
                                   void *stream);

/*
 * Device status of the last score/select/attend/decode step that used `workspace` (the word is
 * cleared at the start of every such call, in its first kernel): bit 0 (EKV_STATUS_CAPACITY) =
 * some row's candidate set exceeded a kernel capacity -- the exact support did not fit the tau
 * kernel's shared-memory list (more than ~10k support tokens) or, sequence-sharded, more than
 * 8192 candidates per row and rank; such rows get out = NaN, tau = NaN, supp_count = -1.
 * Bit 1 (EKV_STATUS_TIMEOUT): in-kernel collectives (ekv_comm.peers) -- a peer's exchange did
 * not arrive within ~2 s; those rows are NaN and the exchange buffers must be re-zeroed.
 * Copies the word to *flags, synchronising `stream` (the one call that does), and returns
 * EKV_ERR_COMM when bit 1 is set, else EKV_ERR_CAPACITY when bit 0 is set, else EKV_OK.  cache / n_q_heads / sel as for
 * entmaxkv_workspace_size.
 */
enum { EKV_STATUS_CAPACITY = 1, EKV_STATUS_TIMEOUT = 2 };
ekv_status entmaxkv_workspace_status(const ekv_cache *cache, int32_t n_q_heads, const ekv_select_params *sel,
                                     const void *workspace, int32_t *flags, void *stream);

/* Number of kernels the last successful entmaxkv_decode / full_attend call on this
 * thread enqueued (for launch accounting). */
int32_t entmaxkv_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* ENTMAXKV_H */
