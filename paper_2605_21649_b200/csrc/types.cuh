// types.cuh -- constants and plain structs shared by the host launch code and the kernels
// of libentmaxkv (no kernels here, so every translation unit may include it).
#pragma once
#include <stdint.h>
#include <stddef.h>

namespace ekv {

constexpr int kD = 128;   // head_dim = value_dim (R1)
constexpr int kP = 16;    // page size
constexpr float kCd = 0x1.6a09e6p-4f;   // fl32(1/sqrt(128)) (R2)

struct CacheView {
    int dtype, B, Hkv, maxp, nphys;
    const void *K, *V;
    void *Kw, *Vw;            // writable aliases (append)
    void *kmin, *kmax;        // bound: 0 = KV dtype, 1 = e4m3 outward-rounded (uint8)
    float *ksum, *ksumsq;
    void *kavg, *kvar;        // stat: 0 = fp32, 1 = bf16 (RNE)
    const int32_t *page_table;
    int32_t *seq_lens;
    int bound, stat;
};

// ---------------------------------------------------------------- a2 top-k
constexpr int kTkKPT = 16;          // keys per thread; NT = 512 (8192 pages per CTA, <= 8 CTAs)
constexpr int kTkCap = 4096;        // sample-pivot candidates per row (u64 composites, x2 in smem)

// ---------------------------------------------------------------- a3 / a5 candidates and tau
constexpr int kCpc = 1024;          // candidates per chunk region (k_candidates)
constexpr int kCap = 12288;         // eval-list capacity per row
constexpr int kPr = 2048;           // pruned-list capacity (tau solver)

struct TauArgs {
    const float *scores; size_t ntok;
    const uint32_t *rowmax; const int *ccount; const float *cand_s; const int32_t *cand_j; int nch;
    const int32_t *page_idx; const int32_t *n_sel; int sel_stride; int full;
    int Hq, G; float alpha; int transform;
    float *out; double *tau_out; int32_t *supp_out;
    int32_t *tok_list; double *p_list; int32_t *n_list; int list_cap;     // eval list
    int no_pv;                                                            // tau/supp only (dense-V)
    int cap, pr;                                                          // tau kernel capacities
    int approx_h;                                                         // > 0: approximate tau, Halley steps
    const double *tau_init;                                               // approx: start, else histogram
    int var;                                                              // list lengths vary (slices from n_sel)
    int32_t *supp_tok; int supp_cap;                                      // support token list (decode stats)
    uint32_t *status;                                                     // workspace status word (EKV_STATUS_*)
    int32_t *retry; int retry_pass;   // reduced-capacity rows that overflowed -> re-run at kTsCap (pass 1)
};
constexpr uint32_t kStatusCapacity = 1u;   // a row's candidates overflowed a kernel capacity (row NaN)

constexpr int kTsNT = 256;
constexpr int kTsCap = 10240;       // candidates in shared memory
constexpr int kTsSup = 1024;        // support entries per gather round
constexpr int kTsVpre = 64;         // V rows staged for short lists
constexpr int kTsU = 4;             // float4 items per thread per round (x 4 ranks: 1024 pages)
template <typename T> constexpr int ts_smem() {
    return (4 + 4 + 4 + 1) * kTsCap + (8 + 4) * kPr + kTsVpre * kD * (int)sizeof(T);
}
constexpr int kSmxPages = 32;       // list pages per CTA of the split dense-V / softmax pass

// ---------------------------------------------------------------- a4 delta_bar
constexpr int kDbChunk = 8192;      // pages per CTA: 256 threads x 8 groups of 4 pages
struct DbConst {                    // per-call constants of alpha (host-computed)
    double a, beta, inv_a;          // a = alpha - 1, beta = 1/a
    int ib;                         // integer beta in 1..4, else 0
};

// ---------------------------------------------------------------- P2 sequence sharding
constexpr int kShT = 62;            // interior probes per multisection round (6 bits)
constexpr int kShP = kShT + 2;      // probe points incl. the bracket ends
constexpr int kShCap = 8192;        // local candidates per row
constexpr int kShSums = 5;          // S_0 .. S_4
constexpr int kShMergeNT = 1024;
constexpr int kShMergeKPT = 16;     // W * kc <= 16384
constexpr int kMaxPeers = 8;        // in-kernel collectives (N2): ranks per exchange
constexpr uint32_t kStatusTimeout = 2u;    // a peer's flag did not arrive in time (row NaN)
// Rank q's exchange buffer (entmaxkv_peer_buffer_size): [ctr: rows x u64][flag: W x rows x u64]
// (padded to 256 B) then [data: 2 parities x W senders x rows x pay bytes].
struct PeerSet {
    unsigned char *buf[kMaxPeers];   // every rank's exchange buffer, as mapped in this process
    int W, rk, rows;
    uint32_t pay;                    // payload bytes per (parity, sender, row), multiple of 16
};
struct ShardRow {                   // per-row multisection state (device)
    double lo, hi;                  // F(lo) >= 1 > F(hi)
    double cgt_lo, cge_hi;          // #{z > lo}, #{z >= hi} (global)
    int done, rounds;
};

// debug builds (-DEKV_STAMPS): each translation unit registers a reader of its stamp buffers
typedef void (*DebugReader)(int what, void *out, int reset);
void debug_register(DebugReader r);   // entmaxkv.cu

}  // namespace ekv
