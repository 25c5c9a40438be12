// kernels_shard.cuh -- sequence-sharded decode (north star: "sequence
// sharding of the page cache across 2/4/8 GPUs over NVLink with NCCL allreduce of per-head
// partial sum (z - tau)_+^{1/(alpha-1)} during tau bisection and of partial
// numerator/denominator outputs").
//
// Striping: rank r of W holds the global pages p = r + i W (local page i); only the global
// last page can be partial and it is its owner's last local page, so a rank's pages form an
// ordinary local cache of L_r tokens.  The collectives are issued by the host between these
// kernels (entmaxkv_decode_sharded), through the caller's communicator callbacks:
//   1. local top-k (the ordinary kernels) -> k_shard_pack: (box score, global page) of the
//      rank's k best pages -> ALL-GATHER -> k_shard_merge: the global top-k with R3's
//      tie-break (score desc, global page asc) -> this rank's share, ascending local ids.
//   2. K scores of the share (ordinary kernels) -> k_shard_zmax -> ALL-REDUCE(MAX) of z_max.
//   3. k_shard_cand: local candidates {z > z_max - 1} (tau >= z_max - 1, R9), fp64 z.
//   4. multisection on F(x) = sum (z - x)_+^beta (F decreasing; F(z_max - 1) >= 1 >
//      F(z_max) = 0): each round k_shard_probe evaluates, at T + 2 points lo = x_0 < ... <
//      x_{T+1} = hi, the partial F and the counts #{z > x}, #{z >= x} -> ALL-REDUCE(SUM) ->
//      the next round's k_shard_probe first narrows [lo, hi] to the adjacent probes with
//      F(lo) >= 1 > F(hi).  A row is done when no z lies strictly between lo and hi
//      (#{z > lo} == #{z >= hi}): then the support is exactly {z > lo} = {z >= hi}, i.e.
//      R9's F(z_j) < 1 test (z >= hi: F(z) <= F(hi) < 1; z <= lo: F(z) >= F(lo) >= 1).
//   5. k_shard_sums: S_m = sum_{z > lo} (z - lo)^m, m <= 4 -> ALL-REDUCE(SUM) -> tau = lo +
//      delta with sum_S (w - delta)^beta = 1 (w = z - lo): closed forms for beta = 1, 2,
//      Newton on the expanded polynomial for beta = 3, 4 (integer beta only).
//   6. k_shard_pv: numerator sum p_j v_j (fp32) and denominator sum p_j (fp64) of the
//      local support -> ALL-REDUCE(SUM) -> k_shard_out: out = num / den (R12).
#pragma once
#include "common.cuh"

namespace ekv {


// 1a. (score, global page) of the rank's selected pages; padding: -inf / -1
static __global__ void __launch_bounds__(256) k_shard_pack(const float *__restrict__ box, int maxp,
                                                    const int32_t *__restrict__ page_idx,
                                                    const int32_t *__restrict__ n_sel, int stride, int kc,
                                                    int rank, int world, float *__restrict__ cs,
                                                    int32_t *__restrict__ cg) {
    const int row = blockIdx.x;
    const int n = n_sel[row];
    for (int i = threadIdx.x; i < kc; i += 256) {
        float s = -INFINITY;
        int g = -1;
        if (i < n) {
            const int lp = page_idx[(size_t)row * stride + i];
            s = box[(size_t)row * maxp + lp];
            g = lp * world + rank;
        }
        cs[(size_t)row * kc + i] = s;
        cg[(size_t)row * kc + i] = g;
    }
}

// ============================================================================ N2: in-kernel collectives
// (SURVEY 8(f) N2).  Every rank owns an exchange buffer (PeerSet layout, types.cuh) that all
// ranks can address (CUDA IPC + NVLink peer access across GPUs; plain pointers for virtual
// ranks on one GPU).  Exchange e of a row: each rank writes its payload into slot
// [e & 1][own rank][row] of EVERY rank's buffer (remote stores), fences at system scope and
// raises flag[own rank][row] = e there (release); a reader spins on its own buffer's W
// flags (acquire) and reduces the W payloads in rank order -- identical bits on every rank,
// so the ranks' data-dependent control flow (multisection rounds) stays in lockstep with no
// host involvement.  Double buffering is safe: a rank writes exchange e + 1 only after it
// has received every rank's exchange e, which each sent only after consuming e - 1.  The
// per-row exchange counter lives in the own buffer (ctr[row]) and persists across calls, so
// the step is CUDA-graph capturable.  A flag not raised within ~2 s marks the row failed
// (kStatusTimeout) instead of hanging the device.
__device__ __forceinline__ size_t px_hdr(const PeerSet &P) {
    return ((size_t)8 * P.rows * (1 + P.W) + 255) & ~(size_t)255;
}
__device__ __forceinline__ uint64_t *px_ctr(const PeerSet &P, int row) {
    return reinterpret_cast<uint64_t *>(P.buf[P.rk]) + row;
}
__device__ __forceinline__ uint64_t *px_flag(const PeerSet &P, int q, int sender, int row) {
    return reinterpret_cast<uint64_t *>(P.buf[q]) + P.rows + (size_t)sender * P.rows + row;
}
__device__ __forceinline__ unsigned char *px_data(const PeerSet &P, int q, uint64_t e, int sender, int row) {
    return P.buf[q] + px_hdr(P) + (((size_t)(e & 1) * P.W + sender) * P.rows + row) * P.pay;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t px_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// raise exchange e's flag of `row` at every rank (after this CTA's payload stores)
__device__ __forceinline__ void px_signal(const PeerSet &P, int row, uint64_t e) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < P.W) st_release_sys(px_flag(P, threadIdx.x, P.rk, row), e);
}
// push nb bytes (16-byte multiple, shared memory) as exchange e of `row` to every rank
__device__ __forceinline__ void px_push(const PeerSet &P, int row, uint64_t e, const void *src, int nb) {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    for (int q = 0; q < P.W; ++q) {
        uint4 *d = reinterpret_cast<uint4 *>(px_data(P, q, e, P.rk, row));
        for (int i = threadIdx.x; i < nb / 16; i += blockDim.x) __stcg(d + i, s4[i]);
    }
    px_signal(P, row, e);
}
// wait until every rank's exchange e of `row` has arrived; false (on every thread) on timeout
__device__ __forceinline__ bool px_wait(const PeerSet &P, int row, uint64_t e) {
    bool ok = true;
    if (threadIdx.x < P.W) {
        const uint64_t *f = px_flag(P, P.rk, threadIdx.x, row);
        const uint64_t t0 = px_now();
        while (ld_acquire_sys(f) < e) {
            if (px_now() - t0 > 2000000000ull) { ok = false; break; }
        }
    }
    return __syncthreads_and(ok) != 0;
}

// 1a'. (in-kernel mode) the pack of 1a written straight into every rank's exchange buffer:
//      payload = kc floats (scores) then kc int32 (global pages)
static __global__ void __launch_bounds__(256) k_shard_pack_push(const float *__restrict__ box, int maxp,
                                                                const int32_t *__restrict__ page_idx,
                                                                const int32_t *__restrict__ n_sel, int stride,
                                                                int kc, PeerSet P) {
    const int row = blockIdx.x;
    const int n = n_sel[row];
    const uint64_t e = *px_ctr(P, row) + 1;
    for (int i = threadIdx.x; i < kc; i += 256) {
        float s = -INFINITY;
        int g = -1;
        if (i < n) {
            const int lp = page_idx[(size_t)row * stride + i];
            s = box[(size_t)row * maxp + lp];
            g = lp * P.W + P.rk;
        }
        for (int q = 0; q < P.W; ++q) {
            unsigned char *d = px_data(P, q, e, P.rk, row);
            __stcg(reinterpret_cast<float *>(d) + i, s);
            __stcg(reinterpret_cast<int32_t *>(d) + kc + i, g);
        }
    }
    px_signal(P, row, e);
    if (threadIdx.x == 0) *px_ctr(P, row) = e;
}

// 1b. global top-k among the W gathered lists (recv_s / recv_g: [W][rows][kc]); this rank's
// selected entries come from its own (ascending) segment, so the output stays ascending.
static __global__ void __launch_bounds__(kShMergeNT) k_shard_merge(const float *__restrict__ recv_s,
                                                            const int32_t *__restrict__ recv_g, int rows,
                                                            int kc, int k, int rank, int world,
                                                            const int32_t *__restrict__ gseq,
                                                            int32_t *__restrict__ page_idx,
                                                            int32_t *__restrict__ n_sel, int stride, int Hq, int G,
                                                            uint32_t *__restrict__ umask, int W, PeerSet P,
                                                            uint32_t *__restrict__ status) {
    __shared__ uint32_t hist[256];
    __shared__ int sh[kShMergeNT / 32 + 2];
    const int row = blockIdx.x;
    // in-kernel collective mode (P.W > 0): the W lists arrive in this rank's exchange buffer
    // (k_shard_pack_push); wait for them, then read them from there
    uint64_t ep = 0;
    if (P.W > 0) {
        ep = *px_ctr(P, row);
        if (!px_wait(P, row, ep)) {
            if (threadIdx.x == 0) { n_sel[row] = 0; atomicOr(status, kStatusTimeout); }
            return;
        }
    }
    auto lst_s = [&](int w, int i) -> float {
        return P.W > 0 ? __ldcg(reinterpret_cast<const float *>(px_data(P, P.rk, ep, w, row)) + i)
                       : recv_s[((size_t)w * rows + row) * kc + i];
    };
    auto lst_g = [&](int w, int i) -> int32_t {
        return P.W > 0 ? __ldcg(reinterpret_cast<const int32_t *>(px_data(P, P.rk, ep, w, row)) + kc + i)
                       : recv_g[((size_t)w * rows + row) * kc + i];
    };
    const int ntot = world * kc;
    const int Mg = n_pages_of(gseq[row / Hq]);         // global pages of the sequence
    const int keff = min(k, Mg);
    uint32_t key[kShMergeKPT], inv[kShMergeKPT];
#pragma unroll
    for (int j = 0; j < kShMergeKPT; ++j) {
        const int e = threadIdx.x + kShMergeNT * j;
        key[j] = 0u;
        inv[j] = 0u;
        if (e < ntot) {
            const int w = e / kc, i = e - w * kc;
            const int g = lst_g(w, i);
            if (g >= 0) {
                key[j] = f2key(lst_s(w, i));
                inv[j] = 0xffffffffu - (uint32_t)g;      // larger = lower global page (R3)
            }
        }
    }
    int n_gt = 0;
    uint32_t T = 0u, Ic = 0u;
    int nvalid = 0;
#pragma unroll
    for (int j = 0; j < kShMergeKPT; ++j) nvalid += key[j] != 0u;
    nvalid = block_sum_i<kShMergeNT>(nvalid, sh);
    const int kk = min(keff, nvalid);
    if (kk > 0) {
        T = block_kth_largest<kShMergeNT, kShMergeKPT>(key, kk, hist, sh, &n_gt);
        const int need = kk - n_gt;              // equal keys to take, lowest global pages first
        uint32_t eq[kShMergeKPT];
#pragma unroll
        for (int j = 0; j < kShMergeKPT; ++j) eq[j] = (key[j] == T && key[j] != 0u) ? inv[j] : 0u;
        int dummy;
        Ic = block_kth_largest<kShMergeNT, kShMergeKPT>(eq, need, hist, sh, &dummy);
    }
    // this rank's segment, in its ascending order
    int32_t *out = page_idx + (size_t)row * stride;
    const int unit = (row / Hq) * (Hq / G) + (row % Hq) / G, gh = (row % Hq) % G;
    uint32_t *um = umask + (size_t)unit * W;
    int base = 0;
    for (int i0 = 0; i0 < kc; i0 += kShMergeNT) {
        const int i = i0 + threadIdx.x;
        bool s = false;
        int lp = 0;
        if (i < kc && kk > 0) {
            const int g = lst_g(rank, i);
            if (g >= 0) {
                const uint32_t kv = f2key(lst_s(rank, i)), iv = 0xffffffffu - (uint32_t)g;
                s = kv > T || (kv == T && iv >= Ic);
                lp = g / world;
            }
        }
        int tot;
        const int pos = base + block_excl_scan<kShMergeNT>(s ? 1 : 0, sh, &tot);
        if (s) {
            out[pos] = lp;
            union_mark(um, lp, gh);
        }
        base += tot;
    }
    if (threadIdx.x == 0) n_sel[row] = base;
}

// 2. local row max (ordered key, 0 = empty) -> fp32 (-inf when empty)
static __global__ void k_shard_zmax(const uint32_t *__restrict__ rowmax, int rows, float *__restrict__ zmax) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) zmax[i] = rowmax[i] ? key2f(rowmax[i]) : -INFINITY;
}


// 3. local candidates {z > z_max - 1} of the row's score list (list-ordered reads);
//    initialises the bracket [a z_max - 1 - eps, a z_max] (block function, 256 threads)
__device__ __forceinline__ void shard_cand_row(int row, float zm, const float *__restrict__ scores, size_t ntok,
                                               const int32_t *__restrict__ page_idx,
                                               const int32_t *__restrict__ n_sel, int stride,
                                               const int32_t *__restrict__ seq_lens,
                                               const int32_t *__restrict__ ptab, int maxp, int Hq, float alpha,
                                               double *__restrict__ cz, int32_t *__restrict__ cj,
                                               int32_t *__restrict__ cph, int32_t *__restrict__ ncand,
                                               ShardRow *__restrict__ st, int *sh) {
    const int b = row / Hq;
    const int L = seq_lens[b];
    const int nl = n_sel[row];
    const double a = (double)alpha - 1.0;
    const double zmax = a * (double)zm;
    const double tlo = zmax - 1.0 - 1e-12 * fmax(1.0, fabs(zmax));
    if (threadIdx.x == 0) {
        ShardRow s;
        s.lo = tlo; s.hi = zmax; s.cgt_lo = -1.0; s.cge_hi = -1.0; s.done = (zm == -INFINITY) ? 2 : 0; s.rounds = 0;
        st[row] = s;
    }
    const float *srow = scores + (size_t)row * ntok;
    const int32_t *plist = page_idx + (size_t)row * stride;
    int n = 0;
    if (zm != -INFINITY) {
        for (int e0 = 0; e0 < nl * kP; e0 += 256) {
            const int e = e0 + threadIdx.x;
            bool in = false;
            float s = 0.f;
            int j = 0, pg = 0;
            if (e < nl * kP) {
                pg = plist[e / kP];
                j = pg * kP + e % kP;
                s = srow[j];
                in = j < L && s != -INFINITY && a * (double)s > tlo;
            }
            int tot;
            const int pos = n + block_excl_scan<256>(in ? 1 : 0, sh, &tot);
            if (in && pos < kShCap) {
                const size_t o = (size_t)row * kShCap + pos;
                cz[o] = a * (double)s;
                cj[o] = j;
                cph[o] = ptab[(size_t)b * maxp + pg];
            }
            n += tot;
        }
    }
    if (threadIdx.x == 0) ncand[row] = n;          // > kShCap: overflow (row reported NaN)
}
static __global__ void __launch_bounds__(256) k_shard_cand(const float *__restrict__ scores, size_t ntok,
                                                    const int32_t *__restrict__ page_idx,
                                                    const int32_t *__restrict__ n_sel, int stride,
                                                    const int32_t *__restrict__ seq_lens, const int32_t *__restrict__ ptab,
                                                    int maxp, int Hq, const float *__restrict__ zmax_g, float alpha,
                                                    double *__restrict__ cz, int32_t *__restrict__ cj,
                                                    int32_t *__restrict__ cph, int32_t *__restrict__ ncand,
                                                    ShardRow *__restrict__ st) {
    __shared__ int sh[9];
    shard_cand_row(blockIdx.x, zmax_g[blockIdx.x], scores, ntok, page_idx, n_sel, stride, seq_lens, ptab, maxp, Hq,
                   alpha, cz, cj, cph, ncand, st, sh);
}

template <int IB> __device__ __forceinline__ double sh_pow(double x, double beta) {
    if constexpr (IB == 1) return x;
    else if constexpr (IB == 2) return x * x;
    else if constexpr (IB == 3) return x * x * x;
    else { const double x2 = x * x; return x2 * x2; }
}

// probe point t of [lo, hi] (identical arithmetic on every rank)
__device__ __forceinline__ double probe_x(double lo, double hi, int t) {
    if (t == 0) return lo;
    if (t == kShP - 1) return hi;
    return lo + (hi - lo) * ((double)t / (double)(kShP - 1));
}

// narrow [lo, hi] with the all-reduced partials r[kShP][3] of the current bracket (thread 0)
__device__ __forceinline__ void shard_narrow(ShardRow &s, const double *r) {
    // F decreasing: last probe with F >= 1 and the next one
    int t1 = 0;
    for (int t = 0; t < kShP; ++t) if (r[3 * t] >= 1.0) t1 = t;
    const int t2 = min(t1 + 1, kShP - 1);
    const double nlo = probe_x(s.lo, s.hi, t1), nhi = probe_x(s.lo, s.hi, t2);
    s.cgt_lo = r[3 * t1 + 1];
    s.cge_hi = r[3 * t2 + 2];
    s.lo = nlo;
    s.hi = nhi;
    s.rounds += 1;
    if (s.cgt_lo == s.cge_hi) s.done = 1;                 // no z strictly inside
    else if (!(nhi > nlo) || s.rounds >= 12) s.done = 3;   // fp64 resolution reached
}

// this rank's partials (F, #>, #>=) at the kShP probes of [s.lo, s.hi] into acc (shared):
// warp w evaluates probes w, w + 8, ...: lanes stride over the candidates, fixed-order
// xor-shuffle sums (deterministic); no block barrier per probe.  Ends with a barrier.
template <int IB>
__device__ __forceinline__ void shard_partials(const double *__restrict__ czr, int n, const ShardRow &s, double beta,
                                               double (*acc)[3]) {
    for (int i = threadIdx.x; i < kShP * 3; i += 256) (&acc[0][0])[i] = 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t = warp; t < kShP && !s.done; t += 8) {
        const double x = probe_x(s.lo, s.hi, t);
        double f = 0.0, cg = 0.0, ce = 0.0;
        for (int i = lane; i < n; i += 32) {
            const double z = czr[i];
            const double d = z - x;
            if (d > 0.0) { f += sh_pow<IB>(d, beta); cg += 1.0; }
            if (d >= 0.0) ce += 1.0;
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            f += __shfl_xor_sync(0xffffffffu, f, o);
            cg += __shfl_xor_sync(0xffffffffu, cg, o);
            ce += __shfl_xor_sync(0xffffffffu, ce, o);
        }
        if (lane == 0) { acc[t][0] = f; acc[t][1] = cg; acc[t][2] = ce; }
    }
    __syncthreads();
}

// 4. one multisection round.  red (nullable) = the previous round's all-reduced partials
//    [rows][kShP][3] (F, #>, #>=): narrow the bracket first.  part = this round's partials.
//    Capacity: a rank holding more than kShCap candidates of a row marks the row's first
//    partial F(lo) = +inf; the all-reduce carries it to every rank, which all mark the row
//    done = 4 (NaN out / tau, supp -1, EKV_STATUS_CAPACITY) in the same round -- the ranks'
//    control flow and collectives stay in lockstep.
template <int IB>
__global__ void __launch_bounds__(256) k_shard_probe(const double *__restrict__ cz, const int32_t *__restrict__ ncand,
                                                     double beta, ShardRow *__restrict__ st,
                                                     const double *__restrict__ red, double *__restrict__ part,
                                                     uint32_t *__restrict__ status) {
    __shared__ ShardRow s;
    __shared__ double acc[kShP][3];
    const int row = blockIdx.x;
    if (threadIdx.x == 0) {
        s = st[row];
        if (red && !s.done && red[(size_t)row * kShP * 3] == INFINITY) {
            s.done = 4;                                           // some rank overflowed
            st[row] = s;
            if (status) atomicOr(status, kStatusCapacity);
        } else if (red && !s.done) {
            shard_narrow(s, red + (size_t)row * kShP * 3);
            st[row] = s;
        }
    }
    __syncthreads();
    shard_partials<IB>(cz + (size_t)row * kShCap, min(ncand[row], kShCap), s, beta, acc);
    if (threadIdx.x == 0 && !red && ncand[row] > kShCap) acc[0][0] = INFINITY;   // capacity overflow marker
    __syncthreads();
    for (int i = threadIdx.x; i < kShP * 3; i += 256) part[(size_t)row * kShP * 3 + i] = (&acc[0][0])[i];
}

// host-visible convergence summary: number of rows still open
// (open[0] = rows still open, open[1] = rows marked capacity-overflowed)
static __global__ void k_shard_open(const ShardRow *__restrict__ st, int rows, int *__restrict__ open) {
    __shared__ int sh[9];
    int c = 0, o = 0;
    for (int i = threadIdx.x; i < rows; i += 256) { c += st[i].done == 0; o += st[i].done == 4; }
    c = block_sum_i<256>(c, sh);
    o = block_sum_i<256>(o, sh);
    if (threadIdx.x == 0) { open[0] = c; open[1] = o; }
}

// 5a. power sums of w = z - lo over the local support (block function; result in S_out[0..4]
//     of thread 0 via the shared wp)
__device__ __forceinline__ void shard_sums_row(const double *__restrict__ czr, int n, const ShardRow &s,
                                               double (*wp)[kShSums], double *S_out) {
    double S[kShSums] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (s.done == 1) {
        for (int i = threadIdx.x; i < n; i += 256) {
            const double w = czr[i] - s.lo;
            if (w > 0.0) { double p = 1.0; for (int m = 0; m < kShSums; ++m) { S[m] += p; p *= w; } }
        }
    }
#pragma unroll
    for (int m = 0; m < kShSums; ++m)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) S[m] += __shfl_xor_sync(0xffffffffu, S[m], o);
    if ((threadIdx.x & 31) == 0)
        for (int m = 0; m < kShSums; ++m) wp[threadIdx.x >> 5][m] = S[m];
    __syncthreads();
    if (threadIdx.x < kShSums) {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v += wp[w][threadIdx.x];
        S_out[threadIdx.x] = v;
    }
}
static __global__ void __launch_bounds__(256) k_shard_sums(const double *__restrict__ cz, const int32_t *__restrict__ ncand,
                                                    const ShardRow *__restrict__ st, double *__restrict__ sums) {
    __shared__ double wp[8][kShSums];
    const int row = blockIdx.x;
    const ShardRow s = st[row];
    shard_sums_row(cz + (size_t)row * kShCap, min(ncand[row], kShCap), s, wp, sums + (size_t)row * kShSums);
}

// 5b. tau from the all-reduced power sums: sum_m C(beta, m) (-delta)^(beta - m) S_m = 1
__device__ __forceinline__ double shard_tau_of(const double *S, int ib, const ShardRow &s) {
    double t = NAN;
    if (s.done == 1 && S[0] > 0.0) {
        double d;
        if (ib == 1) d = (S[1] - 1.0) / S[0];
        else if (ib == 2) {
            const double disc = fmax(0.0, S[1] * S[1] - S[0] * (S[2] - 1.0));
            d = (S[1] - sqrt(disc)) / S[0];
        } else {
            // P(d) = sum_m C(b,m) (-d)^(b-m) S_m - 1, decreasing on [0, min w); P(0) >= 0
            d = 0.0;
            for (int it = 0; it < 100; ++it) {
                double P, dP;
                if (ib == 3) {
                    P = S[3] - 3.0 * d * S[2] + 3.0 * d * d * S[1] - d * d * d * S[0] - 1.0;
                    dP = -3.0 * S[2] + 6.0 * d * S[1] - 3.0 * d * d * S[0];
                } else {
                    P = S[4] - 4.0 * d * S[3] + 6.0 * d * d * S[2] - 4.0 * d * d * d * S[1] + d * d * d * d * S[0] - 1.0;
                    dP = -4.0 * S[3] + 12.0 * d * S[2] - 12.0 * d * d * S[1] + 4.0 * d * d * d * S[0];
                }
                if (!(dP < 0.0)) break;
                const double step = -P / dP;
                d += step;
                if (!(fabs(step) > 1e-16 * fmax(1.0, fabs(d)))) break;
            }
        }
        t = s.lo + d;
    }
    return t;
}
static __global__ void k_shard_tau(const double *__restrict__ sums, int ib, ShardRow *__restrict__ st, int rows,
                            double *__restrict__ tau, int32_t *__restrict__ supp) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= rows) return;
    const ShardRow s = st[row];
    const double *S = sums + (size_t)row * kShSums;
    tau[row] = shard_tau_of(S, ib, s);
    if (supp) supp[row] = (s.done == 1) ? (int32_t)S[0] : -1;
}

// 6a. local numerator / denominator of the support {z > lo} (block function): num[kD] fp32
//     and den in shared memory (fixed-order sums over the 8 warps)
template <typename T, int IB>
__device__ __forceinline__ void shard_pv_row(const CacheView &c, int kvh, const double *__restrict__ czr,
                                             const int32_t *__restrict__ cjr, const int32_t *__restrict__ cphr,
                                             int n, const ShardRow &s, double t, double beta,
                                             float (*red)[kD], double *wd, float *num, double *den) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T *Vb = reinterpret_cast<const T *>(c.V);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    double ps = 0.0;
    if (s.done == 1 && t == t) {
        for (int i = warp; i < n; i += 8) {
            const double z = czr[i];
            if (!(z > s.lo)) continue;
            const double d = z - t;
            const double p = d > 0.0 ? sh_pow<IB>(d, beta) : 0.0;
            const int j = cjr[i];
            float vx[4];
            const T *vr = Vb + (((size_t)cphr[i] * c.Hkv + kvh) * kP + (j % kP)) * kD + 4 * lane;
            if constexpr (sizeof(T) == 2) {
                const uint2 w = *reinterpret_cast<const uint2 *>(vr);
                vx[0] = bf_lo(w.x); vx[1] = bf_hi(w.x); vx[2] = bf_lo(w.y); vx[3] = bf_hi(w.y);
            } else {
                const float4 w = *reinterpret_cast<const float4 *>(vr);
                vx[0] = w.x; vx[1] = w.y; vx[2] = w.z; vx[3] = w.w;
            }
            const float pf = (float)p;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = __fmaf_rn(pf, vx[q], acc[q]);
            if (lane == 0) ps += p;
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) red[warp][4 * lane + q] = acc[q];
    if (lane == 0) wd[warp] = ps;
    __syncthreads();
    if (threadIdx.x < kD) {
        float o = 0.f;
        for (int w = 0; w < 8; ++w) o = __fadd_rn(o, red[w][threadIdx.x]);
        num[threadIdx.x] = o;
    }
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v += wd[w];
        *den = v;
    }
}
template <typename T, int IB>
__global__ void __launch_bounds__(256) k_shard_pv(CacheView c, const double *__restrict__ cz,
                                                  const int32_t *__restrict__ cj, const int32_t *__restrict__ cph,
                                                  const int32_t *__restrict__ ncand, const ShardRow *__restrict__ st,
                                                  const double *__restrict__ tau, double beta, int Hq, int G,
                                                  float *__restrict__ num, double *__restrict__ den) {
    __shared__ float red[8][kD];
    __shared__ double wd[8];
    const int row = blockIdx.x, kvh = (row % Hq) / G;
    const size_t o = (size_t)row * kShCap;
    shard_pv_row<T, IB>(c, kvh, cz + o, cj + o, cph + o, min(ncand[row], kShCap), st[row], tau[row], beta, red, wd,
                        num + (size_t)row * kD, den + row);
}

// 6b. out = num / den; NaN rows (overflow / unconverged) stay NaN
static __global__ void k_shard_out(const float *__restrict__ num, const double *__restrict__ den,
                            const double *__restrict__ tau, int rows, float *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * kD) return;
    const int row = i / kD;
    const double t = tau[row];
    out[i] = (t == t) ? (float)((double)num[i] / den[row]) : NAN;
}

}  // namespace ekv

namespace ekv {
// 2'-6'. (in-kernel mode) one CTA per row runs the rest of the step with its collectives
// inside: all-reduce(max) of z_max, local candidates, the multisection rounds (all-reduce(sum)
// of the kShP x 3 partials per round, until the row converges -- identically on every rank),
// all-reduce of the power sums -> tau, all-reduce of numerator / denominator -> out.
template <typename T, int IB>
__global__ void __launch_bounds__(256) k_shard_dsolve(CacheView c, PeerSet P, const float *__restrict__ scores,
                                                      size_t ntok, const int32_t *__restrict__ page_idx,
                                                      const int32_t *__restrict__ n_sel, int stride,
                                                      const uint32_t *__restrict__ rowmax, int Hq, int G,
                                                      float alpha, double beta, double *__restrict__ cz,
                                                      int32_t *__restrict__ cj, int32_t *__restrict__ cph,
                                                      int32_t *__restrict__ ncand, ShardRow *__restrict__ st,
                                                      double *__restrict__ tau_out, int32_t *__restrict__ supp_out,
                                                      float *__restrict__ out, uint32_t *__restrict__ status) {
    __shared__ __align__(16) double acc[kShP][3];
    __shared__ double red[kShP][3];
    __shared__ __align__(16) struct { float num[kD]; double den; double pad; } pv;
    __shared__ __align__(16) double sx[8];
    __shared__ float redv[8][kD];
    __shared__ double wd[8];
    __shared__ double wp[8][kShSums];
    __shared__ ShardRow s;
    __shared__ float zm_sh;
    __shared__ int sh[9];
    const int row = blockIdx.x;
    uint64_t e = *px_ctr(P, row);
    bool dead = false;
    // all-reduce(max) of the row maxima
    if (threadIdx.x == 0) { sx[0] = rowmax[row] ? (double)key2f(rowmax[row]) : -INFINITY; sx[1] = 0.0; }
    __syncthreads();
    px_push(P, row, ++e, sx, 16);
    dead = !px_wait(P, row, e);
    if (threadIdx.x == 0) {
        double m = -INFINITY;
        for (int q = 0; q < P.W; ++q) m = fmax(m, __ldcg(reinterpret_cast<const double *>(px_data(P, P.rk, e, q, row))));
        zm_sh = (float)m;
    }
    __syncthreads();
    shard_cand_row(row, dead ? -INFINITY : zm_sh, scores, ntok, page_idx, n_sel, stride, c.seq_lens, c.page_table,
                   c.maxp, Hq, alpha, cz, cj, cph, ncand, st, sh);
    __syncthreads();
    if (threadIdx.x == 0) s = st[row];
    __syncthreads();
    const int nc = ncand[row], n = min(nc, kShCap);
    const double *czr = cz + (size_t)row * kShCap;
    // multisection rounds
    for (bool first = true; !s.done && !dead; first = false) {
        shard_partials<IB>(czr, n, s, beta, acc);
        if (threadIdx.x == 0 && first && nc > kShCap) acc[0][0] = INFINITY;   // capacity overflow marker
        __syncthreads();
        px_push(P, row, ++e, acc, kShP * 3 * 8);
        if (!px_wait(P, row, e)) { dead = true; break; }
        for (int i = threadIdx.x; i < kShP * 3; i += 256) {
            double v = 0.0;
            for (int q = 0; q < P.W; ++q) v += __ldcg(reinterpret_cast<const double *>(px_data(P, P.rk, e, q, row)) + i);
            (&red[0][0])[i] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (first && red[0][0] == INFINITY) { s.done = 4; atomicOr(status, kStatusCapacity); }
            else shard_narrow(s, &red[0][0]);
        }
        __syncthreads();
    }
    // power sums -> tau
    double t = NAN;
    int supp = -1;
    if (!dead) {
        shard_sums_row(czr, n, s, wp, sx);
        if (threadIdx.x >= kShSums && threadIdx.x < 8) sx[threadIdx.x] = 0.0;
        __syncthreads();
        px_push(P, row, ++e, sx, 64);
        dead = !px_wait(P, row, e);
        if (!dead) {
            double S[kShSums];
#pragma unroll
            for (int m = 0; m < kShSums; ++m) {
                S[m] = 0.0;
                for (int q = 0; q < P.W; ++q) S[m] += __ldcg(reinterpret_cast<const double *>(px_data(P, P.rk, e, q, row)) + m);
            }
            t = shard_tau_of(S, IB, s);
            supp = (s.done == 1) ? (int)S[0] : -1;
        }
        __syncthreads();
    }
    // numerator / denominator -> out
    if (!dead) {
        const size_t o = (size_t)row * kShCap;
        shard_pv_row<T, IB>(c, (row % Hq) / G, czr, cj + o, cph + o, n, s, t, beta, redv, wd, pv.num, &pv.den);
        __syncthreads();
        px_push(P, row, ++e, &pv, (int)sizeof(pv));
        dead = !px_wait(P, row, e);
    }
    if (threadIdx.x < kD) {
        float num = 0.f;
        double den = 0.0;
        if (!dead) {
            for (int q = 0; q < P.W; ++q) {
                const unsigned char *d = px_data(P, P.rk, e, q, row);
                num = __fadd_rn(num, __ldcg(reinterpret_cast<const float *>(d) + threadIdx.x));
                den += __ldcg(reinterpret_cast<const double *>(d + kD * 4));
            }
        }
        out[(size_t)row * kD + threadIdx.x] = (!dead && t == t) ? (float)((double)num / den) : NAN;
    }
    if (threadIdx.x == 0) {
        if (dead) { t = NAN; supp = -1; atomicOr(status, kStatusTimeout); }
        if (tau_out) tau_out[row] = t;
        if (supp_out) supp_out[row] = supp;
        *px_ctr(P, row) = e;
    }
}
}  // namespace ekv

namespace ekv {
// global |C_page| = min(k, global pages) per row
static __global__ void k_shard_nsel(const int32_t *__restrict__ gseq, int Hq, int rows, int k, int32_t *__restrict__ n_sel) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row < rows) n_sel[row] = min(k, n_pages_of(gseq[row / Hq]));
}
}  // namespace ekv
