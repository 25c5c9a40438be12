// shard.cu -- sequence-sharded decode: host orchestration of the
// kernels_shard.cuh kernels and the caller's collectives.
#include <algorithm>
#include <cmath>
#include "host.h"
#include "kernels_shard.cuh"

using namespace ekvh;

namespace {
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
    S.open = take(8);
    S.total = o;
    return S;
}

// in-kernel collectives (N2): payload bytes per (parity, sender, row) and buffer bytes
uint32_t peer_pay(int kc) {
    size_t p = std::max<size_t>({(size_t)8 * kc, (size_t)kShP * 3 * 8, (size_t)kD * 4 + 16, 64});
    return (uint32_t)((p + 15) & ~(size_t)15);
}
size_t peer_bytes(int rows, int world, int kc) {
    const size_t hdr = ((size_t)8 * rows * (1 + world) + 255) & ~(size_t)255;
    return hdr + (size_t)2 * world * rows * peer_pay(kc);
}

ekv_status comm_allreduce(const ekv_comm *cm, void *buf, size_t count, int dtype, int op, cudaStream_t st) {
    if (cm->world <= 1) return EKV_OK;
    if (cm->allreduce(buf, count, dtype, op, cm->user, st) != 0) return fail(EKV_ERR_COMM, "allreduce callback failed");
    return EKV_OK;
}
// the step with in-kernel collectives (N2): no callback, no host synchronisation
ekv_status decode_sharded_dev(const ekv_cache *cache, const CacheView &v, const Layout &L, const ShardLayout &S,
                              const PeerSet &P, const int32_t *global_seq_lens, const void *q, int Hq,
                              const ekv_select_params *sel, const ekv_attn_params *attn, int ib, double beta,
                              float *out, ekv_decode_stats *stats, void *workspace, cudaStream_t st) {
    const int rows = P.rows, Gq = Hq / cache->n_kv_heads, maxp = cache->max_pages_per_seq;
    float *box = at<float>(workspace, L.box);
    int32_t *pi = at<int32_t>(workspace, L.page_idx);
    int32_t *ns = at<int32_t>(workspace, L.n_sel);
    uint32_t *um = at<uint32_t>(workspace, L.umask);
    uint32_t *status = at<uint32_t>(workspace, L.status);
    // (local box scores and local top-k already enqueued by the caller)
    k_shard_pack_push<<<rows, 256, 0, st>>>(box, maxp, pi, ns, L.cap, S.kc, P);
    EKV_TRY(check_launch("k_shard_pack_push"));
    k_shard_merge<<<rows, kShMergeNT, 0, st>>>(nullptr, nullptr, rows, S.kc, sel->k_pages, P.rk, P.W, global_seq_lens,
                                               pi, ns, L.cap, Hq, Gq, um, L.W, P, status);
    EKV_TRY(check_launch("k_shard_merge"));
    float *scores = at<float>(workspace, L.scores);
    uint32_t *rowmax = at<uint32_t>(workspace, L.rowmax);
    EKV_TRY(launch_scores(v, q, Hq, um, L.W, pi, ns, L.cap, scores, rowmax, 0, st));
    double *cz = at<double>(workspace, S.cz);
    int32_t *cj = at<int32_t>(workspace, S.cj), *cph = at<int32_t>(workspace, S.cph), *nc = at<int32_t>(workspace, S.ncand);
    ShardRow *rst = at<ShardRow>(workspace, S.rowst);
    double *tau = (stats && stats->tau) ? stats->tau : at<double>(workspace, S.tau);
    int32_t *supp = stats ? stats->supp_count : nullptr;
    auto solve = [&](auto tag) {
        using T = decltype(tag);
#define EKV_DSOLVE(IB) k_shard_dsolve<T, IB><<<rows, 256, 0, st>>>(v, P, scores, (size_t)maxp * kP, pi, ns, L.cap, rowmax, \
                                                                    Hq, Gq, attn->alpha, beta, cz, cj, cph, nc, rst, tau, \
                                                                    supp, out, status)
        switch (ib) {
        case 1: EKV_DSOLVE(1); break;
        case 2: EKV_DSOLVE(2); break;
        case 3: EKV_DSOLVE(3); break;
        default: EKV_DSOLVE(4); break;
        }
#undef EKV_DSOLVE
    };
    if (cache->dtype == EKV_BF16) solve(__nv_bfloat16());
    else solve(0.0f);
    EKV_TRY(check_launch("k_shard_dsolve"));
    if (stats && stats->n_sel) {
        k_shard_nsel<<<(rows + 127) / 128, 128, 0, st>>>(global_seq_lens, Hq, rows, sel->k_pages, stats->n_sel);
        EKV_TRY(check_launch("k_shard_nsel"));
    }
    return EKV_OK;
}
}  // namespace

extern "C" {

size_t entmaxkv_peer_buffer_size(const ekv_cache *local, int32_t n_q_heads, const ekv_select_params *sel,
                                 int32_t world) {
    if (check_cache(local, n_q_heads) != EKV_OK || world < 1 || world > kMaxPeers) return 0;
    return peer_bytes(local->batch * n_q_heads, world, sel_cap(local, sel));
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
    EKV_CALL("entmaxkv_decode_sharded");
    EKV_TRY(check_cache(cache, n_q_heads));
    EKV_TRY(check_attn(attn));
    EKV_TRY(check_sel(sel, attn->alpha));
    if (!q || !out || !workspace || !comm || !global_seq_lens) return fail(EKV_ERR_INVALID_ARG, "NULL argument");
    EKV_TRY(check_q(q));
    const bool dev = comm->peers[0] != nullptr;     // in-kernel collectives (N2)
    if (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world ||
        (!dev && comm->world > 1 && (!comm->allreduce || !comm->allgather)))
        return fail(EKV_ERR_INVALID_ARG, "bad communicator (rank %d, world %d)", comm->rank, comm->world);
    if (dev) {
        if (comm->world > kMaxPeers) return fail(EKV_ERR_UNSUPPORTED, "in-kernel collectives: world %d > %d", comm->world, kMaxPeers);
        for (int r = 0; r < comm->world; ++r)
            if (!comm->peers[r]) return fail(EKV_ERR_INVALID_ARG, "in-kernel collectives: peers[%d] is NULL", r);
    }
    if (sel->policy != EKV_TOPK || attn->transform != EKV_ENTMAX)
        return fail(EKV_ERR_UNSUPPORTED, "sharded decode supports top-k selection with entmax");
    const double beta = 1.0 / ((double)attn->alpha - 1.0);
    const int ib = (std::fabs(beta - std::rint(beta)) < 1e-9 && beta <= 4.5 && beta >= 0.5) ? (int)std::rint(beta) : 0;
    if (ib < 1 || ib > 4)
        return fail(EKV_ERR_UNSUPPORTED, "sharded decode needs integer beta = 1/(alpha-1) in {1,2,3,4} (alpha=%g)",
                    (double)attn->alpha);
    const int W = comm->world, rk = comm->rank;
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
    EKV_TRY(launch_score(v, q, n_q_heads, EKV_SCORE_BOX, box, nullptr, nullptr, nullptr, 0, st));
    EKV_TRY(launch_topk(box, cache->batch, n_q_heads, maxp, cache->seq_lens, sel->k_pages, pi, ns, L.cap, Gq,
                        UnionOut{nullptr, 0}, st));
    PeerSet P;
    memset(&P, 0, sizeof(P));
    if (dev) {
        for (int r = 0; r < W; ++r) P.buf[r] = static_cast<unsigned char *>(comm->peers[r]);
        P.W = W; P.rk = rk; P.rows = rows; P.pay = peer_pay(S.kc);
        return decode_sharded_dev(cache, v, L, S, P, global_seq_lens, q, n_q_heads, sel, attn, ib, beta, out, stats,
                                  workspace, st);
    }
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
                                               n_q_heads, Gq, um, L.W, P, at<uint32_t>(workspace, L.status));
    EKV_TRY(check_launch("k_shard_merge"));
    // 2. K scores of the local share, global z_max
    float *scores = at<float>(workspace, L.scores);
    uint32_t *rowmax = at<uint32_t>(workspace, L.rowmax);
    EKV_TRY(launch_scores(v, q, n_q_heads, um, L.W, pi, ns, L.cap, scores, rowmax, 0, st));
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
    uint32_t *status = at<uint32_t>(workspace, L.status);
    auto probe = [&](const double *red) -> ekv_status {
        switch (ib) {
        case 1: k_shard_probe<1><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part, status); break;
        case 2: k_shard_probe<2><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part, status); break;
        case 3: k_shard_probe<3><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part, status); break;
        default: k_shard_probe<4><<<rows, 256, 0, st>>>(cz, nc, beta, rst, red, part, status); break;
        }
        return check_launch("k_shard_probe");
    };
    EKV_TRY(probe(nullptr));
    // adaptive (fixed_rounds = 0): stop once every row has converged, one small device->host read
    // per round from the second on; fixed_rounds = R: exactly R rounds, no host read (rows that
    // converge early idle), so the whole step can be captured in a CUDA graph.  12 rounds of
    // 63-way multisection exhaust fp64 (R20), so R >= 12 always converges.
    const int fixed = comm->fixed_rounds;
    int overflow = 0;
    for (int round = 0; round < (fixed > 0 ? fixed : 13); ++round) {
        EKV_TRY(comm_allreduce(comm, part, (size_t)rows * kShP * 3, 1, 0, st));
        EKV_TRY(probe(part));
        if (fixed > 0 || round < 1) continue;   // two rounds (12 bits) before the first check
        k_shard_open<<<1, 256, 0, st>>>(rst, rows, openp);
        EKV_TRY(check_launch("k_shard_open"));
        int open[2] = {0, 0};
        if (cudaMemcpyAsync(open, openp, 2 * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(EKV_ERR_CUDA, "round sync: %s", cudaGetErrorString(cudaGetLastError()));
        overflow = open[1];
        if (open[0] == 0) break;
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
    if (overflow > 0)   // every rank finished the step's collectives; the rows are NaN on all of them
        return fail(EKV_ERR_CAPACITY, "%d row(s) exceed %d candidates per rank (NaN out/tau, supp -1)", overflow, kShCap);
    return EKV_OK;
}

}  // extern "C"
