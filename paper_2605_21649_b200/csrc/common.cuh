// common.cuh -- device helpers for libentmaxkv (sm_100a).
// Numerics follow DESIGN.md section 2 (R1 canonical dot16x8, R5 metadata, R9 support).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include "types.cuh"

namespace ekv {

__device__ __forceinline__ int n_pages_of(int L) { return (L + kP - 1) / kP; }

// union mark of one selected page: bit g of the page's byte (fire-and-forget atomic)
__device__ __forceinline__ void union_mark(uint32_t *um, int p, int g) {
    atomicOr(um + (p >> 2), 1u << ((p & 3) * 8 + g));
}

// ---------------------------------------------------------------- element access
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
    // 8 consecutive elements starting at p (16-byte aligned) -> fp32 (exact)
    static __device__ __forceinline__ void load8(const __nv_bfloat16 *p, float (&x)[8]) {
        uint4 v = *reinterpret_cast<const uint4 *>(p);
        x[0] = bf_lo(v.x); x[1] = bf_hi(v.x); x[2] = bf_lo(v.y); x[3] = bf_hi(v.y);
        x[4] = bf_lo(v.z); x[5] = bf_hi(v.z); x[6] = bf_lo(v.w); x[7] = bf_hi(v.w);
    }
    static __device__ __forceinline__ void load8_nc(const __nv_bfloat16 *p, float (&x)[8]) {
        uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
        x[0] = bf_lo(v.x); x[1] = bf_hi(v.x); x[2] = bf_lo(v.y); x[3] = bf_hi(v.y);
        x[4] = bf_lo(v.z); x[5] = bf_hi(v.z); x[6] = bf_lo(v.w); x[7] = bf_hi(v.w);
    }
    static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    static __device__ __forceinline__ __nv_bfloat16 from_f(float f) { return __float2bfloat16_rn(f); }
};
template <> struct Elem<float> {
    static __device__ __forceinline__ void load8(const float *p, float (&x)[8]) {
        float4 a = *reinterpret_cast<const float4 *>(p);
        float4 b = *reinterpret_cast<const float4 *>(p + 4);
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
    static __device__ __forceinline__ void load8_nc(const float *p, float (&x)[8]) {
        float4 a = __ldg(reinterpret_cast<const float4 *>(p));
        float4 b = __ldg(reinterpret_cast<const float4 *>(p + 4));
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
    static __device__ __forceinline__ float to_f(float v) { return v; }
    static __device__ __forceinline__ float from_f(float f) { return f; }
};

// ---------------------------------------------------------------- R1: 16-lane reduce-scatter tree
// Each lane of a 16-lane group holds the fma-chain partial of its 8-dim chunk
// c = lane & 15 for G heads.  The tree pairs lanes (c, c^8), (c, c^4), (c, c^2),
// (c, c^1) exactly like a butterfly; instead of reducing every head on every lane,
// each split step keeps half of the heads (reduce-scatter), so G = 4 costs 5
// shuffles instead of 16.  fp32 addition is commutative, so the result of head h is
// bit-identical to the butterfly/oracle tree.
template <int G, int O> struct RS {
    static __device__ __forceinline__ void run(float *v, int lane) {
        if constexpr (G > 1) {
            const bool up = (lane & O) != 0;
#pragma unroll
            for (int i = 0; i < G / 2; ++i) {
                float send = up ? v[i] : v[i + G / 2];
                float keep = up ? v[i + G / 2] : v[i];
                v[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, O));
            }
            if constexpr (O > 1) RS<G / 2, O / 2>::run(v, lane);
        } else {
            v[0] = __fadd_rn(v[0], __shfl_xor_sync(0xffffffffu, v[0], O));
            if constexpr (O > 1) RS<1, O / 2>::run(v, lane);
        }
    }
};
template <int G> __device__ __forceinline__ float rs_reduce16(float (&v)[G], int lane) {
    RS<G, 8>::run(v, lane);
    return v[0];
}
// head index held by `lane` after rs_reduce16<G>
template <int G> __device__ __forceinline__ int rs_head(int lane) {
    int h = 0, n = G;
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        if (n > 1) { if (lane & o) h += n / 2; n >>= 1; }
    }
    return h;
}
// lanes that write (one per head per 16-lane group)
template <int G> __device__ __forceinline__ bool rs_writer(int lane) {
    return (lane & (16 / G - 1)) == 0;
}

// ---------------------------------------------------------------- ordered keys (R3)
__device__ __forceinline__ uint32_t f2key(float f) {
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;             // -0 == +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint32_t ordered_f(float f) { return f2key(f); }
__device__ __forceinline__ float key2f(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(u);
}

// ---------------------------------------------------------------- powers (R9)
__device__ __forceinline__ double powb(double x, double beta, int ib) {
    switch (ib) {
    case 1: return x;
    case 2: return x * x;
    case 3: return (x * x) * x;
    case 4: { double x2 = x * x; return x2 * x2; }
    default: return pow(x, beta);
    }
}
__device__ __forceinline__ double powbm1(double x, double beta, int ib) {  // x^(beta-1)
    switch (ib) {
    case 1: return 1.0;
    case 2: return x;
    case 3: return x * x;
    case 4: return (x * x) * x;
    default: return pow(x, beta - 1.0);
    }
}

// fp32 versions (steering iterations only; never decide support or tau)
__device__ __forceinline__ float powbf(float x, float beta, int ib) {
    switch (ib) {
    case 1: return x;
    case 2: return x * x;
    case 3: return (x * x) * x;
    case 4: { float x2 = x * x; return x2 * x2; }
    default: return __powf(x, beta);
    }
}
__device__ __forceinline__ float powbm1f(float x, float beta, int ib) {
    switch (ib) {
    case 1: return 1.0f;
    case 2: return x;
    case 3: return x * x;
    case 4: return (x * x) * x;
    default: return __powf(x, beta - 1.0f);
    }
}

// ---------------------------------------------------------------- block reductions (deterministic)
template <int NT> __device__ __forceinline__ double block_sum_d(double v, double *sh) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (l < NT / 32) ? sh[l] : 0.0;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (l == 0) sh[0] = r;
    }
    __syncthreads();
    return sh[0];
}
template <int NT> __device__ __forceinline__ void block_sum2_d(double &a, double &b, double *sh) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { sh[2 * w] = a; sh[2 * w + 1] = b; }
    __syncthreads();
    if (w == 0) {
        double x = (l < NT / 32) ? sh[2 * l] : 0.0, y = (l < NT / 32) ? sh[2 * l + 1] : 0.0;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            x += __shfl_xor_sync(0xffffffffu, x, o);
            y += __shfl_xor_sync(0xffffffffu, y, o);
        }
        if (l == 0) { sh[0] = x; sh[1] = y; }
    }
    __syncthreads();
    a = sh[0]; b = sh[1];
}
template <int NT> __device__ __forceinline__ float block_max_f(float v, float *sh) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        float r = (l < NT / 32) ? sh[l] : -INFINITY;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, o));
        if (l == 0) sh[0] = r;
    }
    __syncthreads();
    return sh[0];
}
template <int NT> __device__ __forceinline__ int block_sum_i(int v, int *sh) {
    v = __reduce_add_sync(0xffffffffu, v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        int r = (l < NT / 32) ? sh[l] : 0;
        r = __reduce_add_sync(0xffffffffu, r);
        if (l == 0) sh[0] = r;
    }
    __syncthreads();
    return sh[0];
}
// exclusive block scan of ints; returns exclusive prefix, total via *tot
// the same scan on 64-bit words (used with packed 16-bit count fields)
template <int NT>
__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v, unsigned long long *sh,
                                                                  unsigned long long *tot) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (l >= o) x += y;
    }
    __syncthreads();
    if (l == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long s = (l < NT / 32) ? sh[l] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (l >= o) s += y;
        }
        if (l < NT / 32) sh[l] = s;
    }
    __syncthreads();
    const unsigned long long base = (w > 0) ? sh[w - 1] : 0ull;
    *tot = sh[NT / 32 - 1];
    return base + x - v;
}
// Exclusive block scan with one barrier: warp scans, warp totals published to wb[NT/32], every
// warp sums the lower warps' totals itself.  The caller keeps a barrier between a scan's reads of
// wb and the next write of the same buffer.
template <int NT> __device__ __forceinline__ int block_excl_scan1(int v, int *wb, int *tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    if (lane == 31) wb[w] = x;
    __syncthreads();
    const int wv = lane < NT / 32 ? wb[lane] : 0;
    *tot = __reduce_add_sync(0xffffffffu, wv);
    return __reduce_add_sync(0xffffffffu, lane < w ? wv : 0) + x - v;
}

template <int NT> __device__ __forceinline__ int block_excl_scan(int v, int *sh, int *tot) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (l >= o) x += y;
    }
    __syncthreads();
    if (l == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = (l < NT / 32) ? sh[l] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (l >= o) s += y;
        }
        if (l < NT / 32) sh[l] = s;        // inclusive warp totals
    }
    __syncthreads();
    int base = (w > 0) ? sh[w - 1] : 0;
    *tot = sh[NT / 32 - 1];
    return base + x - v;
}

// ---------------------------------------------------------------- TMA bulk copy + mbarrier (sm_90+/sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
#ifndef EKV_MBAR_HINT
#define EKV_MBAR_HINT 0
#endif
// streaming bulk copy: the source lines are marked evict-first in L2 (data read once per step
// -- page metadata, K tiles -- must not push out what the next kernels re-read: box scores,
// page tables, score rows).  EKV_EF=0 builds plain copies (A/B).
#ifndef EKV_EF
#define EKV_EF 1
#endif
__device__ __forceinline__ void bulk_g2s_stream(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
#if EKV_EF
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
#else
    bulk_g2s(dst, src, bytes, bar);
#endif
}
// bulk L2 prefetch (no shared memory, no completion): warms L2 for a later TMA read
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
#if EKV_MBAR_HINT
    // try_wait with a suspend-time hint (ns): the warp may sleep until the phase completes
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase), "r"((unsigned)EKV_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#endif
}

}  // namespace ekv

namespace ekv {
// ---------------------------------------------------------------- packed fp32x2 FMA (sm_100: FFMA2)
// {a.x*b + c.x, a.y*b + c.y}, each an IEEE fma with round-to-nearest: bit-identical to two
// __fmaf_rn; ptxas folds the broadcast of b into the FFMA2 operand.
__device__ __forceinline__ float2 ffma2(float2 a, float b, float2 c) {
    unsigned long long ra, rb, rc, rd;
    asm("mov.b64 %0, {%1,%2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%1};" : "=l"(rb) : "f"(b));
    asm("mov.b64 %0, {%1,%2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
    float2 d;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}

// bitonic sort of n (power of two) u64 keys in shared memory, ascending; all threads call.
template <int NT> __device__ __forceinline__ void bitonic_sort_u64(unsigned long long *a, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += NT) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long x = a[i], y = a[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}
template <int NT> __device__ __forceinline__ void bitonic_sort_u32_desc(uint32_t *a, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += NT) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t x = a[i], y = a[ixj];
                    const bool up = (i & k) == 0;
                    if ((x < y) == up) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}
__device__ __forceinline__ int next_pow2(int x) { int p = 1; while (p < x) p <<= 1; return p; }
}  // namespace ekv

namespace ekv {
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
}  // namespace ekv

// ---------------------------------------------------------------- programmatic dependent launch
// Kernels of the decode chain are launched with programmatic stream serialisation: a kernel
// lets its successor be scheduled early (launch_dependents) and waits for its predecessor's
// completion and memory (wait) before touching anything the predecessor wrote.  Both are
// no-ops when the launch carries no programmatic dependency.
namespace ekv {
// floor(n / d) for 0 <= n < 2^22, 1 <= d < 2^10 from a precomputed fp32 reciprocal (one
// correction step each way): no integer-division sequence on latency-critical paths
__device__ __forceinline__ int qdiv_small(int n, int d, float inv) {
    int q = __float2int_rz((float)n * inv);
    q += ((q + 1) * d <= n) ? 1 : 0;
    q -= (q * d > n) ? 1 : 0;
    return q;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }
// Every kernel of the decode chain starts with pdl_enter(): it waits for its predecessor (the
// successor is scheduled when this kernel's CTAs exit -- an explicit early trigger was measured
// slower: the successor's resident CTAs took SM slots from this kernel, C4 step 119.7 -> 129.7 us).
// Invariant: a CTA of kernel n starts only after every CTA of kernel n-1 has exited, and n-1
// passed its own wait only after n-2 completed, so a prologue placed BEFORE pdl_enter() may read
// data written two or more launches back (not n-1's).
__device__ __forceinline__ void pdl_enter() { pdl_wait(); }
// Per-kernel early trigger (bit KID of EKV_PDL_TRIG; trace ids): kernels whose grid is one
// partial wave let their successor be launched right away, so its CTAs are resident (waiting
// in pdl_enter) when this grid completes -- the launch latency leaves the critical path.
#ifndef EKV_PDL_TRIG
#define EKV_PDL_TRIG 65   /* append (0) and tau (6): measured 112.3 -> 111.7 us; other kernels slower */
#endif
template <int KID> __device__ __forceinline__ void pdl_trigger() {
    if constexpr (((EKV_PDL_TRIG) >> KID) & 1) pdl_launch();
}
}  // namespace ekv

// ---------------------------------------------------------------- optional in-kernel phase stamps
// Built with -DEKV_STAMPS: block 0 / thread 0 of an instrumented kernel writes %globaltimer
// (ns) at checkpoints into ekv_stamps[kernel_slot][i]; read with entmaxkv_debug_stamps().
namespace ekv {
#ifdef EKV_STAMPS
static __device__ unsigned long long ekv_stamps[8][32];
__device__ __forceinline__ void stamp(int k, int i) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ekv_stamps[k][i] = t;
        ekv_stamps[k][16 + i] = clock64();
    }
}
__device__ __forceinline__ void stamp_if(bool cond, int k, int i) {
    if (cond && blockIdx.x == 0 && blockIdx.y == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ekv_stamps[k][i] = t;
    }
}
// per-CTA timeline of one instrumented kernel (id EKV_CTA_KERNEL: 1 = K-score, 2 = score_pages):
// [0] start, [1] first data, [2] end, [3] count
#ifndef EKV_CTA_KERNEL
#define EKV_CTA_KERNEL 1
#endif
static __device__ unsigned long long ekv_cta[4][1024];
template <int KID> __device__ __forceinline__ void stamp_cta(bool cond, int which) {
    if (KID == EKV_CTA_KERNEL && cond && blockIdx.x < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ekv_cta[which][blockIdx.x] = t;
    }
}
template <int KID> __device__ __forceinline__ void count_cta(bool cond, unsigned long long v) {
    if (KID == EKV_CTA_KERNEL && cond && blockIdx.x < 1024) ekv_cta[3][blockIdx.x] = v;
}
// per-CTA phase times of one kernel (id EKV_PH_KERNEL: 6 = tau_sparse, 2 = topk) and two
// per-CTA counters: ekv_ph[phase][cta] (ns), ekv_phc[which][cta]
#ifndef EKV_PH_KERNEL
#define EKV_PH_KERNEL 6
#endif
static __device__ unsigned long long ekv_ph[8][1024];
static __device__ long long ekv_phc[8][1024];
template <int KID> __device__ __forceinline__ void ph_stamp(int phase) {
    if (KID == EKV_PH_KERNEL && threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ekv_ph[phase][blockIdx.x] = t;
    }
}
template <int KID> __device__ __forceinline__ void ph_stamp_if(bool cond, int phase) {
    if (KID == EKV_PH_KERNEL && cond && blockIdx.x < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ekv_ph[phase][blockIdx.x] = t;
    }
}
template <int KID> __device__ __forceinline__ void ph_count(int which, long long v) {
    if (KID == EKV_PH_KERNEL && (threadIdx.x & 31) == 0 && blockIdx.x < 1024) ekv_phc[which][blockIdx.x] = v;
}
// whole-kernel trace: first CTA start (min) and last CTA end (max, thread 0 of each CTA)
static __device__ unsigned long long ekv_trace[16][2];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
struct TraceScope {
    int k;
    __device__ __forceinline__ explicit TraceScope(int kid) : k(kid) {
        if (threadIdx.x == 0 && threadIdx.y == 0) atomicMin(&ekv_trace[k][0], gtimer());
    }
    __device__ __forceinline__ ~TraceScope() {
        if (threadIdx.x == 0 && threadIdx.y == 0) atomicMax(&ekv_trace[k][1], gtimer());
    }
};
#define EKV_TRACE(kid) ::ekv::TraceScope ekv_trace_scope_(kid)
// host side: every translation unit has its own (static) stamp buffers and registers a
// reader for them; the entmaxkv_debug_* calls merge the readers' results
static void tu_debug_read(int what, void *out, int reset) {
    switch (what) {
    case 0:
        if (reset) {
            unsigned long long init[16][2];
            for (int i = 0; i < 16; ++i) { init[i][0] = ~0ull; init[i][1] = 0ull; }
            cudaMemcpyToSymbol(ekv_trace, init, sizeof(init));
        } else {
            cudaMemcpyFromSymbol(out, ekv_trace, sizeof(ekv_trace));
        }
        break;
    case 1: cudaMemcpyFromSymbol(out, ekv_cta, sizeof(ekv_cta)); break;
    case 2: cudaMemcpyFromSymbol(out, ekv_ph, sizeof(ekv_ph)); break;
    case 3: cudaMemcpyFromSymbol(out, ekv_phc, sizeof(ekv_phc)); break;
    default: cudaMemcpyFromSymbol(out, ekv_stamps, sizeof(ekv_stamps)); break;
    }
}
static struct TuDebugReg { TuDebugReg() { debug_register(&tu_debug_read); } } tu_debug_reg;
#else
#define EKV_TRACE(kid) do {} while (0)
template <int KID> __device__ __forceinline__ void ph_stamp(int) {}
template <int KID> __device__ __forceinline__ void ph_stamp_if(bool, int) {}
template <int KID> __device__ __forceinline__ void ph_count(int, long long) {}
__device__ __forceinline__ void stamp(int, int) {}
__device__ __forceinline__ void stamp_if(bool, int, int) {}
template <int KID> __device__ __forceinline__ void stamp_cta(bool, int) {}
template <int KID> __device__ __forceinline__ void count_cta(bool, unsigned long long) {}
#endif
}  // namespace ekv

namespace ekv {
// Block sum of two doubles with ONE barrier: warp shuffle tree, per-warp partials in a
// double-buffered shared slot (buf[2][2*NW]), then every thread adds the NW partials in
// the same fixed order (deterministic; no second barrier needed before the next call
// because the next call writes the other buffer).
template <int NT> struct BlockRed2 {
    double *buf;   // [2][2 * NT/32]
    int ph;
    __device__ __forceinline__ void sum(double &a, double &b) {
        constexpr int NW = NT / 32;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        double *s = buf + ph * 2 * NW;
        ph ^= 1;
        if ((threadIdx.x & 31) == 0) { s[2 * (threadIdx.x >> 5)] = a; s[2 * (threadIdx.x >> 5) + 1] = b; }
        __syncthreads();
        double x = 0.0, y = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) { x += s[2 * w]; y += s[2 * w + 1]; }
        a = x; b = y;
    }
};
}  // namespace ekv

namespace ekv {
// Block-wide k-th largest of per-thread uint32 keys (CPT slots per thread, 0 = no key):
// MSB-first radix select with 8-bit digits; each round builds a 256-bin shared histogram
// of the digits of the keys that match the prefix found so far (warp-aggregated with
// __match_any_sync), and warp 0 locates the digit holding the k-th key with a suffix scan.
// Returns T* = the k-th largest key; *n_gt = number of keys > T*.  Requires
// 1 <= k <= number of keys.  hist: 256 words of shared memory; sh: >= 2 ints.
template <int NT, int CPT>
__device__ uint32_t block_kth_largest(const uint32_t (&key)[CPT], int k, uint32_t *hist, int *sh, int *n_gt) {
    uint32_t prefix = 0u, pmask = 0u;
    int kk = k, above = 0;
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0u;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const uint32_t x = key[j];
            const bool act = x != 0u && (x & pmask) == prefix;
            if (__ballot_sync(0xffffffffu, act) == 0u) continue;      // warp-uniform skip
            const uint32_t d = act ? ((x >> shift) & 255u) : (256u + lane);
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (act && lane == __ffs(peers) - 1) atomicAdd(&hist[d], (uint32_t)__popc(peers));
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            int v[8], s = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) { v[e] = (int)hist[255 - 8 * lane - e]; s += v[e]; }
            int incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int excl = incl - s;
            int D = -1, cab = 0, cum = excl;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (D < 0 && cum + v[e] >= kk) { D = 255 - 8 * lane - e; cab = cum; }
                cum += v[e];
            }
            const unsigned bm = __ballot_sync(0xffffffffu, D >= 0 && excl < kk);
            const int src = __ffs(bm) - 1;
            D = __shfl_sync(0xffffffffu, D, src);
            cab = __shfl_sync(0xffffffffu, cab, src);
            if (lane == 0) { sh[0] = D; sh[1] = cab; }
        }
        __syncthreads();
        const uint32_t D = (uint32_t)sh[0];
        const int cab = sh[1];
        prefix |= D << shift;
        pmask |= 255u << shift;
        above += cab;
        kk -= cab;
        __syncthreads();
    }
    *n_gt = above;
    return prefix;
}
}  // namespace ekv

namespace ekv {
// fp32 accumulate of a bf16 x bf16 product (sm_100: FHFMA.BF16, half selectors folded):
// both operands widen exactly to fp32 and their product is exact in fp32, so this is
// bit-identical to fmaf(float(a), float(b), c) -- the R1 chain step.
__device__ __forceinline__ float fma_bf16lo(uint32_t a, uint32_t b, float c) {
    unsigned short al, ah, bl, bh;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(al), "=h"(ah) : "r"(a));
    asm("mov.b32 {%0,%1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b));
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(c) : "h"(al), "h"(bl));
    return c;
}
__device__ __forceinline__ float fma_bf16hi(uint32_t a, uint32_t b, float c) {
    unsigned short al, ah, bl, bh;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(al), "=h"(ah) : "r"(a));
    asm("mov.b32 {%0,%1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b));
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(c) : "h"(ah), "h"(bh));
    return c;
}
// PRMT byte select: bytes 0-3 of a, 4-7 of b (selector nibbles in the low 16 bits)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
// packed fp32x2 add (sm_100: FADD2): two independent IEEE round-to-nearest adds
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long ra, rb, rd;
    asm("mov.b64 %0, {%1,%2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    float2 d;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}
}  // namespace ekv

namespace ekv {
// ---------------------------------------------------------------- fp8 e4m3 page bounds (R24, §8(f) N3)
// OCP e4m3 "FN": sign-magnitude byte, bias 7, no infinities, 0x7f/0xff NaN, max finite 448.
// Positive codes 0x00..0x7e are ordered by value, negative codes 0x80..0xfe by magnitude.
__device__ __forceinline__ float e4m3_to_f(uint32_t code) {
    uint32_t h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"((unsigned short)(code & 0xffu)));
    return __half2float(__ushort_as_half((unsigned short)(h2 & 0xffffu)));
}
// round to nearest (saturating to +-448)
__device__ __forceinline__ uint32_t e4m3_rn(float x) {
    unsigned short r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(0.0f), "f"(x));
    return (uint32_t)r & 0xffu;
}
// largest e4m3 value <= x (kmin, rounded down); |x| <= 448 (precondition)
__device__ __forceinline__ uint32_t e4m3_rd(float x) {
    uint32_t c = e4m3_rn(x);
    if (e4m3_to_f(c) > x) {
        const uint32_t mag = c & 0x7fu;
        if (!(c & 0x80u)) c = mag ? c - 1u : 0x81u;     // positive: one step down; +0 -> -2^-9
        else if (mag == 0u) c = 0x81u;                  // -0 -> -2^-9
        else if (mag < 0x7eu) c = c + 1u;               // negative: magnitude one step up
    }
    return c;
}
// smallest e4m3 value >= x (kmax, rounded up); |x| <= 448 (precondition)
__device__ __forceinline__ uint32_t e4m3_ru(float x) {
    uint32_t c = e4m3_rn(x);
    if (e4m3_to_f(c) < x) {
        const uint32_t mag = c & 0x7fu;
        if (c & 0x80u) c = mag > 1u ? c - 1u : 0x00u;   // negative: magnitude one step down (-2^-9 -> 0)
        else if (mag < 0x7eu) c = c + 1u;               // positive / +0: one step up
    }
    return c;
}
// 8 consecutive e4m3 bytes (8-byte aligned, shared memory) -> 8 exact fp32 values
__device__ __forceinline__ void load8_e4m3(const unsigned char *p, float (&x)[8]) {
    const uint2 w = *reinterpret_cast<const uint2 *>(p);
    const uint32_t ws[2] = {w.x, w.y};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t h2;
            asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"((unsigned short)(ws[j] >> (16 * h))));
            const __half2 hh = *reinterpret_cast<const __half2 *>(&h2);
            const float2 f = __half22float2(hh);
            x[4 * j + 2 * h] = f.x;
            x[4 * j + 2 * h + 1] = f.y;
        }
    }
}
}  // namespace ekv

namespace ekv {
// two e4m3 bytes (low 16 bits) -> f16x2 (exact: every e4m3 value is an f16 value; F2FP unpack)
__device__ __forceinline__ uint32_t e4m3x2_to_h2(uint32_t two) {
    uint32_t h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"((unsigned short)(two & 0xffffu)));
    return h2;
}
// fp32 accumulate of an f16 x f16 product (FHFMA, half selectors folded): the operands widen
// exactly and the product is exact in fp32, so this is fmaf(float(a), float(b), c) -- the R1
// chain step.  Used for the e4m3 box path with q converted to f16 when that is exact.
__device__ __forceinline__ float fma_h_lo(uint32_t a, uint32_t b, float c) {
    unsigned short al, ah, bl, bh;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(al), "=h"(ah) : "r"(a));
    asm("mov.b32 {%0,%1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b));
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"(al), "h"(bl));
    return c;
}
__device__ __forceinline__ float fma_h_hi(uint32_t a, uint32_t b, float c) {
    unsigned short al, ah, bl, bh;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(al), "=h"(ah) : "r"(a));
    asm("mov.b32 {%0,%1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b));
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"(ah), "h"(bh));
    return c;
}
// bf16x2 word -> f16x2 word; *exact = both values representable in f16 (|v| in [2^-17, 65504] or 0)
__device__ __forceinline__ uint32_t bf2_to_h2(uint32_t w, bool &exact) {
    const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xffff0000u);
    const __half2 h = __floats2half2_rn(lo, hi);
    const float2 back = __half22float2(h);
    exact = exact && back.x == lo && back.y == hi;
    return *reinterpret_cast<const uint32_t *>(&h);
}
}  // namespace ekv
