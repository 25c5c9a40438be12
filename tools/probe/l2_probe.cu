// Per-SM load latency / bandwidth probe: CTAs each read a private contiguous chunk (float4 per
// thread, all loads in flight), data either L2-resident (just written) or cold (HBM).
// Reports the in-kernel duration (globaltimer, first start -> last end) per configuration.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_t0, g_t1;
__global__ void writer(float4 *p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_float4(1.f, 2.f, 3.f, (float)(i & 7));
}
template <int U>
__global__ void reader(const float4 *p, size_t chunk_f4, size_t stride_f4, float *sink) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) atomicMin(&g_t0, t);
    const float4 *q = p + blockIdx.x * stride_f4;
    float acc = 0.f;
    for (size_t base = 0; base < chunk_f4; base += (size_t)U * blockDim.x) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            size_t i = base + threadIdx.x + (size_t)u * blockDim.x;
            v[u] = i < chunk_f4 ? q[i] : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
    }
    if (acc == -1.f) *sink = acc;
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) atomicMax(&g_t1, t);
}
// scattered 64-byte pieces (4 threads per piece), random piece order
__global__ void scatter_reader(const float4 *p, const int *idx, int npieces, float *sink) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) atomicMin(&g_t0, t);
    float acc = 0.f;
    const int *ix = idx + blockIdx.x * npieces;
    for (int e = threadIdx.x; e < npieces * 4; e += blockDim.x) {
        const float4 v = p[(size_t)ix[e >> 2] * 4 + (e & 3)];
        acc += v.x;
    }
    if (acc == -1.f) *sink = acc;
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) atomicMax(&g_t1, t);
}
template <typename F> double timed(F launch) {
    unsigned long long a = ~0ull, b = 0;
    cudaMemcpyToSymbol(g_t0, &a, 8); cudaMemcpyToSymbol(g_t1, &b, 8);
    launch();
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&a, g_t0, 8); cudaMemcpyFromSymbol(&b, g_t1, 8);
    return (b - a) / 1e3;
}
int main() {
    const size_t big = (size_t)512 << 20;   // 512 MB (flush)
    float4 *buf, *flush; float *sink; int *idx;
    cudaMalloc(&buf, (size_t)64 << 20); cudaMalloc(&flush, big); cudaMalloc(&sink, 4);
    cudaMalloc(&idx, sizeof(int) * 256 * 4096);
    int *h = new int[256 * 4096];
    unsigned s = 1;
    for (int i = 0; i < 256 * 4096; ++i) { s = s * 1664525u + 1013904223u; h[i] = (int)(s % (1u << 20)); }  // 64B pieces in 64 MB
    cudaMemcpy(idx, h, sizeof(int) * 256 * 4096, cudaMemcpyHostToDevice);
    const size_t n64 = ((size_t)64 << 20) / 16;
    for (int hot = 1; hot >= 0; --hot) {
        for (int ctas : {32, 128, 256}) {
            for (int thr : {256, 1024}) {
                for (int kb : {8, 32}) {
                    const size_t chunk = (size_t)kb * 1024 / 16;
                    writer<<<592, 512>>>(hot ? buf : flush, hot ? n64 : big / 16);
                    if (!hot) writer<<<592, 512>>>(flush, big / 16);
                    cudaDeviceSynchronize();
                    double us = timed([&] { reader<4><<<ctas, thr>>>(buf, chunk, chunk, sink); });
                    printf("%s ctas=%3d thr=%4d chunk=%2d KB/CTA contiguous: %7.2f us  (%.1f GB/s total)\n", hot ? "L2 " : "HBM", ctas,
                           thr, kb, us, ctas * kb * 1024.0 / us / 1e3);
                }
            }
        }
        for (int ctas : {32, 256}) for (int np : {656, 82}) for (int thr : {256, 1024}) {
            writer<<<592, 512>>>(hot ? buf : flush, hot ? n64 : big / 16);
            if (!hot) writer<<<592, 512>>>(flush, big / 16);
            cudaDeviceSynchronize();
            double us = timed([&] { scatter_reader<<<ctas, thr>>>(buf, idx, np, sink); });
            printf("%s ctas=%3d thr=%4d scattered 64B pieces=%4d/CTA: %7.2f us\n", hot ? "L2 " : "HBM", ctas, thr, np, us);
        }
    }
    return 0;
}
