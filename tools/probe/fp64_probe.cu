// Throughput probe: fp64 DFMA, F2F.F64.F32 conversion, fp32 FFMA, match.any, shared atomics.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_probe tools/probe/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double *o, int n) {
    double a = threadIdx.x * 1e-3, b = 1.0000001, c0 = 0.5, c1 = 0.25, c2 = 0.125, c3 = 0.0625;
    for (int i = 0; i < n; ++i) { c0 = fma(c0, b, a); c1 = fma(c1, b, a); c2 = fma(c2, b, a); c3 = fma(c3, b, a); }
    o[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3;
}
__global__ void k_ffma(float *o, int n) {
    float a = threadIdx.x * 1e-3f, b = 1.0000001f, c0 = 0.5f, c1 = 0.25f, c2 = 0.125f, c3 = 0.0625f;
    for (int i = 0; i < n; ++i) { c0 = fmaf(c0, b, a); c1 = fmaf(c1, b, a); c2 = fmaf(c2, b, a); c3 = fmaf(c3, b, a); }
    o[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3;
}
__global__ void k_cvt(double *o, int n) {
    float f0 = threadIdx.x * 1e-3f, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
    double s = 0;
    for (int i = 0; i < n; ++i) {
        s += (double)f0; s += (double)f1; s += (double)f2; s += (double)f3;
        f0 += 1.0f; f1 += 1.0f; f2 += 1.0f; f3 += 1.0f;
    }
    o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_match(unsigned *o, int n) {
    unsigned v = threadIdx.x & 3, acc = 0;
    for (int i = 0; i < n; ++i) { acc += __match_any_sync(0xffffffffu, v); v = (v * 1664525u + acc) & 7; }
    o[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_satom(unsigned *o, int n) {
    __shared__ unsigned h[256];
    h[threadIdx.x & 255] = 0; __syncthreads();
    for (int i = 0; i < n; ++i) atomicAdd(&h[(i * 7) & 255], 1u);   // all lanes same address
    __syncthreads();
    o[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x & 255];
}
template <typename K, typename T> void run(const char *name, K k, int blocks, int threads, int n, double ops_per_iter) {
    T *o; cudaMalloc(&o, sizeof(T) * blocks * threads);
    k<<<blocks, threads>>>(o, 10); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<<<blocks, threads>>>(o, n); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double lane_ops = (double)blocks * threads * n * ops_per_iter;
    printf("%-8s blocks=%4d threads=%4d : %8.3f ms  %10.2f G lane-ops/s  %8.2f lane-ops/clk/SM(1.965GHz,148)\n", name, blocks,
           threads, ms, lane_ops / ms / 1e6, lane_ops / (ms * 1e-3) / 1.965e9 / 148);
    cudaFree(o);
}
int main() {
    for (int th : {32, 1024}) {
        run<decltype(&k_dfma), double>("dfma", k_dfma, 148, th, 4096, 4);
        run<decltype(&k_ffma), float>("ffma", k_ffma, 148, th, 4096, 4);
        run<decltype(&k_cvt), double>("cvt+dadd", k_cvt, 148, th, 4096, 4);
        run<decltype(&k_match), unsigned>("match", k_match, 148, th, 4096, 1);
        run<decltype(&k_satom), unsigned>("satom", k_satom, 148, th, 4096, 1);
    }
    return 0;
}
