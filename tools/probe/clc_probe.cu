#include <cstdint>
__global__ void k(int *out) {
    __shared__ __align__(16) uint4 resp;
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int tile = blockIdx.x;
    uint32_t ph = 0;
    while (true) {
        if (threadIdx.x == 0) atomicAdd(out + tile, 1);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
            asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
                         :: "r"((uint32_t)__cvta_generic_to_shared(&resp)), "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        }
        asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(ph) : "memory");
        ph ^= 1;
        uint32_t ok, x;
        asm volatile("{\n\t.reg .pred p;\n\t.reg .b128 h;\n\tld.shared.b128 h, [%2];\n\t"
                     "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, h;\n\tselp.u32 %0, 1, 0, p;\n\t"
                     "clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, h;\n\t}"
                     : "=r"(ok), "=r"(x) : "r"((uint32_t)__cvta_generic_to_shared(&resp)) : "memory");
        __syncthreads();
        if (!ok) break;
        tile = (int)x;
    }
}

#include <cstdio>
__global__ void cnt_k(int *ctas) { if (threadIdx.x == 0) atomicAdd(ctas, 1); }
int main() {
    const int N = 20000;
    int *d; cudaMalloc(&d, N * 4); cudaMemset(d, 0, N * 4);
    k<<<N, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    int *h = new int[N]; cudaMemcpy(h, d, N * 4, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < N; ++i) bad += h[i] != 1;
    printf("clc probe: %s, tiles wrong: %d of %d\n", cudaGetErrorString(e), bad, N);
    return bad != 0;
}
