// Fixed per-launch cost of the ingredients of the product kernels (back-to-back launches).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_empty() {}
__global__ void k_dyn_smem() { extern __shared__ uint8_t s[]; if (threadIdx.x == 999) s[0] = 1; }
__global__ void k_tmem() {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(slot));
}
__global__ void k_tmem_dyn() {
    extern __shared__ uint8_t s[];
    __shared__ uint32_t slot;
    if (threadIdx.x == 999) s[0] = 1;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(slot));
}

template <typename F>
float time_it(F launch, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / reps;
}

int main() {
    const int smem = 151 * 1024;
    cudaFuncSetAttribute(k_dyn_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tmem_dyn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int grid : {3, 144}) {
        printf("grid %3d: empty %.2f us | dyn smem 151KB %.2f us | tmem alloc/dealloc %.2f us | both %.2f us\n", grid,
               time_it([&] { k_empty<<<grid, 128>>>(); }, 2000),
               time_it([&] { k_dyn_smem<<<grid, 128, smem>>>(); }, 2000),
               time_it([&] { k_tmem<<<grid, 128>>>(); }, 2000),
               time_it([&] { k_tmem_dyn<<<grid, 128, smem>>>(); }, 2000));
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
