// Micro test: cycles per tcgen05.mma (f16, SS mode, operands resident in smem, no TMA) for the
// shapes of the few-tile / small-n kernels, one CTA per SM:
//   * a chain of MMAs into ONE accumulator vs the same MMAs alternating between TWO accumulators
//     (is a dependent accumulation chain latency-bound at small N?)
//   * with an mbarrier commit + wait after every 4 MMAs (the ring handshake of the 1-CTA kernel)
//     or after every MMA group of a chain step (the small-n kernel's per-product wait)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_chain tools/micro/mma_chain.cu
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2507_09165_b200/csrc/ptx.cuh"

using namespace psd;

// kAcc accumulators (MMA i of a group goes to accumulator i % kAcc); kWait: commit + wait after
// every group of kGroup MMAs (unrolled, descriptors precomputed as in the product kernels)
template <int M, int N, int kGroup, int kAcc, bool kWait>
__global__ void __launch_bounds__(128, 1) chain_kernel(int iters, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    // operands: zeros are fine for timing
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1);
        ptx::fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) ptx::tmem_alloc<512>(slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x < 32 && ptx::elect_one()) {
        constexpr uint32_t idesc = ptx::make_idesc(0, M, N);
        const uint64_t ad = ptx::smem_desc_sw128_kmajor(ptx::smem_u32(smem));
        const uint64_t bd = ptx::smem_desc_sw128_kmajor(ptx::smem_u32(smem + 32 * 1024));
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; it += kGroup) {
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
                const uint32_t d = tmem + static_cast<uint32_t>((k % kAcc) * 128);
                ptx::mma_f16(d, ad + ((k & 3) * 2), bd + ((k & 3) * 2), idesc, (it | k) >= kAcc ? 1u : 0u);
            }
            if (kWait) {
                ptx::mma_commit(bar);
                ptx::mbar_wait(bar, ph);
                ph ^= 1;
            }
        }
        ptx::mma_commit(bar);
        ptx::mbar_wait(bar, ph);
        const long long t1 = clock64();
        atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

template <int M, int N, int kGroup, int kAcc, bool kWait>
void run(int grid, int iters) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 64 * 1024 + 2048;
    auto k = chain_kernel<M, N, kGroup, kAcc, kWait>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, 128, smem>>>(iters, d);    // warm-up
    cudaMemset(d, 0, 8);
    k<<<grid, 128, smem>>>(iters, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    printf("M=%3d N=%3d grid %3d  %d acc  group %2d %s: %7.1f cycles per MMA %s\n", M, N, grid, kAcc, kGroup,
           kWait ? "+wait" : "     ", static_cast<double>(c) / grid / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    const int iters = 4096;
    for (int grid : {1, 148}) {
        run<128, 64, 4, 1, false>(grid, iters);
        run<128, 64, 4, 2, false>(grid, iters);
        run<128, 64, 4, 1, true>(grid, iters);
        run<128, 64, 4, 2, true>(grid, iters);
        run<128, 64, 8, 1, true>(grid, iters);
        run<128, 64, 8, 2, true>(grid, iters);
        run<128, 128, 4, 1, false>(grid, iters);
        run<128, 128, 4, 1, true>(grid, iters);
        run<128, 256, 4, 1, false>(grid, iters);
        run<64, 64, 8, 1, false>(grid, iters);
        run<64, 64, 8, 2, false>(grid, iters);
        run<64, 64, 8, 2, true>(grid, iters);
        run<64, 64, 8, 1, true>(grid, iters);
        run<64, 128, 8, 1, false>(grid, iters);
    }
    return 0;
}
