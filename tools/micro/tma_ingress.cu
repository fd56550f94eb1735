// Micro test: L2 -> shared-memory bulk-copy (TMA engine) throughput per SM, one CTA per SM, the
// source resident in L2 (16 MB).  A producer thread keeps a ring of kStages x 24 KB stages in flight
// (cp.async.bulk, 3 x 8 KB per stage, mbarrier complete_tx); a consumer thread waits on each stage
// and frees it at once.  Prints bytes per SM clock per SM and the whole-chip figure, for several grid
// sizes -- is the few-tile product kernel (c3: 72 CTAs, 24 KB per 64-wide K block) bound by what one
// SM can ingest?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_ingress tools/micro/tma_ingress.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2507_09165_b200/csrc/ptx.cuh"

using namespace psd;

constexpr int kChunk = 8192;
constexpr int kStageBytes = 3 * kChunk;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(ptx::smem_u32(dst)), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)) : "memory");
}

template <int kStages>
__global__ void __launch_bounds__(64, 1) ingress_kernel(const uint8_t* __restrict__ src, size_t src_bytes, int iters,
                                                        unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const size_t nchunks = src_bytes / kChunk;
    const long long t0 = clock64();
    if (threadIdx.x == 0) {                      // producer
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            ptx::mbar_wait(&empty[st], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&full[st], kStageBytes);
            for (int c = 0; c < 3; ++c) {
                const size_t chunk = (static_cast<size_t>(blockIdx.x) * 977 + static_cast<size_t>(it) * 3 + c) % nchunks;
                bulk_g2s(smem + st * kStageBytes + c * kChunk, src + chunk * kChunk, kChunk, &full[st]);
            }
        }
    } else if (threadIdx.x == 32) {              // consumer
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            ptx::mbar_wait(&full[st], ph);
            ptx::mbar_arrive(&empty[st]);
        }
        const long long t1 = clock64();
        atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    }
}


// the same with 2D tensor-map loads shaped like the 1-CTA kernel's stage: a 128 x 64 A box (16 KB)
// and a 64 x 64 B box (8 KB), SW128, from a 2048 x 4096 fp16 tensor (16 MB, L2-resident)
template <int kStages, int kBoxes>
__global__ void __launch_bounds__(64, 1) ingress2d_kernel(const __grid_constant__ CUtensorMap mA,
                                                          const __grid_constant__ CUtensorMap mB, int iters,
                                                          unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint64_t pol = ptx::policy_evict_last();
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            ptx::mbar_wait(&empty[st], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&full[st], kStageBytes);
            const int kx = (it % 64) * 64;
            const int row = (blockIdx.x % 16) * 128;
            if (kBoxes == 2) {
                ptx::tma_load_2d(smem + st * kStageBytes, &mA, &full[st], kx, row, pol);
                ptx::tma_load_2d(smem + st * kStageBytes + 16384, &mB, &full[st], kx, (blockIdx.x % 32) * 64, pol);
            } else {                             // kBoxes x (24 KB / kBoxes) boxes of mB's shape
                constexpr int kRowsPer = 24576 / kBoxes / 128;
                for (int q = 0; q < kBoxes; ++q)
                    ptx::tma_load_2d(smem + st * kStageBytes + q * kRowsPer * 128, &mB, &full[st], kx,
                                     (blockIdx.x % 8) * 256 + q * kRowsPer, pol);
            }
        }
    } else if (threadIdx.x == 32) {
        for (int it = 0; it < iters; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (it / kStages) & 1;
            ptx::mbar_wait(&full[st], ph);
            ptx::mbar_arrive(&empty[st]);
        }
        const long long t1 = clock64();
        atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int kStages, int kBoxes>
void run2d(const CUtensorMap& mA, const CUtensorMap& mB, int grid) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = kStages * kStageBytes + 2048;
    cudaFuncSetAttribute(ingress2d_kernel<kStages, kBoxes>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    ingress2d_kernel<kStages, kBoxes><<<grid, 64, smem>>>(mA, mB, iters, d);
    cudaMemset(d, 0, 8);
    ingress2d_kernel<kStages, kBoxes><<<grid, 64, smem>>>(mA, mB, iters, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double per_sm = static_cast<double>(iters) * kStageBytes / (static_cast<double>(c) / grid);
    printf("2D tensor %d boxes stages %d grid %3d: %6.1f B/cycle per SM, %7.0f B/cycle chip %s\n", kBoxes, kStages, grid, per_sm,
           per_sm * grid, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}


// the 1-CTA product kernel's mainloop in isolation: producer thread (2D TMA, A 128 x 64 + B 64 x 64
// per stage), MMA thread (wait full, 4 x tcgen05.mma M=128 N=64 K=16, commit to empty), `iters` K
// blocks; cycles from the first TMA issue to the last MMA's completion
template <int kStages>
__global__ void __launch_bounds__(64, 1) pipe_kernel(const __grid_constant__ CUtensorMap mA,
                                                     const __grid_constant__ CUtensorMap mB, int iters,
                                                     unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_barrier_init();
    }
    if (threadIdx.x >= 32) ptx::tmem_alloc<64>(slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *slot;
    const long long t0 = clock64();
    if (threadIdx.x < 32) {
        if (ptx::elect_one()) {
            const uint64_t pol = ptx::policy_evict_last();
            for (int it = 0; it < iters; ++it) {
                const int st = it % kStages;
                const uint32_t ph = (it / kStages) & 1;
                ptx::mbar_wait(&empty[st], ph ^ 1);
                ptx::mbar_arrive_expect_tx(&full[st], kStageBytes);
                const int kx = (it % 64) * 64;
                ptx::tma_load_2d(smem + st * kStageBytes, &mA, &full[st], kx, (blockIdx.x % 16) * 128, pol);
                ptx::tma_load_2d(smem + st * kStageBytes + 16384, &mB, &full[st], kx, (blockIdx.x % 32) * 64, pol);
            }
        }
        __syncwarp();
    } else {
        if (ptx::elect_one()) {
            constexpr uint32_t idesc = ptx::make_idesc(0, 128, 64);
            for (int it = 0; it < iters; ++it) {
                const int st = it % kStages;
                const uint32_t ph = (it / kStages) & 1;
                ptx::mbar_wait(&full[st], ph);
                ptx::tc_fence_after();
                const uint64_t ad = ptx::smem_desc_sw128_kmajor(ptx::smem_u32(smem + st * kStageBytes));
                const uint64_t bd = ptx::smem_desc_sw128_kmajor(ptx::smem_u32(smem + st * kStageBytes + 16384));
#pragma unroll
                for (int k = 0; k < 4; ++k) ptx::mma_f16(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
                ptx::mma_commit(&empty[st]);
            }
            ptx::mma_commit(done);
            ptx::mbar_wait(done, 0);
            const long long t1 = clock64();
            atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
        }
        __syncwarp();
        ptx::tc_fence_before();
        ptx::tmem_dealloc<64>(tmem);
    }
}

template <int kStages>
void runpipe(const CUtensorMap& mA, const CUtensorMap& mB, int grid, int iters) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = kStages * kStageBytes + 2048;
    cudaFuncSetAttribute(pipe_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    pipe_kernel<kStages><<<grid, 64, smem>>>(mA, mB, iters, d);
    cudaMemset(d, 0, 8);
    pipe_kernel<kStages><<<grid, 64, smem>>>(mA, mB, iters, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("pipeline stages %d grid %3d K blocks %4d: %7.1f cycles per K block (%8.0f total) %s\n", kStages, grid, iters,
           static_cast<double>(c) / grid / iters, static_cast<double>(c) / grid, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

template <int kStages>
void run(const uint8_t* src, size_t bytes, int grid) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = kStages * kStageBytes + 2048;
    cudaFuncSetAttribute(ingress_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    ingress_kernel<kStages><<<grid, 64, smem>>>(src, bytes, iters, d);
    cudaMemset(d, 0, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    ingress_kernel<kStages><<<grid, 64, smem>>>(src, bytes, iters, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = static_cast<double>(c) / grid;
    const double per_sm = static_cast<double>(iters) * kStageBytes / cyc;
    printf("stages %d grid %3d: %6.1f B/cycle per SM, %7.0f B/cycle chip, %6.2f TB/s (event) %s\n", kStages, grid, per_sm,
           per_sm * grid, static_cast<double>(iters) * kStageBytes * grid / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    const size_t bytes = 16ull << 20;
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    for (int grid : {1, 148}) run<8>(src, bytes, grid);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(p);
    auto mk = [&](CUtensorMap* m, uint32_t box_rows) {
        cuuint64_t dims[2] = {4096, 2048};
        cuuint64_t str[1] = {4096 * 2};
        cuuint32_t box[2] = {64, box_rows};
        cuuint32_t es[2] = {1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap mA, mB, m64, m32;
    if (mk(&mA, 128) != CUDA_SUCCESS || mk(&mB, 64) != CUDA_SUCCESS || mk(&m64, 64) != CUDA_SUCCESS ||
        mk(&m32, 32) != CUDA_SUCCESS) { printf("encode failed\n"); return 1; }
    for (int grid : {1, 72, 148})
        for (int iters : {16, 2000}) {
            runpipe<5>(mA, mB, grid, iters);
            runpipe<8>(mA, mB, grid, iters);
        }
    for (int grid : {1, 72, 148}) {
        run2d<5, 2>(mA, mB, grid);
        run2d<8, 2>(mA, mB, grid);
        run2d<5, 3>(mA, m64, grid);
        run2d<8, 3>(mA, m64, grid);
        run2d<5, 6>(mA, m32, grid);
        run2d<8, 6>(mA, m32, grid);
    }
    return 0;
}
