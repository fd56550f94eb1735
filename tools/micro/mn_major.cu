// Micro test: tcgen05.mma with an MN-major (transposed) SW128 operand loaded by TMA as two
// 64x64 boxes -- which LBO / SBO the smem descriptor needs.  D[m][n] = sum_k A[m][k] B[n][k] with
// A given transposed in global memory (At[k][m]); B K-major.  Prints the max error per variant.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2507_09165_b200/csrc/ptx.cuh"

using namespace psd;

__device__ void wait_bounded(uint64_t* bar, uint32_t ph, int tag, float* out) {
    const unsigned long long t0 = ptx::globaltimer();
    while (!ptx::mbar_try_wait(bar, ph)) {
        if (ptx::globaltimer() - t0 > 200000000ull) { if (out) out[0] = -1000.0f - tag; asm volatile("trap;"); }
    }
}

__global__ void __launch_bounds__(128) kern(const __grid_constant__ CUtensorMap mAt, const __grid_constant__ CUtensorMap mB,
                                            float* out, uint32_t lbo, uint32_t sbo, int a_mn, int b_mn,
                                            const __grid_constant__ CUtensorMap mBt) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = ptx::align_smem_1024(raw);
    uint8_t* sA = smem;             // 16 KB
    uint8_t* sB = smem + 16384;     // 16 KB
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint64_t* mbar = bar + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::mbar_init(mbar, 1); ptx::fence_barrier_init(); }
    if (warp == 0) ptx::tmem_alloc<128>(tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(bar, 32768);
        if (a_mn) {   // At rows k 0..63, cols m 0..63 and 64..127
            ptx::tma_load_2d(sA, &mAt, bar, 0, 0, ptx::policy_evict_first());
            ptx::tma_load_2d(sA + 8192, &mAt, bar, 64, 0, ptx::policy_evict_first());
        }
        if (b_mn) {
            ptx::tma_load_2d(sB, &mBt, bar, 0, 0, ptx::policy_evict_first());
            ptx::tma_load_2d(sB + 8192, &mBt, bar, 64, 0, ptx::policy_evict_first());
        } else {
            ptx::tma_load_2d(sB, &mB, bar, 0, 0, ptx::policy_evict_first());
            ptx::tma_load_2d(sB + 8192, &mB, bar, 0, 64, ptx::policy_evict_first());
        }
        wait_bounded(bar, 0, 1, out);
        ptx::tc_fence_after();
        const uint32_t idesc = ptx::make_idesc(0, 128, 128) | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u);
        for (int k = 0; k < 4; ++k) {
            uint64_t ad, bd;
            auto mn_desc = [&](uint32_t base) {
                uint64_t d = ptx::smem_desc_sw128_kmajor(base + k * 2048);   // 16 K-rows of 128 B
                d &= ~((uint64_t(0x3FFF) << 16) | (uint64_t(0x3FFF) << 32));
                d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
                d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
                return d;
            };
            ad = a_mn ? mn_desc(ptx::smem_u32(sA)) : ptx::smem_desc_sw128_kmajor(ptx::smem_u32(sA) + k * 32);
            bd = b_mn ? mn_desc(ptx::smem_u32(sB)) : ptx::smem_desc_sw128_kmajor(ptx::smem_u32(sB) + k * 32);
            ptx::mma_f16(tmem, ad, bd, idesc, k != 0);
        }
        ptx::mma_commit(mbar);
    }
    __syncwarp();
    wait_bounded(mbar, 0, 2, out);
    ptx::tc_fence_after();
    for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + (uint32_t(warp * 32) << 16) + c0, r);
        ptx::tmem_ld_wait();
        for (int i = 0; i < 32; ++i) out[(warp * 32 + (threadIdx.x & 31)) * 128 + c0 + i] = __uint_as_float(r[i]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc<128>(tmem); }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int M = 128, N = 128, K = 64;
    std::vector<__half> At(K * M), B(N * K), Bt(K * N);
    std::vector<float> A(M * K), Bf(N * K);
    srand(1);
    for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) { float v = (rand() % 17 - 8) / 8.0f; A[m * K + k] = v; At[k * M + m] = __float2half(v); }
    for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) { float v = (rand() % 13 - 6) / 4.0f; Bf[n * K + k] = v; B[n * K + k] = __float2half(v); Bt[k * N + n] = __float2half(v); }
    std::vector<__half> Ak(M * K);
    for (int i = 0; i < M * K; ++i) Ak[i] = __float2half(A[i]);
    __half *dAt, *dB, *dBt, *dAk; float* dO;
    cudaMalloc(&dAt, K * M * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dBt, K * N * 2); cudaMalloc(&dAk, M * K * 2); cudaMalloc(&dO, M * N * 4);
    cudaMemcpy(dAt, At.data(), K * M * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dBt, Bt.data(), K * N * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dAk, Ak.data(), M * K * 2, cudaMemcpyHostToDevice);
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    auto mk = [&](CUtensorMap* m, void* base, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br) {
        cuuint64_t dims[2] = {cols, rows}; cuuint64_t str[1] = {cols * 2}; cuuint32_t box[2] = {bc, br}; cuuint32_t es[2] = {1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap mAt, mB, mBt, mAk;
    mk(&mAt, dAt, M, K, 64, 64);    // At: K rows x M cols, box 64 x 64
    mk(&mB, dB, K, N, 64, 64);      // B: N rows x K cols, box 64 cols x 64 rows
    mk(&mBt, dBt, N, K, 64, 64);
    mk(&mAk, dAk, K, M, 64, 64);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
    std::vector<float> ref(M * N);
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * Bf[n * K + k]; ref[m * N + n] = (float)s; }
    std::vector<float> o(M * N);
    uint32_t lbos[] = {8192, 1024, 16, 2048, 128};
    uint32_t sbos[] = {1024, 8192, 2048, 128};
    for (int amn = 1; amn >= 0; --amn) for (int bmn = 0; bmn <= 1; ++bmn) {
        if (!amn && !bmn) continue;
        for (uint32_t lbo : lbos) for (uint32_t sbo : sbos) {
            printf("run a_mn %d b_mn %d lbo %u sbo %u ... ", amn, bmn, lbo, sbo); fflush(stdout);
            cudaMemset(dO, 0, M * N * 4);
            kern<<<1, 128, 40960>>>(mAt, mB, dO, lbo, sbo, amn, bmn, mBt);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("a_mn %d b_mn %d lbo %u sbo %u: %s\n", amn, bmn, lbo, sbo, cudaGetErrorString(e)); return 1; }
            cudaMemcpy(o.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
            double err = 0; for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(o[i] - ref[i]));
            printf("max err %g\n", err); fflush(stdout);
        }
    }
    return 0;
}
