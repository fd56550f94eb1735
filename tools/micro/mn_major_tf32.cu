// NEGATIVE RESULT (B200): with kind::tf32 the MN-major bit gives the same wrong product for every
// LBO / SBO tried (max err 13.9 vs 0 for the K-major reference) -- transposed operands are a 16-bit
// feature here, so the tf32 paths keep full (mirrored) operand storage.
// Micro test: tcgen05.mma with an MN-major (transposed) SW128 operand loaded by TMA as two
// 64x64 boxes -- which LBO / SBO the smem descriptor needs.  D[m][n] = sum_k A[m][k] B[n][k] with
// A given transposed in global memory (At[k][m]); B K-major.  Prints the max error per variant.
#include <cuda.h>
#include <cuda_fp16.h>
// TF32 VARIANT: fp32 storage, kind::tf32, K = 32 per load (128 B), 8 per MMA
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
        // A: 128 (M) x 32 (K) fp32 = 16 KB; MN-major: 4 boxes of 32 M x 32 K (4 KB each)
        for (int c = 0; c < 4; ++c) ptx::tma_load_2d(sA + c * 4096, &mAt, bar, 32 * c, 0, ptx::policy_evict_first());
        // B: 128 (N) x 32 (K) K-major: 4 boxes of 32 rows x 32 K
        for (int c = 0; c < 4; ++c) ptx::tma_load_2d(sB + c * 4096, &mB, bar, 0, 32 * c, ptx::policy_evict_first());
        wait_bounded(bar, 0, 1, out);
        ptx::tc_fence_after();
        const uint32_t idesc = ptx::make_idesc(2, 128, 128) | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u);
        for (int k = 0; k < 4; ++k) {
            uint64_t ad, bd;
            auto mn_desc = [&](uint32_t base) {
                uint64_t d = ptx::smem_desc_sw128_kmajor(base + k * 1024);   // 8 K-rows of 128 B
                d &= ~((uint64_t(0x3FFF) << 16) | (uint64_t(0x3FFF) << 32));
                d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
                d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
                return d;
            };
            ad = a_mn ? mn_desc(ptx::smem_u32(sA)) : ptx::smem_desc_sw128_kmajor(ptx::smem_u32(sA) + k * 32);
            bd = b_mn ? mn_desc(ptx::smem_u32(sB)) : ptx::smem_desc_sw128_kmajor(ptx::smem_u32(sB) + k * 32);
            ptx::mma_tf32(tmem, ad, bd, idesc, k != 0);
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
    const int M = 128, N = 128, K = 32;
    std::vector<float> At(K * M), B(N * K), Bt(K * N);
    std::vector<float> A(M * K), Bf(N * K);
    srand(1);
    for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) { float v = (rand() % 17 - 8) / 8.0f; A[m * K + k] = v; At[k * M + m] = v; }
    for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) { float v = (rand() % 13 - 6) / 4.0f; Bf[n * K + k] = v; B[n * K + k] = v; Bt[k * N + n] = v; }
    float *dAt, *dB, *dBt; float* dO;
    cudaMalloc(&dAt, K * M * 4); cudaMalloc(&dB, N * K * 4); cudaMalloc(&dBt, K * N * 4); cudaMalloc(&dO, M * N * 4);
    cudaMemcpy(dAt, At.data(), K * M * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), N * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBt, Bt.data(), K * N * 4, cudaMemcpyHostToDevice);
    void* p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)p;
    auto mk = [&](CUtensorMap* m, void* base, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br) {
        cuuint64_t dims[2] = {cols, rows}; cuuint64_t str[1] = {cols * 4}; cuuint32_t box[2] = {bc, br}; cuuint32_t es[2] = {1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUtensorMap mAt, mB, mBt;
    mk(&mAt, dAt, M, K, 32, 32);    // At: K rows x M cols, box 32 x 32
    mk(&mB, dB, K, N, 32, 32);      // B: N rows x K cols, box 32 cols x 32 rows
    mk(&mBt, dBt, N, K, 32, 32);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
    std::vector<float> ref(M * N);
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < K; ++k) { float a = A[m * K + k], bq = Bf[n * K + k]; s += (double)a * bq; } ref[m * N + n] = (float)s; }
    std::vector<float> o(M * N);
    uint32_t lbos[] = {4096, 1024, 8192};
    uint32_t sbos[] = {1024, 4096};
    for (int amn = 1; amn >= 1; --amn) for (int bmn = 0; bmn <= 0; ++bmn) {
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
