// sym_gemm.cu -- symmetric product C = alpha * (A B) + beta * D on sm_100a tensor cores.
//
// Every product of the composite filter (Algorithm 2) multiplies two
// commuting symmetric matrices (powers/polynomials of the same X), so
// C is symmetric: only upper tiles (I <= J) are computed and each is stored twice
// (direct + transposed), which halves the MMA work and makes C exactly symmetric.
// A and B are symmetric, so both operands are read as row panels ("K-major"):
// A tile = rows I*128.., B^T tile = rows J*128.. of B (B^T = B).
//
// Pipeline per CTA (one 128x128 upper tile):
//   warp 0 / 1 elected lane : TMA producer  -> kStages-deep smem ring (mbarrier full/empty)
//   warp 1 / 1 elected lane : tcgen05.mma.cta_group::1 (M=128, N=128) into TMEM
//   warps 0-3               : epilogue  tcgen05.ld -> alpha*acc + beta*D -> mirrored stores
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "epilogue.cuh"
#include "kernels.h"
#include "optraits.cuh"
#include "ptx.cuh"

namespace psd {

namespace {

constexpr int kThreads = 128;
constexpr int kTileBytes = kTile * kBlockKBytes;                 // 16 KB per operand tile
constexpr int kRingBytes1 = 128 * 1024;
template <bool kSplit> struct Ring1 {
    static constexpr int kStageBytes = (kSplit ? 4 : 2) * kTileBytes;   // A, B (+ A_lo, B_lo)
    static constexpr int kStages = kRingBytes1 / kStageBytes;           // 4 or 2
};
constexpr int kSmemBytes = kRingBytes1 + 1024 + 256 + 4 * kEpiWarpSmemBytes;  // ring, align, barriers, staging

__device__ __forceinline__ void upper_tile_coords(int t, int nt, int& I, int& J) {
    // row-major enumeration of {(I, J): 0 <= I <= J < nt}
    int i = 0;
    int rem = t;
    while (rem >= nt - i) { rem -= nt - i; ++i; }
    I = i;
    J = i + rem;
}

template <OpType T, bool kSplit>
__global__ void __launch_bounds__(kThreads, 1)
sym_gemm_kernel(const __grid_constant__ OperandMaps tm, const GemmShape s, const EpiParams e) {
    using Tr = OpTraits<T>;
    constexpr int kStages = Ring1<kSplit>::kStages;
    constexpr int kStageBytes = Ring1<kSplit>::kStageBytes;
    constexpr int kBK = kBlockKBytes / Tr::kBytes;     // K elements per block (64 f16 / 32 tf32)
    constexpr int kUmmaK = 32 / Tr::kBytes;            // K per tcgen05.mma (16 f16 / 8 tf32)
    constexpr uint32_t kIdesc = ptx::make_idesc(Tr::kFmt, kTile, kTile);

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = smem;                                         // stage: A | B | A_lo | B_lo
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes1);
    uint64_t* empty = full + kStages;
    uint64_t* accum_full = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_full + 1);
    uint8_t* epi_smem = smem + kRingBytes1 + 256;                   // 4 x kEpiWarpSmemBytes

    const int warp = threadIdx.x >> 5;
    const int nt = s.npad / kTile;
    const int b = blockIdx.y;
    int I, J;
    upper_tile_coords(blockIdx.x, nt, I, J);

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::tma_prefetch_desc(&tm.a);
            ptx::tma_prefetch_desc(&tm.b);
            for (int i = 0; i < kStages; ++i) {
                ptx::mbar_init(&full[i], 1);
                ptx::mbar_init(&empty[i], 1);
            }
            ptx::mbar_init(accum_full, 1);
            ptx::fence_barrier_init();
        }
        __syncwarp();
    } else if (warp == 1) {
        ptx::tmem_alloc<kTile>(tmem_slot);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_kb = s.npad / kBK;
    const int rowA = b * s.npad + I * kTile;
    const int rowB = b * s.npad + J * kTile;

    if (warp == 0) {
        if (ptx::elect_one()) {
            const uint64_t pol = ptx::policy_evict_last();
            for (int kb = 0; kb < num_kb; ++kb) {
                const int st = kb % kStages;
                const uint32_t ph = (kb / kStages) & 1;
                ptx::mbar_wait(&empty[st], ph ^ 1);
                uint8_t* sa = ring + st * kStageBytes;
                ptx::mbar_arrive_expect_tx(&full[st], kStageBytes);
                ptx::tma_load_2d(sa, &tm.a, &full[st], kb * kBK, rowA, pol);
                ptx::tma_load_2d(sa + kTileBytes, &tm.b, &full[st], kb * kBK, rowB, pol);
                if constexpr (kSplit) {
                    ptx::tma_load_2d(sa + 2 * kTileBytes, &tm.a_lo, &full[st], kb * kBK, rowA, pol);
                    ptx::tma_load_2d(sa + 3 * kTileBytes, &tm.b_lo, &full[st], kb * kBK, rowB, pol);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (ptx::elect_one()) {
            for (int kb = 0; kb < num_kb; ++kb) {
                const int st = kb % kStages;
                const uint32_t ph = (kb / kStages) & 1;
                ptx::mbar_wait(&full[st], ph);
                ptx::tc_fence_after();
                const uint32_t sa = ptx::smem_u32(ring + st * kStageBytes);
                const uint64_t adesc = ptx::smem_desc_sw128_kmajor(sa);
                const uint64_t bdesc = ptx::smem_desc_sw128_kmajor(sa + kTileBytes);
                auto mma = [&](uint64_t a, uint64_t bb, uint32_t accumulate) {
                    if constexpr (T == OpType::TF32)
                        ptx::mma_tf32(tmem_base, a, bb, kIdesc, accumulate);
                    else
                        ptx::mma_f16(tmem_base, a, bb, kIdesc, accumulate);
                };
#pragma unroll
                for (int k = 0; k < kBK / kUmmaK; ++k) {
                    const uint64_t koff = static_cast<uint64_t>((k * 32) >> 4);   // 32 B per K step
                    mma(adesc + koff, bdesc + koff, (kb | k) != 0);
                    if constexpr (kSplit) {
                        const uint64_t alo = ptx::smem_desc_sw128_kmajor(sa + 2 * kTileBytes);
                        const uint64_t blo = ptx::smem_desc_sw128_kmajor(sa + 3 * kTileBytes);
                        mma(adesc + koff, blo + koff, 1u);            // A_hi B_lo
                        mma(alo + koff, bdesc + koff, 1u);            // A_lo B_hi
                    }
                }
                ptx::mma_commit(&empty[st]);
            }
            ptx::mma_commit(accum_full);
        }
        __syncwarp();
    }

    // ------------------------------------------------------------------ epilogue
    ptx::mbar_wait(accum_full, 0);
    ptx::tc_fence_after();

    const int gi0 = I * kTile + warp * 32;          // this warp's first row (TMEM lanes 32w..)
    const bool diag = (I == J);
    float alpha = e.alpha;
    if (e.alpha_dev) alpha *= static_cast<float>(e.alpha_dev[b]);
    uint8_t* wsmem = epi_smem + warp * kEpiWarpSmemBytes;

#pragma unroll 1
    for (int c0 = 0; c0 < kTile; c0 += 32) {
        const int gj0 = J * kTile + c0;
        if (diag && gj0 + 31 < gi0) continue;       // chunk below the diagonal for the whole warp
        uint32_t raw[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + c0, raw);
        ptx::tmem_ld_wait();
        epilogue_chunk<T>(e, alpha, b, s.npad, gi0, gj0, diag, raw, wsmem);
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kTile>(tmem_base);
    }
}

template <OpType T, bool kSplit>
cudaError_t launch_t(const OperandMaps& m, const GemmShape& s, const EpiParams& e, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t err = cudaFuncSetAttribute(sym_gemm_kernel<T, kSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        if (err != cudaSuccess) return err;
        attr_set = true;
    }
    const int nt = s.npad / kTile;
    dim3 grid(nt * (nt + 1) / 2, s.batch);
    sym_gemm_kernel<T, kSplit><<<grid, kThreads, kSmemBytes, stream>>>(m, s, e);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_sym_gemm(OpType t, bool split, const OperandMaps& m, const GemmShape& s, const EpiParams& e,
                            cudaStream_t stream) {
    switch (t) {
        case OpType::F16: return split ? launch_t<OpType::F16, true>(m, s, e, stream)
                                       : launch_t<OpType::F16, false>(m, s, e, stream);
        case OpType::BF16: return split ? launch_t<OpType::BF16, true>(m, s, e, stream)
                                        : launch_t<OpType::BF16, false>(m, s, e, stream);
        case OpType::TF32: return split ? launch_t<OpType::TF32, true>(m, s, e, stream)
                                        : launch_t<OpType::TF32, false>(m, s, e, stream);
    }
    return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ TMA descriptors
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}
}  // namespace

bool make_operand_tmap(CUtensorMap* map, const void* base, OpType t, int npad, int batch) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const int bytes = (t == OpType::TF32) ? 4 : 2;
    const CUtensorMapDataType dt = (t == OpType::F16) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                 : (t == OpType::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(npad), static_cast<cuuint64_t>(npad) * batch};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(npad) * bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBlockKBytes / bytes), static_cast<cuuint32_t>(kTile)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace psd
