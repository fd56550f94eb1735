// small_batch.cu -- batched small-n path (n <= 64): the whole of Algorithm 2 for a
// pair of matrices per CTA iteration, on-chip, HBM touched once for X and once for P.
//
//   * bound + scale in-kernel: a CTA stages the two 64x64 fp32 inputs
//     in smem, reduces ||X||_F per matrix in fp64 (deterministic fixed order) and writes X_0 in
//     the operand format (SW128 K-major fp16, hi/lo for the split path);
//   * every product of the chain is tcgen05.mma.cta_group::1 M=64 N=64 K=16 from smem
//     descriptors into TMEM; the two matrices of the pair use the two half-subpartition
//     interleaves of one 64-column accumulator (lanes 32w+[0,16) and 32w+[16,32)), so one
//     tcgen05.ld 32x32b gives each thread one row of one matrix;
//   * epilogue: alpha*acc + beta*D (D = the rounded operand copy in smem, reading R18), written
//     back in place into the operand slot (the MMA has completed), fence.proxy.async, barrier;
//   * reconstruction P = 1/2 X + 1/2 lambda~ X_0 S: X_0 is re-staged from X, and the
//     result is symmetrised through smem (exact symmetry) and stored to HBM.
// Two CTAs per SM (96 KB smem each) so one CTA's epilogue overlaps the other's MMAs.
#include <cuda_fp16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace psd {

namespace {

constexpr int kN = 64;                  // padded matrix edge
constexpr int kSlotBytes = kN * 128;    // 64 rows x 128 B (fp16), one SW128 atom wide
constexpr int kThreadsS = 256;        // 8 warps: TMEM quadrant = warp & 3, column half = warp >> 2

// byte offset of element (row, col) in a SW128 K-major 64x64 fp16 slot
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
    return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

template <bool kSplit>
struct SmallLayout {
    // per matrix: Z slot, Y slot (hi [+ lo]), U slot (always 16 KB: hi + lo, or fp32 staging)
    static constexpr int kParts = kSplit ? 2 : 1;
    static constexpr int kZ = 0;
    static constexpr int kY = kParts * kSlotBytes;
    static constexpr int kU = 2 * kParts * kSlotBytes;
    static constexpr int kPerMatrix = kU + 2 * kSlotBytes;
    static constexpr int kBytes = 2 * kPerMatrix + 1024 + 256;   // + align slack, barrier, tmem slot, 2x8 partial sums
};

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <bool kSplit, bool kScale = true>
__device__ __forceinline__ void store_row(uint8_t* slot, int row, int half, const float (&v)[32], float s) {
    // hi = rn(v s) [, lo = rn(v s - hi)] into the swizzled slot row, columns [32 half, 32 half + 32)
    // (kScale false: s is already folded into v)
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const int c = 4 * half + cc;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float a = kScale ? v[8 * cc + 2 * h] * s : v[8 * cc + 2 * h];
            const float b = kScale ? v[8 * cc + 2 * h + 1] * s : v[8 * cc + 2 * h + 1];
            const __half2 hh = __floats2half2_rn(a, b);
            hi[h] = *reinterpret_cast<const uint32_t*>(&hh);
            if constexpr (kSplit) {
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(a - hf.x, b - hf.y);
                lo[h] = *reinterpret_cast<const uint32_t*>(&ll);
            }
        }
        *reinterpret_cast<uint4*>(slot + swz(row, c)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        if constexpr (kSplit)
            *reinterpret_cast<uint4*>(slot + kSlotBytes + swz(row, c)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
}

// Exact symmetry of a stored operand: row `row` takes its lower part (col < row) from the
// upper part of the rows above it (reads touch only the upper triangle, writes only the lower).
// Without it the rounding-level antisymmetric part of the products grows like prod_t c_{t,0}
// along the chain (it is not damped by the sign dynamics).
template <bool kSplit>
__device__ __forceinline__ void mirror_lower(uint8_t* slot, int row) {
    for (int c = 0; c < row; ++c) {
        const uint32_t src = static_cast<uint32_t>(c * 128 + ((((row >> 3) ^ (c & 7))) << 4) + (row & 7) * 2);
        const uint32_t dst = static_cast<uint32_t>(row * 128 + ((((c >> 3) ^ (row & 7))) << 4) + (c & 7) * 2);
        *reinterpret_cast<uint16_t*>(slot + dst) = *reinterpret_cast<const uint16_t*>(slot + src);
        if constexpr (kSplit)
            *reinterpret_cast<uint16_t*>(slot + kSlotBytes + dst) = *reinterpret_cast<const uint16_t*>(slot + kSlotBytes + src);
    }
}

// Block version: the 64x64 fp16 part(s) of a slot as 8x8 blocks of 8x8 elements; block (bi, bj),
// bi > bj, becomes the transpose of block (bj, bi); a diagonal block takes its lower triangle from
// its upper triangle.  36 block tasks per matrix part, one per thread (16-byte smem accesses).
__device__ __forceinline__ void mirror_block_task(uint8_t* part, int task) {
    // task -> (bi >= bj): row-major over the lower triangle of the 8 x 8 block grid
    int bi = 0, rem = task;
    while (rem > bi) { rem -= bi + 1; ++bi; }
    const int bj = rem;
    uint16_t blk[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int row = 8 * bj + r;                    // source: block (bj, bi) (upper)
        const uint4 q = *reinterpret_cast<const uint4*>(part + swz(row, bi));
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&q);
#pragma unroll
        for (int c = 0; c < 8; ++c) blk[r][c] = h[c];
    }
    if (bi != bj) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            __align__(16) uint16_t o[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) o[c] = blk[c][r];   // transpose
            *reinterpret_cast<uint4*>(part + swz(8 * bi + r, bj)) = *reinterpret_cast<const uint4*>(o);
        }
    } else {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            __align__(16) uint16_t o[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) o[c] = (c >= r) ? blk[r][c] : blk[c][r];
            *reinterpret_cast<uint4*>(part + swz(8 * bi + r, bj)) = *reinterpret_cast<const uint4*>(o);
        }
    }
}

// The same mirror, four 8x8 blocks per warp instruction: ldmatrix.x4.trans reads upper blocks
// (bj, bi) transposed and stmatrix.x4 writes them as blocks (bi, bj); lanes 8q..8q+7 address the
// rows of block q.  Group g of a 64x64 part: g < 7 the off-diagonal blocks 4g..4g+3 (row-major over
// the strict lower block triangle), g = 7, 8 the diagonal blocks 4(g-7)..+3, which merge their
// plain and transposed loads (upper part kept).  The 8 row addresses of a block hit 8 distinct
// 16-byte chunks of the SW128 rows: conflict-free.  Fragment of lane t: row t/4, columns 2(t%4)+{0,1}.
constexpr int kMirrorGroups = 9;
__device__ __forceinline__ void mirror_group_warp(uint8_t* part, int g, int lane) {
    const int q = lane >> 3, rr = lane & 7;
    int bi, bj;
    if (g < 7) {
        const int k = 4 * g + q;                       // 0..27
        bi = 1;
        while (k >= bi * (bi + 1) / 2) ++bi;
        bj = k - bi * (bi - 1) / 2;
    } else {
        bi = bj = 4 * (g - 7) + q;
    }
    const uint32_t src = ptx::smem_u32(part + swz(8 * bj + rr, bi));
    const uint32_t dst = ptx::smem_u32(part + swz(8 * bi + rr, bj));
    uint32_t t[4];
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]) : "r"(src) : "memory");
    if (g >= 7) {
        uint32_t nrm[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(nrm[0]), "=r"(nrm[1]), "=r"(nrm[2]), "=r"(nrm[3]) : "r"(src) : "memory");
        const int r = lane >> 2, c = 2 * (lane & 3);
        const uint32_t mask = ((c >= r) ? 0xFFFFu : 0u) | ((c + 1 >= r) ? 0xFFFF0000u : 0u);
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] = (nrm[i] & mask) | (t[i] & ~mask);
    }
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};"
                 :: "r"(dst), "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]) : "memory");
}

template <bool kSplit>
__device__ __forceinline__ void add_row(const uint8_t* slot, int row, int half, float beta, float (&v)[32]) {
    // v += beta * (hi [+ lo]) of the slot row, columns [32 half, 32 half + 32)
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const int c = 4 * half + cc;
        const uint4 h = *reinterpret_cast<const uint4*>(slot + swz(row, c));
        const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
        float2 lf[4];
        if constexpr (kSplit) {
            const uint4 l = *reinterpret_cast<const uint4*>(slot + kSlotBytes + swz(row, c));
            const uint32_t lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) lf[q] = __half22float2(*reinterpret_cast<const __half2*>(&lw[q]));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 f = __half22float2(*reinterpret_cast<const __half2*>(&hw[q]));
            if constexpr (kSplit) {
                f.x += lf[q].x;
                f.y += lf[q].y;
            }
            v[8 * cc + 2 * q] += beta * f.x;
            v[8 * cc + 2 * q + 1] += beta * f.y;
        }
    }
}

__device__ __forceinline__ float4 load_row4(const float* base, int64_t roff, int n, int q) {
    // columns 4q..4q+3 of a row (zero past n)
    const float* xr = base + roff;
    if (n == kN) return __ldg(reinterpret_cast<const float4*>(xr) + q);
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    const int c = 4 * q;
    if (c + 0 < n) x.x = __ldg(xr + c + 0);
    if (c + 1 < n) x.y = __ldg(xr + c + 1);
    if (c + 2 < n) x.z = __ldg(xr + c + 2);
    if (c + 3 < n) x.w = __ldg(xr + c + 3);
    return x;
}

// resident CTAs per SM (8 warps each): 3 for the single-pass layout (80 registers, a 136-byte spill:
// measured 0.289 -> 0.271 ms at c2 vs 2 CTAs), 2 for the split one (smem)
template <bool kSplit> constexpr int kSmallCtasPerSm = kSplit ? 2 : 3;

template <bool kSplit>
__global__ void __launch_bounds__(kThreadsS, kSmallCtasPerSm<kSplit>)
small_batch_kernel(const float* __restrict__ X, float* __restrict__ out, int n, int batch,
                   double* __restrict__ lambda_out, unsigned* __restrict__ status, const SmallPlan plan) {
    using L = SmallLayout<kSplit>;
    constexpr int kWarps = kThreadsS / 32;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* mma_bar = reinterpret_cast<uint64_t*>(smem + 2 * L::kPerMatrix);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_bar + 1);
    double* red = reinterpret_cast<double*>(mma_bar + 2);     // [2 matrices][8 warps]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int quad = warp & 3;                   // TMEM lane quadrant: rows 16 quad .. 16 quad + 15
    const int half = warp >> 2;                  // column half: [32 half, 32 half + 32)
    const int m = lane >> 4;                     // matrix of the pair this thread serves
    const int row = 16 * quad + (lane & 15);     // its row
    const int c0 = 32 * half;                    // its first column
    uint8_t* mat = smem + m * L::kPerMatrix;

    if (threadIdx.x == 0) {
        ptx::mbar_init(mma_bar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<64>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t kIdesc = ptx::make_idesc(0, 64, 64);   // f16 x f16 -> f32, M=64, N=64
    uint32_t mma_phase = 0;

    const int pairs = (batch + 1) / 2;
    for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
        const int b = 2 * pr + m;
        const bool valid = b < batch;
        float* stage = reinterpret_cast<float*>(mat + L::kU);   // 64 x 64 fp32 staging (16 KB)

        // ---- stage X (zero padded) for both matrices of the pair into the U slots: coalesced loads
        auto stage_X = [&]() {
            const int64_t base = static_cast<int64_t>(2 * pr) * n * n;
            const int nvalid = min(2, batch - 2 * pr);
            for (int e = threadIdx.x; e < 2 * kN * kN / 4; e += kThreadsS) {
                const int mm = e / (kN * kN / 4);
                const int rem = e - mm * (kN * kN / 4);
                const int r = rem >> 4, q = rem & 15;
                float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                if (mm < nvalid && r < n) {
                    const int64_t roff = base + static_cast<int64_t>(mm) * n * n + static_cast<int64_t>(r) * n;
                    x = load_row4(X, roff, n, q);
                    if (plan.form.Xk) {           // ADMM: M = C - X_k / sigma - Diag(y) (R22)
                        const float4 k = load_row4(plan.form.Xk, roff, n, q);
                        x.x = __fsub_rn(x.x, __fmul_rn(k.x, plan.form.inv_sigma));
                        x.y = __fsub_rn(x.y, __fmul_rn(k.y, plan.form.inv_sigma));
                        x.z = __fsub_rn(x.z, __fmul_rn(k.z, plan.form.inv_sigma));
                        x.w = __fsub_rn(x.w, __fmul_rn(k.w, plan.form.inv_sigma));
                        if (plan.form.y && (r >> 2) == q) {
                            const float yv = plan.form.y[static_cast<int64_t>(2 * pr + mm) * n + r];
                            const int d = r & 3;
                            if (d == 0) x.x = __fsub_rn(x.x, yv);
                            if (d == 1) x.y = __fsub_rn(x.y, yv);
                            if (d == 2) x.z = __fsub_rn(x.z, yv);
                            if (d == 3) x.w = __fsub_rn(x.w, yv);
                        }
                    }
                }
                // XOR-swizzle float4 columns by row to keep the transposed reads conflict-light
                reinterpret_cast<float4*>(smem + mm * L::kPerMatrix + L::kU)[r * 16 + (q ^ (r & 15))] = x;
            }
            __syncthreads();
        };
        auto stage_at = [&](int r, int c) -> float {      // swizzled staging read
            return stage[r * kN + (((c >> 2) ^ (r & 15)) << 2) + (c & 3)];
        };
        stage_X();
        double ss = 0.0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int c = c0 + i;
            if (c >= row) {
                const double x = stage_at(row, c);                         // upper triangle (R10)
                ss += (c == row ? 1.0 : 2.0) * x * x;
            }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);   // within 16 lanes
        if ((lane & 15) == 0) red[m * kWarps + warp] = ss;
        __syncthreads();
        double lsum = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) lsum += red[m * kWarps + w];             // fixed order
        double lam = sqrt(lsum);
        if (!isfinite(lam)) {
            if ((lane & 15) == 0 && warp == 0 && valid) atomicOr(status, 1u);
            lam = __longlong_as_double(0x7ff8000000000000LL);
        }
        if (valid && warp == 0 && (lane & 15) == 0 && lambda_out) lambda_out[b] = lam;
        const double inv = lam > 0.0 ? 1.0 / lam : (lam == 0.0 ? 0.0 : lam);
        auto store_x0 = [&](int slot_off) {               // X_0 = sym_upper(X) / lambda~ from staging
            float x0[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int c = c0 + i;
                const float x = (c >= row) ? stage_at(row, c) : stage_at(c, row);
                x0[i] = static_cast<float>(static_cast<double>(x) * inv);
            }
            store_row<kSplit>(mat + slot_off, row, half, x0, plan.s_x0);
        };
        store_x0(L::kZ);
        fence_proxy_async_smem();
        __syncthreads();

        // ---- the chain of products
        for (int si = 0; si < plan.nsteps; ++si) {
            const SmallStep st = plan.steps[si];
            if (st.reload_x0) {
                // X_0 back into the Y slot for the reconstruction product (Z slot holds S; the
                // U slots are free again and serve as staging)
                stage_X();
                store_x0(L::kY);
                fence_proxy_async_smem();
                __syncthreads();
            }
            const long long t_a = kDebug ? clock64() : 0;
            if (threadIdx.x == 0) {
                ptx::tc_fence_after();
#pragma unroll 1
                for (int mm = 0; mm < 2; ++mm) {
                    uint8_t* mb = smem + mm * L::kPerMatrix;
                    const uint32_t a = ptx::smem_u32(mb + st.slot_a);
                    const uint32_t bb = ptx::smem_u32(mb + st.slot_b);
                    const uint64_t ad = ptx::smem_desc_sw128_kmajor(a), bd = ptx::smem_desc_sw128_kmajor(bb);
                    const uint32_t d = tmem + (static_cast<uint32_t>(16 * mm) << 16);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t koff = static_cast<uint64_t>((k * 32) >> 4);
                        ptx::mma_f16(d, ad + koff, bd + koff, kIdesc, k != 0);
                        if constexpr (kSplit) {
                            const uint64_t al = ptx::smem_desc_sw128_kmajor(a + kSlotBytes);
                            const uint64_t bl = ptx::smem_desc_sw128_kmajor(bb + kSlotBytes);
                            ptx::mma_f16(d, ad + koff, bl + koff, kIdesc, 1u);
                            ptx::mma_f16(d, al + koff, bd + koff, kIdesc, 1u);
                        }
                    }
                }
                ptx::mma_commit(mma_bar);
            }
            ptx::mbar_wait(mma_bar, mma_phase);
            mma_phase ^= 1;
            ptx::tc_fence_after();
            const long long t_b = kDebug ? clock64() : 0;

            // a chain product's operand scale (a power of two, compute_scales) is folded into alpha
            // and beta: (alpha acc + beta D) s == (alpha s) acc + (beta s) D exactly
            const bool fold = st.final_mode == 0 && !plan.nofold;
            const float alpha = fold ? st.alpha * st.out_scale : st.alpha;
            const float beta = fold ? st.beta * st.out_scale : st.beta;
            float v[32];
            {
                uint32_t raw[32];
                ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(32 * quad) << 16) + c0, raw);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = alpha * __uint_as_float(raw[i]);
            }
            ptx::tc_fence_before();
            const long long t_c = kDebug ? clock64() : 0;
            if (st.slot_d >= 0) add_row<kSplit>(mat + st.slot_d, row, half, beta, v);
            if (st.final_mode == 0) {
                // in place: the MMA that read this slot has completed (mma_bar)
                if (fold)
                    store_row<kSplit, false>(mat + st.slot_out, row, half, v, 1.0f);
                else
                    store_row<kSplit>(mat + st.slot_out, row, half, v, st.out_scale);
                if (st.mirror) {
                    // the stage output Z must be exactly symmetric: its antisymmetric part would
                    // grow like prod c_{t,0} over the stages (R20); Y and U need not be (their
                    // rounding-level asymmetry is not amplified -- rounding model)
                    __syncthreads();
                    constexpr int kParts = kSplit ? 2 : 1;
                    if (plan.mirror_scalar) {     // A/B baseline (PSD_SMALL_MIRROR_SCALAR)
                        for (int task = threadIdx.x; task < 2 * kParts * 36; task += kThreadsS) {
                            const int mm = task / (kParts * 36);
                            const int part = (task / 36) % kParts;
                            mirror_block_task(smem + mm * L::kPerMatrix + st.slot_out + part * kSlotBytes, task % 36);
                        }
                    } else {
                        for (int task = warp; task < 2 * kParts * kMirrorGroups; task += kWarps) {
                            const int mm = task / (kParts * kMirrorGroups);
                            const int part = (task / kMirrorGroups) % kParts;
                            mirror_group_warp(smem + mm * L::kPerMatrix + st.slot_out + part * kSlotBytes,
                                              task % kMirrorGroups, lane);
                        }
                    }
                }
                fence_proxy_async_smem();
                __syncthreads();
                if (kDebug && plan.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
                    const long long t_d = clock64();
                    atomicAdd(plan.dbg + 0, static_cast<unsigned long long>(t_b - t_a));   // MMA issue + wait
                    atomicAdd(plan.dbg + 1, static_cast<unsigned long long>(t_c - t_b));   // TMEM loads
                    atomicAdd(plan.dbg + 2, static_cast<unsigned long long>(t_d - t_c));   // epilogue + mirror + sync
                    atomicAdd(plan.dbg + 3, 1ull);
                }
            } else {
                // final: 1/2 X + 1/2 lambda~ X0 S  (mode 1)  or  S (mode 2); symmetrise via staging
                // the input element (row, c), c >= row: X, or the ADMM argument M (R22)
                const int64_t roff = static_cast<int64_t>(b) * n * n + static_cast<int64_t>(row) * n;
                const float yv = (plan.form.Xk && plan.form.y && valid && row < n)
                                     ? plan.form.y[static_cast<int64_t>(b) * n + row] : 0.0f;
                auto input_at = [&](int c) -> float {
                    const bool in = valid && row < n && c < n && c >= row;
                    float x = in ? __ldg(X + roff + c) : 0.0f;
                    if (plan.form.Xk) {
                        const float k = in ? __ldg(plan.form.Xk + roff + c) : 0.0f;
                        x = __fsub_rn(x, __fmul_rn(k, plan.form.inv_sigma));
                        if (c == row) x = __fsub_rn(x, yv);
                    }
                    return x;
                };
                if (st.final_mode == 1) {
                    // + beta X[row][c] for c >= row (the lower part is replaced by the mirror below)
                    const float a = static_cast<float>(lam);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = a * v[i] + st.beta * input_at(c0 + i);
                }
                float4* srow = reinterpret_cast<float4*>(stage + row * kN);
                // ADMM: X_next = sigma (P - M) is stored first, while the inputs (which the
                // outputs may overwrite: in place) are still intact; then P
                const bool two = st.final_mode == 1 && plan.out2;
                for (int pass = two ? 1 : 0; pass >= 0; --pass) {
                    if (pass == 1) {
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq) {
                            const int c = c0 + 4 * qq;
                            srow[(8 * half + qq) ^ (row & 15)] =
                                make_float4(plan.sigma2 * (v[4 * qq] - input_at(c)),
                                            plan.sigma2 * (v[4 * qq + 1] - input_at(c + 1)),
                                            plan.sigma2 * (v[4 * qq + 2] - input_at(c + 2)),
                                            plan.sigma2 * (v[4 * qq + 3] - input_at(c + 3)));
                        }
                    } else {
#pragma unroll
                        for (int qq = 0; qq < 8; ++qq)
                            srow[(8 * half + qq) ^ (row & 15)] =
                                make_float4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
                    }
                    __syncthreads();
                    float* dst = pass == 0 ? out : plan.out2;
                    if (valid && row < n) {
                        float* orow = dst + static_cast<int64_t>(b) * n * n + static_cast<int64_t>(row) * n;
                        if (n == kN) {
#pragma unroll
                            for (int qq = 0; qq < 8; ++qq) {
                                const int c = c0 + 4 * qq;
                                float4 o;
                                o.x = (c + 0 >= row) ? stage_at(row, c + 0) : stage_at(c + 0, row);
                                o.y = (c + 1 >= row) ? stage_at(row, c + 1) : stage_at(c + 1, row);
                                o.z = (c + 2 >= row) ? stage_at(row, c + 2) : stage_at(c + 2, row);
                                o.w = (c + 3 >= row) ? stage_at(row, c + 3) : stage_at(c + 3, row);
                                __stcs(reinterpret_cast<float4*>(orow + c), o);
                            }
                        } else {
                            for (int c = c0; c < min(c0 + 32, n); ++c)
                                orow[c] = (c >= row) ? stage_at(row, c) : stage_at(c, row);
                        }
                    }
                    __syncthreads();
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<64>(tmem);
    }
}

template <bool kSplit>
cudaError_t launch_small_t(const float* X, float* out, int n, int batch, double* lambda_out, unsigned* status,
                           const SmallPlan& plan, cudaStream_t stream) {
    using L = SmallLayout<kSplit>;
    static int num_sms = 0;
    if (!num_sms) {
        cudaError_t err = cudaFuncSetAttribute(small_batch_kernel<kSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               L::kBytes);
        if (err != cudaSuccess) return err;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int pairs = (batch + 1) / 2;
    int grid = kSmallCtasPerSm<kSplit> * num_sms;
    if (grid > pairs) grid = pairs;
    small_batch_kernel<kSplit><<<grid, kThreadsS, L::kBytes, stream>>>(X, out, n, batch, lambda_out, status, plan);
    return cudaGetLastError();
}

}  // namespace

int small_slot_offset(bool split, int slot) {
    if (split) {
        using L = SmallLayout<true>;
        return slot == 0 ? L::kZ : (slot == 1 ? L::kY : L::kU);
    }
    using L = SmallLayout<false>;
    return slot == 0 ? L::kZ : (slot == 1 ? L::kY : L::kU);
}

cudaError_t launch_small_batch(bool split, const float* X, float* out, int n, int batch, double* lambda_out,
                               unsigned* status, const SmallPlan& plan, cudaStream_t stream) {
    return split ? launch_small_t<true>(X, out, n, batch, lambda_out, status, plan, stream)
                 : launch_small_t<false>(X, out, n, batch, lambda_out, status, plan, stream);
}

}  // namespace psd
