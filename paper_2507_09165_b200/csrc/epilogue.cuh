// epilogue.cuh -- fused symmetric epilogue shared by the product kernels.
//
// One warp owns 32 consecutive output rows gi0..gi0+31 of an upper tile (I <= J); lane l
// holds row gi = gi0 + l and processes 32 accumulator columns gj0..gj0+31 at a time (one
// tcgen05.ld 32x32b.x32, or a DSMEM-reduced split-K partial):
//     v = alpha * acc + beta * D[gi][gj]         D: the operand-precision copy of the addend
//                                                (Z or Y; hi + lo on the split path) or, for
//                                                the reconstruction, the fp32 input X
//     operand copy: out_op[gi][gj] = v, and out_op[gj][gi] = v unless upper-only storage
//                   skips the mirror of an off-diagonal tile (the loaders then read the lower
//                   triangle as the transpose of the stored upper tile: exactly symmetric either way)
//     final output: outF[gi][gj]  = outF[gj][gi]  = v     (fp32, masked to n)
// Chunks are 32-aligned, so a chunk is either strictly above the diagonal (gj0 > gi0: direct
// rows + the mirrored block through a per-warp 32x32 smem transpose) or a diagonal 32x32
// block (gj0 == gi0: the block is symmetrised from its upper triangle through smem and
// written as full rows).  Callers skip blocks below the diagonal.  Blocks are staged in the
// warp's smem and drained with coalesced row-segment stores.  This is where the polynomial's
// axpy terms (c_j Y, c_0 Z) and the reconstruction 1/2 X + 1/2 lambda~ X_0 S of Algorithm 2
// are fused -- and the ADMM formation / X update -- so no separate elementwise
// pass touches HBM.
#pragma once
#include "kernels.h"
#include "optraits.cuh"

namespace psd {

// per-warp staging: 32 rows x (32 + 4) fp32 words (row stride 144 B keeps LDS.128 of
// 8-lane phases conflict-free); reused as 32 x 40 fp16 (row stride 80 B)
constexpr int kEpiWarpSmemBytes = 32 * 36 * 4;

// Symmetrise a diagonal 32x32 block in registers: lane r keeps row r of upper(v) + mirror.
__device__ __forceinline__ void symmetrize_block(float (&v)[32], uint8_t* wsmem) {
    const int lane = threadIdx.x & 31;
    float* S = reinterpret_cast<float*>(wsmem);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 32; ++c) S[lane * 36 + c] = v[c];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 32; ++c)
        if (c < lane) v[c] = S[c * 36 + lane];          // element (lane, c) := computed (c, lane)
    __syncwarp();
}

// Coalesced block stores: the 32x32 block is staged in the warp's smem (row-major, 16-byte
// aligned rows) and read back so that each warp store instruction writes whole row segments of
// several rows (16-bit: 8 rows x 64 B; 32-bit: 4 rows x 128 B) instead of one 16-byte piece of 32
// different rows -- 4x fewer L1/L2 store transactions for the same bytes (measured at c4: 5% more
// throughput under the power cap, tools/ab_probe.py).
// `rowbase(r)` is the global address of row r of the block's destination (already at its column).
template <int kBytes, typename RowAddr>
__device__ __forceinline__ void drain_staged_block(const uint8_t* S, int stride_bytes, RowAddr rowbase) {
    const int lane = threadIdx.x & 31;
    constexpr int kChunks = 2 * kBytes;                 // 16-byte chunks per 32-element row
    constexpr int kRowsPerInst = 32 / kChunks;
#pragma unroll
    for (int i = 0; i < kChunks; ++i) {
        const int r = i * kRowsPerInst + lane / kChunks, c = lane % kChunks;
        const uint4 x = *reinterpret_cast<const uint4*>(S + r * stride_bytes + c * 16);
        __stcs(reinterpret_cast<uint4*>(rowbase(r)) + c, x);
    }
}

// Stage the operand-precision conversion of v (lane = row) into the warp's smem rows.
template <OpType T>
__device__ __forceinline__ void stage_op_rows(const float (&v)[32], uint8_t* wsmem, int stride) {
    using Tr = OpTraits<T>;
    const int lane = threadIdx.x & 31;
    if constexpr (Tr::kBytes == 2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) w[h] = Tr::pack2(v[q * 8 + 2 * h], v[q * 8 + 2 * h + 1]);
            *reinterpret_cast<uint4*>(wsmem + lane * stride + q * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(wsmem + lane * stride + q * 16) =
                make_float4(Tr::cvt(v[4 * q]), Tr::cvt(v[4 * q + 1]), Tr::cvt(v[4 * q + 2]), Tr::cvt(v[4 * q + 3]));
    }
}

// Stage the transpose: element (c, lane) = v[c].
template <OpType T>
__device__ __forceinline__ void stage_op_cols(const float (&v)[32], uint8_t* wsmem, int stride) {
    using Tr = OpTraits<T>;
    using op_t = typename Tr::type;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < 32; ++c) *reinterpret_cast<op_t*>(wsmem + c * stride + lane * Tr::kBytes) = Tr::cvt(v[c]);
}

// Store a 32x32 block (rows gi0.., columns gj0..) in operand precision and mirror it to
// (gj0.., gi0..) unless it is a (symmetrised) diagonal block -- both through the coalesced drain.
template <OpType T>
__device__ __forceinline__ void store_op_block(void* out, int64_t opBase, int npad, int gi0, int gj0, bool diag32,
                                               const float (&v)[32], uint8_t* wsmem, bool mirror = true) {
    using Tr = OpTraits<T>;
    using op_t = typename Tr::type;
    op_t* out_op = reinterpret_cast<op_t*>(out);
    constexpr int kStride = Tr::kBytes == 2 ? 80 : 144;     // conflict-free staging row strides
    __syncwarp();
    stage_op_rows<T>(v, wsmem, kStride);
    __syncwarp();
    drain_staged_block<Tr::kBytes>(wsmem, kStride, [&](int r) {
        return out_op + opBase + static_cast<int64_t>(gi0 + r) * npad + gj0;
    });
    if (!diag32 && mirror) {
        __syncwarp();
        stage_op_cols<T>(v, wsmem, kStride);
        __syncwarp();
        drain_staged_block<Tr::kBytes>(wsmem, kStride, [&](int r) {
            return out_op + opBase + static_cast<int64_t>(gj0 + r) * npad + gi0;
        });
    }
    __syncwarp();
}

// Same block stored into every destination of `dsts` (peer-memory row-panel mode): staged once
// (direct, then mirrored) and drained npeers times through the coalesced drain.
template <OpType T>
__device__ __forceinline__ void store_op_block_peers(void* const* dsts, int nd, int64_t opBase, int npad, int gi0,
                                                     int gj0, bool diag32, const float (&v)[32], uint8_t* wsmem,
                                                     bool mirror = true) {
    using Tr = OpTraits<T>;
    using op_t = typename Tr::type;
    constexpr int kStride = Tr::kBytes == 2 ? 80 : 144;
    __syncwarp();
    stage_op_rows<T>(v, wsmem, kStride);
    __syncwarp();
    for (int p = 0; p < nd; ++p) {
        op_t* base = reinterpret_cast<op_t*>(dsts[p]);
        drain_staged_block<Tr::kBytes>(wsmem, kStride, [&](int r) {
            return base + opBase + static_cast<int64_t>(gi0 + r) * npad + gj0;
        });
    }
    if (!diag32 && mirror) {
        __syncwarp();
        stage_op_cols<T>(v, wsmem, kStride);
        __syncwarp();
        for (int p = 0; p < nd; ++p) {
            op_t* base = reinterpret_cast<op_t*>(dsts[p]);
            drain_staged_block<Tr::kBytes>(wsmem, kStride, [&](int r) {
                return base + opBase + static_cast<int64_t>(gj0 + r) * npad + gi0;
            });
        }
    }
    __syncwarp();
}

// kCg: load through L2 only (ld.global.cg) -- the persistent chain kernel rewrites the addend
// buffers between its products, so a line this SM cached in L1 earlier may be stale.
template <OpType T, bool kCg = false>
__device__ __forceinline__ void add_op_row(const void* D, int64_t opBase, int npad, int gi, int gj0, float beta,
                                           float (&v)[32]) {
    using Tr = OpTraits<T>;
    using op_t = typename Tr::type;
    const op_t* drow = reinterpret_cast<const op_t*>(D) + opBase + static_cast<int64_t>(gi) * npad + gj0;
    if constexpr (Tr::kBytes == 2) {
        const uint4* d4 = reinterpret_cast<const uint4*>(drow);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 d = kCg ? __ldcg(d4 + q) : d4[q];
            const uint32_t w[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                float lo, hi;
                Tr::unpack2(w[h], lo, hi);
                v[q * 8 + 2 * h] += beta * lo;
                v[q * 8 + 2 * h + 1] += beta * hi;
            }
        }
    } else {
        const float4* d4 = reinterpret_cast<const float4*>(drow);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 d = kCg ? __ldcg(d4 + q) : d4[q];
            v[4 * q] += beta * d.x;
            v[4 * q + 1] += beta * d.y;
            v[4 * q + 2] += beta * d.z;
            v[4 * q + 3] += beta * d.w;
        }
    }
}

// Addend words of one chunk fetched ahead of time (the chain kernel loads them while the MMAs
// run): the 16-byte row segments of the primary addend, Dop (4 words for 16-bit operands, 8 for
// tf32) or the fp32 X (8 words).  Returns false (nothing loaded) where the masked path is needed.
template <OpType T>
__device__ __forceinline__ bool prefetch_addend(const EpiParams& e, int b, int npad, int gi, int gj0, uint4 (&pre)[8]) {
    using Tr = OpTraits<T>;
    if (e.Dop) {
        const uint4* d4 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(e.Dop) +
                                                         (static_cast<int64_t>(b) * npad * npad +
                                                          static_cast<int64_t>(gi) * npad + gj0) * Tr::kBytes);
#pragma unroll
        for (int q = 0; q < 2 * Tr::kBytes; ++q) pre[q] = __ldcg(d4 + q);
        return true;
    }
    if (e.Df && !e.Df2 && gi < e.nDf && gj0 + 32 <= e.nDf && (e.ldDf & 3) == 0) {
        const uint4* d4 = reinterpret_cast<const uint4*>(e.Df + static_cast<int64_t>(b) * e.strideDf +
                                                         static_cast<int64_t>(gi) * e.ldDf + gj0);
#pragma unroll
        for (int q = 0; q < 8; ++q) pre[q] = __ldcs(d4 + q);
        return true;
    }
    return false;
}

// Store a 32x32 fp32 block (rows gi0.., columns gj0..) of the final output F (ld, masked to nF),
// mirrored to (gj0.., gi0..) unless it is a (symmetrised) diagonal block.
__device__ __forceinline__ void store_f32_block(float* F, int64_t ld, int nF, int gi0, int gj0, bool diag32,
                                                const float (&v)[32], uint8_t* wsmem) {
    const int lane = threadIdx.x & 31;
    const int gi = gi0 + lane;
    const bool fast = (ld & 3) == 0 && gi0 + 32 <= nF && gj0 + 32 <= nF;
    if (fast) {                                      // coalesced drain (see drain_staged_block)
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(wsmem + lane * 144 + q * 16) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
        drain_staged_block<4>(wsmem, 144, [&](int r) { return F + static_cast<int64_t>(gi0 + r) * ld + gj0; });
        if (!diag32) {
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 32; ++c) reinterpret_cast<float*>(wsmem + c * 144)[lane] = v[c];
            __syncwarp();
            drain_staged_block<4>(wsmem, 144, [&](int r) { return F + static_cast<int64_t>(gj0 + r) * ld + gi0; });
        }
        __syncwarp();
    } else if (gi < nF) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int gj = gj0 + i;
            if (gj >= nF) continue;
            F[static_cast<int64_t>(gi) * ld + gj] = v[i];
            if (!diag32) F[static_cast<int64_t>(gj) * ld + gi] = v[i];
        }
    }
}

// store_f32_block with separate bases for the direct block (rows gi0..) and the mirrored one
// (rows gj0..): the peer-memory row-panel path sends each to the rank owning the rows.
__device__ __forceinline__ void store_f32_block_split(float* Fd, float* Fm, int64_t ld, int nF, int gi0, int gj0,
                                                      bool diag32, const float (&v)[32], uint8_t* wsmem) {
    const int lane = threadIdx.x & 31;
    const int gi = gi0 + lane;
    const bool fast = (ld & 3) == 0 && gi0 + 32 <= nF && gj0 + 32 <= nF;
    if (fast) {
        float4* dst = reinterpret_cast<float4*>(Fd + static_cast<int64_t>(gi) * ld + gj0);
#pragma unroll
        for (int q = 0; q < 8; ++q) __stcs(dst + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        if (!diag32) {
            float* S = reinterpret_cast<float*>(wsmem);
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 32; ++c) S[c * 36 + lane] = v[c];
            __syncwarp();
            const float4* src = reinterpret_cast<const float4*>(S + lane * 36);
            float4* tdst = reinterpret_cast<float4*>(Fm + static_cast<int64_t>(gj0 + lane) * ld + gi0);
#pragma unroll
            for (int q = 0; q < 8; ++q) __stcs(tdst + q, src[q]);
            __syncwarp();
        }
    } else if (gi < nF) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int gj = gj0 + i;
            if (gj >= nF) continue;
            Fd[static_cast<int64_t>(gi) * ld + gj] = v[i];
            if (!diag32) Fm[static_cast<int64_t>(gj) * ld + gi] = v[i];
        }
    }
}

// fp32 row segment [gj0, gj0 + 32) of row gi of F (ld, masked to nF: zero outside)
__device__ __forceinline__ void load_f32_row(const float* F, int64_t ld, int nF, int gi, int gj0, float (&d)[32]) {
    const float* row = F + static_cast<int64_t>(gi) * ld;
    if (gi < nF && gj0 + 32 <= nF && (ld & 3) == 0) {
        const float4* d4 = reinterpret_cast<const float4*>(row + gj0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 x = __ldcs(d4 + q);
            d[4 * q] = x.x;
            d[4 * q + 1] = x.y;
            d[4 * q + 2] = x.z;
            d[4 * q + 3] = x.w;
        }
    } else {
        const bool row_ok = gi < nF;
#pragma unroll
        for (int i = 0; i < 32; ++i) d[i] = (row_ok && gj0 + i < nF) ? row[gj0 + i] : 0.0f;
    }
}

// L2 prefetch of this thread's addend row segment(s) [gj0, gj0 + ncols) of row gi, issued before
// the epilogue waits for its accumulator: the addends (e.g. the fp32 input X of the reconstruction,
// 2 GB at config c4, not L2-resident) then arrive while the MMAs of the tile still run.
template <OpType T>
__device__ __forceinline__ void prefetch_addend_l2(const EpiParams& e, int b, int npad, int gi, int gj0, int ncols) {
    using Tr = OpTraits<T>;
    auto pf = [](const void* p) { asm volatile("prefetch.global.L2 [%0];" :: "l"(p)); };
    if (e.Dop) {
        const int64_t off = static_cast<int64_t>(b) * npad * npad + static_cast<int64_t>(gi) * npad + gj0;
        for (int c = 0; c < ncols * Tr::kBytes; c += 128) {
            pf(reinterpret_cast<const uint8_t*>(e.Dop) + off * Tr::kBytes + c);
            if (e.Dop_lo) pf(reinterpret_cast<const uint8_t*>(e.Dop_lo) + off * Tr::kBytes + c);
        }
    } else if (e.Df && gi < e.nDf) {
        const int64_t off = static_cast<int64_t>(b) * e.strideDf + static_cast<int64_t>(gi) * e.ldDf + gj0;
        const int cols = min(ncols, e.nDf - gj0);
        for (int c = 0; c < cols; c += 32) {
            pf(e.Df + off + c);
            if (e.Df2) pf(e.Df2 + off + c);
        }
    }
}

template <OpType T, bool kCg = false>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& e, float alpha, int b, int npad, int gi0, int gj0,
                                               bool tile_diag, const uint32_t (&raw)[32], uint8_t* wsmem,
                                               int64_t packed_off = -1, const uint4* pre = nullptr) {
    using Tr = OpTraits<T>;
    using op_t = typename Tr::type;
    const int lane = threadIdx.x & 31;
    const int gi = gi0 + lane;
    const bool diag32 = (gi0 == gj0);                   // diagonal 32x32 block
    const int64_t opBase = static_cast<int64_t>(b) * npad * npad;
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = alpha * __uint_as_float(raw[i]);

    // addends: full 32-element row segments (the values left of the diagonal are discarded
    // by the symmetrisation of a diagonal block)
    if (pre && e.Dop) {                              // prefetched primary addend
        if constexpr (Tr::kBytes == 2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t w[4] = {pre[q].x, pre[q].y, pre[q].z, pre[q].w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    float lo, hi;
                    Tr::unpack2(w[h], lo, hi);
                    v[q * 8 + 2 * h] += e.beta * lo;
                    v[q * 8 + 2 * h + 1] += e.beta * hi;
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[4 * q] += e.beta * __uint_as_float(pre[q].x);
                v[4 * q + 1] += e.beta * __uint_as_float(pre[q].y);
                v[4 * q + 2] += e.beta * __uint_as_float(pre[q].z);
                v[4 * q + 3] += e.beta * __uint_as_float(pre[q].w);
            }
        }
        if (e.Dop_lo) add_op_row<T, kCg>(e.Dop_lo, opBase, npad, gi, gj0, e.beta, v);
    } else if (pre && e.Df) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            v[4 * q] += e.beta * __uint_as_float(pre[q].x);
            v[4 * q + 1] += e.beta * __uint_as_float(pre[q].y);
            v[4 * q + 2] += e.beta * __uint_as_float(pre[q].z);
            v[4 * q + 3] += e.beta * __uint_as_float(pre[q].w);
        }
    } else if (e.Dop) {
        add_op_row<T, kCg>(e.Dop, opBase, npad, gi, gj0, e.beta, v);
        if (e.Dop_lo) add_op_row<T, kCg>(e.Dop_lo, opBase, npad, gi, gj0, e.beta, v);
    } else if (e.Df) {                               // fp32 addend (the input X), masked to nDf
        float m[32];
        load_f32_row(e.Df + static_cast<int64_t>(b) * e.strideDf, e.ldDf, e.nDf, gi, gj0, m);
        if (e.Df2) {
            // ADMM: m = C - X_k / sigma - Diag(y), one rounding per operation (as the bound and
            // scale kernels form it, R22)
            float k[32];
            load_f32_row(e.Df2 + static_cast<int64_t>(b) * e.strideDf, e.ldDf, e.nDf, gi, gj0, k);
#pragma unroll
            for (int i = 0; i < 32; ++i) m[i] = __fsub_rn(m[i], __fmul_rn(k[i], e.df2_scale));
            if (e.ddiag && diag32 && gi < e.nDf) {
                const float yv = e.ddiag[static_cast<int64_t>(b) * e.nDf + gi];
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i == lane) m[i] = __fsub_rn(m[i], yv);
            }
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += e.beta * m[i];
        if (e.outF2) {
            // X_next = sigma (S - M) (P:L934-936 with M = C - A*y - X_k / sigma), stored like outF
#pragma unroll
            for (int i = 0; i < 32; ++i) m[i] = e.outF2_scale * (v[i] - m[i]);
            if (diag32) symmetrize_block(m, wsmem);
            store_f32_block(e.outF2 + static_cast<int64_t>(b) * e.strideF, e.ldF, e.nF, gi0, gj0, diag32, m, wsmem);
        }
    }
    if (kDebug && e.dbg_all && threadIdx.x == 0) {       // debug timeline: addend loaded and added
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        // the compiler must not hoist the stamp above the addend's use: make it depend on v
        if (v[0] == 1234.5f && v[31] == 1234.5f) t += 1;
        e.dbg_all[8 * (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) + 7] = t;
    }
    if (diag32) symmetrize_block(v, wsmem);
    if (kDebug && e.dbg_nostore) {                             // debug experiment only: keep v live, store nothing
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += v[i];
        if (acc == 12345.678f) reinterpret_cast<volatile float*>(wsmem)[0] = acc;
        return;
    }

    if (packed_off >= 0) {
        // row-panel mode: this warp's 32 x 32 block of the tile, unmirrored, row-major tile slot
        // (row stride 256)
        const int64_t o = packed_off + static_cast<int64_t>(lane) * 256;
        if (e.packed_f32) {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.packed) + o);
#pragma unroll
            for (int q = 0; q < 8; ++q) __stcs(dst + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        } else if constexpr (Tr::kBytes == 2) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<op_t*>(e.packed) + o);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t w[4];
#pragma unroll
                for (int h = 0; h < 4; ++h)
                    w[h] = Tr::pack2(v[q * 8 + 2 * h] * e.out_scale, v[q * 8 + 2 * h + 1] * e.out_scale);
                __stcs(dst + q, make_uint4(w[0], w[1], w[2], w[3]));
            }
        } else {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<op_t*>(e.packed) + o);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                __stcs(dst + q, make_float4(Tr::cvt(v[4 * q] * e.out_scale), Tr::cvt(v[4 * q + 1] * e.out_scale),
                                            Tr::cvt(v[4 * q + 2] * e.out_scale), Tr::cvt(v[4 * q + 3] * e.out_scale)));
        }
        return;
    }

    if (e.out_op) {
        float w[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) w[i] = v[i] * e.out_scale;
        if (e.out_lo) {
            // split precision: hi = rn(w), lo = rn(w - hi); both stored mirrored
            float lo[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float h = Tr::to_float(Tr::cvt(w[i]));
                lo[i] = w[i] - h;
                w[i] = h;
            }
            store_op_block<T>(e.out_lo, opBase, npad, gi0, gj0, diag32, lo, wsmem, !(e.upper_only && !tile_diag));
        }
        if (e.npeers > 0)
            store_op_block_peers<T>(e.out_peers, e.npeers, opBase, npad, gi0, gj0, diag32, w, wsmem,
                                    !(e.upper_only && !tile_diag));
        else
            store_op_block<T>(e.out_op, opBase, npad, gi0, gj0, diag32, w, wsmem, !(e.upper_only && !tile_diag));
    }

    if (e.peer_rows > 0) {
        // peer-memory row panels: each 32-row block goes to the rank owning those rows
        // (rows past n -- padding -- are never stored; clamp the owner index for them)
        const int od = min(gi0 / e.peer_rows, kMaxPeers - 1), om = min(gj0 / e.peer_rows, kMaxPeers - 1);
        store_f32_block_split(e.outF_peers[od], e.outF_peers[om], e.ldF, e.nF, gi0, gj0, diag32, v, wsmem);
    } else if (e.outF) {
        store_f32_block(e.outF + static_cast<int64_t>(b) * e.strideF, e.ldF, e.nF, gi0, gj0, diag32, v, wsmem);
    }
}

}  // namespace psd
