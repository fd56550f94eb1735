// small_batch.cu -- batched small-n path (n <= 64): the whole of Algorithm 2 for a
// pair of matrices per CTA iteration, on-chip; HBM is touched once for X (upper triangle only,
// reading R10) and once for P.
//
//   * bound + scale in-kernel: each thread loads the upper part of its
//     own row straight into registers, the CTA reduces ||X||_F per matrix in fp64 (fixed order,
//     deterministic) and writes X_0 in the operand format (SW128 K-major fp16, hi/lo for the split
//     path); the lower triangle is then filled from the upper one in shared memory (R20);
//   * every product of the chain is tcgen05.mma.cta_group::1 M=64 N=64 K=16 from smem
//     descriptors into TMEM; the two matrices of the pair use the two half-subpartition
//     interleaves of one 64-column accumulator (lanes 32w+[0,16) and 32w+[16,32)), so one
//     tcgen05.ld 32x32b gives each thread one row of one matrix;
//   * epilogue (one row of 64 columns per thread): alpha*acc + beta*D with packed f32x2 FMAs
//     (D = the rounded operand copy in smem, reading R18), written back in place into the
//     operand slot (the MMA has completed), fence.proxy.async, barrier;
//   * reconstruction P = 1/2 X + 1/2 lambda~ X_0 S: X is reloaded (L2) into registers,
//     X_0 restaged for the last product, the result symmetrised through smem (exact symmetry) and
//     stored to HBM.
// 4 CTAs of 4 warps per SM on the 16-bit path (2 on the split path): while one CTA waits for its
// MMAs, the others run their epilogues.  Chain products commit each matrix's MMAs separately, so
// matrix 0's epilogue overlaps matrix 1's MMAs (SmallPlan::split_commit).  Only the issuing thread waits on the MMA barrier; the
// other warps sleep in bar.sync (a 256-thread spin on the mbarrier took ~15% of the issue slots
// in the first version, profiles/r2_c2_small_v2.md).
#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"

namespace psd {

namespace {

constexpr int kN = 64;                  // padded matrix edge
constexpr int kSlotBytes = kN * 128;    // 64 rows x 128 B (fp16), one SW128 atom wide
// 4 warps (16-bit: 4 CTAs/SM at 128 registers) or 8 warps (split path: 2 CTAs/SM, two warps per
// TMEM quadrant, each with half the columns and one matrix of the chain epilogue -- measured
// 319 -> 277 us at c2 fp16x3; at fp16 the 8-warp layout needs 64 registers and spills: 139 -> 164 us)
template <bool kSplit> constexpr int kWarpsS = kSplit ? 8 : 4;

// byte offset of the 16-byte chunk `chunk` (8 fp16 columns) of row `row` in a SW128 K-major slot
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
    return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

template <bool kSplit>
struct SmallLayout {
    // per matrix: Z slot, Y slot, U slot (hi [+ lo] each); the fp32 staging of the final product
    // reuses the first 16 KB of the matrix region (its operands are consumed by then)
    static constexpr int kParts = kSplit ? 2 : 1;
    static constexpr int kZ = 0;
    static constexpr int kY = kParts * kSlotBytes;
    static constexpr int kU = 2 * kParts * kSlotBytes;
    static constexpr int kPerMatrix = 3 * kParts * kSlotBytes;
    static constexpr int kBytes = 2 * kPerMatrix + 1024 + 256;   // + align slack, barrier, tmem slot, partial sums
};
// resident CTAs per SM: 4 x 49 KB (16-bit), 2 x 97 KB (split)
template <bool kSplit> constexpr int kSmallCtasPerSm = kSplit ? 2 : 4;

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- packed fp32 pairs (FFMA2 / FMUL2 on sm_100)
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
// float(h) + c for the two halves of a packed fp16 pair (FHADD: one instruction per element)
__device__ __forceinline__ float2 add_h2(uint32_t h, float2 c) {
    float2 d;
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
        "add.rn.f32.f16 %0, lo, %3;\n\tadd.rn.f32.f16 %1, hi, %4;\n\t}"
        : "=f"(d.x), "=f"(d.y) : "r"(h), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// The rounded operand value(s) of 8 consecutive columns: hi [+ lo] (the same copy the tensor
// cores multiply, reading R18)
template <bool kSplit>
__device__ __forceinline__ void load_operand8(const uint8_t* part, uint32_t off, float2 (&d)[4]) {
    const uint4 h = *reinterpret_cast<const uint4*>(part + off);
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w};
    if constexpr (kSplit) {
        const uint4 l = *reinterpret_cast<const uint4*>(part + kSlotBytes + off);
        const uint32_t lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = add_h2(lw[q], __half22float2(*reinterpret_cast<const __half2*>(&hw[q])));
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = __half22float2(*reinterpret_cast<const __half2*>(&hw[q]));
    }
}

// hi = rn(v) [, lo = rn(v - hi)] of 8 consecutive columns into the slot
template <bool kSplit>
__device__ __forceinline__ void store_operand8(uint8_t* part, uint32_t off, const float2 (&v)[4]) {
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        hi[q] = pack_h2(v[q].x, v[q].y);
        if constexpr (kSplit) {
            const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hi[q]));
            lo[q] = pack_h2(v[q].x - hf.x, v[q].y - hf.y);
        }
    }
    *reinterpret_cast<uint4*>(part + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    if constexpr (kSplit)
        *reinterpret_cast<uint4*>(part + kSlotBytes + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

// Exact symmetry of a stored operand (reading R20), four 8x8 blocks per warp instruction:
// ldmatrix.x4.trans reads upper blocks (bj, bi) transposed and stmatrix.x4 writes them as blocks
// (bi, bj); lanes 8q..8q+7 address the rows of block q.  Group g of a 64x64 part: g < 7 the
// strictly-lower blocks 4g..4g+3 (row-major), g = 7, 8 the diagonal blocks 4(g-7)..+3, which merge
// their plain and transposed loads (upper part kept).  The 8 row addresses of a block hit 8
// distinct 16-byte chunks of the SW128 rows: conflict-free.  Fragment of lane t: row t/4, columns
// 2(t%4)+{0,1}.
constexpr int kMirrorGroups = 9;
__device__ __forceinline__ void mirror_group_warp(uint8_t* part, int g, int lane) {
    const int q = lane >> 3, rr = lane & 7;
    int bi, bj;
    if (g < 7) {
        const int k = 4 * g + q;                       // 0..27 over the strict lower block triangle
        bi = 1 + (k >= 1) + (k >= 3) + (k >= 6) + (k >= 10) + (k >= 15) + (k >= 21);
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

// mirror the slot at `slot_off` of both matrices (all parts); caller synchronises before/after
template <bool kSplit>
__device__ __forceinline__ void mirror_slot(uint8_t* smem, int slot_off, int warp, int lane) {
    using L = SmallLayout<kSplit>;
    constexpr int kTasks = 2 * L::kParts * kMirrorGroups;
#pragma unroll 1
    for (int task = warp; task < kTasks; task += kWarpsS<kSplit>) {
        const int mm = task / (L::kParts * kMirrorGroups);
        const int part = (task / kMirrorGroups) % L::kParts;
        mirror_group_warp(smem + mm * L::kPerMatrix + slot_off + part * kSlotBytes, task % kMirrorGroups, lane);
    }
}

// 16 bytes of a row when `p` holds (else zeros), as one predicated load: the 16 loads of a row group
// are issued back to back (a branch around each made the compiler wait for every load in turn)
__device__ __forceinline__ float4 ldg4_pred(const float* ptr, bool p) {
    float4 v;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
                 "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
                 "@q ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "r"(static_cast<int>(p)));
    return v;
}
// the same for rows whose length is not a multiple of 4 (4-byte aligned): up to `rem` elements
__device__ __forceinline__ float4 ldg4_tail(const float* ptr, bool p, int rem) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p) {
        v.x = __ldg(ptr);
        if (rem > 1) v.y = __ldg(ptr + 1);
        if (rem > 2) v.z = __ldg(ptr + 2);
        if (rem > 3) v.w = __ldg(ptr + 3);
    }
    return v;
}

// ---- fragment-layout epilogue of the chain products
// tcgen05.ld 16x256b: 16 TMEM lanes x 8 fp32 columns per repetition; thread t gets lane t/4 cols
// 2(t%4)+{0,1} (regs 0,1) and lane t/4+8, same cols (regs 2,3) -- the 8x8-block fragment layout
// of ldmatrix / stmatrix / movmatrix, so the epilogue reads the addend, writes the output and its
// transpose (the mirror, R20) with one warp instruction per 8x8 block group.
__device__ __forceinline__ void tmem_ld_16x256b_x1(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_16x256b_x2(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&d)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t (&d)[2]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
                 : "=r"(d[0]), "=r"(d[1]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void stsm_x4(uint32_t addr, const uint32_t (&d)[4]) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};"
                 :: "r"(addr), "r"(d[0]), "r"(d[1]), "r"(d[2]), "r"(d[3]) : "memory");
}
__device__ __forceinline__ void stsm_x2(uint32_t addr, uint32_t d0, uint32_t d1) {
    asm volatile("stmatrix.sync.aligned.m8n8.x2.shared.b16 [%0], {%1, %2};" :: "r"(addr), "r"(d0), "r"(d1) : "memory");
}
__device__ __forceinline__ void stsm_x2_trans(uint32_t addr, uint32_t d0, uint32_t d1) {
    asm volatile("stmatrix.sync.aligned.m8n8.x2.trans.shared.b16 [%0], {%1, %2};" :: "r"(addr), "r"(d0), "r"(d1) : "memory");
}
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}

// One 8x8 output block in fragment form: hi [, lo] of alpha acc + beta D (D = hi [+ lo] of the
// addend's fragment, R18); the operand scale is folded into alpha and beta by the caller.
template <bool kSplit>
struct Frag {
    uint32_t hi, lo;
};
template <bool kSplit>
__device__ __forceinline__ Frag<kSplit> combine(uint32_t a0, uint32_t a1, bool has_d, uint32_t dh, uint32_t dl,
                                                float2 alpha, float2 beta) {
    float2 v = make_float2(__uint_as_float(a0), __uint_as_float(a1));
    if (has_d) {
        float2 d = __half22float2(*reinterpret_cast<const __half2*>(&dh));
        if constexpr (kSplit) d = add_h2(dl, d);
        v = fma2(alpha, v, mul2(beta, d));
    } else {
        v = mul2(alpha, v);
    }
    Frag<kSplit> f;
    f.hi = pack_h2(v.x, v.y);
    f.lo = 0;
    if constexpr (kSplit) {
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&f.hi));
        f.lo = pack_h2(v.x - hf.x, v.y - hf.y);
    }
    return f;
}
// a diagonal block made exactly symmetric from its upper triangle (fragment of lane t: row t/4,
// columns 2(t%4)+{0,1})
__device__ __forceinline__ uint32_t diag_upper(uint32_t f, uint32_t mask) {
    const uint32_t t = movmatrix_trans(f);
    return (f & mask) | (t & ~mask);
}

// The chain-product epilogue of warp W (TMEM lane quadrant W = rows 16W..16W+15 of both matrices),
// every block index a compile-time constant.  Only the upper 8x8 blocks are computed; each writes
// itself and its transpose (every product is exactly symmetric, R20).  Warp W owns the 9 unordered
// block pairs {P, Q} with P in its row blocks {2W, 2W+1}: the three inside them, and for every
// other warp b the two (2W, 2b), (2W, 2b+1) if b > W, else (2W, 2b+1), (2W+1, 2b+1) -- the same
// count for every quadrant (SMSP), and every pair exactly once.  In place is safe: a warp reads
// the addend only at the positions it writes.
template <int W, int K> struct Region {
    static constexpr int bq = K + (K >= W ? 1 : 0);   // the other warp
    static constexpr bool kRight = bq > W;           // (R0, 2bq), (R0, 2bq+1)  else  (R0, 2bq+1), (R1, 2bq+1)
};
template <int W, int K>
__device__ __forceinline__ void region_load(uint32_t tb, uint32_t (&a)[8]) {
    using Rg = Region<W, K>;
    if constexpr (Rg::kRight) tmem_ld_16x256b_x2(tb + 16 * Rg::bq, a);
    else tmem_ld_16x256b_x1(tb + 16 * Rg::bq + 8, *reinterpret_cast<uint32_t(*)[4]>(a));
}
// normal and transposed block-row offsets (within a part) of this lane for region K of warp W
template <int W, int K>
__device__ __forceinline__ void region_offsets(uint32_t lrow128, uint32_t lrow, uint32_t lq1, uint32_t& on, uint32_t& ot) {
    using Rg = Region<W, K>;
    constexpr int R0 = 2 * W, bq = Rg::bq;
    if constexpr (Rg::kRight) {
        on = (8 * R0) * 128 + lrow128 + (((2 * bq + lq1) ^ lrow) << 4);
        ot = (8 * 2 * bq) * 128 + lq1 * 1024 + lrow128 + ((R0 ^ lrow) << 4);
    } else {
        on = (8 * R0) * 128 + lq1 * 1024 + lrow128 + (((2 * bq + 1) ^ lrow) << 4);
        ot = (8 * (2 * bq + 1)) * 128 + lrow128 + (((R0 + lq1) ^ lrow) << 4);
    }
}
// the accumulator registers of region K's two blocks
template <int W, int K>
__device__ __forceinline__ void region_acc(const uint32_t (&a)[8], uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    if constexpr (Region<W, K>::kRight) { a0 = a[0]; a1 = a[1]; a2 = a[4]; a3 = a[5]; }
    else { a0 = a[0]; a1 = a[1]; a2 = a[2]; a3 = a[3]; }
}
// accumulator fragments of matrix mm for warp W's blocks (caller waits)
template <int W>
struct EpiFrags {
    uint32_t aW[8], a0[8], a1[8], a2[8];
};
template <int W>
__device__ __forceinline__ void epi_load(uint32_t tmem, int mm, EpiFrags<W>& f) {
    const uint32_t tb = tmem + (static_cast<uint32_t>(32 * W + 16 * mm) << 16);
    tmem_ld_16x256b_x2(tb + 16 * W, f.aW);
    region_load<W, 0>(tb, f.a0);
    region_load<W, 1>(tb, f.a1);
    region_load<W, 2>(tb, f.a2);
}
// the addend's fragments at every block a warp writes (hi [, lo]): all shared-memory reads of the
// epilogue are issued before its first store (the ldmatrix / stmatrix asm is ordered, so a read
// after a store would wait for the store)
struct EpiD {
    uint32_t wh[4], wl[4], rh[3][2], rl[3][2];
};
template <bool kSplit, int W>
__device__ __forceinline__ void epi_load_d(uint32_t pd, bool has_d, uint32_t offW, const uint32_t (&on)[3], EpiD& d) {
#pragma unroll
    for (int i = 0; i < 4; ++i) d.wh[i] = d.wl[i] = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) d.rh[k][0] = d.rh[k][1] = d.rl[k][0] = d.rl[k][1] = 0;
    if (!has_d) return;
    ldsm_x4(pd + offW, d.wh);
    if constexpr (kSplit) ldsm_x4(pd + kSlotBytes + offW, d.wl);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ldsm_x2(pd + on[k], d.rh[k]);
        if constexpr (kSplit) ldsm_x2(pd + kSlotBytes + on[k], d.rl[k]);
    }
}
template <bool kSplit, int W>
__device__ __forceinline__ void epi_store(const EpiFrags<W>& f, const EpiD& d, uint32_t po, uint32_t offW,
                                          const uint32_t (&on)[3], const uint32_t (&ot)[3], bool has_d, float2 alpha,
                                          float2 beta, uint32_t diag_mask) {
    {
        // blocks inside the warp's rows, lane group q: [(R0,R0), (R1,R0), (R0,R1), (R1,R1)]
        const Frag<kSplit> f0 = combine<kSplit>(f.aW[0], f.aW[1], has_d, d.wh[0], d.wl[0], alpha, beta);
        const Frag<kSplit> f2 = combine<kSplit>(f.aW[4], f.aW[5], has_d, d.wh[2], d.wl[2], alpha, beta);
        const Frag<kSplit> f3 = combine<kSplit>(f.aW[6], f.aW[7], has_d, d.wh[3], d.wl[3], alpha, beta);
        const uint32_t h[4] = {diag_upper(f0.hi, diag_mask), movmatrix_trans(f2.hi), f2.hi, diag_upper(f3.hi, diag_mask)};
        stsm_x4(po + offW, h);
        if constexpr (kSplit) {
            const uint32_t l[4] = {diag_upper(f0.lo, diag_mask), movmatrix_trans(f2.lo), f2.lo, diag_upper(f3.lo, diag_mask)};
            stsm_x4(po + kSlotBytes + offW, l);
        }
    }
    auto region = [&](const uint32_t (&a)[8], auto kc) {
        constexpr int K = decltype(kc)::value;
        uint32_t a0, a1, a2, a3;
        region_acc<W, K>(a, a0, a1, a2, a3);
        const Frag<kSplit> g0 = combine<kSplit>(a0, a1, has_d, d.rh[K][0], d.rl[K][0], alpha, beta);
        const Frag<kSplit> g1 = combine<kSplit>(a2, a3, has_d, d.rh[K][1], d.rl[K][1], alpha, beta);
        stsm_x2(po + on[K], g0.hi, g1.hi);
        stsm_x2_trans(po + ot[K], g0.hi, g1.hi);
        if constexpr (kSplit) {
            stsm_x2(po + kSlotBytes + on[K], g0.lo, g1.lo);
            stsm_x2_trans(po + kSlotBytes + ot[K], g0.lo, g1.lo);
        }
    };
    region(f.a0, std::integral_constant<int, 0>{});
    region(f.a1, std::integral_constant<int, 1>{});
    region(f.a2, std::integral_constant<int, 2>{});
}
// the chain-product epilogue of warp W: matrix `mm` (mm < 0: both matrices, their fragments and
// addends loaded before the first store)
template <bool kSplit, int W>
__device__ __forceinline__ void chain_epilogue(uint32_t tmem, int mm, uint32_t pd0, uint32_t po0, uint32_t mat_bytes,
                                               bool has_d, float2 alpha, float2 beta, int lane, uint32_t diag_mask) {
    constexpr int R0 = 2 * W;
    const uint32_t lrow = lane & 7, lq = lane >> 3, lq1 = lq & 1;
    const uint32_t lrow128 = lrow * 128;
    const uint32_t offW = (8 * R0) * 128 + (lq & 1) * 1024 + lrow128 + (((R0 + (lq >> 1)) ^ lrow) << 4);
    uint32_t on[3], ot[3];
    region_offsets<W, 0>(lrow128, lrow, lq1, on[0], ot[0]);
    region_offsets<W, 1>(lrow128, lrow, lq1, on[1], ot[1]);
    region_offsets<W, 2>(lrow128, lrow, lq1, on[2], ot[2]);
    if (mm >= 0) {
        EpiFrags<W> f;
        EpiD d;
        epi_load<W>(tmem, mm, f);
        epi_load_d<kSplit, W>(pd0 + mm * mat_bytes, has_d, offW, on, d);
        ptx::tmem_ld_wait();
        epi_store<kSplit, W>(f, d, po0 + mm * mat_bytes, offW, on, ot, has_d, alpha, beta, diag_mask);
    } else {
        EpiFrags<W> f0, f1;
        EpiD d0, d1;
        epi_load<W>(tmem, 0, f0);
        epi_load<W>(tmem, 1, f1);
        epi_load_d<kSplit, W>(pd0, has_d, offW, on, d0);
        epi_load_d<kSplit, W>(pd0 + mat_bytes, has_d, offW, on, d1);
        ptx::tmem_ld_wait();
        epi_store<kSplit, W>(f0, d0, po0, offW, on, ot, has_d, alpha, beta, diag_mask);
        epi_store<kSplit, W>(f1, d1, po0 + mat_bytes, offW, on, ot, has_d, alpha, beta, diag_mask);
    }
}

template <bool kSplit>
__global__ void __launch_bounds__(32 * kWarpsS<kSplit>, kSmallCtasPerSm<kSplit>)
small_batch_kernel(const float* __restrict__ X, float* __restrict__ out, int n, int batch,
                   double* __restrict__ lambda_out, unsigned* __restrict__ status,
                   const __grid_constant__ SmallPlan plan) {
    using L = SmallLayout<kSplit>;
    constexpr int kWarps = kWarpsS<kSplit>;
    constexpr int kQW = kWarps / 4;              // warps per TMEM quadrant
    constexpr int kCT = kN / kQW;                // columns per thread in the row-per-thread phases
    constexpr int kRW = 16 / kQW;                // rows per warp in the coalesced load / store phases
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint64_t* mma_bar = reinterpret_cast<uint64_t*>(smem + 2 * L::kPerMatrix);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_bar + 1);
    double* red = reinterpret_cast<double*>(mma_bar + 2);     // [2 matrices][8 warps]
    uint64_t* mma_bar1 = mma_bar + 2 + 16;                    // split commits: matrix 1's products

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3;                      // TMEM lane quadrant (warp % 4, the hardware rule)
    const int hw = warp >> 2;                    // 8 warps: column half (row-per-thread phases) / matrix (chain epilogue)
    const int m = lane >> 4;                     // row-per-thread phases: matrix of the pair this thread serves
    const int row = 16 * q + (lane & 15);        // its row (TMEM lane 32 q + lane)
    const int rx = row & 7;                      // its SW128 chunk swizzle
    const uint32_t rbase = static_cast<uint32_t>(row * 128);
    uint8_t* mat = smem + m * L::kPerMatrix;
    const bool vec = (n & 3) == 0;               // float4 rows (X is 16-byte aligned)
    const uint32_t smem_base = ptx::smem_u32(smem);
    // fragment phases: lane t addresses row t & 7 of block t >> 3 in ldmatrix / stmatrix; its
    // fragment is row t/4, cols 2(t%4)+{0,1}
    const uint32_t diag_mask = ((2 * (lane & 3) >= (lane >> 2)) ? 0xFFFFu : 0u) |
                               ((2 * (lane & 3) + 1 >= (lane >> 2)) ? 0xFFFF0000u : 0u);

    if (threadIdx.x == 0) {
        ptx::mbar_init(mma_bar, 1);
        ptx::mbar_init(mma_bar1, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<128>(tmem_slot);   // cols [0,64): accumulator, [64,128): the input rows
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tmem_row = tmem + (static_cast<uint32_t>(32 * q) << 16);
    const uint32_t tmem_x = tmem_row + 64 + kCT * hw;     // this thread's input columns
    constexpr uint32_t kIdesc = ptx::make_idesc(0, 64, 64);   // f16 x f16 -> f32, M=64, N=64
    uint32_t mma_phase = 0, mma_phase1 = 0;

    const int pairs = (batch + 1) / 2;
    for (int pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
        const long long t_pair = kDebug ? clock64() : 0;
        const int b = 2 * pr + m;
        const bool valid = b < batch;

        // X_0 = sym_upper(X) / lambda~ into a slot: this thread's 32 columns of its row (chunks
        // left of the quadrant's first row are below the diagonal for every lane: skipped), then
        // the mirror.  X_0 in fp32: x * fl(1 / lambda~), the operand scale (a power of two) exact.
        auto store_x0 = [&](const float (&xr)[kCT], double inv, int slot_off) {
            const float is = static_cast<float>(inv) * plan.s_x0;
            const float2 invs = make_float2(is, is);
#pragma unroll
            for (int jj = 0; jj < kCT / 8; ++jj) {
                const int j = (kCT / 8) * hw + jj;
                if (j < 2 * q) continue;
                float2 v[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = mul2(make_float2(xr[8 * jj + 2 * e], xr[8 * jj + 2 * e + 1]), invs);
                store_operand8<kSplit>(mat + slot_off, rbase + ((j ^ rx) << 4), v);
            }
            __syncthreads();
            mirror_slot<kSplit>(smem, slot_off, warp, lane);
            fence_proxy_async_smem();
            __syncthreads();
        };
        // the input rows kept in TMEM columns [64, 128) from the first read on (X is read once)
        auto x_from_tmem = [&](float (&xr)[kCT]) {
#pragma unroll
            for (int h = 0; h < kCT / 32; ++h)
                ptx::tmem_ld_32x32b_x32(tmem_x + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(xr + 32 * h));
            ptx::tmem_ld_wait();
        };

        // ---- bound: lambda~ = ||X||_F over the upper triangle, fp64, fixed reduction order
        double lam, inv;
        {
            float xr[kCT];
            // the upper part (c >= r; whole 4-column groups that reach the diagonal) of the input
            // rows -- X, or the ADMM argument M = X - X_k / sigma - Diag(y) (R22); the lower
            // triangle is never read (R10).  Coalesced: per instruction, lanes 0-15 read one row of
            // matrix 0 and lanes 16-31 the same row of matrix 1 (2 x 256 B); warp (q, h) reads rows
            // 16q + 8h .. + 7; the rows reach the row-per-thread layout through fp32 staging in the
            // (still free) Y and U slots.
            {
                float4* xs = reinterpret_cast<float4*>(mat + L::kY);     // 64 x 16 float4, swizzled
                const int cl = lane & 15;
                const int c4 = 4 * cl;
                float4 xv[kRW];
                const int64_t base = static_cast<int64_t>(b) * n * n + c4;
                const int r0 = 16 * q + kRW * hw;
                auto pred = [&](int i) { const int r = r0 + i; return valid && r < n && c4 < n && c4 + 3 >= r; };
                if (vec) {
#pragma unroll
                    for (int i = 0; i < kRW; ++i) xv[i] = ldg4_pred(X + base + static_cast<int64_t>(r0 + i) * n, pred(i));
                } else {
#pragma unroll
                    for (int i = 0; i < kRW; ++i) xv[i] = ldg4_tail(X + base + static_cast<int64_t>(r0 + i) * n, pred(i), n - c4);
                }
                if (plan.form.Xk) {
#pragma unroll
                    for (int i = 0; i < kRW; ++i) {
                        const int r = r0 + i;
                        const float* kp = plan.form.Xk + base + static_cast<int64_t>(r) * n;
                        const float4 k = vec ? ldg4_pred(kp, pred(i)) : ldg4_tail(kp, pred(i), n - c4);
                        float4& x = xv[i];
                        x.x = __fsub_rn(x.x, __fmul_rn(k.x, plan.form.inv_sigma));
                        x.y = __fsub_rn(x.y, __fmul_rn(k.y, plan.form.inv_sigma));
                        x.z = __fsub_rn(x.z, __fmul_rn(k.z, plan.form.inv_sigma));
                        x.w = __fsub_rn(x.w, __fmul_rn(k.w, plan.form.inv_sigma));
                        if (plan.form.y && pred(i) && r >= c4 && r < c4 + 4) {
                            const float yv = plan.form.y[static_cast<int64_t>(b) * n + r];
                            if (r == c4 + 0) x.x = __fsub_rn(x.x, yv);
                            if (r == c4 + 1) x.y = __fsub_rn(x.y, yv);
                            if (r == c4 + 2) x.z = __fsub_rn(x.z, yv);
                            if (r == c4 + 3) x.w = __fsub_rn(x.w, yv);
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < kRW; ++i) {
                    const int r = r0 + i;
                    xs[r * 16 + (cl ^ (r & 15))] = xv[i];
                }
                __syncthreads();                 // the warps of a quadrant wrote its 16 rows
#pragma unroll
                for (int jq = 0; jq < kCT / 4; ++jq) {
                    const int qq = (kCT / 4) * hw + jq;    // float4 column group
                    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (qq >= 4 * q) x = xs[row * 16 + (qq ^ (row & 15))];   // left of the quadrant's rows: lower
                    xr[4 * jq + 0] = x.x;
                    xr[4 * jq + 1] = x.y;
                    xr[4 * jq + 2] = x.z;
                    xr[4 * jq + 3] = x.w;
                }
            }
            const long long t_ld = kDebug ? clock64() : 0;
            // the next pair's matrices into L2 while this pair's chain runs (bulk prefetch: one
            // instruction per contiguous matrix when its start is 16-byte aligned)
            if (pr + static_cast<int>(gridDim.x) < pairs && (lane & 15) == 0 && warp == 0) {
                const int bn = 2 * (pr + gridDim.x) + m;
                if (bn < batch) {
                    const float* nx = X + static_cast<int64_t>(bn) * n * n;
                    if (((n * n) & 3) == 0) {
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(nx), "r"(n * n * 4) : "memory");
                        if (plan.form.Xk)
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                                         :: "l"(plan.form.Xk + static_cast<int64_t>(bn) * n * n), "r"(n * n * 4) : "memory");
                    } else {
                        for (int o = 0; o < n * n; o += 32) asm volatile("prefetch.global.L2 [%0];" :: "l"(nx + o));
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < kCT / 32; ++h)
                ptx::tmem_st_32x32b_x32(tmem_x + 32 * h, *reinterpret_cast<const uint32_t(*)[32]>(xr + 32 * h));
            // sum of x^2 over c > row (counted twice) and the diagonal; four independent fp64
            // accumulators (fixed combination order: deterministic)
            double acc4[4] = {0.0, 0.0, 0.0, 0.0};
            double dg = 0.0;
#pragma unroll
            for (int g = 0; g < kCT / 16; ++g) {
                if (kCT * hw + 16 * g + 15 < 16 * q) continue;         // left of the quadrant's first row
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int cc = 16 * g + i, c = kCT * hw + cc;
                    const double x = xr[cc];
                    if (c > row) acc4[i & 3] = fma(x, x, acc4[i & 3]);
                    if (c == row) dg = x * x;
                }
            }
            double ss = fma(2.0, (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]), dg);
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);   // within 16 lanes
            if ((lane & 15) == 0) red[m * kWarps + warp] = ss;
            ptx::tmem_st_wait();
            __syncthreads();
            double lsum = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) lsum += red[m * kWarps + w];              // fixed order
            lam = sqrt(lsum);
            if (!isfinite(lam)) {
                if (lane == 0 && warp == 0 && valid) atomicOr(status, 1u);
                if (lane == 16 && warp == 0 && valid) atomicOr(status, 1u);
                lam = __longlong_as_double(0x7ff8000000000000LL);
            }
            if (valid && warp == 0 && (lane & 15) == 0 && lambda_out) lambda_out[b] = lam;
            inv = lam > 0.0 ? 1.0 / lam : (lam == 0.0 ? 0.0 : lam);
            const long long t_lam = kDebug ? clock64() : 0;
            store_x0(xr, inv, L::kZ);
            if (kDebug && plan.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
                atomicAdd(plan.dbg + 8, static_cast<unsigned long long>(t_ld - t_pair));    // loads
                if (pr == static_cast<int>(blockIdx.x)) atomicAdd(plan.dbg + 11, static_cast<unsigned long long>(t_ld - t_pair));
                atomicAdd(plan.dbg + 9, static_cast<unsigned long long>(t_lam - t_ld));    // bound
                atomicAdd(plan.dbg + 10, static_cast<unsigned long long>(clock64() - t_lam));   // X_0 + mirror
            }
        }
        if (kDebug && plan.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
            atomicAdd(plan.dbg + 5, static_cast<unsigned long long>(clock64() - t_pair));   // load, bound, X_0
            atomicAdd(plan.dbg + 7, 1ull);
        }

        // ---- the chain of products
#pragma unroll 1
        for (int si = 0; si < plan.nsteps; ++si) {
            const SmallStep& st = plan.steps[si];
            if (st.reload_x0) {
                // X_0 back into the Y slot for the reconstruction product (the Z slot holds S)
                float xr[kCT];
                x_from_tmem(xr);
                store_x0(xr, inv, L::kY);
            }
            const long long t_a = kDebug ? clock64() : 0;
            long long t_i = t_a;
            if (plan.split_commit && st.final_mode == 0) {
                // one commit per matrix: matrix 0's epilogue runs while matrix 1's MMAs finish (the
                // two matrices use disjoint operand slots and TMEM lane halves)
                if (threadIdx.x == 0) {
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(smem + st.slot_a), b0 = ptx::smem_u32(smem + st.slot_b);
                    const uint64_t ad0 = ptx::smem_desc_sw128_kmajor(a0), bd0 = ptx::smem_desc_sw128_kmajor(b0);
                    constexpr uint64_t kMatDesc = static_cast<uint64_t>(L::kPerMatrix >> 4);
                    constexpr uint64_t kLoDesc = static_cast<uint64_t>(kSlotBytes >> 4);
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint64_t koff = static_cast<uint64_t>((k * 32) >> 4);
                            const uint64_t ad = ad0 + mm * kMatDesc + koff, bd = bd0 + mm * kMatDesc + koff;
                            const uint32_t d = tmem + (static_cast<uint32_t>(16 * mm) << 16);
                            ptx::mma_f16(d, ad, bd, kIdesc, k != 0);
                            if constexpr (kSplit) {
                                ptx::mma_f16(d, ad, bd + kLoDesc, kIdesc, 1u);
                                ptx::mma_f16(d, ad + kLoDesc, bd, kIdesc, 1u);
                            }
                        }
                        ptx::mma_commit(mm == 0 ? mma_bar : mma_bar1);
                    }
                }
                const float2 alpha = make_float2(st.alpha * st.out_scale, st.alpha * st.out_scale);
                const float2 beta = make_float2(st.beta * st.out_scale, st.beta * st.out_scale);
                const bool has_d = st.slot_d >= 0;
                const uint32_t pd = smem_base + static_cast<uint32_t>(has_d ? st.slot_d : 0);
                const uint32_t po = smem_base + static_cast<uint32_t>(st.slot_out);
                auto epi = [&](int mm) {
                    switch (q) {
                        case 0: chain_epilogue<kSplit, 0>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                        case 1: chain_epilogue<kSplit, 1>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                        case 2: chain_epilogue<kSplit, 2>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                        default: chain_epilogue<kSplit, 3>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                    }
                };
                if (kQW == 2) {                          // 8 warps: warp half hw serves matrix hw
                    ptx::mbar_wait(hw == 0 ? mma_bar : mma_bar1, hw == 0 ? mma_phase : mma_phase1);
                    ptx::tc_fence_after();
                    epi(hw);
                } else {
                    ptx::mbar_wait(mma_bar, mma_phase);
                    ptx::tc_fence_after();
                    epi(0);
                    ptx::mbar_wait(mma_bar1, mma_phase1);
                    ptx::tc_fence_after();
                    epi(1);
                }
                mma_phase ^= 1;
                mma_phase1 ^= 1;
                ptx::tc_fence_before();
                fence_proxy_async_smem();
                __syncthreads();
                continue;
            }
            if (threadIdx.x == 0) {
                ptx::tc_fence_after();
                // the two matrices' K steps interleaved: two independent accumulation chains in
                // flight (each MMA of a chain waits for the previous one's accumulator)
                const uint32_t a0 = ptx::smem_u32(smem + st.slot_a), b0 = ptx::smem_u32(smem + st.slot_b);
                const uint64_t ad0 = ptx::smem_desc_sw128_kmajor(a0), bd0 = ptx::smem_desc_sw128_kmajor(b0);
                constexpr uint64_t kMatDesc = static_cast<uint64_t>(L::kPerMatrix >> 4);   // next matrix
                constexpr uint64_t kLoDesc = static_cast<uint64_t>(kSlotBytes >> 4);       // lo part
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t koff = static_cast<uint64_t>((k * 32) >> 4);
#pragma unroll
                    for (int mm = 0; mm < 2; ++mm) {
                        const uint64_t ad = ad0 + mm * kMatDesc + koff, bd = bd0 + mm * kMatDesc + koff;
                        const uint32_t d = tmem + (static_cast<uint32_t>(16 * mm) << 16);
                        ptx::mma_f16(d, ad, bd, kIdesc, k != 0);
                        if constexpr (kSplit) {
                            ptx::mma_f16(d, ad, bd + kLoDesc, kIdesc, 1u);
                            ptx::mma_f16(d, ad + kLoDesc, bd, kIdesc, 1u);
                        }
                    }
                }
                ptx::mma_commit(mma_bar);
                if (kDebug) t_i = clock64();
                ptx::mbar_wait(mma_bar, mma_phase);    // only the issuer polls; the rest sleep in bar.sync
                ptx::tc_fence_before();
            }
            mma_phase ^= 1;
            __syncthreads();
            ptx::tc_fence_after();
            const long long t_b = kDebug ? clock64() : 0;

            if (st.final_mode == 0) {
                // chain product: (alpha acc + beta D) s, the operand scale s (a power of two,
                // compute_scales) folded into alpha and beta exactly; in place (the MMA that read
                // the slots has completed).  Warp (q, h) runs quadrant q's epilogue of matrix h: only
                // the upper 8x8 blocks, each written with its transpose (every product exactly
                // symmetric, R20); the quadrant's 9 block pairs are the same count for every SMSP.
                const float2 alpha = make_float2(st.alpha * st.out_scale, st.alpha * st.out_scale);
                const float2 beta = make_float2(st.beta * st.out_scale, st.beta * st.out_scale);
                const bool has_d = st.slot_d >= 0;
                const uint32_t pd = smem_base + static_cast<uint32_t>(has_d ? st.slot_d : 0);
                const uint32_t po = smem_base + static_cast<uint32_t>(st.slot_out);
                const int mm = kQW == 2 ? hw : -1;       // 8 warps: one matrix per warp; 4 warps: both
                switch (q) {
                    case 0: chain_epilogue<kSplit, 0>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                    case 1: chain_epilogue<kSplit, 1>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                    case 2: chain_epilogue<kSplit, 2>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                    default: chain_epilogue<kSplit, 3>(tmem, mm, pd, po, L::kPerMatrix, has_d, alpha, beta, lane, diag_mask); break;
                }
                const long long t_c = kDebug ? clock64() : 0;
                ptx::tc_fence_before();
                fence_proxy_async_smem();
                __syncthreads();
                if (kDebug && plan.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
                    const long long t_d = clock64();
                    atomicAdd(plan.dbg + 0, static_cast<unsigned long long>(t_i - t_a));   // MMA issue
                    atomicAdd(plan.dbg + 1, static_cast<unsigned long long>(t_b - t_i));   // MMA completion wait + barrier
                    atomicAdd(plan.dbg + 2, static_cast<unsigned long long>(t_c - t_b));   // epilogue (warp 0)
                    atomicAdd(plan.dbg + 4, static_cast<unsigned long long>(t_d - t_c));   // fences + barrier
                    atomicAdd(plan.dbg + 3, 1ull);
                }
            } else {
                const long long t_f = kDebug ? clock64() : 0;
                // final: P = lambda~ alpha acc + beta X  (mode 1, R5)  or
                //        S = alpha acc + beta D          (mode 2; the sign output)
                // computed on this row's upper part (row per thread, 32 columns, 32x32b loads), staged
                // as fp32 in the (consumed) operand region, and stored whole: the lower part is read
                // back transposed (exact symmetry)
                float* stage = reinterpret_cast<float*>(mat);          // 64 x 64 fp32, float4-swizzled
                float4* srow = reinterpret_cast<float4*>(stage + row * kN);
                const bool live = kCT * hw + kCT - 1 >= 16 * q;       // columns at or right of the quadrant's rows
                auto stage_at = [&](int r, int c) -> float {
                    return stage[r * kN + (((c >> 2) ^ (r & 15)) << 2) + (c & 3)];
                };
                auto store_staged = [&](float* dst) {                  // after a barrier
                    // coalesced: per instruction lanes 0-15 write one row of matrix 0, lanes 16-31
                    // the same row of matrix 1; the lower part is the transpose of the upper
                    if (!valid) return;
                    const int cl = lane & 15;
                    const int c4 = 4 * cl;
#pragma unroll 4
                    for (int i = 0; i < kRW; ++i) {
                        const int r = 16 * q + kRW * hw + i;
                        if (r >= n) break;
                        float* orow = dst + static_cast<int64_t>(b) * n * n + static_cast<int64_t>(r) * n;
                        if (vec) {
                            if (c4 < n) {
                                float4 o = reinterpret_cast<const float4*>(stage)[r * 16 + (cl ^ (r & 15))];
                                if (c4 + 0 < r) o.x = stage_at(c4 + 0, r);
                                if (c4 + 1 < r) o.y = stage_at(c4 + 1, r);
                                if (c4 + 2 < r) o.z = stage_at(c4 + 2, r);
                                if (c4 + 3 < r) o.w = stage_at(c4 + 3, r);
                                __stcs(reinterpret_cast<float4*>(orow + c4), o);
                            }
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (c4 + e < n) orow[c4 + e] = (c4 + e >= r) ? stage_at(r, c4 + e) : stage_at(c4 + e, r);
                        }
                    }
                };
                if (st.final_mode == 1) {
                    // the epilogue reads no operand slot: staging may start at once (the MMA has
                    // completed).  ADMM: X_next = sigma (P - M) first, then P; both from
                    // the accumulator and the input rows kept in TMEM.
                    const float lamf = static_cast<float>(lam);
#pragma unroll 1
                    for (int pass = plan.out2 ? 1 : 0; pass >= 0; --pass) {
                        if (live) {
#pragma unroll
                            for (int h = 0; h < kCT / 16; ++h) {
                                uint32_t r[16], xh[16];
                                asm volatile(
                                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                                    : "r"(tmem_row + kCT * hw + 16 * h));
                                asm volatile(
                                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                                    : "=r"(xh[0]), "=r"(xh[1]), "=r"(xh[2]), "=r"(xh[3]), "=r"(xh[4]), "=r"(xh[5]), "=r"(xh[6]), "=r"(xh[7]),
                                      "=r"(xh[8]), "=r"(xh[9]), "=r"(xh[10]), "=r"(xh[11]), "=r"(xh[12]), "=r"(xh[13]), "=r"(xh[14]), "=r"(xh[15])
                                    : "r"(tmem_x + 16 * h));
                                ptx::tmem_ld_wait();
#pragma unroll
                                for (int qq = 0; qq < 4; ++qq) {
                                    float o[4];
#pragma unroll
                                    for (int e = 0; e < 4; ++e) {
                                        const float x = __uint_as_float(xh[4 * qq + e]);
                                        const float p = lamf * (st.alpha * __uint_as_float(r[4 * qq + e])) + st.beta * x;
                                        o[e] = pass == 1 ? plan.sigma2 * (p - x) : p;
                                    }
                                    srow[((kCT / 4) * hw + 4 * h + qq) ^ (row & 15)] = make_float4(o[0], o[1], o[2], o[3]);
                                }
                            }
                        }
                        __syncthreads();
                        store_staged(pass == 0 ? out : plan.out2);
                        __syncthreads();
                    }
                } else {
                    float v[kCT];
                    if (live) {
#pragma unroll
                        for (int h = 0; h < kCT / 32; ++h) {
                            uint32_t r[32];
                            ptx::tmem_ld_32x32b_x32(tmem_row + kCT * hw + 32 * h, r);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[32 * h + i] = st.alpha * __uint_as_float(r[i]);
                        }
                        if (st.slot_d >= 0) {
#pragma unroll
                            for (int jj = 0; jj < kCT / 8; ++jj) {
                                float2 d[4];
                                load_operand8<kSplit>(mat + st.slot_d, rbase + ((((kCT / 8) * hw + jj) ^ rx) << 4), d);
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    v[8 * jj + 2 * e] += st.beta * d[e].x;
                                    v[8 * jj + 2 * e + 1] += st.beta * d[e].y;
                                }
                            }
                        }
                    }
                    __syncthreads();             // every operand read is done: staging may overwrite
                    if (live) {
#pragma unroll
                        for (int qq = 0; qq < kCT / 4; ++qq)
                            srow[((kCT / 4) * hw + qq) ^ (row & 15)] = make_float4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
                    }
                    __syncthreads();
                    store_staged(out);
                    __syncthreads();
                }
                if (kDebug && plan.dbg && blockIdx.x == 0 && threadIdx.x == 0)
                    atomicAdd(plan.dbg + 6, static_cast<unsigned long long>(clock64() - t_f + (t_b - t_a)));   // final product
                ptx::tc_fence_before();
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<128>(tmem);
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
    int per_sm = kSmallCtasPerSm<kSplit>;
    if (const char* v = debug_env("PSD_SMALL_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(v)));   // A/B only
    int grid = per_sm * num_sms;
    if (grid > pairs) grid = pairs;
    small_batch_kernel<kSplit><<<grid, 32 * kWarpsS<kSplit>, L::kBytes, stream>>>(X, out, n, batch, lambda_out, status, plan);
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
