// sym_gemm.cu -- symmetric product C = alpha * (A B) + beta * D on sm_100a tensor cores, 128x128
// upper tiles: the path for small and few-tile problems (configs c1 padded, c3: one n = 1024).
//
// Every product of the composite filter (Algorithm 2) multiplies two commuting
// symmetric matrices (powers/polynomials of the same X), so C is symmetric: only
// upper tiles (I <= J) are computed.  A and B are symmetric, so both operands are read as row
// panels: K-major from the stored tiles, or -- with upper-only storage (GemmShape::upper_only,
// 16-bit operands), where each tile is stored once and only the 128x128 diagonal blocks whole --
// transposed (MN-major, 64 x 64 TMA boxes) left of the row block's diagonal block.  Tiles
// (128 x 128, or 128 x 64 for few-tile problems) meeting the diagonal are stored mirrored.
//
// A cluster of KS CTAs (KS = 1, 2, 4; cluster split-K) owns one 128x128 upper tile:
//   warp 0 / elected lane : TMA producer over this CTA's K slice -> kStages smem ring
//   warp 1 / elected lane : tcgen05.mma.cta_group::1 (M = N = 128) into TMEM
//   KS = 1 : warps 0-7 run the epilogue straight from TMEM (tcgen05.ld 32x32b): warps w and w + 4
//            share TMEM lane quadrant w % 4 and take alternate 32-column chunks
//   KS > 1 : every CTA parks its partial accumulator in its own (now idle) ring smem; after a
//            cluster barrier CTA k sums rows [k*128/KS, (k+1)*128/KS) over the KS partials with
//            ld.shared::cluster (DSMEM) and runs the epilogue for those rows -- KS x more SMs
//            busy on few-tile problems (n = 1024: 36 tiles -> 144 CTAs) and a KS x shorter
//            epilogue per CTA.
// Launched with programmatic dependent launch: the prologue (barrier init, TMEM alloc,
// descriptor prefetch) overlaps the previous kernel; griddepcontrol.wait precedes any read of
// the previous kernel's outputs.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "epilogue.cuh"
#include "kernels.h"
#include "optraits.cuh"
#include "ptx.cuh"

namespace psd {

namespace {

constexpr int kWarps = 8;                       // producer, MMA issuer; all 8 run the epilogue
constexpr int kThreads = 32 * kWarps;
constexpr int kTileBytes = kTile * kBlockKBytes;                 // 16 KB per operand tile
constexpr int kRingBytes1 = 128 * 1024;
template <bool kSplit, int BN> struct Ring1 {
    static constexpr int kBBytes = BN * kBlockKBytes;                   // B tile: BN rows
    static constexpr int kStageBytes = (kSplit ? 2 : 1) * (kTileBytes + kBBytes);   // A, B (+ A_lo, B_lo)
    static constexpr int kStages = kRingBytes1 / kStageBytes;
};
constexpr int kSmemBytes = kRingBytes1 + 1024 + 256 + kWarps * kEpiWarpSmemBytes;  // ring, align, barriers, staging
// cluster split-K with KS = 2: the peer's partial of this CTA's half of the tile rows (64 x BN fp32)
template <int KS, int BN> constexpr int kRecvBytes = KS == 2 ? 64 * BN * 4 : 0;
template <int KS, int BN> constexpr int kSmemBytesKs = kSmemBytes + kRecvBytes<KS, BN>;

// receive-buffer layout: row r (0..63) of BN fp32, float4 column q stored at q ^ (r & 15) -- the 8 lanes
// of a 128-bit access phase (8 consecutive rows, same q) hit 8 different 16-byte bank groups
template <int BN>
__device__ __forceinline__ uint32_t recv_off(int r, int q) {
    return static_cast<uint32_t>((r * (BN / 4) + (q ^ (r & 15))) * 16);
}

// 16 bytes into a peer CTA's shared memory, completion counted on the peer's mbarrier (bytes)
__device__ __forceinline__ void st_async_v4(uint32_t cluster_addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                 :: "r"(cluster_addr), "r"(a), "r"(b), "r"(c), "r"(d), "r"(cluster_bar) : "memory");
}

// Row-major enumeration of the 128 x BN tiles (row block I, column block J) that hold any
// upper-triangle element: J >= I * (128 / BN).
template <int BN>
__device__ __forceinline__ void upper_tile_coords(int t, int npad, int& I, int& J) {
    constexpr int r = kTile / BN;
    const int ncb = npad / BN;
    int i = 0;
    int rem = t;
    while (rem >= ncb - i * r) { rem -= ncb - i * r; ++i; }
    I = i;
    J = i * r + rem;
}

// Tile t of this launch (GemmShape::sub_mode) -> (I, J) in 128-row / BN-column units of the npad matrix
template <int BN>
__device__ __forceinline__ void tile_coords(const GemmShape& s, int t, int& I, int& J) {
    if (s.sub_mode == 0) {
        upper_tile_coords<BN>(t, s.npad, I, J);
    } else if (s.sub_mode == 3) {                  // upper tiles of the top-left sub_m block
        upper_tile_coords<BN>(t, s.sub_m, I, J);
    } else if (s.sub_mode == 1) {                  // upper tiles of the bottom-right sub_m block
        upper_tile_coords<BN>(t, s.sub_m, I, J);
        I += s.sub_m / kTile;
        J += s.sub_m / BN;
    } else {                                       // every tile of the top-right sub_m block
        const int ncb = s.sub_m / BN;
        I = t / ncb;
        J = ncb + t % ncb;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define DBG_STAMP(i) do { if (kDebug && e.dbg && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) e.dbg[i] = gtimer(); } while (0)
// every CTA's thread 0: [0] start, [1] after griddepcontrol.wait, [2] accumulator complete, [3] end,
// [4] / [5] before / after its first epilogue_chunk (0 if thread 0 runs none), [6] after the final barrier
#define DBG_ALL(i) do { if (kDebug && e.dbg_all && threadIdx.x == 0) \
    e.dbg_all[8 * (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) + (i)] = gtimer(); } while (0)

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// partial-accumulator layout in smem: row-major 128 x 128 fp32, float4 column q of row r stored at
// q ^ (r & 31) so that 32 lanes reading 32 different rows at the same q hit 32 different banks
__device__ __forceinline__ uint32_t part_off(int r, int q) {
    return static_cast<uint32_t>((r * 32 + (q ^ (r & 31))) * 16);
}

__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t cluster_addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(cluster_addr) : "memory");
    return v;
}

template <OpType T, bool kSplit, int KS, int BN>
__global__ void __launch_bounds__(kThreads, 1)
sym_gemm_kernel(const __grid_constant__ OperandMaps tm, const GemmShape s, const EpiParams e) {
    using Tr = OpTraits<T>;
    constexpr int kStages = Ring1<kSplit, BN>::kStages;
    constexpr int kStageBytes = Ring1<kSplit, BN>::kStageBytes;
    constexpr int kBBytes = Ring1<kSplit, BN>::kBBytes;
    constexpr int kBK = kBlockKBytes / Tr::kBytes;     // K elements per block (64 f16 / 32 tf32)
    constexpr int kUmmaK = 32 / Tr::kBytes;            // K per tcgen05.mma (16 f16 / 8 tf32)
    constexpr uint32_t kIdesc = ptx::make_idesc(Tr::kFmt, kTile, BN);
    // split precisions (KS = 1): the K range is cut into up to 512 / BN runs, each accumulated from
    // zero in its own TMEM columns and summed round-to-nearest in the epilogue (GemmShape::kchunk)
    // (single pass: two runs of npad / 2 when the planner sets kchunk = npad / 2, the K split of the
    // KS = 2 cluster launch, so batch sizes that do and do not take the cluster agree bitwise)
    constexpr bool kRuns = KS == 1;
    constexpr uint32_t kCols = kRuns ? 512 : BN;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint8_t* ring = smem;                                         // stage: A | B | A_lo | B_lo
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes1);
    uint64_t* empty = full + kStages;
    uint64_t* accum_full = empty + kStages;
    uint64_t* recv_bar = accum_full + 1;                          // KS == 2: the peer's partial landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);
    uint8_t* epi_smem = smem + kRingBytes1 + 256;                   // kWarps x kEpiWarpSmemBytes
    uint8_t* recv = epi_smem + kWarps * kEpiWarpSmemBytes;          // KS == 2: kRecvBytes

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    const int krank = (KS > 1) ? static_cast<int>(ptx::cluster_ctarank()) : 0;
    int I, J;
    tile_coords<BN>(s, blockIdx.x / KS, I, J);
    DBG_STAMP(0);
    DBG_ALL(0);

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::tma_prefetch_desc(&tm.a);
            ptx::tma_prefetch_desc(&tm.b);
            for (int i = 0; i < kStages; ++i) {
                ptx::mbar_init(&full[i], 1);
                ptx::mbar_init(&empty[i], 1);
            }
            ptx::mbar_init(accum_full, 1);
            if constexpr (KS == 2) {
                // phase 0 completes when the peer's kRecvBytes have landed (its st.async complete_tx)
                ptx::mbar_init(recv_bar, 1);
                ptx::mbar_arrive_expect_tx(recv_bar, kRecvBytes<KS, BN>);
            }
            ptx::fence_barrier_init();
        }
        __syncwarp();
    } else if (warp == 1) {
        ptx::tmem_alloc<kCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if constexpr (KS == 2) ptx::cluster_sync();      // both CTAs' recv_bar initialised before any st.async
    const uint32_t tmem_base = *tmem_slot;
    DBG_STAMP(1);
    grid_dep_wait();                                  // the operands are the previous kernel's output
    DBG_STAMP(2);
    DBG_ALL(1);

    const int kbeg = s.k_begin / kBK;                 // K range (whole npad unless sub_mode products)
    const int kend = (s.k_end > 0 ? s.k_end : s.npad) / kBK;
    const int num_kb = (kend - kbeg) / KS;            // this CTA's K slice
    const int kb0 = kbeg + krank * num_kb;
    const int rowA = b * s.npad + I * kTile;
    const int rowB = b * s.npad + J * BN;
    int nruns = 1;
    if (kRuns && s.kchunk > 0) nruns = min(static_cast<int>(kCols / BN), ((kend - kbeg) * kBK + s.kchunk - 1) / s.kchunk);
    const int run_kb = (num_kb + nruns - 1) / nruns;    // K blocks per accumulation run
    nruns = (num_kb + run_kb - 1) / run_kb;

    if (warp == 0) {
        if (ptx::elect_one()) {
            const uint64_t pol = ptx::policy_evict_last();
            int st = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < num_kb; ++kb, st = (st + 1 == kStages) ? 0 : st + 1, ph ^= (st == 0)) {
                ptx::mbar_wait(&empty[st], ph ^ 1);
                uint8_t* sa = ring + st * kStageBytes;
                const int kx = (kb0 + kb) * kBK;
                ptx::mbar_arrive_expect_tx(&full[st], kStageBytes);
                // upper-only storage (16-bit, no split-K): left of the 128-row block's diagonal block a
                // panel is the stored upper block transposed -- 64 x 64 boxes read as an MN-major operand
                auto load = [&](uint8_t* dst, const CUtensorMap* mk, const CUtensorMap* mt, int rows, int row0,
                                int diag0, int row) {
                    if (Tr::kBytes == 2 && s.upper_only && kx < diag0) {
                        for (int c = 0; c < rows; c += 64)
                            ptx::tma_load_2d(dst + c * kBlockKBytes, mt, &full[st], row0 + c, b * s.npad + kx, pol);
                    } else {
                        ptx::tma_load_2d(dst, mk, &full[st], kx, row, pol);
                    }
                };
                const int jdiag = (J * BN / kTile) * kTile;          // 128-row block holding B's rows
                load(sa, &tm.a, &tm.a_t, kTile, I * kTile, I * kTile, rowA);
                load(sa + kTileBytes, &tm.b, &tm.b_t, BN, J * BN, jdiag, rowB);
                if constexpr (kSplit) {
                    load(sa + kTileBytes + kBBytes, &tm.a_lo, &tm.a_lo_t, kTile, I * kTile, I * kTile, rowA);
                    load(sa + 2 * kTileBytes + kBBytes, &tm.b_lo, &tm.b_lo_t, BN, J * BN, jdiag, rowB);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (ptx::elect_one()) {
            // the issue loop is the mainloop's critical path at N = 64 (4 MMAs = 192 tensor cycles per
            // K block): ring position, run position and the MN-major switch are kept as counters and
            // bounds instead of per-block divisions (tools/micro/tma_ingress.cu: the same pipeline with
            // a lean issue loop runs a K block in ~280 cycles)
            const bool up = Tr::kBytes == 2 && s.upper_only;
            const int a_mn_end = up ? I * kTile : 0;                      // kx below: MN-major (transposed)
            const int b_mn_end = up ? (J * BN / kTile) * kTile : 0;
            const uint32_t ring0 = ptx::smem_u32(ring);
            int st = 0, kr = 0, run = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < num_kb; ++kb) {
                ptx::mbar_wait(&full[st], ph);
                ptx::tc_fence_after();
                const uint32_t sa = ring0 + static_cast<uint32_t>(st * kStageBytes);
                const int kx = (kb0 + kb) * kBK;
                const bool a_mn = kx < a_mn_end;
                const bool b_mn = kx < b_mn_end;
                // MN-major (transposed) operands: 64-element MN chunks 8 KB apart, 8-row K groups 1 KB
                // apart, one K step of 16 = 2 KB (tools/micro/mn_major.cu)
                auto desc = [&](uint32_t addr, bool mn) {
                    return mn ? ptx::smem_desc_sw128_mnmajor(addr, 8192, 1024) : ptx::smem_desc_sw128_kmajor(addr);
                };
                const uint64_t adesc = desc(sa, a_mn);
                const uint64_t bdesc = desc(sa + kTileBytes, b_mn);
                const uint32_t idesc = kIdesc | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u);
                const uint64_t astep = a_mn ? (2048 >> 4) : (32 >> 4), bstep = b_mn ? (2048 >> 4) : (32 >> 4);
                auto mma = [&](uint32_t d, uint64_t a, uint64_t bb, uint32_t accumulate) {
                    if constexpr (T == OpType::TF32)
                        ptx::mma_tf32(d, a, bb, kIdesc, accumulate);
                    else
                        ptx::mma_f16(d, a, bb, idesc, accumulate);
                };
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(run * BN);
#pragma unroll
                for (int k = 0; k < kBK / kUmmaK; ++k) {
                    mma(d_tmem, adesc + k * astep, bdesc + k * bstep, (kr | k) != 0);
                    if constexpr (kSplit) {
                        const uint64_t alo = desc(sa + kTileBytes + kBBytes, a_mn);
                        const uint64_t blo = desc(sa + 2 * kTileBytes + kBBytes, b_mn);
                        mma(d_tmem, adesc + k * astep, blo + k * bstep, 1u);    // A_hi B_lo
                        mma(d_tmem, alo + k * astep, bdesc + k * bstep, 1u);    // A_lo B_hi
                    }
                }
                ptx::mma_commit(&empty[st]);
                if (++st == kStages) { st = 0; ph ^= 1; }
                if (++kr == run_kb) { kr = 0; ++run; }            // next accumulation run (split precisions)
            }
            ptx::mma_commit(accum_full);
        }
        __syncwarp();
    }

    // ------------------------------------------------------------------ epilogue
    ptx::mbar_wait(accum_full, 0);
    ptx::tc_fence_after();
    DBG_STAMP(3);
    DBG_ALL(2);
    grid_dep_launch();                               // the next kernel may start its prologue

    const bool diag = (I * kTile < J * BN + BN) && (J * BN < I * kTile + kTile);   // tile meets the diagonal
    float alpha = e.alpha;
    if (e.alpha_dev) alpha *= static_cast<float>(e.alpha_dev[b]);
    uint8_t* wsmem = epi_smem + warp * kEpiWarpSmemBytes;

    if constexpr (KS == 1) {
        const int quad = warp & 3;                  // TMEM lanes 32 quad .. (a warp reaches only its quadrant)
        const int gi0 = I * kTile + quad * 32;      // this warp's first row
#pragma unroll 1
        for (int c0 = (warp >> 2) * 32; c0 < BN; c0 += 64) {
            const int gj0 = J * BN + c0;
            if (diag && gj0 + 31 < gi0) continue;   // chunk below the diagonal for the whole warp
            uint32_t raw[32];
            const uint32_t tl = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + c0;
            ptx::tmem_ld_32x32b_x32(tl, raw);
            ptx::tmem_ld_wait();
            if constexpr (kRuns) {
                // the K runs in order, round-to-nearest fp32 adds
                for (int r = 1; r < nruns; ++r) {
                    uint32_t part[32];
                    ptx::tmem_ld_32x32b_x32(tl + static_cast<uint32_t>(r * BN), part);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        raw[i] = __float_as_uint(__fadd_rn(__uint_as_float(raw[i]), __uint_as_float(part[i])));
                }
            }
            if (c0 < 32) DBG_ALL(4);
            epilogue_chunk<T>(e, alpha, b, s.npad, gi0, gj0, diag, raw, wsmem);
            if (c0 < 32) DBG_ALL(5);
        }
    } else if constexpr (KS == 2) {
        // Push reduction: CTA k finishes rows [64k, 64k + 64) of the tile (TMEM quadrants 2k, 2k + 1).
        // The warps on the other two quadrants send this CTA's partial of the peer's rows straight into
        // the peer's receive buffer (st.async, counted on the peer's recv_bar) while the warps on this
        // CTA's own quadrants load their partial from TMEM, wait for the peer's, add the two in rank
        // order -- p0 + p1, the arithmetic of the single-CTA K-run sum -- and run the epilogue.  No parking
        // of the own partial, no cluster barrier after the mainloop, all 8 warps busy.
        const int quad = warp & 3;
        const int rr = (quad & 1) * 32 + lane;                 // row within a 64-row half
        const bool mine = (quad >> 1) == krank;
        if (!mine) {
            const uint32_t peer = static_cast<uint32_t>(krank ^ 1);
            const uint32_t rbuf = ptx::mapa_shared(ptx::smem_u32(recv), peer);
            const uint32_t rbar = ptx::mapa_shared(ptx::smem_u32(recv_bar), peer);
#pragma unroll 1
            for (int c0 = (warp >> 2) * 32; c0 < BN; c0 += 64) {
                uint32_t raw[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + c0, raw);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    st_async_v4(rbuf + recv_off<BN>(rr, c0 / 4 + q), raw[4 * q], raw[4 * q + 1], raw[4 * q + 2],
                                raw[4 * q + 3], rbar);
            }
        } else {
            const int gi0 = I * kTile + quad * 32;
            bool waited = false;
#pragma unroll 1
            for (int c0 = (warp >> 2) * 32; c0 < BN; c0 += 64) {
                const int gj0 = J * BN + c0;
                if (diag && gj0 + 31 < gi0) continue;
                uint32_t own[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + c0, own);
                ptx::tmem_ld_wait();
                if (!waited) {
                    ptx::mbar_wait(recv_bar, 0);
                    waited = true;
                }
                uint32_t raw[32];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(recv + recv_off<BN>(rr, c0 / 4 + q));
                    const float pv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float mine_v = __uint_as_float(own[4 * q + i]);
                        const float p0 = krank == 0 ? mine_v : pv[i];
                        const float p1 = krank == 0 ? pv[i] : mine_v;
                        raw[4 * q + i] = __float_as_uint(__fadd_rn(p0, p1));
                    }
                }
                if (c0 < 32) DBG_ALL(4);
                epilogue_chunk<T>(e, alpha, b, s.npad, gi0, gj0, diag, raw, wsmem);
                if (c0 < 32) DBG_ALL(5);
            }
            // a CTA must not exit while the peer's st.async into its receive buffer is in flight
            if (!waited) ptx::mbar_wait(recv_bar, 0);
        }
    } else {
        // park this CTA's partial accumulator (all MMAs done -> the ring is free)
        const int r = (warp & 3) * 32 + lane;
#pragma unroll 1
        for (int c0 = (warp >> 2) * 32; c0 < BN; c0 += 64) {
            uint32_t raw[32];
            ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + c0, raw);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 8; ++q)
                *reinterpret_cast<uint4*>(ring + part_off(r, c0 / 4 + q)) =
                    make_uint4(raw[4 * q], raw[4 * q + 1], raw[4 * q + 2], raw[4 * q + 3]);
        }
        ptx::cluster_sync();
        // CTA k reduces row groups [k * 4/KS, (k+1) * 4/KS) x BN/32 column chunks; warp w takes chunks w, w+8, ..
        constexpr int kGroups = 4 / KS;
        constexpr int kCC = BN / 32;                 // 32-column chunks of the tile
        const uint32_t ring_u = ptx::smem_u32(ring);
        uint32_t peer[KS];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) peer[kk] = ptx::mapa_shared(ring_u, static_cast<uint32_t>(kk));
#pragma unroll 1
        for (int ch = warp; ch < kGroups * kCC; ch += kWarps) {
            const int rg = krank * kGroups + ch / kCC;
            const int cc = ch % kCC;
            const int gi0 = I * kTile + rg * 32;
            const int gj0 = J * BN + cc * 32;
            if (diag && gj0 + 31 < gi0) continue;
            const int row = rg * 32 + lane;
            float acc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = 0.0f;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 v = ld_dsmem_f4(peer[kk] + part_off(row, cc * 8 + q));
                    acc[4 * q] += v.x;
                    acc[4 * q + 1] += v.y;
                    acc[4 * q + 2] += v.z;
                    acc[4 * q + 3] += v.w;
                }
            }
            uint32_t raw[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) raw[i] = __float_as_uint(acc[i]);
            epilogue_chunk<T>(e, alpha, b, s.npad, gi0, gj0, diag, raw, wsmem);
        }
        ptx::cluster_sync();                         // peers' partials stay valid until all read
    }

    DBG_STAMP(4);
    ptx::tc_fence_before();
    __syncthreads();
    DBG_ALL(6);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kCols>(tmem_base);
    }
    DBG_STAMP(5);
    DBG_ALL(3);
}

template <OpType T, bool kSplit, int KS, int BN>
cudaError_t launch_t(const OperandMaps& m, const GemmShape& s, const EpiParams& e, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t err = cudaFuncSetAttribute(sym_gemm_kernel<T, kSplit, KS, BN>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytesKs<KS, BN>);
        if (err != cudaSuccess) return err;
        attr_set = true;
    }
    const int edge = s.sub_mode ? s.sub_m : s.npad;
    const int nrb = edge / kTile, ncb = edge / BN;
    const int tiles = s.sub_mode == 2 ? nrb * ncb : nrb * ncb - (kTile / BN) * nrb * (nrb - 1) / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(tiles * KS, s.batch);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytesKs<KS, BN>;
    cfg.stream = stream;
    cudaLaunchAttribute attrs[2];
    int na = 0;
    static const bool pdl = !debug_env("PSD_NO_PDL");
    if (pdl) {
        attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (KS > 1) {
        attrs[na].id = cudaLaunchAttributeClusterDimension;
        attrs[na].val.clusterDim.x = KS;
        attrs[na].val.clusterDim.y = 1;
        attrs[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, sym_gemm_kernel<T, kSplit, KS, BN>, m, s, e);
}

template <OpType T, bool kSplit>
cudaError_t launch_ks(int ks, int bn, const OperandMaps& m, const GemmShape& s, const EpiParams& e,
                      cudaStream_t stream) {
    if (bn == 64) return ks == 2 ? launch_t<T, kSplit, 2, 64>(m, s, e, stream) : launch_t<T, kSplit, 1, 64>(m, s, e, stream);
    switch (ks) {
        case 4: return launch_t<T, kSplit, 4, kTile>(m, s, e, stream);
        case 2: return launch_t<T, kSplit, 2, kTile>(m, s, e, stream);
        default: return launch_t<T, kSplit, 1, kTile>(m, s, e, stream);
    }
}

}  // namespace

// Split-K factor for a few-tile problem.  KS = 2 (a cluster of two CTAs per tile, each accumulating
// one K half; the halves meet through the st.async push reduction) is taken when the CTA pairs fill
// at most one wave AND the K range is exactly two accumulation chunks (npad == 2 kchunk), so each CTA
// accumulates one chunk from zero and the reduction adds the two in order -- the arithmetic of the
// single-CTA K-run sum (bit-identical; the planner sets kchunk = npad / 2 for the single-pass 1-CTA
// path at npad = 1024).  Measured at c3 (n = 1024, 19 products; profiles/r2s3/push/): fp16 KS = 1 149
// vs KS = 2 142 us (debug build), fp16x3 229 -> 197 us and tf32x3 328 -> 295 us with the push
// reduction (the round-2 DSMEM pull reduction had made single-pass KS = 2 slower: 175 vs 154 us).
int sym_gemm_split_k(int npad, int batch, OpType t, bool split, int kchunk) {
    static const int forced = debug_env("PSD_SPLITK") ? std::atoi(debug_env("PSD_SPLITK")) : 0;
    if (forced == 1 || forced == 2 || forced == 4) return forced;
    (void)t;
    (void)split;
    if (kchunk <= 0 || npad != 2 * kchunk) return 1;
    const int bn = sym_gemm_bn(npad, batch);
    const int nrb = npad / kTile, ncb = npad / bn;
    const int tiles = (nrb * ncb - (kTile / bn) * nrb * (nrb - 1) / 2) * batch;
    return tiles * 2 <= 148 ? 2 : 1;
}

// 128 x 64 tiles for few-tile problems: twice the CTAs, half the MMA and epilogue per CTA.
int sym_gemm_bn(int npad, int batch) {
    static const int forced = debug_env("PSD_BN") ? std::atoi(debug_env("PSD_BN")) : 0;
    if (forced == 64 || forced == 128) return forced;
    const int nt = npad / kTile;
    return (nt * (nt + 1) / 2 * batch < 100) ? 64 : 128;
}

cudaError_t launch_sym_gemm(OpType t, bool split, const OperandMaps& m, const GemmShape& s, const EpiParams& e,
                            cudaStream_t stream) {
    const int ks = s.sub_mode ? 1 : sym_gemm_split_k(s.npad, s.batch, t, split, s.kchunk);
    const int bn = sym_gemm_bn(s.npad, s.batch);
    switch (t) {
        case OpType::F16: return split ? launch_ks<OpType::F16, true>(ks, bn, m, s, e, stream)
                                       : launch_ks<OpType::F16, false>(ks, bn, m, s, e, stream);
        case OpType::BF16: return split ? launch_ks<OpType::BF16, true>(ks, bn, m, s, e, stream)
                                        : launch_ks<OpType::BF16, false>(ks, bn, m, s, e, stream);
        case OpType::TF32: return split ? launch_ks<OpType::TF32, true>(ks, bn, m, s, e, stream)
                                        : launch_ks<OpType::TF32, false>(ks, bn, m, s, e, stream);
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

bool make_operand_tmap(CUtensorMap* map, const void* base, OpType t, int npad, int batch, int box_rows) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const int bytes = (t == OpType::TF32) ? 4 : 2;
    const CUtensorMapDataType dt = (t == OpType::F16) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                 : (t == OpType::BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(npad), static_cast<cuuint64_t>(npad) * batch};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(npad) * bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBlockKBytes / bytes), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace psd
