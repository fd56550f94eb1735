// sym_gemm_2cta.cu -- persistent CTA-pair (cta_group::2) symmetric product for large n.
//
// Same product and epilogue as sym_gemm.cu (C = alpha A B + beta D over upper tiles;
// Algorithm 2's products), re-tiled for full tensor-core
// rate on sm_100a:
//   * a cluster of 2 CTAs (one TPC) owns a 256 x 256 upper output tile; tcgen05.mma
//     .cta_group::2 with M = 256, N = 256, K = 16: CTA r holds A rows [r*128, r*128+128)
//     and B^T rows [r*128, r*128+128) of the tile in its smem, and the accumulator rows
//     [r*128, +128) x 256 columns in its TMEM -- half the operand bytes per CTA of a 1-SM
//     tile of the same size (64 B/clk/SM of L2->SMEM traffic at full MMA rate);
//   * persistent: grid = 2 x (#SMs / 2); cluster c walks tiles c, c + #clusters, ...;
//   * warp roles: w0 TMA producer, w1 MMA issuer (leader CTA only), w2 TMEM allocator,
//     w4..w7 epilogue (one TMEM lane quadrant each);
//   * TMEM holds two 256-column fp32 accumulators (all 512 columns), so the epilogue of
//     tile i overlaps the mainloop of tile i+1; split precisions instead use columns [0, 256) for
//     K-chunk runs (accumulated from zero every GemmShape::kchunk K elements) and [256, 512) for
//     their round-to-nearest sum, folded by the epilogue warps while the next run accumulates;
//   * kStages-deep smem ring, 32 KB per stage per CTA (A 16 KB + B 16 KB, SW128);
//   * dynamic tile scheduler: the leader's producer takes tile ids from a global counter and
//     broadcasts them to both CTAs through an mbarrier-guarded smem ring;
//   * upper-only operand storage (GemmShape::upper_only, 16-bit): K blocks left of a row block's
//     diagonal tile are loaded transposed (two 64 x 64 boxes of the stored upper tile) and fed to
//     tcgen05 as MN-major operands; the epilogue then skips the mirror of off-diagonal tiles.
#include "epilogue.cuh"
#include "kernels.h"
#include "optraits.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <cstdlib>
#include <string>

namespace psd {

namespace {

constexpr int kT2 = 256;                       // output tile edge per CTA pair
constexpr int kRowsPerCta = 128;
constexpr int kThreads2 = 256;                 // 8 warps
constexpr int kRingBytes = 192 * 1024;         // operand ring per CTA
// stage = A + B halves (32 KB), or A_hi, B_hi, A_lo, B_lo for split precision (64 KB)
template <bool kSplit> struct Ring2 {
    static constexpr int kStageBytes = (kSplit ? 4 : 2) * kRowsPerCta * kBlockKBytes;
    static constexpr int kStages = kRingBytes / kStageBytes;   // 6 or 3
};
constexpr int kSmem2 = kRingBytes + 1024 + 512 + 4 * kEpiWarpSmemBytes;  // ring, align, barriers+ids, staging
constexpr uint32_t kTmemCols = 512;            // 2 accumulators x 256 fp32 columns

__device__ __forceinline__ void decode_tile(int t, const GemmShape& s, int& b, int& I, int& J) {
    b = t / s.tiles_per_matrix;
    const uint32_t code = __ldg(s.tiles + (t - b * s.tiles_per_matrix));
    I = static_cast<int>(code >> 16);
    J = static_cast<int>(code & 0xFFFFu);
}

template <OpType T, bool kSplit>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
sym_gemm_2cta_kernel(const __grid_constant__ OperandMaps tm, const GemmShape s, const EpiParams e) {
    using Tr = OpTraits<T>;
    constexpr int kStages2 = Ring2<kSplit>::kStages;
    constexpr int kStageBytes = Ring2<kSplit>::kStageBytes;
    constexpr int kBK = kBlockKBytes / Tr::kBytes;
    constexpr int kUmmaK = 32 / Tr::kBytes;
    constexpr uint32_t kIdesc = ptx::make_idesc(Tr::kFmt, kT2, kT2);
    constexpr int kTileBytes1 = kRowsPerCta * kBlockKBytes;   // 16 KB
    constexpr int kRing = 4;                                  // tile-id ring depth
    // consumers of each tile id that release a ring slot (arrivals on the leader's tile_empty):
    // leader MMA thread, 4 leader epilogue warps, peer producer, 4 peer epilogue warps
    constexpr uint32_t kTileConsumers = 10;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = ptx::align_smem_1024(smem_raw);
    uint8_t* ring = smem;                                       // stage st: A at +0, B at +16 KB
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes);
    uint64_t* empty = full + kStages2;
    uint64_t* tmem_full = empty + kStages2;                     // [2]
    uint64_t* tmem_empty = tmem_full + 2;                       // [2]
    uint64_t* tile_full = tmem_empty + 2;                       // [kRing]
    uint64_t* tile_empty = tile_full + kRing;                   // [kRing]
    uint32_t* tile_id = reinterpret_cast<uint32_t*>(tile_empty + kRing);   // [kRing]
    uint32_t* tmem_slot = tile_id + kRing;
    uint8_t* epi_smem = smem + kRingBytes + 512;                // 4 x kEpiWarpSmemBytes

    const int warp = threadIdx.x >> 5;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = (rank == 0);
    const int total_tiles = s.tiles_per_matrix * s.batch;
    const int kbeg = s.k_begin / kBK;                 // K range (whole npad unless psd_polar's block products)
    const int num_kb = (s.k_end > 0 ? s.k_end : s.npad) / kBK - kbeg;
    // K blocks per accumulation run: split precisions restart the accumulator every s.kchunk K
    // elements (GemmShape::kchunk); otherwise one run per tile
    const int chunk_kb = (kSplit && s.kchunk >= kBK) ? s.kchunk / kBK : num_kb;

    if (warp == 0 && ptx::elect_one()) {
        ptx::tma_prefetch_desc(&tm.a);
        ptx::tma_prefetch_desc(&tm.b);
        if constexpr (kSplit) {
            ptx::tma_prefetch_desc(&tm.a_lo);
            ptx::tma_prefetch_desc(&tm.b_lo);
        }
        for (int i = 0; i < kStages2; ++i) {
            ptx::mbar_init(&full[i], 2);          // leader arrive.expect_tx + peer arrive
            ptx::mbar_init(&empty[i], 1);         // one multicast MMA commit
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tmem_full[i], 1);     // one multicast MMA commit
            ptx::mbar_init(&tmem_empty[i], 2 * 4);     // every epilogue warp of both CTAs
        }
        for (int i = 0; i < kRing; ++i) {
            ptx::mbar_init(&tile_full[i], 1);     // the fetcher's (local or remote) arrive
            ptx::mbar_init(&tile_empty[i], kTileConsumers);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc_pair<kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t tile_empty_leader = ptx::mapa_shared(ptx::smem_u32(tile_empty), 0);

    // Tile ids come from a global counter (dynamic scheduling keeps the tiles in flight a
    // contiguous window of the visiting order, so the operand panels they share stay in L2).
    // The leader's producer fetches; everybody else reads the id from its CTA's ring.
    auto next_tile = [&](int i) -> int {
        const int slot = i & (kRing - 1);
        ptx::mbar_wait_cluster(&tile_full[slot], (i / kRing) & 1);
        return static_cast<int>(tile_id[slot]);
    };
    auto release_tile = [&](int i) {
        ptx::mbar_arrive_remote(tile_empty_leader + 8u * static_cast<uint32_t>(i & (kRing - 1)));
    };

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer (+ fetcher)
        if (ptx::elect_one()) {
            int st = 0;
            uint32_t ph = 0;
            const uint32_t full_leader0 = ptx::mapa_shared(ptx::smem_u32(full), 0);
            for (int i = 0;; ++i) {
                int t;
                if (leader) {
                    const int slot = i & (kRing - 1);
                    ptx::mbar_wait(&tile_empty[slot], ((i / kRing) & 1) ^ 1);
                    t = atomicAdd(s.counter, 1);
                    if (t > total_tiles) t = total_tiles;
                    tile_id[slot] = static_cast<uint32_t>(t);
                    ptx::st_shared_cluster_u32(ptx::mapa_shared(ptx::smem_u32(&tile_id[slot]), 1), static_cast<uint32_t>(t));
                    ptx::mbar_arrive_remote_release(ptx::mapa_shared(ptx::smem_u32(&tile_full[slot]), 1));
                    ptx::mbar_arrive_remote_release(ptx::mapa_shared(ptx::smem_u32(&tile_full[slot]), 0));
                } else {
                    t = next_tile(i);
                    release_tile(i);
                }
                if (t >= total_tiles) break;
                int b, I, J;
                decode_tile(t, s, b, I, J);
                const int rowA = b * s.npad + I * kT2 + rank * kRowsPerCta;
                const int rowB = b * s.npad + J * kT2 + rank * kRowsPerCta;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&empty[st], ph ^ 1);
                    const uint32_t full_leader = full_leader0 + 8u * static_cast<uint32_t>(st);
                    uint8_t* sa = ring + st * kStageBytes;
                    if (leader) ptx::mbar_arrive_expect_tx(&full[st], 2 * kStageBytes);
                    else ptx::mbar_arrive_remote(full_leader);
                    const int k0 = (kbeg + kb) * kBK;
                    // upper-only storage: left of block `blk`'s diagonal tile the panel is the stored
                    // upper tile transposed -- two 64x64 boxes (rows k0.., this CTA's 128 columns) that
                    // the MMA reads as an MN-major operand
                    auto load = [&](uint8_t* dst, const CUtensorMap* mk, const CUtensorMap* mt, int blk, int row) {
                        if (Tr::kBytes == 2 && s.upper_only && k0 < blk * kT2) {
                            const int x = blk * kT2 + static_cast<int>(rank) * kRowsPerCta;
                            ptx::tma_load_2d_pair_nohint(dst, mt, full_leader, x, b * s.npad + k0);
                            ptx::tma_load_2d_pair_nohint(dst + kTileBytes1 / 2, mt, full_leader, x + 64, b * s.npad + k0);
                        } else {
                            ptx::tma_load_2d_pair_nohint(dst, mk, full_leader, k0, row);
                        }
                    };
                    load(sa, &tm.a, &tm.a_t, I, rowA);
                    load(sa + kTileBytes1, &tm.b, &tm.b_t, J, rowB);
                    if constexpr (kSplit) {
                        load(sa + 2 * kTileBytes1, &tm.a_lo, &tm.a_lo_t, I, rowA);
                        load(sa + 3 * kTileBytes1, &tm.b_lo, &tm.b_lo_t, J, rowB);
                    }
                    if (++st == kStages2) { st = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (leader)
        if (leader && ptx::elect_one()) {
            int st = 0;
            uint32_t ph = 0;
            int it = 0;
            int cc = 0;                  // accumulation runs issued (one per tile, or per K chunk)
            // debug build only: cycles waiting for a tile id, a free accumulator, operand stages;
            // total cycles in the loop
            unsigned long long w_tile = 0, w_tmem = 0, w_full = 0, t_start = 0, g_start = 0;
            if (kDebug && e.dbg) {
                t_start = clock64();
                g_start = ptx::globaltimer();
            }
            for (;; ++it) {
                unsigned long long c0 = (kDebug && e.dbg) ? clock64() : 0;
                const int t = next_tile(it);
                release_tile(it);
                if (kDebug && e.dbg) { const unsigned long long c1 = clock64(); w_tile += c1 - c0; c0 = c1; }
                if (t >= total_tiles) break;
                int tb, tI, tJ;
                decode_tile(t, s, tb, tI, tJ);
                int acc = 0;
                uint32_t d_tmem = tmem_base;
                for (int kb = 0; kb < num_kb; ++kb) {
                    const int kc = kb % chunk_kb;          // position in the accumulation run
                    if (kc == 0) {
                        // a run starts from zero in a free accumulator: the split path's single chunk
                        // buffer (the epilogue folds every run into its sum), else the tile ping-pong
                        acc = kSplit ? 0 : (cc & 1);
                        const uint32_t acc_ph = kSplit ? (cc & 1) : ((cc >> 1) & 1);
                        if (kDebug && e.dbg) c0 = clock64();
                        ptx::mbar_wait(&tmem_empty[acc], acc_ph ^ 1);
                        if (kDebug && e.dbg) w_tmem += clock64() - c0;
                        ptx::tc_fence_after();
                        d_tmem = tmem_base + acc * kT2;
                    }
                    if (kDebug && e.dbg) {
                        const unsigned long long c2 = clock64();
                        ptx::mbar_wait(&full[st], ph);
                        w_full += clock64() - c2;
                    } else {
                        ptx::mbar_wait(&full[st], ph);
                    }
                    ptx::tc_fence_after();
                    const uint32_t sa = ptx::smem_u32(ring + st * kStageBytes);
                    // upper-only storage: operands left of their diagonal tile arrive transposed
                    // (MN-major: 64-element MN chunks 8 KB apart = LBO, 8-row K groups 1 KB apart = SBO;
                    // one K step of 16 = 2 KB); the instruction descriptor says which is which
                    const bool a_mn = Tr::kBytes == 2 && s.upper_only && (kbeg + kb) * kBK < tI * kT2;
                    const bool b_mn = Tr::kBytes == 2 && s.upper_only && (kbeg + kb) * kBK < tJ * kT2;
                    const uint64_t adesc = a_mn ? ptx::smem_desc_sw128_mnmajor(sa, kTileBytes1 / 2, 1024)
                                                : ptx::smem_desc_sw128_kmajor(sa);
                    const uint64_t bdesc = b_mn ? ptx::smem_desc_sw128_mnmajor(sa + kTileBytes1, kTileBytes1 / 2, 1024)
                                                : ptx::smem_desc_sw128_kmajor(sa + kTileBytes1);
                    const uint32_t idesc = kIdesc | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u);
                    const uint64_t astep = a_mn ? (2048 >> 4) : (32 >> 4), bstep = b_mn ? (2048 >> 4) : (32 >> 4);
                    auto mma = [&](uint64_t a, uint64_t bb, uint32_t accumulate) {
                        if constexpr (T == OpType::TF32)
                            ptx::mma_tf32_pair(d_tmem, a, bb, kIdesc, accumulate);
                        else
                            ptx::mma_f16_pair(d_tmem, a, bb, idesc, accumulate);
                    };
#pragma unroll
                    for (int k = 0; k < kBK / kUmmaK; ++k) {
                        mma(adesc + k * astep, bdesc + k * bstep, (kc | k) != 0);
                        if constexpr (kSplit) {
                            const uint64_t alo = a_mn ? ptx::smem_desc_sw128_mnmajor(sa + 2 * kTileBytes1, kTileBytes1 / 2, 1024)
                                                      : ptx::smem_desc_sw128_kmajor(sa + 2 * kTileBytes1);
                            const uint64_t blo = b_mn ? ptx::smem_desc_sw128_mnmajor(sa + 3 * kTileBytes1, kTileBytes1 / 2, 1024)
                                                      : ptx::smem_desc_sw128_kmajor(sa + 3 * kTileBytes1);
                            mma(adesc + k * astep, blo + k * bstep, 1u);        // A_hi B_lo
                            mma(alo + k * astep, bdesc + k * bstep, 1u);        // A_lo B_hi
                        }
                    }
                    ptx::mma_commit_pair(&empty[st], 0x3);
                    if (kc == chunk_kb - 1 || kb == num_kb - 1) {
                        ptx::mma_commit_pair(&tmem_full[acc], 0x3);
                        ++cc;
                    }
                    if (++st == kStages2) { st = 0; ph ^= 1; }
                }
            }
            if (kDebug && e.dbg) {
                atomicAdd(e.dbg + 0, w_tile);
                atomicAdd(e.dbg + 1, w_tmem);
                atomicAdd(e.dbg + 2, w_full);
                atomicAdd(e.dbg + 3, clock64() - t_start);
                atomicAdd(e.dbg + 4, static_cast<unsigned long long>(it));
                const unsigned long long g_end = ptx::globaltimer();
                atomicAdd(e.dbg + 7, 1ull);                                   // clusters
                atomicMin(e.dbg + 8, g_start);                                // first start
                atomicMax(e.dbg + 9, g_start);                                // last start
                atomicMax(e.dbg + 10, g_end);                                 // last end
                atomicMin(e.dbg + 11, static_cast<unsigned long long>(it));   // fewest tiles
                atomicMax(e.dbg + 12, static_cast<unsigned long long>(it));   // most tiles
            }
            // drain: the last accumulators must be read out before the pair tears down
            if constexpr (kSplit) {
                if (cc > 0) ptx::mbar_wait(&tmem_empty[0], (cc - 1) & 1);
            } else {
                for (int last = cc - 2; last < cc; ++last)
                    if (last >= 0) ptx::mbar_wait(&tmem_empty[last & 1], (last >> 1) & 1);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;                        // TMEM lane quadrant
        uint8_t* wsmem = epi_smem + q * kEpiWarpSmemBytes;
        const uint32_t tmem_empty_leader0 = ptx::mapa_shared(ptx::smem_u32(&tmem_empty[0]), 0);
        const uint32_t tmem_empty_leader1 = ptx::mapa_shared(ptx::smem_u32(&tmem_empty[1]), 0);
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const int nchunks = (num_kb + chunk_kb - 1) / chunk_kb;
        int cc = 0;                                    // accumulation runs consumed
        for (int it = 0;; ++it) {
            const int t = next_tile(it);
            __syncwarp();
            if (ptx::elect_one()) release_tile(it);
            __syncwarp();
            if (t >= total_tiles) break;
            int b, I, J;
            decode_tile(t, s, b, I, J);
            {
                // addend rows of this thread (row gi0 + lane) for the whole tile into L2 while the
                // tile's MMAs run (first column at or right of the diagonal on a diagonal tile)
                const int gi = I * kT2 + static_cast<int>(rank) * kRowsPerCta + q * 32 + (threadIdx.x & 31);
                const int c_lo = (I == J) ? ((gi - J * kT2) & ~31) : 0;
                prefetch_addend_l2<T>(e, b, s.npad, gi, J * kT2 + c_lo, kT2 - c_lo);
            }
            const int gi0 = I * kT2 + static_cast<int>(rank) * kRowsPerCta + q * 32;
            const bool diag = (I == J);
            const unsigned long long e0 = (kDebug && e.dbg && q == 0 && ptx::elect_one()) ? clock64() : 0;
            uint32_t tsum;                             // TMEM columns the stores read the tile from
            if constexpr (kSplit) {
                // every K chunk's run lands in the chunk buffer (columns [0, 256)); fold it into the
                // running sum (columns [256, 512)) with round-to-nearest fp32 adds and hand the
                // buffer back, so the next run starts while this warp keeps folding / storing
                const uint32_t tC = tmem_base + lane_off, tS = tmem_base + kT2 + lane_off;
                for (int ch = 0; ch < nchunks; ++ch, ++cc) {
                    ptx::mbar_wait(&tmem_full[0], cc & 1);
                    ptx::tc_fence_after();
                    // 64 columns per TMEM round trip (four loads in flight per wait); blocks wholly
                    // below the diagonal of a diagonal tile are never stored, so never folded
                    const int c_first = diag ? max(0, (gi0 - J * kT2) & ~31) : 0;
#pragma unroll 1
                    for (int c0 = c_first & ~63; c0 < kT2; c0 += 64) {
                        const bool lo_live = c0 >= c_first;            // block c0 (block c0 + 32 always is)
                        uint32_t a0[32], a1[32], s0[32], s1[32];
                        if (lo_live) ptx::tmem_ld_32x32b_x32(tC + c0, a0);
                        ptx::tmem_ld_32x32b_x32(tC + c0 + 32, a1);
                        if (ch) {
                            if (lo_live) ptx::tmem_ld_32x32b_x32(tS + c0, s0);
                            ptx::tmem_ld_32x32b_x32(tS + c0 + 32, s1);
                        }
                        ptx::tmem_ld_wait();
                        if (ch) {
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                a0[i] = __float_as_uint(__fadd_rn(__uint_as_float(s0[i]), __uint_as_float(a0[i])));
                                a1[i] = __float_as_uint(__fadd_rn(__uint_as_float(s1[i]), __uint_as_float(a1[i])));
                            }
                        }
                        if (lo_live) ptx::tmem_st_32x32b_x32(tS + c0, a0);
                        ptx::tmem_st_32x32b_x32(tS + c0 + 32, a1);
                    }
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (ptx::elect_one()) ptx::mbar_arrive_remote(tmem_empty_leader0);
                }
                tsum = tS;
            } else {
                const int acc = it & 1;
                ptx::mbar_wait(&tmem_full[acc], (it >> 1) & 1);
                ptx::tc_fence_after();
                tsum = tmem_base + acc * kT2 + lane_off;
            }
            const unsigned long long e1 = e0 ? clock64() : 0;
            float alpha = e.alpha;
            if (e.alpha_dev) alpha *= static_cast<float>(e.alpha_dev[b]);
#pragma unroll 1
            for (int c0 = 0; c0 < kT2; c0 += 32) {
                const int gj0 = J * kT2 + c0;
                if (diag && gj0 + 31 < gi0) continue;   // chunk below the diagonal for the whole warp
                uint32_t raw[32];
                ptx::tmem_ld_32x32b_x32(tsum + c0, raw);
                ptx::tmem_ld_wait();
                const int64_t pk = e.packed ? static_cast<int64_t>(t) * (kT2 * kT2) +
                                              static_cast<int64_t>(gi0 - I * kT2) * kT2 + c0
                                            : -1;
                epilogue_chunk<T>(e, alpha, b, s.npad, gi0, gj0, diag, raw, wsmem, pk);
            }
            if constexpr (!kSplit) {
                ptx::tc_fence_before();
                __syncwarp();
                if (ptx::elect_one()) ptx::mbar_arrive_remote((it & 1) ? tmem_empty_leader1 : tmem_empty_leader0);
            }
            if (kDebug && e0) {
                atomicAdd(e.dbg + 5, e1 - e0);                 // epilogue warp 4 waiting for / folding accumulators
                atomicAdd(e.dbg + 6, clock64() - e1);          // its store work per tile
            }
        }
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair<kTmemCols>(tmem_base);
    }
}

template <OpType T, bool kSplit>
cudaError_t launch2_t(const OperandMaps& m, const GemmShape& s, const EpiParams& e, cudaStream_t stream) {
    static int num_sms = 0;
    if (!num_sms) {
        cudaError_t err = cudaFuncSetAttribute(sym_gemm_2cta_kernel<T, kSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
        if (err != cudaSuccess) return err;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int total = s.tiles_per_matrix * s.batch;
    int clusters = num_sms / 2;
    if (clusters > total) clusters = total;
    sym_gemm_2cta_kernel<T, kSplit><<<2 * clusters, kThreads2, kSmem2, stream>>>(m, s, e);
    return cudaGetLastError();
}

}  // namespace

void make_tile_order(int nt, const char* order, uint32_t* out) {
    int k = 0;
    auto put = [&](int I, int J) { out[k++] = (static_cast<uint32_t>(I) << 16) | static_cast<uint32_t>(J); };
    const std::string o = order ? order : "row";
    if (o == "col") {
        for (int J = 0; J < nt; ++J)
            for (int I = 0; I <= J; ++I) put(I, J);
    } else if (o.rfind("grouped", 0) == 0) {
        int G = std::atoi(o.c_str() + 7);
        if (G < 1) G = 4;
        const int nb = (nt + G - 1) / G;
        for (int BI = 0; BI < nb; ++BI)
            for (int BJ = BI; BJ < nb; ++BJ)
                for (int I = BI * G; I < std::min(nt, BI * G + G); ++I)
                    for (int J = BJ * G; J < std::min(nt, BJ * G + G); ++J)
                        if (I <= J) put(I, J);
    } else {
        for (int I = 0; I < nt; ++I)
            for (int J = I; J < nt; ++J) put(I, J);
    }
}

bool use_pair_kernel(int64_t n, int64_t batch) {
    const int64_t nt = (n + kT2 - 1) / kT2;
    return n >= 1024 && nt * (nt + 1) / 2 * batch >= 74;
}

int64_t padded_n(int64_t n, int64_t batch) {
    const int64_t m = use_pair_kernel(n, batch) ? kT2 : kTile;
    return (n + m - 1) / m * m;
}

cudaError_t launch_sym_gemm_2cta(OpType t, bool split, const OperandMaps& m, const GemmShape& s,
                                 const EpiParams& e, cudaStream_t stream) {
    switch (t) {
        case OpType::F16: return split ? launch2_t<OpType::F16, true>(m, s, e, stream)
                                       : launch2_t<OpType::F16, false>(m, s, e, stream);
        case OpType::BF16: return split ? launch2_t<OpType::BF16, true>(m, s, e, stream)
                                        : launch2_t<OpType::BF16, false>(m, s, e, stream);
        case OpType::TF32: return split ? launch2_t<OpType::TF32, true>(m, s, e, stream)
                                        : launch2_t<OpType::TF32, false>(m, s, e, stream);
    }
    return cudaErrorInvalidValue;
}

}  // namespace psd
