// rowpanel.cu -- device side of the row-panel (multi-GPU) path, SURVEY.md section 8(e) config c5.
//
// Every product of Algorithm 2 is split over the ranks by upper 256-tiles: rank r
// computes a balanced, disjoint share of the upper tiles (I <= J) and writes them packed and
// unmirrored (epilogue packed mode); an in-place all-gather of the packed buffers gives every
// rank every upper tile (the upper triangle only: half the bytes of gathering row panels);
// this unpack kernel rebuilds the full, exactly symmetric operand on every rank -- the same
// deterministic rule everywhere, so all ranks hold bit-identical operands.  Exact symmetry of
// the operands is required: a rounding-level antisymmetric part grows like prod_t c_{t,0}
// along the chain (reading R20).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kernels.h"

#include <vector>

namespace psd {

namespace {

constexpr int kT = 256;
constexpr int kBand = 32;        // rows of a tile per block

// One block per (tile, 32-row band): direct copy of the band into full[I*256 + band rows][J*256 ..]
// and the transposed band into full[J*256 ..][I*256 + band rows] through smem.
template <typename E>
__global__ void __launch_bounds__(256)
unpack_tiles_kernel(const E* __restrict__ packed, const uint32_t* __restrict__ codes, int ntiles, E* __restrict__ full,
                    int64_t ld, bool mirror) {
    __shared__ E S[kBand][kT + 16 / sizeof(E)];
    const int tile = blockIdx.x / (kT / kBand);
    const int band = blockIdx.x % (kT / kBand);
    if (tile >= ntiles) return;
    const uint32_t code = codes[tile];
    if (code == 0xFFFFFFFFu) return;          // padding slot of a rank with fewer tiles
    const int I = static_cast<int>(code >> 16), J = static_cast<int>(code & 0xFFFFu);
    const E* src = packed + static_cast<int64_t>(tile) * kT * kT;
    const int r0 = band * kBand;
    constexpr int kVec = 16 / sizeof(E);     // elements per 16-byte vector
    constexpr int kRowVecs = kT / kVec;
    if (I != J) {
        for (int v = threadIdx.x; v < kBand * kRowVecs; v += 256) {
            const int r = v / kRowVecs, q = v % kRowVecs;
            const uint4 x = reinterpret_cast<const uint4*>(src + static_cast<int64_t>(r0 + r) * kT)[q];
            reinterpret_cast<uint4*>(full + static_cast<int64_t>(I * kT + r0 + r) * ld + J * kT)[q] = x;
            const E* xe = reinterpret_cast<const E*>(&x);
#pragma unroll
            for (int k = 0; k < kVec; ++k) S[r][q * kVec + k] = xe[k];
        }
        if (!mirror) return;             // upper-only operand storage: no transposed band
        __syncthreads();
        // transposed: output row J*256 + c, columns I*256 + r0 .. + kBand
        constexpr int kOutVecs = kBand / kVec;
        for (int v = threadIdx.x; v < kT * kOutVecs; v += 256) {
            const int c = v / kOutVecs, q = v % kOutVecs;
            __align__(16) E tmp[kVec];
#pragma unroll
            for (int k = 0; k < kVec; ++k) tmp[k] = S[q * kVec + k][c];
            reinterpret_cast<uint4*>(full + static_cast<int64_t>(J * kT + c) * ld + I * kT + r0)[q] =
                *reinterpret_cast<const uint4*>(tmp);
        }
    } else {
        // diagonal tile: element (r, c) = packed[min][max] (the upper part is the computed one)
        for (int e = threadIdx.x; e < kBand * kT; e += 256) {
            const int r = r0 + e / kT, c = e % kT;
            const E x = (c >= r) ? src[static_cast<int64_t>(r) * kT + c] : src[static_cast<int64_t>(c) * kT + r];
            full[static_cast<int64_t>(I * kT + r) * ld + I * kT + c] = x;
        }
    }
}

__global__ void peer_signal_kernel(unsigned long long* const* __restrict__ flags, int nranks, int rank,
                                   unsigned long long epoch) {
    // every store of this rank's previous kernels (the product epilogue's peer stores) is ordered
    // before the flag by the system-scope fence; the flag store itself is a release
    __threadfence_system();
    const int p = threadIdx.x;
    if (p < nranks)
        asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(flags[p] + rank), "l"(epoch) : "memory");
}

__global__ void peer_wait_kernel(const unsigned long long* __restrict__ my_flags, int nranks, unsigned long long epoch,
                                 unsigned long long timeout_ns, unsigned* __restrict__ status) {
    const int p = threadIdx.x;
    if (p < nranks) {
        unsigned long long t0, t, v;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + p) : "memory");
            if (v >= epoch) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                // a peer never arrived: record it (psd_status -> PSD_ETIMEOUT) and let the stream
                // go on (the result is invalid), never hang or trap the context
                atomicOr(status, 2u);
                break;
            }
            __nanosleep(256);
        }
    }
    __syncthreads();
    // the next kernels read the peers' stores through TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

}  // namespace

cudaError_t launch_peer_signal(unsigned long long* const* flags_dev, int nranks, int rank, unsigned long long epoch,
                               cudaStream_t stream) {
    peer_signal_kernel<<<1, 32, 0, stream>>>(flags_dev, nranks, rank, epoch);
    return cudaGetLastError();
}

cudaError_t launch_peer_wait(const unsigned long long* my_flags, int nranks, unsigned long long epoch,
                             unsigned long long timeout_ns, unsigned* status, cudaStream_t stream) {
    peer_wait_kernel<<<1, 32, 0, stream>>>(my_flags, nranks, epoch, timeout_ns, status);
    return cudaGetLastError();
}

cudaError_t launch_unpack_tiles(int elem_bytes, const void* packed, const uint32_t* codes, int ntiles, void* full,
                                int64_t ld, cudaStream_t stream, bool mirror) {
    const int blocks = ntiles * (kT / kBand);
    if (blocks == 0) return cudaSuccess;
    if (elem_bytes == 2)
        unpack_tiles_kernel<uint16_t><<<blocks, 256, 0, stream>>>(static_cast<const uint16_t*>(packed), codes, ntiles,
                                                                  static_cast<uint16_t*>(full), ld, mirror);
    else
        unpack_tiles_kernel<float><<<blocks, 256, 0, stream>>>(static_cast<const float*>(packed), codes, ntiles,
                                                               static_cast<float*>(full), ld, mirror);
    return cudaGetLastError();
}

// Balanced assignment of the upper tiles (row-major order t) of an nt x nt tile grid:
// rank r takes t = r, r + P, r + 2P, ...; every rank's list is padded to ceil(T / P) slots.
int rowpanel_tiles(int nt, int nranks, int rank, uint32_t* codes, int cap) {
    const int T = nt * (nt + 1) / 2;
    const int per = (T + nranks - 1) / nranks;
    if (!codes) return per;
    // the upper tiles in the single-GPU visiting order (8 x 8 super-tiles beyond 16 tile rows, for
    // L2 reuse of the panels), dealt round robin: every rank's list keeps that locality
    std::vector<uint32_t> order(T);
    make_tile_order(nt, nt > 16 ? "grouped8" : "row", order.data());
    int k = 0;
    for (int t = 0; t < T; ++t)
        if (t % nranks == rank && k < cap) codes[k++] = order[t];
    const int actual = k;
    while (k < per && k < cap) codes[k++] = 0xFFFFFFFFu;
    return actual;
}

}  // namespace psd
