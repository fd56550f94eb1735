// polar.cu -- the polar factor of a general square A through the symmetric path (
// the polar factor generalises the matrix sign).
//
// The Jordan-Wielandt embedding H = [[0, A], [A^T, 0]] (2n x 2n, symmetric) has H^2 =
// diag(A A^T, A^T A), so any odd polynomial f(x) = x q(x^2) gives f(H) = [[0, A q(A^T A)],
// [A^T q(A A^T), 0]]: the top-right block of the composite filter's sign output on H is exactly the
// filter's polar iterate f_T o ... o f_1 (A / lambda~).  psd_polar therefore writes the upper
// triangle of H (the sign path reads only the upper triangle, R10), computes lambda~ = ||A||_F
// (>= ||A||_2 = ||H||_2; deterministic fp64 partials), runs psd_sign on H with that bound and copies
// the top-right block out.  H's structure is exploited in the product loop (psd_api.cu, R25): every
// iterate is block off-diagonal and Y, U block diagonal, so each product runs only over its nonzero
// block (Y, U: the bottom-right block = the A^T A side; Z': the top-right block) and its nonzero K
// half -- the flops of a direct nonsymmetric chain.  A is zero-padded to m = a multiple of 128 so the
// block boundary is a tile boundary (zero singular values map to 0); a rectangular rows x cols A is
// padded the same way (f(A) = A q(A^T A) is rows x cols).
#include <cstdint>

#include "kernels.h"

namespace psd {

namespace {

constexpr int kPolarThreads = 256;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// H = [[0, A'], [A'^T, 0]] of edge 2m, A' = A zero-padded to m x m (m >= n, a multiple of the tile edge:
// the block boundary falls on a tile boundary).  Block k of matrix b covers rows [k * rows_per, ...) of
// the top half: H row i < m gets zeros in [0, m) and A row i (zero-extended) in [m, 2m); H row m + i
// gets zeros in [m, 2m) (the lower-left block is never read).  partial[b][k] = sum of a^2 (fp64, fixed
// order).
__global__ void __launch_bounds__(kPolarThreads)
polar_embed_kernel(const float* __restrict__ A, int rows, int cols, int m, int rows_per, float* __restrict__ H,
                   double* __restrict__ partial) {
    const int b = blockIdx.y, k = blockIdx.x;
    const int64_t N = 2 * static_cast<int64_t>(m);
    const float* Ab = A + static_cast<int64_t>(b) * rows * cols;
    float* Hb = H + static_cast<int64_t>(b) * N * N;
    const int r0 = k * rows_per, r1 = min(m, r0 + rows_per);
    double s = 0.0;
    for (int i = r0; i < r1; ++i) {
        const float* arow = Ab + static_cast<int64_t>(i) * cols;
        float* top = Hb + static_cast<int64_t>(i) * N;
        float* bot = Hb + (static_cast<int64_t>(m) + i) * N + m;
        for (int j = threadIdx.x; j < m; j += kPolarThreads) {
            const float a = (i < rows && j < cols) ? arow[j] : 0.0f;
            s = fma(static_cast<double>(a), static_cast<double>(a), s);
            top[m + j] = a;
            top[j] = 0.0f;
            bot[j] = 0.0f;
        }
    }
    __shared__ double red[kPolarThreads / 32];
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kPolarThreads / 32; ++w) t += red[w];      // fixed order: deterministic
        partial[static_cast<int64_t>(b) * gridDim.x + k] = t;
    }
}

// out[b][i][j] = S[b][i][m + j] for i < rows, j < cols: one block per output row (blockIdx.x =
// b * rows + i), float4 when rows are 16-byte aligned
__global__ void __launch_bounds__(kPolarThreads)
polar_extract_kernel(const float* __restrict__ S, int rows, int cols, int m, float* __restrict__ out) {
    const int64_t N = 2 * static_cast<int64_t>(m);
    const int64_t row = blockIdx.x;                       // b * rows + i
    const int64_t b = row / rows, i = row - b * rows;
    const float* src = S + b * N * N + i * N + m;
    float* dst = out + row * cols;
    if ((cols & 3) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (int j = threadIdx.x; j < cols / 4; j += kPolarThreads) d4[j] = s4[j];
    } else {
        for (int j = threadIdx.x; j < cols; j += kPolarThreads) dst[j] = src[j];
    }
}

}  // namespace

int polar_blocks_per_matrix(int m, int batch) {
    int k = (m + 7) / 8;                                  // ~8 rows per block
    const int fill = (4 * 148 + batch - 1) / batch;      // a few blocks per SM over the batch
    if (k < fill) k = fill;
    if (k > m) k = m;
    return k < 1 ? 1 : (k > 512 ? 512 : k);
}

cudaError_t launch_polar_embed(const float* A, int rows, int cols, int m, int batch, float* H, double* partial,
                               int nblk, cudaStream_t stream) {
    const int rows_per = (m + nblk - 1) / nblk;
    polar_embed_kernel<<<dim3(nblk, batch), kPolarThreads, 0, stream>>>(A, rows, cols, m, rows_per, H, partial);
    return cudaGetLastError();
}

cudaError_t launch_polar_extract(const float* S, int rows, int cols, int m, int batch, float* out, cudaStream_t stream) {
    polar_extract_kernel<<<static_cast<unsigned>(static_cast<int64_t>(batch) * rows), kPolarThreads, 0, stream>>>(
        S, rows, cols, m, out);
    return cudaGetLastError();
}

}  // namespace psd
