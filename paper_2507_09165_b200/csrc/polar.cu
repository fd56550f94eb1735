// polar.cu -- the polar factor of a general square A through the symmetric path (
// the polar factor generalises the matrix sign).
//
// The Jordan-Wielandt embedding H = [[0, A], [A^T, 0]] (2n x 2n, symmetric) has H^2 =
// diag(A A^T, A^T A), so any odd polynomial f(x) = x q(x^2) gives f(H) = [[0, A q(A^T A)],
// [A^T q(A A^T), 0]]: the top-right block of the composite filter's sign output on H is exactly the
// filter's polar iterate f_T o ... o f_1 (A / lambda~).  psd_polar therefore writes the upper
// triangle of H (the sign path reads only the upper triangle, R10), computes lambda~ = ||A||_F
// (>= ||A||_2 = ||H||_2; deterministic fp64 partials), runs psd_sign on H with that bound and copies
// the top-right block out.  Cost: the chain runs on 2n (about 6x the flops of a direct
// nonsymmetric chain, which needs general-output and Gram-product modes in the product kernels:
// DESIGN.md, next).
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

// Block k of matrix b: rows [k * rows_per, ...) of A.  H row i (< n): [0 .. n) zeros, [n .. 2n) = A row i;
// H row n + i: [n .. 2n) zeros (the lower-left block is never read).  partial[b][k] = sum of a^2 over the
// block's rows (fp64, fixed order).
__global__ void __launch_bounds__(kPolarThreads)
polar_embed_kernel(const float* __restrict__ A, int n, int rows_per, float* __restrict__ H, double* __restrict__ partial) {
    const int b = blockIdx.y, k = blockIdx.x;
    const int64_t N = 2 * static_cast<int64_t>(n);
    const float* Ab = A + static_cast<int64_t>(b) * n * n;
    float* Hb = H + static_cast<int64_t>(b) * N * N;
    const int r0 = k * rows_per, r1 = min(n, r0 + rows_per);
    double s = 0.0;
    for (int i = r0; i < r1; ++i) {
        const float* arow = Ab + static_cast<int64_t>(i) * n;
        float* top = Hb + static_cast<int64_t>(i) * N;
        float* bot = Hb + (static_cast<int64_t>(n) + i) * N + n;
        for (int j = threadIdx.x; j < n; j += kPolarThreads) {
            const float a = arow[j];
            s = fma(static_cast<double>(a), static_cast<double>(a), s);
            top[n + j] = a;
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

// out[b][i][j] = S[b][i][n + j]: one block per output row (blockIdx.x = b * n + i), float4 when rows
// are 16-byte aligned
__global__ void __launch_bounds__(kPolarThreads)
polar_extract_kernel(const float* __restrict__ S, int n, float* __restrict__ out) {
    const int64_t N = 2 * static_cast<int64_t>(n);
    const int64_t row = blockIdx.x;                       // b * n + i
    const int64_t b = row / n, i = row - b * n;
    const float* src = S + b * N * N + i * N + n;
    float* dst = out + row * n;
    if ((n & 3) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (int j = threadIdx.x; j < n / 4; j += kPolarThreads) d4[j] = s4[j];
    } else {
        for (int j = threadIdx.x; j < n; j += kPolarThreads) dst[j] = src[j];
    }
}

}  // namespace

int polar_blocks_per_matrix(int n, int batch) {
    int k = (n + 7) / 8;                                  // ~8 rows per block
    const int fill = (4 * 148 + batch - 1) / batch;      // a few blocks per SM over the batch
    if (k < fill) k = fill;
    if (k > n) k = n;
    return k < 1 ? 1 : (k > 512 ? 512 : k);
}

cudaError_t launch_polar_embed(const float* A, int n, int batch, float* H, double* partial, int nblk,
                               cudaStream_t stream) {
    const int rows_per = (n + nblk - 1) / nblk;
    polar_embed_kernel<<<dim3(nblk, batch), kPolarThreads, 0, stream>>>(A, n, rows_per, H, partial);
    return cudaGetLastError();
}

cudaError_t launch_polar_extract(const float* S, int n, int batch, float* out, cudaStream_t stream) {
    polar_extract_kernel<<<static_cast<unsigned>(static_cast<int64_t>(batch) * n), kPolarThreads, 0, stream>>>(S, n, out);
    return cudaGetLastError();
}

}  // namespace psd
