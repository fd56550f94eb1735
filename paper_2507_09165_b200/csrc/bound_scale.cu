// bound_scale.cu -- the two HBM-bound steps before the products of Algorithm 2:
//   (a1) lambda~ = ||X||_F  (reading R4), fp32 loads, fp64 accumulation,
//        warp-shuffle + block tree, fixed-order (deterministic) grid reduction;
//   (a2) X_0 = X / lambda~ fused with the conversion to the operand
//        precision (P:L794 times "data type conversion") and the symmetrisation from
//        the upper triangle (reading R10): one read of the upper triangle, mirrored writes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kernels.h"

namespace psd {

namespace {

constexpr int kBoundThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kBoundThreads)
frobenius_partials_kernel(const float* __restrict__ X, int n, int nblk, double* __restrict__ partial) {
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* Xb = X + static_cast<int64_t>(b) * n * n;
    double acc = 0.0;
    // rows i == blockIdx.x (mod nblk), one warp per row, upper part j >= i
    for (int i = blockIdx.x + nblk * warp; i < n; i += nblk * (kBoundThreads / 32)) {
        const float* row = Xb + static_cast<int64_t>(i) * n;
        for (int j = i + lane; j < n; j += 32) {
            const double x = row[j];
            acc += (j == i ? 1.0 : 2.0) * x * x;
        }
    }
    acc = warp_sum(acc);
    __shared__ double red[kBoundThreads / 32];
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        double v = lane < kBoundThreads / 32 ? red[lane] : 0.0;
        v = warp_sum(v);
        if (lane == 0) partial[static_cast<int64_t>(b) * nblk + blockIdx.x] = v;
    }
}

__global__ void finalize_bound_kernel(const double* __restrict__ partial, int nblk, double* lambda,
                                      double* lambda_out, unsigned* status) {
    const int b = blockIdx.x, lane = threadIdx.x;
    double v = 0.0;
    for (int k = lane; k < nblk; k += 32) v += partial[static_cast<int64_t>(b) * nblk + k];
    v = warp_sum(v);
    if (lane == 0) {
        double lam = sqrt(v);
        if (!isfinite(lam)) {
            atomicOr(status, 1u);
            lam = __longlong_as_double(0x7ff8000000000000LL);   // NaN propagates to the output
        }
        lambda[b] = lam;
        if (lambda_out) lambda_out[b] = lam;
    }
}

template <OpType T> struct Cvt;
template <> struct Cvt<OpType::F16> {
    using type = __half;
    __device__ static type f(float v) { return __float2half_rn(v); }
};
template <> struct Cvt<OpType::BF16> {
    using type = __nv_bfloat16;
    __device__ static type f(float v) { return __float2bfloat16_rn(v); }
};
template <> struct Cvt<OpType::TF32> {
    using type = float;
    __device__ static type f(float v) {
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
        return __uint_as_float(r);
    }
};

constexpr int kST = 32;   // scale tile

__device__ __forceinline__ void upper_coords(int t, int nt, int& I, int& J) {
    // closed form for row-major upper-triangle enumeration, with a fix-up step
    int i = static_cast<int>((2.0 * nt + 1.0 - sqrt((2.0 * nt + 1.0) * (2.0 * nt + 1.0) - 8.0 * t)) / 2.0);
    if (i < 0) i = 0;
    auto start = [nt](int r) { return r * nt - (r * (r - 1)) / 2; };
    while (i > 0 && start(i) > t) --i;
    while (start(i + 1) <= t) ++i;
    I = i;
    J = i + (t - start(i));
}

template <OpType T>
__global__ void __launch_bounds__(kST * 8)
scale_convert_kernel(const float* __restrict__ X, int n, int npad, const double* __restrict__ lambda,
                     double scale, typename Cvt<T>::type* __restrict__ out_op, float* __restrict__ out32,
                     float* __restrict__ outF, double post) {
    using op_t = typename Cvt<T>::type;
    __shared__ float S[kST][kST + 1];
    const int b = blockIdx.y;
    const int ntile = npad / kST;
    int I, J;
    upper_coords(blockIdx.x, ntile, I, J);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float* Xb = X + static_cast<int64_t>(b) * n * n;

    double inv = scale;
    if (lambda) {
        const double lam = lambda[b];
        inv = (lam > 0.0) ? 1.0 / lam : (lam == 0.0 ? 0.0 : lam);   // NaN stays NaN; 0 -> zeros
    }
    for (int r = ty; r < kST; r += 8) {
        const int gi = I * kST + r, gj = J * kST + tx;
        float x = 0.0f;
        if (gi < n && gj < n) x = Xb[static_cast<int64_t>(gi) * n + gj];
        S[r][tx] = static_cast<float>(static_cast<double>(x) * inv);
    }
    __syncthreads();
    const int64_t base = static_cast<int64_t>(b) * npad * npad;
    for (int r = ty; r < kST; r += 8) {
        // direct tile (I, J): element (r, tx); on the diagonal tile the lower half mirrors
        const float vd = (I == J && tx < r) ? S[tx][r] : S[r][tx];
        const int64_t od = base + static_cast<int64_t>(I * kST + r) * npad + J * kST + tx;
        if (out_op) out_op[od] = Cvt<T>::f(vd);
        if (out32) out32[od] = vd;
        // transposed tile (J, I): element (r, tx) = S[tx][r]
        if (I != J) {
            const float vt = S[tx][r];
            const int64_t ot = base + static_cast<int64_t>(J * kST + r) * npad + I * kST + tx;
            if (out_op) out_op[ot] = Cvt<T>::f(vt);
        }
        if (outF) {
            float* F = outF + static_cast<int64_t>(b) * n * n;
            const int gi = I * kST + r, gj = J * kST + tx;
            if (gi < n && gj < n) F[static_cast<int64_t>(gi) * n + gj] = static_cast<float>(vd * post);
            const int ti = J * kST + r, tj = I * kST + tx;
            if (I != J && ti < n && tj < n) F[static_cast<int64_t>(ti) * n + tj] = static_cast<float>(S[tx][r] * post);
        }
    }
}

}  // namespace

int bound_blocks_per_matrix(int n) {
    int k = (n + 15) / 16;
    return k < 1 ? 1 : (k > 256 ? 256 : k);
}

cudaError_t launch_frobenius_partials(const float* X, int n, int batch, double* partial, int nblk,
                                      cudaStream_t stream) {
    dim3 grid(nblk, batch);
    frobenius_partials_kernel<<<grid, kBoundThreads, 0, stream>>>(X, n, nblk, partial);
    return cudaGetLastError();
}

cudaError_t launch_finalize_bound(const double* partial, int nblk, int batch, double* lambda,
                                  double* lambda_out, unsigned* status, cudaStream_t stream) {
    finalize_bound_kernel<<<batch, 32, 0, stream>>>(partial, nblk, lambda, lambda_out, status);
    return cudaGetLastError();
}

cudaError_t launch_scale_convert(OpType t, const float* X, int n, int npad, int batch,
                                 const double* lambda, double scale, void* out_op, float* out32,
                                 float* outF, double post, cudaStream_t stream) {
    const int nt = npad / kST;
    dim3 grid(nt * (nt + 1) / 2, batch);
    switch (t) {
        case OpType::F16:
            scale_convert_kernel<OpType::F16><<<grid, kST * 8, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<__half*>(out_op), out32, outF, post);
            break;
        case OpType::BF16:
            scale_convert_kernel<OpType::BF16><<<grid, kST * 8, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<__nv_bfloat16*>(out_op), out32, outF, post);
            break;
        case OpType::TF32:
            scale_convert_kernel<OpType::TF32><<<grid, kST * 8, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<float*>(out_op), out32, outF, post);
            break;
    }
    return cudaGetLastError();
}

}  // namespace psd
