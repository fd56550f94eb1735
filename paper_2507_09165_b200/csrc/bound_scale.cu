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
    __device__ static float back(type v) { return __half2float(v); }
};
template <> struct Cvt<OpType::BF16> {
    using type = __nv_bfloat16;
    __device__ static type f(float v) { return __float2bfloat16_rn(v); }
    __device__ static float back(type v) { return __bfloat162float(v); }
};
template <> struct Cvt<OpType::TF32> {
    using type = float;
    __device__ static type f(float v) {
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
        return __uint_as_float(r);
    }
    __device__ static float back(type v) { return v; }
};

constexpr int kST = 64;   // scale tile (64 x 64, 256 threads)

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

// One block per upper 64x64 tile pair (I <= J) of the padded matrix: reads tile (I, J) of X
// once (upper triangle; on a diagonal tile the lower half mirrors the upper), writes the
// operand copy of tiles (I, J) and (J, I), zero in the padding.
template <OpType T>
__global__ void __launch_bounds__(256)
scale_convert_kernel(const float* __restrict__ X, int n, int npad, const double* __restrict__ lambda,
                     double scale, typename Cvt<T>::type* __restrict__ out_op, typename Cvt<T>::type* __restrict__ out_lo,
                     float op_scale, float* __restrict__ outF, double post) {
    using op_t = typename Cvt<T>::type;
    __shared__ float S[kST][kST + 1];
    const int b = blockIdx.y;
    const int ntile = npad / kST;
    int I, J;
    upper_coords(blockIdx.x, ntile, I, J);
    const int tid = threadIdx.x;
    const float* Xb = X + static_cast<int64_t>(b) * n * n;

    double inv = scale;
    if (lambda) {
        const double lam = lambda[b];
        inv = (lam > 0.0) ? 1.0 / lam : (lam == 0.0 ? 0.0 : lam);   // NaN stays NaN; 0 -> zeros
    }
    const int r0 = I * kST, c0 = J * kST;
    if ((n & 3) == 0 && r0 + kST <= n && c0 + kST <= n) {
        // 64 rows x 16 float4; 4 per thread, coalesced
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int idx = tid + 256 * k;
            const int r = idx >> 4, q = idx & 15;
            const float4 x = __ldcs(reinterpret_cast<const float4*>(Xb + static_cast<int64_t>(r0 + r) * n + c0) + q);
            S[r][4 * q] = static_cast<float>(static_cast<double>(x.x) * inv);
            S[r][4 * q + 1] = static_cast<float>(static_cast<double>(x.y) * inv);
            S[r][4 * q + 2] = static_cast<float>(static_cast<double>(x.z) * inv);
            S[r][4 * q + 3] = static_cast<float>(static_cast<double>(x.w) * inv);
        }
    } else {
        for (int idx = tid; idx < kST * kST; idx += 256) {
            const int r = idx >> 6, c = idx & 63;
            const int gi = r0 + r, gj = c0 + c;
            const float x = (gi < n && gj < n) ? Xb[static_cast<int64_t>(gi) * n + gj] : 0.0f;
            S[r][c] = static_cast<float>(static_cast<double>(x) * inv);
        }
    }
    __syncthreads();
    const int64_t base = static_cast<int64_t>(b) * npad * npad;
    // each thread: one row segment of 16 elements of the direct tile and of the mirrored tile
    const int r = tid >> 2, cs = (tid & 3) * 16;
    if (out_op) {
        constexpr int kVec = 16 / sizeof(op_t);   // elements per 16-byte store
        for (int part = 0; part < (out_lo ? 2 : 1); ++part) {
            __align__(16) op_t vd[16];
            __align__(16) op_t vt[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int c = cs + i;
                const float xd = ((I == J && c < r) ? S[c][r] : S[r][c]) * op_scale;
                const float xt = S[c][r] * op_scale;
                const op_t hd = Cvt<T>::f(xd), ht = Cvt<T>::f(xt);
                // part 0: hi = rn(x s); part 1: lo = rn(x s - hi)
                vd[i] = part == 0 ? hd : Cvt<T>::f(xd - Cvt<T>::back(hd));
                vt[i] = part == 0 ? ht : Cvt<T>::f(xt - Cvt<T>::back(ht));
            }
            op_t* dstb = part == 0 ? out_op : out_lo;
            uint4* od = reinterpret_cast<uint4*>(dstb + base + static_cast<int64_t>(r0 + r) * npad + c0 + cs);
#pragma unroll
            for (int q = 0; q < 16 / kVec; ++q) od[q] = *reinterpret_cast<const uint4*>(vd + q * kVec);
            if (I != J) {
                uint4* ot = reinterpret_cast<uint4*>(dstb + base + static_cast<int64_t>(c0 + r) * npad + r0 + cs);
#pragma unroll
                for (int q = 0; q < 16 / kVec; ++q) ot[q] = *reinterpret_cast<const uint4*>(vt + q * kVec);
            }
        }
    }
    if (outF) {
        float* F = outF + static_cast<int64_t>(b) * n * n;
        for (int i = 0; i < 16; ++i) {
            const int c = cs + i;
            const float vd = (I == J && c < r) ? S[c][r] : S[r][c];
            const int gi = r0 + r, gj = c0 + c;
            if (gi < n && gj < n) F[static_cast<int64_t>(gi) * n + gj] = static_cast<float>(vd * post);
            const int ti = c0 + r, tj = r0 + c;
            if (I != J && ti < n && tj < n) F[static_cast<int64_t>(ti) * n + tj] = static_cast<float>(S[c][r] * post);
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
                                 const double* lambda, double scale, void* out_op, void* out_lo,
                                 double op_scale, float* outF, double post, cudaStream_t stream) {
    const int nt = npad / kST;
    dim3 grid(nt * (nt + 1) / 2, batch);
    switch (t) {
        case OpType::F16:
            scale_convert_kernel<OpType::F16><<<grid, 256, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<__half*>(out_op), static_cast<__half*>(out_lo),
                static_cast<float>(op_scale), outF, post);
            break;
        case OpType::BF16:
            scale_convert_kernel<OpType::BF16><<<grid, 256, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<__nv_bfloat16*>(out_op),
                static_cast<__nv_bfloat16*>(out_lo), static_cast<float>(op_scale), outF, post);
            break;
        case OpType::TF32:
            scale_convert_kernel<OpType::TF32><<<grid, 256, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<float*>(out_op), static_cast<float*>(out_lo),
                static_cast<float>(op_scale), outF, post);
            break;
    }
    return cudaGetLastError();
}

}  // namespace psd
