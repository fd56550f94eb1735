// bound_scale.cu -- the two HBM-bound steps before the products of Algorithm 2:
//   (a1) lambda~ = ||X||_F  (reading R4), fp32 loads, fp64 accumulation,
//        warp-shuffle + block tree, fixed-order (deterministic) grid reduction;
//   (a2) X_0 = X / lambda~ fused with the conversion to the operand
//        precision (P:L794 times "data type conversion") and the symmetrisation from
//        the upper triangle (reading R10): one read of the upper triangle, mirrored writes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kernels.h"

#include <utility>

namespace psd {

namespace {

constexpr int kBoundThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ADMM input formation (psd_admm_update): m = (x - xk * inv_sigma) - [i == j] y_i, fp32 with one
// rounding per operation (no contraction), the same wherever the input is read (R22).
__device__ __forceinline__ float form_m(float x, float xk, float inv_sigma) {
    return __fsub_rn(x, __fmul_rn(xk, inv_sigma));
}

__global__ void __launch_bounds__(kBoundThreads)
frobenius_partials_kernel(const float* __restrict__ X, int n, int nblk, double* __restrict__ partial,
                          const InputForm form) {
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* Xb = X + static_cast<int64_t>(b) * n * n;
    const float* Kb = form.Xk ? form.Xk + static_cast<int64_t>(b) * n * n : nullptr;
    double acc = 0.0;
    // rows i == blockIdx.x (mod nblk), one warp per row, upper part j >= i
    const bool vec = (n & 3) == 0;                   // rows 16-byte aligned: float4 loads
    for (int i = blockIdx.x + nblk * warp; i < n; i += nblk * (kBoundThreads / 32)) {
        const float* row = Xb + static_cast<int64_t>(i) * n;
        const float* krow = Kb ? Kb + static_cast<int64_t>(i) * n : nullptr;
        const float yi = (Kb && form.y) ? form.y[static_cast<int64_t>(b) * n + i] : 0.0f;
        if (vec) {
            // 4 columns per lane per step (independent accumulations), from the float4 holding i
            double a4[4] = {0.0, 0.0, 0.0, 0.0};
            for (int c = (i & ~3) + 4 * lane; c < n; c += 128) {
                float4 x4 = __ldg(reinterpret_cast<const float4*>(row + c));
                if (krow) {
                    const float4 k4 = __ldg(reinterpret_cast<const float4*>(krow + c));
                    x4.x = form_m(x4.x, k4.x, form.inv_sigma);
                    x4.y = form_m(x4.y, k4.y, form.inv_sigma);
                    x4.z = form_m(x4.z, k4.z, form.inv_sigma);
                    x4.w = form_m(x4.w, k4.w, form.inv_sigma);
                }
                const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int j = c + q;
                    float m = xs[q];
                    if (krow && j == i) m = __fsub_rn(m, yi);
                    const double x = m;
                    a4[q] += (j < i) ? 0.0 : (j == i ? 1.0 : 2.0) * x * x;
                }
            }
            acc += (a4[0] + a4[1]) + (a4[2] + a4[3]);
        } else {
            for (int j = i + lane; j < n; j += 32) {
                float m = row[j];
                if (krow) {
                    m = form_m(m, krow[j], form.inv_sigma);
                    if (j == i) m = __fsub_rn(m, yi);
                }
                const double x = m;
                acc += (j == i ? 1.0 : 2.0) * x * x;
            }
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
                     float op_scale, float* __restrict__ outF, double post, const InputForm form, int mirror_block) {
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
    const float* Kb = form.Xk ? form.Xk + static_cast<int64_t>(b) * n * n : nullptr;
    const float* yb = (form.Xk && form.y) ? form.y + static_cast<int64_t>(b) * n : nullptr;
    if ((n & 3) == 0 && r0 + kST <= n && c0 + kST <= n) {
        // 64 rows x 16 float4; 4 per thread, coalesced
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int idx = tid + 256 * k;
            const int r = idx >> 4, q = idx & 15;
            float4 x = __ldcs(reinterpret_cast<const float4*>(Xb + static_cast<int64_t>(r0 + r) * n + c0) + q);
            if (Kb) {        // ADMM: M = C - Xk / sigma - Diag(y)
                const float4 k4 = __ldcs(reinterpret_cast<const float4*>(Kb + static_cast<int64_t>(r0 + r) * n + c0) + q);
                x.x = form_m(x.x, k4.x, form.inv_sigma);
                x.y = form_m(x.y, k4.y, form.inv_sigma);
                x.z = form_m(x.z, k4.z, form.inv_sigma);
                x.w = form_m(x.w, k4.w, form.inv_sigma);
                if (yb && r0 == c0) {
                    const int d = r - 4 * q;           // which component sits on the diagonal
                    const float yv = yb[r0 + r];
                    if (d == 0) x.x = __fsub_rn(x.x, yv);
                    if (d == 1) x.y = __fsub_rn(x.y, yv);
                    if (d == 2) x.z = __fsub_rn(x.z, yv);
                    if (d == 3) x.w = __fsub_rn(x.w, yv);
                }
            }
            S[r][4 * q] = static_cast<float>(static_cast<double>(x.x) * inv);
            S[r][4 * q + 1] = static_cast<float>(static_cast<double>(x.y) * inv);
            S[r][4 * q + 2] = static_cast<float>(static_cast<double>(x.z) * inv);
            S[r][4 * q + 3] = static_cast<float>(static_cast<double>(x.w) * inv);
        }
    } else {
        for (int idx = tid; idx < kST * kST; idx += 256) {
            const int r = idx >> 6, c = idx & 63;
            const int gi = r0 + r, gj = c0 + c;
            float x = (gi < n && gj < n) ? Xb[static_cast<int64_t>(gi) * n + gj] : 0.0f;
            if (Kb && gi < n && gj < n) {
                x = form_m(x, Kb[static_cast<int64_t>(gi) * n + gj], form.inv_sigma);
                if (yb && gi == gj) x = __fsub_rn(x, yb[gi]);
            }
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
            // upper-only operand storage (mirror_block > 0): the product kernels read the lower triangle
            // only inside the diagonal mirror_block x mirror_block blocks, so the mirrored tile is
            // written there alone (half the operand-copy writes of the scale pass)
            if (I != J && (mirror_block == 0 || r0 / mirror_block == c0 / mirror_block)) {
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

int bound_blocks_per_matrix(int n, int batch) {
    // about 16 rows per block, but at least two blocks per SM over the whole batch (small batches:
    // one row per warp in flight), at most 256 partial sums per matrix (the workspace) and one
    // row per block
    int k = (n + 15) / 16;
    const int fill = (2 * 148 + batch - 1) / batch;
    if (k < fill) k = fill;
    if (k > n) k = n;
    return k < 1 ? 1 : (k > 256 ? 256 : k);
}

cudaError_t launch_frobenius_partials(const float* X, int n, int batch, double* partial, int nblk,
                                      cudaStream_t stream, const InputForm& form) {
    dim3 grid(nblk, batch);
    frobenius_partials_kernel<<<grid, kBoundThreads, 0, stream>>>(X, n, nblk, partial, form);
    return cudaGetLastError();
}

cudaError_t launch_finalize_bound(const double* partial, int nblk, int batch, double* lambda,
                                  double* lambda_out, unsigned* status, cudaStream_t stream) {
    finalize_bound_kernel<<<batch, 32, 0, stream>>>(partial, nblk, lambda, lambda_out, status);
    return cudaGetLastError();
}

cudaError_t launch_scale_convert(OpType t, const float* X, int n, int npad, int batch,
                                 const double* lambda, double scale, void* out_op, void* out_lo,
                                 double op_scale, float* outF, double post, cudaStream_t stream,
                                 const InputForm& form, int mirror_block) {
    const int nt = npad / kST;
    dim3 grid(nt * (nt + 1) / 2, batch);
    switch (t) {
        case OpType::F16:
            scale_convert_kernel<OpType::F16><<<grid, 256, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<__half*>(out_op), static_cast<__half*>(out_lo),
                static_cast<float>(op_scale), outF, post, form, mirror_block);
            break;
        case OpType::BF16:
            scale_convert_kernel<OpType::BF16><<<grid, 256, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<__nv_bfloat16*>(out_op),
                static_cast<__nv_bfloat16*>(out_lo), static_cast<float>(op_scale), outF, post, form, mirror_block);
            break;
        case OpType::TF32:
            scale_convert_kernel<OpType::TF32><<<grid, 256, 0, stream>>>(
                X, n, npad, lambda, scale, static_cast<float*>(out_op), static_cast<float*>(out_lo),
                static_cast<float>(op_scale), outF, post, form, mirror_block);
            break;
    }
    return cudaGetLastError();
}


// ---------------------------------------------------------------------------------------------
// Lanczos bound: Algorithm 2 line 1 with Theorem 2.  The north star's
// "power-iteration bound" is taken in the paper's form -- a k-step Krylov (Lanczos) run on X^2,
// which contains the k-step power iterate and costs the same two matrix-vector products per
// step (reading R21).  Everything runs on the symmetric operand copy X0 = X / lambda_F (entries
// |.| <= 1, so fp16 is safe; the chain itself runs on this rounded matrix):
//   v_0 = h / ||h||  (h: fixed counter-hash start vector, the oracle implements the same hash)
//   k = 0..m-1:  w = X0 (X0 v_k) (two SYMVs over the upper 128-blocks of X0: half the bytes of
//                a GEMV);  two classical Gram-Schmidt passes against v_0..v_k
//                (alpha_k = the v_k coefficients); beta_k = ||w||; v_{k+1} = w / beta_k
//   (theta, y) = largest eigenpair of the tridiagonal T_m (bisection + inverse iteration)
//   q = V y;  sigma = q^T X0^2 q / q^T q;  r = || X0^2 q / |q| - sigma q / |q| ||
//   lambda~ = lambda_F * min(1, sqrt(sigma + r) / s0 * safety)   (never looser than Frobenius)
// All reductions are fixed-order (per-block partials summed in index order): deterministic.
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int kLzThreads = 1024;
constexpr int kMaxLz = 64;

template <typename E>
__device__ __forceinline__ float elem_to_float(E v);
template <> __device__ __forceinline__ float elem_to_float<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float elem_to_float<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ float elem_to_float<float>(float v) { return v; }

__device__ __forceinline__ double sum_partials(const double* p, int count) {
    double s = 0.0;
    for (int i = 0; i < count; ++i) s += p[i];          // fixed order: identical in every block
    return s;
}

// block-wide sum (fixed order), every thread gets the result; red: >= 32 doubles of smem
__device__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) t += red[w];
    return t;
}

// Symmetric matrix-vector product from the upper 128-blocks of X0 only (half the bytes of a
// full GEMV; every operand layout of the chain -- whole, or upper-only with whole diagonal
// blocks -- holds them).  Block (I, J), I <= J, contributes X_IJ x_J to y_I and, for I < J,
// X_IJ^T x_I to y_J; each contribution goes to its own partial slot P[b][row block][col block]
// and lz_symv_reduce_kernel sums the slots of a row block in block order (deterministic).
constexpr int kSymvB = 128;          // block edge
constexpr int kSymvThreads = 256;    // 16 threads per block row (8 elements each), 16 rows per pass

// x scale: 1 / sqrt(sum of xpart[b][0..xparts)) when xpart != nullptr
__device__ __forceinline__ float symv_xscale(const double* xpart, int xparts, int b) {
    if (!xpart) return 1.0f;
    const double nn = sum_partials(xpart + static_cast<int64_t>(b) * xparts, xparts);
    return static_cast<float>(nn > 0.0 ? 1.0 / sqrt(nn) : 0.0);
}

template <typename E>
__global__ void __launch_bounds__(kSymvThreads, 4)
lz_symv_kernel(const E* __restrict__ A, int npad, int nb, const float* __restrict__ x, int64_t xstride,
               const double* __restrict__ xpart, int xparts, float* __restrict__ P, int reverse) {
    // blockIdx.x enumerates the upper blocks row-major: (I, J), I <= J.  Consecutive launches walk
    // the batch in opposite directions, so a launch starts on the matrices the previous one read
    // last (still in L2)
    const int b = reverse ? static_cast<int>(gridDim.y) - 1 - static_cast<int>(blockIdx.y) : static_cast<int>(blockIdx.y);
    int I = 0, rem = blockIdx.x;
    while (rem >= nb - I) { rem -= nb - I; ++I; }
    const int J = I + rem;
    __shared__ float xI[kSymvB], xJ[kSymvB];
    __shared__ float colp[kSymvThreads / 16][kSymvB];       // column partials of the 16 row groups
    const float sc = symv_xscale(xpart, xparts, b);
    const float* xb = x + static_cast<int64_t>(b) * xstride;
    if (threadIdx.x < kSymvB) xJ[threadIdx.x] = xb[J * kSymvB + threadIdx.x] * sc;
    else xI[threadIdx.x - kSymvB] = xb[I * kSymvB + threadIdx.x - kSymvB] * sc;
    __syncthreads();
    const int cq = threadIdx.x & 15;               // 8-column chunk of this thread
    const int rg = threadIdx.x >> 4;               // row group: rows rg, rg + 16, ...
    constexpr int kEl = 8;
    const E* blk = A + (static_cast<int64_t>(b) * npad + static_cast<int64_t>(I) * kSymvB) * npad +
                   static_cast<int64_t>(J) * kSymvB + cq * kEl;
    float cs[kEl];
#pragma unroll
    for (int e = 0; e < kEl; ++e) cs[e] = 0.0f;
    float xj[kEl];
#pragma unroll
    for (int e = 0; e < kEl; ++e) xj[e] = xJ[cq * kEl + e];
    float* Pb = P + static_cast<int64_t>(b) * nb * npad;
    constexpr int kRows = kSymvB / 16;            // 8 rows per thread
    constexpr int kWords = kEl * sizeof(E) / 16;  // 16-byte loads per row chunk (1 or 2)
    uint4 raw[kRows][kWords];
#pragma unroll
    for (int k = 0; k < kRows; ++k) {             // all loads in flight first
        const uint4* rp = reinterpret_cast<const uint4*>(blk + static_cast<int64_t>(rg + 16 * k) * npad);
#pragma unroll
        for (int w = 0; w < kWords; ++w) raw[k][w] = __ldg(rp + w);
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
        const int i = rg + 16 * k;
        float rs = 0.0f;
        const float xi = xI[i];
        const E* ev = reinterpret_cast<const E*>(raw[k]);
#pragma unroll
        for (int e = 0; e < kEl; ++e) {
            const float a = elem_to_float<E>(ev[e]);
            rs = fmaf(a, xj[e], rs);
            cs[e] = fmaf(a, xi, cs[e]);
        }
        // row sum over the 16 threads of the row (lanes 16h .. 16h + 15 of the warp), fixed order
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
        if (cq == 0) Pb[static_cast<int64_t>(J) * npad + I * kSymvB + i] = rs;   // slot (row block I, col J)
    }
    if (I == J) return;
#pragma unroll
    for (int e = 0; e < kEl; ++e) colp[rg][cq * kEl + e] = cs[e];
    __syncthreads();
    if (threadIdx.x < kSymvB) {
        float t = 0.0f;
#pragma unroll
        for (int g = 0; g < kSymvThreads / 16; ++g) t += colp[g][threadIdx.x];
        Pb[static_cast<int64_t>(I) * npad + J * kSymvB + threadIdx.x] = t;         // slot (row block J, col I)
    }
}

// y[b][rows of block I] = sum over column blocks J of P[b][J][rows] (J = 0..nb-1, fixed order);
// ypart[b][I] = sum of y^2 over the block (fp64)
__global__ void __launch_bounds__(kSymvB)
lz_symv_reduce_kernel(const float* __restrict__ P, int npad, int nb, float* __restrict__ y, double* __restrict__ ypart) {
    __shared__ double red[kSymvB / 32];
    const int b = blockIdx.y, I = blockIdx.x;
    const int i = I * kSymvB + threadIdx.x;
    const float* Pb = P + static_cast<int64_t>(b) * nb * npad;
    float t = 0.0f;
    for (int J = 0; J < nb; ++J) t += Pb[static_cast<int64_t>(J) * npad + i];
    y[static_cast<int64_t>(b) * npad + i] = t;
    double s2 = static_cast<double>(t) * t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s2;
    __syncthreads();
    if (threadIdx.x == 0) ypart[static_cast<int64_t>(b) * nb + I] = ((red[0] + red[1]) + red[2]) + red[3];
}

__device__ __forceinline__ float start_hash(int j) {
    // counter-based start vector, entries in [0.5, 1.5) (oracle: same hash, oracle/bound.py)
    uint32_t h = static_cast<uint32_t>(j) * 2654435761u + 0x9E3779B9u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    return 0.5f + static_cast<float>(h & 0xFFFFu) / 65536.0f;
}

// V: [batch][m+1][npad]; v_0 = h / ||h|| on the first n entries
__global__ void __launch_bounds__(kLzThreads) lz_init_kernel(float* __restrict__ V, int n, int npad, int64_t vstride) {
    __shared__ double red[32];
    float* v = V + static_cast<int64_t>(blockIdx.x) * vstride;
    double s = 0.0;
    for (int j = threadIdx.x; j < n; j += kLzThreads) {
        const double hj = start_hash(j);
        s += hj * hj;
    }
    const double inv = 1.0 / sqrt(block_sum(s, red));
    for (int j = threadIdx.x; j < npad; j += kLzThreads) v[j] = j < n ? static_cast<float>(start_hash(j) * inv) : 0.0f;
}

// one Lanczos step for matrix blockIdx.x: w (= X0^2 v_k, in W) orthogonalised against v_0..v_k
// (CGS2), alpha_k / beta_k recorded, v_{k+1} = w / beta_k.  Dot products: warp i handles the
// basis vectors i, i + 32, ... (warp-shuffle reductions, no block barrier per vector).
__global__ void __launch_bounds__(kLzThreads)
lz_step_kernel(float* __restrict__ V, float* __restrict__ W, int npad, int64_t vstride, int k, double* __restrict__ AB) {
    __shared__ double c[kMaxLz + 1];
    __shared__ double red[32];
    const int b = blockIdx.x;
    float* Vb = V + static_cast<int64_t>(b) * vstride;
    float* w = W + static_cast<int64_t>(b) * npad;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n4 = npad >> 2;                    // float4 groups (npad is a multiple of 128)
    double alpha = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
        // c_i = v_i . w: warp i (i, i + 32, ...), float4 loads, lane partials in fp64, fixed order
        for (int i = warp; i <= k; i += kLzThreads / 32) {
            const float4* vi = reinterpret_cast<const float4*>(Vb + static_cast<int64_t>(i) * npad);
            const float4* w4 = reinterpret_cast<const float4*>(w);
            double s = 0.0;
            for (int j = lane; j < n4; j += 32) {
                const float4 a = vi[j], x = w4[j];
                s += (static_cast<double>(a.x) * x.x + static_cast<double>(a.y) * x.y) +
                     (static_cast<double>(a.z) * x.z + static_cast<double>(a.w) * x.w);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) c[i] = s;
        }
        __syncthreads();
        // w -= sum_i c_i v_i, four consecutive entries per thread
        for (int j = threadIdx.x; j < n4; j += kLzThreads) {
            const float4 x = reinterpret_cast<const float4*>(w)[j];
            double t0 = x.x, t1 = x.y, t2 = x.z, t3 = x.w;
            for (int i = 0; i <= k; ++i) {
                const float4 a = reinterpret_cast<const float4*>(Vb + static_cast<int64_t>(i) * npad)[j];
                t0 -= c[i] * a.x;
                t1 -= c[i] * a.y;
                t2 -= c[i] * a.z;
                t3 -= c[i] * a.w;
            }
            reinterpret_cast<float4*>(w)[j] = make_float4(static_cast<float>(t0), static_cast<float>(t1),
                                                          static_cast<float>(t2), static_cast<float>(t3));
        }
        alpha += c[k];
        __syncthreads();
    }
    double s = 0.0;
    for (int j = threadIdx.x; j < n4; j += kLzThreads) {
        const float4 x = reinterpret_cast<const float4*>(w)[j];
        s += (static_cast<double>(x.x) * x.x + static_cast<double>(x.y) * x.y) +
             (static_cast<double>(x.z) * x.z + static_cast<double>(x.w) * x.w);
    }
    const double beta = sqrt(block_sum(s, red));
    const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
    float4* vn = reinterpret_cast<float4*>(Vb + static_cast<int64_t>(k + 1) * npad);
    for (int j = threadIdx.x; j < n4; j += kLzThreads) {
        const float4 x = reinterpret_cast<const float4*>(w)[j];
        vn[j] = make_float4(static_cast<float>(x.x * inv), static_cast<float>(x.y * inv),
                            static_cast<float>(x.z * inv), static_cast<float>(x.w * inv));
    }
    if (threadIdx.x == 0) {
        AB[static_cast<int64_t>(b) * 2 * kMaxLz + k] = alpha;
        AB[static_cast<int64_t>(b) * 2 * kMaxLz + kMaxLz + k] = beta;
    }
}

// number of eigenvalues of the tridiagonal (a, e) smaller than x (Sturm sequence)
__device__ int sturm_count(const double* a, const double* e, int m, double x) {
    int cnt = 0;
    double d = a[0] - x;
    if (d < 0.0) ++cnt;
    for (int i = 1; i < m; ++i) {
        if (d == 0.0) d = 1e-300;
        d = (a[i] - x) - e[i - 1] * e[i - 1] / d;
        if (d < 0.0) ++cnt;
    }
    return cnt;
}

// Largest Ritz pair of T_m (thread 0: bisection + two inverse-iteration solves with partial
// pivoting), then q = V y by the whole block; qn2 = ||q||^2.
__global__ void __launch_bounds__(kLzThreads)
lz_ritz_kernel(const float* __restrict__ V, int npad, int64_t vstride, int m, const double* __restrict__ AB,
               float* __restrict__ q, double* __restrict__ qn2) {
    __shared__ double a[kMaxLz], e[kMaxLz], y[kMaxLz];
    __shared__ double d[kMaxLz], du[kMaxLz], du2[kMaxLz], dl[kMaxLz];
    __shared__ double red[32];
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < m; ++i) {
            a[i] = AB[static_cast<int64_t>(b) * 2 * kMaxLz + i];
            e[i] = AB[static_cast<int64_t>(b) * 2 * kMaxLz + kMaxLz + i];   // e[m-1] unused
        }
        double lo = a[0], hi = a[0];
        for (int i = 0; i < m; ++i) {
            const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < m - 1 ? fabs(e[i]) : 0.0);
            lo = fmin(lo, a[i] - r);
            hi = fmax(hi, a[i] + r);
        }
        for (int it = 0; it < 200 && hi - lo > 1e-15 * fmax(fabs(lo), fabs(hi)); ++it) {
            const double mid = 0.5 * (lo + hi);
            if (sturm_count(a, e, m, mid) <= m - 1) lo = mid; else hi = mid;
        }
        const double theta = hi;
        const double mu = theta + 1e-12 * fmax(fabs(theta), 1e-300);
        for (int i = 0; i < m; ++i) y[i] = 1.0;
        for (int rep = 0; rep < 2; ++rep) {
            for (int i = 0; i < m; ++i) {
                d[i] = a[i] - mu;
                du[i] = e[i];
                dl[i] = e[i];
                du2[i] = 0.0;
            }
            for (int i = 0; i < m - 1; ++i) {
                if (fabs(d[i]) >= fabs(dl[i])) {
                    if (d[i] == 0.0) d[i] = 1e-300;
                    const double f = dl[i] / d[i];
                    d[i + 1] -= f * du[i];
                    y[i + 1] -= f * y[i];
                } else {
                    const double f = d[i] / dl[i];
                    const double t = d[i + 1];
                    d[i] = dl[i];
                    d[i + 1] = du[i] - f * t;
                    if (i < m - 2) {
                        du2[i] = du[i + 1];
                        du[i + 1] = -f * du2[i];
                    }
                    du[i] = t;
                    const double bt = y[i];
                    y[i] = y[i + 1];
                    y[i + 1] = bt - f * y[i];
                }
            }
            if (d[m - 1] == 0.0) d[m - 1] = 1e-300;
            y[m - 1] /= d[m - 1];
            if (m > 1) y[m - 2] = (y[m - 2] - du[m - 2] * y[m - 1]) / d[m - 2];
            for (int i = m - 3; i >= 0; --i) y[i] = (y[i] - du[i] * y[i + 1] - du2[i] * y[i + 2]) / d[i];
            double nn = 0.0;
            for (int i = 0; i < m; ++i) nn += y[i] * y[i];
            const double inv = nn > 0.0 && isfinite(nn) ? 1.0 / sqrt(nn) : 0.0;
            for (int i = 0; i < m; ++i) y[i] *= inv;
        }
    }
    __syncthreads();
    const float* Vb = V + static_cast<int64_t>(b) * vstride;
    double s = 0.0;
    for (int j = threadIdx.x; j < npad; j += kLzThreads) {
        double t = 0.0;
        for (int i = 0; i < m; ++i) t += y[i] * Vb[static_cast<int64_t>(i) * npad + j];
        q[static_cast<int64_t>(b) * npad + j] = static_cast<float>(t);
        s += t * t;
    }
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) qn2[b] = tot;
}

// r^2 partials: || |w| z - sigma q / |q| ||^2 with w = X0 q/|q| (partials wpart: sigma = |w|^2)
// and z = X0 w / |w|, so X0^2 q/|q| = |w| z.
__global__ void lz_residual_kernel(const float* __restrict__ q, const double* __restrict__ qn2, const float* __restrict__ z,
                                   const double* __restrict__ wpart, int parts, int npad, double* __restrict__ rpart) {
    __shared__ double red[32];
    const int b = blockIdx.y;
    const double invq = qn2[b] > 0.0 ? 1.0 / sqrt(qn2[b]) : 0.0;
    const double sigma = sum_partials(wpart + static_cast<int64_t>(b) * parts, parts);
    const double wn = sqrt(sigma);
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += gridDim.x * blockDim.x) {
        const double dd = wn * z[static_cast<int64_t>(b) * npad + i] - sigma * q[static_cast<int64_t>(b) * npad + i] * invq;
        acc += dd * dd;
    }
    const double tot = block_sum(acc, red);
    if (threadIdx.x == 0) rpart[static_cast<int64_t>(b) * gridDim.x + blockIdx.x] = tot;
}

__global__ void lz_finalize_kernel(const double* __restrict__ wpart, int parts, const double* __restrict__ rpart,
                                   int rparts, double s0, double safety, double* lambda, double* lambda_out) {
    const int b = blockIdx.x;
    const double sigma = sum_partials(wpart + static_cast<int64_t>(b) * parts, parts);
    const double r = sqrt(sum_partials(rpart + static_cast<int64_t>(b) * rparts, rparts));
    // ||X0||_2 <= sqrt(sigma + r) / s0 (Thm 2); never looser than Frobenius (||X0||_F = 1)
    double f = sqrt(sigma + r) / s0 * safety;
    if (!(f < 1.0)) f = 1.0;
    if (!(f > 0.0)) f = 1.0;                             // zero matrix / NaN: keep lambda_F
    const double lam = lambda[b] * f;
    lambda[b] = lam;
    if (lambda_out) lambda_out[b] = lam;
}

template <typename E>
void symv_launch(const void* A, int npad, int batch, const float* x, int64_t xstride, const double* xpart, int xparts,
                 float* P, float* y, double* ypart, int reverse, cudaStream_t stream) {
    const int nb = npad / kSymvB;
    lz_symv_kernel<E><<<dim3(nb * (nb + 1) / 2, batch), kSymvThreads, 0, stream>>>(
        static_cast<const E*>(A), npad, nb, x, xstride, xpart, xparts, P, reverse);
    lz_symv_reduce_kernel<<<dim3(nb, batch), kSymvB, 0, stream>>>(P, npad, nb, y, ypart);
}

}  // namespace

void lanczos_prepare() {}

int lanczos_parts(int npad) { return npad / kSymvB; }

int lanczos_launches(int steps, int n) { return 5 * (steps < n ? steps : n) + 8; }

size_t lanczos_scratch_bytes(int npad, int batch, int steps) {
    const size_t parts = static_cast<size_t>(lanczos_parts(npad));
    return static_cast<size_t>(batch) * npad * 4 * (steps + 1 + 4) +           // V, t, w, q, z
           static_cast<size_t>(batch) * npad * 4 * parts +                    // SYMV partials
           static_cast<size_t>(batch) * 8 * (2 * kMaxLz + 2 * parts + 16 + 1) + 256;
}

cudaError_t launch_lanczos_bound(OpType t, const void* X0, double s0, int n, int npad, int batch, int steps,
                                 double safety, void* scratch, double* lambda, double* lambda_out, cudaStream_t stream) {
    if (npad % kSymvB != 0 || steps < 1 || steps > kMaxLz) return cudaErrorInvalidValue;
    const int m = steps < n ? steps : n;
    const int parts = lanczos_parts(npad);
    const int64_t vstride = static_cast<int64_t>(m + 1) * npad;
    float* V = static_cast<float*>(scratch);
    float* tv = V + static_cast<int64_t>(batch) * vstride;
    float* wv = tv + static_cast<int64_t>(batch) * npad;
    float* qv = wv + static_cast<int64_t>(batch) * npad;
    float* zv = qv + static_cast<int64_t>(batch) * npad;
    float* P = zv + static_cast<int64_t>(batch) * npad;
    double* AB = reinterpret_cast<double*>(P + static_cast<int64_t>(batch) * npad * parts);
    double* pa = AB + static_cast<int64_t>(batch) * 2 * kMaxLz;
    double* pb = pa + static_cast<int64_t>(batch) * parts;
    double* pr = pb + static_cast<int64_t>(batch) * parts;
    double* qn2 = pr + static_cast<int64_t>(batch) * 16;
    int dir = 0;
    auto symv = [&](const float* x, int64_t xs, const double* xp, int xps, float* y, double* yp) {
        switch (t) {
            case OpType::F16: symv_launch<__half>(X0, npad, batch, x, xs, xp, xps, P, y, yp, dir, stream); break;
            case OpType::BF16: symv_launch<__nv_bfloat16>(X0, npad, batch, x, xs, xp, xps, P, y, yp, dir, stream); break;
            case OpType::TF32: symv_launch<float>(X0, npad, batch, x, xs, xp, xps, P, y, yp, dir, stream); break;
        }
        dir ^= 1;
    };
    lz_init_kernel<<<batch, kLzThreads, 0, stream>>>(V, n, npad, vstride);
    for (int k = 0; k < m; ++k) {
        symv(V + static_cast<int64_t>(k) * npad, vstride, nullptr, 0, tv, pa);   // t = X0 v_k
        symv(tv, npad, nullptr, 0, wv, pa);                                      // w = X0 t
        lz_step_kernel<<<batch, kLzThreads, 0, stream>>>(V, wv, npad, vstride, k, AB);
    }
    lz_ritz_kernel<<<batch, kLzThreads, 0, stream>>>(V, npad, vstride, m, AB, qv, qn2);
    symv(qv, npad, qn2, 1, wv, pa);        // w = X0 q / |q|,  sigma = |w|^2
    symv(wv, npad, pa, parts, zv, pb);     // z = X0 w / |w|
    constexpr int kRBlocks = 16;
    lz_residual_kernel<<<dim3(kRBlocks, batch), 256, 0, stream>>>(qv, qn2, zv, pa, parts, npad, pr);
    lz_finalize_kernel<<<batch, 1, 0, stream>>>(pa, parts, pr, kRBlocks, s0, safety, lambda, lambda_out);
    return cudaGetLastError();
}

}  // namespace psd
