// certificate.cu -- the filter's scalar worst-case errors on the device (Eq. comp:error-approx,
// P:L583-590; Eq. comp:minimax-sign):
//     relu_err = max over every float32 x in [0, 1] of 1/2 x |1 - s(x)|
//     sign_err = max over every float32 x in [eps, 1] of |s(x) - 1|
// with s = f_T o ... o f_1 the chain the handle holds (stabilisation folded), evaluated in fp64.
// s is odd, so both maxima over [-1, 1] equal the maxima over [0, 1]: bit patterns
// 0x00000000 .. 0x3F800000, about 1.07e9 values -- one pass of this kernel (a few ms), where a
// CPU takes seconds.  Deterministic: per-block maxima (ties to the smaller x), then a fixed-order
// reduction.
#include "kernels.h"

#include <cmath>
#include <cstring>
#include <vector>

namespace psd {

namespace {

constexpr int kCertThreads = 256;
constexpr int kMaxCoef = 64;

struct CertChain {
    int T;
    int ncoef[32];
    double c[kMaxCoef];
};

__device__ __forceinline__ double scalar_chain(double x, const CertChain& ch) {
    int k = 0;
    for (int t = 0; t < ch.T; ++t) {
        const double x2 = x * x;
        double acc = ch.c[k + ch.ncoef[t] - 1];
        for (int j = ch.ncoef[t] - 2; j >= 0; --j) acc = acc * x2 + ch.c[k + j];   // Horner in x^2
        x = acc * x;
        k += ch.ncoef[t];
    }
    return x;
}

__device__ __forceinline__ void better(double& v, double& x, double v2, double x2) {
    if (v2 > v || (v2 == v && x2 < x)) { v = v2; x = x2; }
}

// mode 0: relu error over [0, 1]; mode 1: sign error over [first, 1]
__global__ void __launch_bounds__(kCertThreads)
certify_kernel(const CertChain ch, int mode, uint32_t first, double* __restrict__ part_v, double* __restrict__ part_x) {
    const uint32_t last = 0x3F800000u;
    double bv = -1.0, bx = 0.0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t u = first + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u <= last; u += stride) {
        const double x = static_cast<double>(__uint_as_float(static_cast<uint32_t>(u)));
        const double s = scalar_chain(x, ch);
        const double e = mode == 0 ? 0.5 * x * fabs(1.0 - s) : fabs(s - 1.0);
        better(bv, bx, e, x);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o), x2 = __shfl_xor_sync(0xffffffffu, bx, o);
        better(bv, bx, v2, x2);
    }
    __shared__ double sv[kCertThreads / 32], sx[kCertThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { sv[warp] = bv; sx[warp] = bx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kCertThreads / 32; ++w) better(bv, bx, sv[w], sx[w]);
        part_v[blockIdx.x] = bv;
        part_x[blockIdx.x] = bx;
    }
}

}  // namespace

// Host: both maxima for the chain `coeffs` (stage-major, ncoef[t] coefficients of x, x^3, ...).
cudaError_t certify_chain(const std::vector<std::vector<double>>& coeffs, double eps, double* relu_err,
                          double* relu_argmax, double* sign_err, double* sign_argmax) {
    CertChain ch{};
    ch.T = static_cast<int>(coeffs.size());
    int k = 0;
    for (int t = 0; t < ch.T; ++t) {
        if (t >= 32 || k + static_cast<int>(coeffs[t].size()) > kMaxCoef) return cudaErrorInvalidValue;
        ch.ncoef[t] = static_cast<int>(coeffs[t].size());
        for (double c : coeffs[t]) ch.c[k++] = c;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8;
    double* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 2 * blocks * sizeof(double));
    if (e != cudaSuccess) return e;
    std::vector<double> v(blocks), x(blocks);
    float fe = static_cast<float>(eps);
    if (static_cast<double>(fe) < eps) fe = std::nextafter(fe, 2.0f);     // first float32 >= eps
    uint32_t first_sign;
    std::memcpy(&first_sign, &fe, 4);
    double out_v[2] = {0, 0}, out_x[2] = {0, 0};
    for (int mode = 0; mode < 2 && e == cudaSuccess; ++mode) {
        certify_kernel<<<blocks, kCertThreads>>>(ch, mode, mode == 0 ? 0u : first_sign, d, d + blocks);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(v.data(), d, blocks * sizeof(double), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(x.data(), d + blocks, blocks * sizeof(double), cudaMemcpyDeviceToHost);
        double bv = -1.0, bx = 0.0;
        for (int i = 0; i < blocks; ++i)
            if (v[i] > bv || (v[i] == bv && x[i] < bx)) { bv = v[i]; bx = x[i]; }
        out_v[mode] = bv;
        out_x[mode] = bx;
    }
    cudaFree(d);
    if (relu_err) *relu_err = out_v[0];
    if (relu_argmax) *relu_argmax = out_x[0];
    if (sign_err) *sign_err = out_v[1];
    if (sign_argmax) *sign_argmax = out_x[1];
    return e;
}

}  // namespace psd
