// Micro test: host -> device transfer of only the upper triangle of fp32 matrices in pinned host
// memory, by a kernel reading the host buffer directly (zero-copy over PCIe), against the copy
// engine moving the whole matrices; both alone and while the copy engine runs a device -> host
// copy of the same size (the e2e pipeline's duplex situation).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc tools/micro/zc_upper.cu && ./zc
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

// one warp per (matrix, row): the float4 groups of row r from column (r & ~3) on; 4 loads in
// flight per lane
__global__ void __launch_bounds__(64) upper_rows_kernel(const float* __restrict__ src, float* __restrict__ dst, int n,
                                                        int batch) {
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x / 32);
    const int w0 = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int64_t rows = static_cast<int64_t>(batch) * n;
    const int nq = n / 4;
    for (int64_t gr = w0; gr < rows; gr += warps) {
        const int r = static_cast<int>(gr % n);
        const float4* s = reinterpret_cast<const float4*>(src + gr * n);
        float4* d = reinterpret_cast<float4*>(dst + gr * n);
        for (int q0 = r / 4 + lane; q0 < nq; q0 += 128) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + 32 * u;
                if (q < nq) v[u] = __ldcs(s + q);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + 32 * u;
                if (q < nq) d[q] = v[u];
            }
        }
    }
}

int main() {
    const int n = 4096, batch = 4;
    const size_t bytes = static_cast<size_t>(batch) * n * n * 4;
    float *h_in, *h_out, *d_in, *d_out;
    CK(cudaHostAlloc(&h_in, bytes, cudaHostAllocDefault));
    CK(cudaHostAlloc(&h_out, bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&d_in, bytes));
    CK(cudaMalloc(&d_out, bytes));
    for (size_t i = 0; i < bytes / 4; ++i) h_in[i] = static_cast<float>(i % 1000);
    float* h_in_dev = nullptr;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_in_dev), h_in, 0));
    printf("mapped pointer %s the host pointer\n", h_in_dev == h_in ? "equals" : "differs from");
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t a, b, c, d;
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c); cudaEventCreate(&d);
    const double upper = static_cast<double>(batch) * (static_cast<double>(n) * n / 2 + n * 2) * 4;
    for (int rep = 0; rep < 2; ++rep) {
        // copy engine, whole matrices
        cudaEventRecord(a, s0);
        CK(cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, s0));
        cudaEventRecord(b, s0);
        CK(cudaStreamSynchronize(s0));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("copy engine H2D whole: %.2f ms, %.1f GB/s\n", ms, bytes / ms / 1e6);
        for (int grid : {148, 296, 592}) {
            cudaEventRecord(a, s0);
            upper_rows_kernel<<<grid, 64, 0, s0>>>(h_in_dev, d_in, n, batch);
            cudaEventRecord(b, s0);
            CK(cudaStreamSynchronize(s0));
            CK(cudaGetLastError());
            cudaEventElapsedTime(&ms, a, b);
            printf("zero-copy upper (grid %d x 64): %.2f ms, %.1f GB/s of upper bytes, %.1f GB/s whole-equivalent\n",
                   grid, ms, upper / ms / 1e6, bytes / ms / 1e6);
        }
        // duplex: D2H of the same size on s1 concurrently
        for (int mode = 0; mode < 2; ++mode) {
            cudaEventRecord(c, s1);
            CK(cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, s1));
            cudaEventRecord(d, s1);
            cudaEventRecord(a, s0);
            if (mode == 0) CK(cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, s0));
            else upper_rows_kernel<<<296, 64, 0, s0>>>(h_in_dev, d_in, n, batch);
            cudaEventRecord(b, s0);
            CK(cudaDeviceSynchronize());
            float m1, m2; cudaEventElapsedTime(&m1, a, b); cudaEventElapsedTime(&m2, c, d);
            printf("duplex (%s H2D): H2D %.2f ms, D2H %.2f ms\n", mode ? "zero-copy upper" : "copy-engine whole", m1, m2);
        }
    }
    // correctness of one row
    CK(cudaMemcpy(h_out, d_in, bytes, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int r = 0; r < n; r += 511)
        for (int col = (r & ~3); col < n; ++col)
            if (h_out[static_cast<size_t>(r) * n + col] != h_in[static_cast<size_t>(r) * n + col]) ++bad;
    printf("mismatches: %d\n", bad);
    return 0;
}
