// optraits.cuh -- operand element types of the symmetric product kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kernels.h"

namespace psd {

template <OpType T> struct OpTraits;
template <> struct OpTraits<OpType::F16> {
    using type = __half;
    static constexpr int kBytes = 2;
    static constexpr uint32_t kFmt = 0;          // tcgen05 instruction-descriptor A/B format
    __device__ static type cvt(float v) { return __float2half_rn(v); }
    __device__ static float to_float(type v) { return __half2float(v); }
    __device__ static uint32_t pack2(float lo, float hi) {
        __half2 h = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static void unpack2(uint32_t w, float& lo, float& hi) {
        const __half2 h = *reinterpret_cast<const __half2*>(&w);
        const float2 f = __half22float2(h);
        lo = f.x;
        hi = f.y;
    }
};
template <> struct OpTraits<OpType::BF16> {
    using type = __nv_bfloat16;
    static constexpr int kBytes = 2;
    static constexpr uint32_t kFmt = 1;
    __device__ static type cvt(float v) { return __float2bfloat16_rn(v); }
    __device__ static float to_float(type v) { return __bfloat162float(v); }
    __device__ static uint32_t pack2(float lo, float hi) {
        __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static void unpack2(uint32_t w, float& lo, float& hi) {
        lo = __uint_as_float(w << 16);
        hi = __uint_as_float(w & 0xFFFF0000u);
    }
};
template <> struct OpTraits<OpType::TF32> {
    using type = float;
    static constexpr int kBytes = 4;
    static constexpr uint32_t kFmt = 2;
    __device__ static type cvt(float v) {        // round-to-nearest (ties away) to tf32
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
        return __uint_as_float(r);
    }
    __device__ static float to_float(type v) { return v; }
    __device__ static uint32_t pack2(float, float) { return 0u; }
    __device__ static void unpack2(uint32_t, float& lo, float& hi) { lo = hi = 0.0f; }
};

}  // namespace psd
