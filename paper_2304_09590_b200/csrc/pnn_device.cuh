// pnn_device.cuh — device helpers shared by the CUDA kernels of the product
// path (NOT shared with oracle/, which has its own C implementation).
#pragma once
#include <cuda_runtime.h>
#include "pnn.h"

// φ (Eqs.3-5; sigmoid/tanh from §5.2).  Accurate libdevice
// expf/tanhf (no fast-math) so the fp32 path tracks the fp32 oracle.
__device__ __forceinline__ float act_fwd(int act, float z) {
    switch (act) {
    case PNN_SIGMOID: return 1.f / (1.f + expf(-z));
    case PNN_TANH: return tanhf(z);
    case PNN_RELU: return z >= 0.f ? z : 0.f;      // Eq.4
    case PNN_LEAKY_RELU: return z >= 0.f ? z : 0.01f * z;   // R30
    default: return z;
    }
}

// φ'(z) from the stored activation x (reading R10; R9: ReLU'(0) = 0).
__device__ __forceinline__ float act_deriv_from_x(int act, float x) {
    switch (act) {
    case PNN_SIGMOID: return x * (1.f - x);
    case PNN_TANH: return 1.f - x * x;
    case PNN_RELU: return x > 0.f ? 1.f : 0.f;
    case PNN_LEAKY_RELU: return x > 0.f ? 1.f : 0.01f;
    default: return 1.f;
    }
}

__device__ __forceinline__ double act_fwd_d(int act, double z) {
    switch (act) {
    case PNN_SIGMOID: return 1.0 / (1.0 + exp(-z));
    case PNN_TANH: return tanh(z);
    case PNN_RELU: return z >= 0.0 ? z : 0.0;
    case PNN_LEAKY_RELU: return z >= 0.0 ? z : (double)0.01f * z;   // fp32 slope, exact product
    default: return z;
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// In-place max-subtracted softmax (Eq.5, reading R4) of z[0..n) by one warp.
__device__ __forceinline__ void softmax_warp(float* z, int n, int lane) {
    float m = -INFINITY;
    for (int k = lane; k < n; k += 32) m = fmaxf(m, z[k]);
    m = warp_max(m);
    float s = 0.f;
    for (int k = lane; k < n; k += 32) {
        float u = expf(z[k] - m);
        z[k] = u;
        s += u;
    }
    s = warp_sum(s);
    for (int k = lane; k < n; k += 32) z[k] = z[k] / s;
}

// Compile-time activation variants (no jump tables on the latency-critical tail).
template <int A> __device__ __forceinline__ float act_fwd_t(float z) {
    if constexpr (A == PNN_SIGMOID) return __frcp_rn(1.f + expf(-z));   // == 1.f/(1+e^-z), IEEE
    else if constexpr (A == PNN_TANH) return tanhf(z);
    else if constexpr (A == PNN_RELU) return z >= 0.f ? z : 0.f;
    else if constexpr (A == PNN_LEAKY_RELU) return z >= 0.f ? z : 0.01f * z;
    else return z;
}
template <int A> __device__ __forceinline__ float act_deriv_t(float x) {
    if constexpr (A == PNN_SIGMOID) return x * (1.f - x);
    else if constexpr (A == PNN_TANH) return 1.f - x * x;
    else if constexpr (A == PNN_RELU) return x > 0.f ? 1.f : 0.f;
    else if constexpr (A == PNN_LEAKY_RELU) return x > 0.f ? 1.f : 0.01f;
    else return 1.f;
}
