// k_merge.cu — the averaging merge ("the average of all
// weights … For the biases the same procedure"; :233-238 "weights, and
// biases are added onto the PNN … scaled by the number of CNs"; reading R18).
//
// HBM-bound: reads K_local·P fp32 once (coalesced: thread i walks child slabs
// c = 0..K_local-1 at the same offset i, 16 loads in flight), writes P fp32 (or fp64 partials for
// the cross-rank all-reduce).  Sums in fp64 in ascending CN order, so K
// identical clones average back to the clone exactly, then divides by K and
// rounds once to fp32.
#include "pnn_internal.h"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double child_sum(const float* __restrict__ ch, int K_local,
                                            long long P, long long i) {
    double s = 0.0;
    int c = 0;
    // 16 independent loads in flight per thread (one element per thread leaves too few bytes in
    // flight per SM for HBM otherwise), summed in ascending c order.
    for (; c + 16 <= K_local; c += 16) {
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcs(ch + (long long)(c + u) * P + i);
#pragma unroll
        for (int u = 0; u < 16; ++u) s += (double)v[u];
    }
    for (; c < K_local; ++c) s += (double)__ldcs(ch + (long long)c * P + i);
    return s;
}

__global__ void __launch_bounds__(kThreads)
merge_sum_kernel(const float* __restrict__ ch, int K_local, long long P, double* __restrict__ sum) {
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < P;
         i += (long long)gridDim.x * kThreads)
        sum[i] = child_sum(ch, K_local, P, i);
}

__global__ void __launch_bounds__(kThreads)
merge_finish_kernel(const double* __restrict__ sum, long long P, int K, float* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < P;
         i += (long long)gridDim.x * kThreads)
        out[i] = (float)(sum[i] / (double)K);
}

__global__ void __launch_bounds__(kThreads)
merge_local_kernel(const float* __restrict__ ch, int K_local, long long P, int K,
                   float* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < P;
         i += (long long)gridDim.x * kThreads)
        out[i] = (float)(child_sum(ch, K_local, P, i) / (double)K);
}

int grid_for(long long P) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (P + kThreads - 1) / kThreads;
    long long cap = (long long)sms * 8;       // 8 resident 256-thread CTAs per SM
    return (int)(blocks < cap ? blocks : cap);
}

}  // namespace

cudaError_t launch_merge_sum(const float* children, int K_local, long long P, double* sum,
                             cudaStream_t st) {
    merge_sum_kernel<<<grid_for(P), kThreads, 0, st>>>(children, K_local, P, sum);
    return cudaGetLastError();
}

cudaError_t launch_merge_finish(const double* sum, long long P, int K, float* merged,
                                cudaStream_t st) {
    merge_finish_kernel<<<grid_for(P), kThreads, 0, st>>>(sum, P, K, merged);
    return cudaGetLastError();
}

cudaError_t launch_merge_local(const float* children, int K_local, long long P, int K,
                               float* merged, cudaStream_t st) {
    merge_local_kernel<<<grid_for(P), kThreads, 0, st>>>(children, K_local, P, K, merged);
    return cudaGetLastError();
}
