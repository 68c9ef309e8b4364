// k_predict.cu — classification readout ("each class is
// represented by one neuron in the last layer … the probabilities of being
// that class"; reading R19: label = argmax_k z^L_k, ties → lowest index).
//
// The forward pass (Eqs.2-3) runs in fp64 from the fp32 parameters (each
// fp32×fp32 product is exact in fp64), so the argmax decision is taken in
// fp64 on both the GPU and the oracle side (R26).  A CTA classifies
// a tile of TILE samples: every weight is read once per tile (warp per
// output neuron, lanes over inputs) and applied to the TILE activations held
// in shared memory (inputs converted to fp64 once per tile).
#include "pnn_internal.h"
#include "pnn_device.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <int TILE, bool EVAL>
__global__ void __launch_bounds__(kThreads, 2)     // <= 128 registers: two CTAs per SM (3: heavy spills)
predict_kernel(NetDesc d, const float* __restrict__ params, const float* __restrict__ X,
               long long n, int32_t* __restrict__ labels, const int32_t* __restrict__ ytrue,
               double* __restrict__ rowstats) {
    extern __shared__ double smd[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n0 = d.n[0];
    int Hm = 1;
    for (int l = 1; l <= d.L; ++l) Hm = d.n[l] > Hm ? d.n[l] : Hm;
    double* hb[2] = {smd, smd + (size_t)TILE * Hm};             // [TILE][Hm] fp64 activations
    double* xin = smd + 2 * (size_t)TILE * Hm;                 // [TILE][n0] inputs, converted once
    for (long long t0 = (long long)blockIdx.x * TILE; t0 < n; t0 += (long long)gridDim.x * TILE) {
        const int nt = (int)((n - t0) < TILE ? (n - t0) : TILE);
        if ((n0 & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
            // 16-byte loads, all of a thread's loads issued before the first conversion (one DRAM
            // round trip per tile instead of one per unrolled group of scalar loads)
            const int n4 = n0 >> 2;
            constexpr int kMaxV = 4;                       // float4 loads in flight per thread
            for (int i0 = tid; i0 < TILE * n4; i0 += kMaxV * kThreads) {
                float4 v[kMaxV];
#pragma unroll
                for (int u = 0; u < kMaxV; ++u) {
                    const int i = i0 + u * kThreads;
                    const int s = i / n4, j4 = i - s * n4;
                    v[u] = (i < TILE * n4 && s < nt)
                               ? *reinterpret_cast<const float4*>(X + (t0 + s) * n0 + 4 * j4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < kMaxV; ++u) {
                    const int i = i0 + u * kThreads;
                    if (i < TILE * n4) {
                        double2* dst = reinterpret_cast<double2*>(xin + 4 * (size_t)i);
                        dst[0] = make_double2((double)v[u].x, (double)v[u].y);
                        dst[1] = make_double2((double)v[u].z, (double)v[u].w);
                    }
                }
            }
        } else {
            for (int i = tid; i < TILE * n0; i += kThreads) {
                int s = i / n0, j = i % n0;
                xin[i] = (s < nt) ? (double)X[(t0 + s) * n0 + j] : 0.0;
            }
        }
        __syncthreads();
        const double* inD = nullptr;
        int W = n0;
        for (int l = 1; l <= d.L; ++l) {
            const int nin = d.n[l - 1], nout = d.n[l];
            const float* Wl = params + d.woff[l];
            const float* bl = Wl + (long long)nout * nin;
            double* out = hb[(l - 1) & 1];
            // a warp forms KB neurons × TILE samples at once (each x value read from shared
            // memory feeds KB fmas); the per-lane partial sums then go through a transpose-reduce
            // whose pairing (xor 16, 8, 4, 2, 1) is that of warp_sum_d, so z is bit-identical
            constexpr int KB = 32 / TILE;
            const double* inp = (l == 1) ? xin : inD;
            for (int k0 = warp * KB; k0 < nout; k0 += kWarps * KB) {
                double acc[KB * TILE];
#pragma unroll
                for (int i = 0; i < KB * TILE; ++i) acc[i] = 0.0;
                // unrolled so each lane has several weight loads in flight (the loop is bound by
                // their latency, not by the DFMAs)
#pragma unroll 4
                for (int j = lane; j < nin; j += 32) {
                    double xv[TILE];
#pragma unroll
                    for (int s = 0; s < TILE; ++s) xv[s] = inp[s * W + j];
#pragma unroll
                    for (int kk = 0; kk < KB; ++kk) {
                        const double wj = (k0 + kk < nout) ? (double)Wl[(long long)(k0 + kk) * nin + j] : 0.0;
#pragma unroll
                        for (int s = 0; s < TILE; ++s) acc[kk * TILE + s] = fma(wj, xv[s], acc[kk * TILE + s]);
                    }
                }
#pragma unroll
                for (int h = 16; h >= 1; h >>= 1) {      // 32 values → lane l holds value l
                    const bool up = lane & h;
#pragma unroll
                    for (int i = 0; i < h; ++i) {
                        const double keep = up ? acc[i + h] : acc[i], give = up ? acc[i] : acc[i + h];
                        acc[i] = keep + __shfl_xor_sync(0xffffffffu, give, h);
                    }
                }
                const int kk = lane / TILE, s = lane % TILE, k = k0 + kk;
                if (k < nout) {
                    const double z = acc[0] + (double)bl[k];
                    // softmax is monotone: the readout only needs z^L (R19)
                    out[s * Hm + k] = (l == d.L) ? z : act_fwd_d(d.act[l - 1], z);
                }
            }
            __syncthreads();
            inD = out;
            W = Hm;
        }
        // argmax over z^L (now in inD), ties → lowest index
        if (tid < nt) {
            const double* z = inD + tid * Hm;
            int best = 0;
            for (int k = 1; k < d.n[d.L]; ++k) if (z[k] > z[best]) best = k;
            if (labels) labels[t0 + tid] = best;
            if constexpr (EVAL) {
                const int O = d.n[d.L], a = d.act[d.L - 1], yv = ytrue[t0 + tid];
                double xmax, xy;
                if (a == PNN_SOFTMAX) {
                    double sum = 0.0;
                    for (int k = 0; k < O; ++k) sum += exp(z[k] - z[best]);
                    xmax = 1.0 / sum;
                    xy = (yv >= 0 && yv < O) ? exp(z[yv] - z[best]) / sum : 0.0;
                } else {
                    xmax = -INFINITY;
                    for (int k = 0; k < O; ++k) xmax = fmax(xmax, act_fwd_d(a, z[k]));
                    xy = (yv >= 0 && yv < O) ? act_fwd_d(a, z[yv]) : 0.0;
                }
                double* r = rowstats + 3 * (t0 + tid);
                r[0] = (best == yv) ? 1.0 : 0.0;
                r[1] = xmax;
                r[2] = -log(fmax(xy, 1e-12));
            }
        }
        __syncthreads();
    }
}

// Mean of each of the 3 row-statistic columns over n rows: one CTA, fixed
// per-thread strides and a fixed tree, so the result is deterministic.
__global__ void __launch_bounds__(1024) eval_reduce(const double* __restrict__ rowstats, long long n,
                                                    double* __restrict__ out) {
    __shared__ double sh[3][1024];
    double a[3] = {0.0, 0.0, 0.0};
    for (long long i = threadIdx.x; i < n; i += 1024)
        for (int c = 0; c < 3; ++c) a[c] += rowstats[3 * i + c];
    for (int c = 0; c < 3; ++c) sh[c][threadIdx.x] = a[c];
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int c = 0; c < 3; ++c) sh[c][threadIdx.x] += sh[c][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 3) out[threadIdx.x] = sh[threadIdx.x][0] / (double)n;
}

template <int TILE, bool EVAL>
size_t pred_smem(const NetDesc& d) {
    int Hm = 1;
    for (int l = 1; l <= d.L; ++l) Hm = d.n[l] > Hm ? d.n[l] : Hm;
    return sizeof(double) * TILE * (2 * (size_t)Hm + (size_t)d.n[0]);
}

template <int TILE, bool EVAL>
cudaError_t launch_pred_t(const NetDesc& d, const float* params, const float* x, long long n, int32_t* labels,
                          const int32_t* ytrue, double* rowstats, cudaStream_t st) {
    const size_t smem = pred_smem<TILE, EVAL>(d);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(predict_kernel<TILE, EVAL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long tiles = (n + TILE - 1) / TILE;
    int per_sm = 1;                                 // CTAs that are actually co-resident
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_kernel<TILE, EVAL>, kThreads, smem) != cudaSuccess
        || per_sm < 1)
        per_sm = 1;
    const int grid = (int)(tiles < (long long)sms * per_sm ? tiles : (long long)sms * per_sm);
    predict_kernel<TILE, EVAL><<<grid, kThreads, smem, st>>>(d, params, x, n, labels, ytrue, rowstats);
    return cudaGetLastError();
}

// The tile (rows per CTA, each weight read once per tile): 8, else 2 when 8 rows of fp64
// inputs + activations do not fit in shared memory.
template <bool EVAL>
cudaError_t launch_pred(const NetDesc& d, const float* params, const float* x, long long n, int32_t* labels,
                        const int32_t* ytrue, double* rowstats, cudaStream_t st) {
    // 8 rows per tile with several CTAs per SM measured faster than 16-32-row tiles at one
    // CTA per SM (C4 readout of 10,000 rows: 0.74 vs 0.86 ms): latency hiding beats reuse.
    // (Round 2: the register cap of 128 makes two CTAs per SM actually co-resident — ncu had
    // shown one, 8 warps, 79 % of cycles with no eligible warp: 314 -> 199 us.)
    constexpr size_t kMax = 220 * 1024;
    if (pred_smem<8, EVAL>(d) <= kMax) return launch_pred_t<8, EVAL>(d, params, x, n, labels, ytrue, rowstats, st);
    if (pred_smem<2, EVAL>(d) <= kMax) return launch_pred_t<2, EVAL>(d, params, x, n, labels, ytrue, rowstats, st);
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_evaluate(const NetDesc& d, const float* params, const float* x, const int32_t* y,
                            long long n, double* rowstats, double* out3, cudaStream_t st) {
    if (n <= 0) return cudaErrorInvalidValue;
    cudaError_t e = launch_pred<true>(d, params, x, n, nullptr, y, rowstats, st);
    if (e != cudaSuccess) return e;
    eval_reduce<<<1, 1024, 0, st>>>(rowstats, n, out3);
    return cudaGetLastError();
}

cudaError_t launch_predict(const NetDesc& d, const float* params, const float* x, long long n,
                           int32_t* labels, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    return launch_pred<false>(d, params, x, n, labels, nullptr, nullptr, st);
}
