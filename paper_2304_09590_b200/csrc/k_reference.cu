// k_reference.cu — reference SGD kernel: one CTA per child network (CN),
// parameters read and written in global memory (L2-resident when they fit),
// one sample at a time, phases separated by __syncthreads.  Valid for every
// shape the C ABI accepts; the resident kernel (k_resident.cu) is the fast path.
//
// Per sample (§3):
//   forward   z^l = W^l x^{l-1} + b^l, x^l = φ_l(z^l)           Eqs.2-5
//   δ^L       softmax+CE: x - e (Eq.10); else (x - e)⊙φ'(z^L)  Eq.9, R11
//   δ^l       ((W^{l+1})^T δ^{l+1}) ⊙ φ'(z^l), pre-update W      Eq.11, R6
//   update    g = η δ;  W -= g x^T;  b -= g                      Eqs.12-13
// Mini-batch (batch > 1): the per-instance gradients are summed with the
// weights fixed, then W -= η·(sum / B_actual) (R14).
#include "pnn_internal.h"
#include "pnn_device.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads)
sgd_reference_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                     const int32_t* __restrict__ Y, long long n_local, int K_local, int s_first,
                     float lr, int batch, float* __restrict__ gscratch) {
    extern __shared__ float sm[];
    const int s = s_first + blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* x0 = sm;                          // [n0]
    float* xs = x0 + d.n[0];                 // [neurons]   activations x^l
    float* ds = xs + d.neurons;              // [neurons]   deltas δ^l
    float* P = children + (long long)s * d.P;
    float* G = batch > 1 ? gscratch + (long long)s * d.P : nullptr;
    long long start, count;
    shard_of(n_local, K_local, s, &start, &count);
    const int n0 = d.n[0];

    for (long long t0 = 0; t0 < count; t0 += batch) {
        const long long bsz = (count - t0 < batch) ? (count - t0) : batch;
        if (G) for (long long i = tid; i < d.P; i += kThreads) G[i] = 0.f;
        for (long long t = t0; t < t0 + bsz; ++t) {
            const long long row = start + t;
            const float* xr = X + row * n0;
            for (int j = tid; j < n0; j += kThreads) x0[j] = xr[j];
            const int label = Y[row];
            __syncthreads();
            // ---- forward (Eqs.2-5) ----
            for (int l = 1; l <= d.L; ++l) {
                const int nin = d.n[l - 1], nout = d.n[l];
                const float* W = P + d.woff[l];
                const float* b = W + (long long)nout * nin;
                const float* xin = (l == 1) ? x0 : xs + d.noff[l - 1];
                float* xo = xs + d.noff[l];
                for (int k = warp; k < nout; k += kWarps) {
                    const float* w = W + (long long)k * nin;
                    float acc = 0.f;
                    for (int j = lane; j < nin; j += 32) acc = fmaf(w[j], xin[j], acc);
                    acc = warp_sum(acc);
                    if (lane == 0) {
                        float z = acc + b[k];
                        xo[k] = (d.act[l - 1] == PNN_SOFTMAX) ? z : act_fwd(d.act[l - 1], z);
                    }
                }
                __syncthreads();
                if (d.act[l - 1] == PNN_SOFTMAX) {
                    if (warp == 0) softmax_warp(xo, nout, lane);
                    __syncthreads();
                }
            }
            // ---- δ^L (Eqs.9-10) ----
            {
                const int nL = d.n[d.L];
                const float* xo = xs + d.noff[d.L];
                float* dL = ds + d.noff[d.L];
                for (int k = tid; k < nL; k += kThreads) {
                    float e = (k == label) ? 1.f : 0.f;
                    dL[k] = (d.act[d.L - 1] == PNN_SOFTMAX)
                                ? xo[k] - e
                                : (xo[k] - e) * act_deriv_from_x(d.act[d.L - 1], xo[k]);
                }
                __syncthreads();
            }
            // ---- δ^l, l = L-1..1 (Eq.11), with the not-yet-updated W^{l+1} ----
            for (int l = d.L - 1; l >= 1; --l) {
                const int nl = d.n[l], nn = d.n[l + 1];
                const float* Wn = P + d.woff[l + 1];
                const float* dn = ds + d.noff[l + 1];
                const float* xl = xs + d.noff[l];
                float* dl = ds + d.noff[l];
                for (int j = tid; j < nl; j += kThreads) {
                    float acc = 0.f;
                    for (int k = 0; k < nn; ++k) acc = fmaf(Wn[(long long)k * nl + j], dn[k], acc);
                    dl[j] = acc * act_deriv_from_x(d.act[l - 1], xl[j]);
                }
                __syncthreads();
            }
            // ---- update (Eqs.12-13) or gradient accumulation ----
            for (int l = 1; l <= d.L; ++l) {
                const int nin = d.n[l - 1], nout = d.n[l];
                float* W = (G ? G : P) + d.woff[l];
                float* b = W + (long long)nout * nin;
                const float* xin = (l == 1) ? x0 : xs + d.noff[l - 1];
                const float* dl = ds + d.noff[l];
                for (int k = warp; k < nout; k += kWarps) {
                    float* w = W + (long long)k * nin;
                    if (G) {
                        const float dk = dl[k];
                        for (int j = lane; j < nin; j += 32) w[j] = fmaf(dk, xin[j], w[j]);
                        if (lane == 0) b[k] += dk;
                    } else {
                        const float g = lr * dl[k];
                        for (int j = lane; j < nin; j += 32) w[j] = fmaf(-g, xin[j], w[j]);
                        if (lane == 0) b[k] -= g;
                    }
                }
            }
            __syncthreads();
        }
        if (G) {
            const float fb = (float)bsz;
            for (long long i = tid; i < d.P; i += kThreads) P[i] = fmaf(-lr, G[i] / fb, P[i]);
            __syncthreads();
        }
    }
}

}  // namespace

cudaError_t launch_sgd_reference(const NetDesc& d, float* children, const float* x,
                                 const int32_t* labels, long long n_local, int K_local,
                                 int s_first, int s_count, float lr, int batch, float* gscratch,
                                 cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    size_t smem = sizeof(float) * (size_t)(d.n[0] + 2 * d.neurons);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(sgd_reference_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    sgd_reference_kernel<<<s_count, kThreads, smem, st>>>(d, children, x, labels, n_local, K_local,
                                                         s_first, lr, batch, gscratch);
    return cudaGetLastError();
}
