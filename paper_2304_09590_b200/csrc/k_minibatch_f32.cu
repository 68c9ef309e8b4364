// k_minibatch_f32.cu — fp32 mini-batch GD for D-H-O nets (the
// paper's own workload, 784-256-10 ReLU + softmax/CE, batch 50; "the
// gradients of all instances are averaged before the updates", :277-279, 336-337).
//
// Per mini-batch step of every CN z (weights fixed over the batch; bsz = rows of the
// batch, short last batch averaged over its size, R14):
//   fwd1   A1[b][h] = φ1(Σ_d W1[h][d]·x_b[d] + b1[h])           (Eqs.2-3; SIMT GEMM tile)
//   out    z2 = W2·a1_b + b2, x2 = φ2(z2) (softmax: R4), δ2_b = x2 − e (Eq.10) or
//          (x2 − e)⊙φ2'(x2) (Eq.9, R11); 0 for rows past the batch
//   hid    δ1[b][h] = (Σ_o W2[o][h]·δ2[b][o]) ⊙ φ1'(A1[b][h])   (Eq.11, pre-update W2, R6)
//          W2 −= η·(Σ_b δ2ᵀa1 / bsz), b2 −= η·(Σ_b δ2 / bsz), b1 −= η·(Σ_b δ1 / bsz)
//   upd1   W1[h][d] −= η·(Σ_b δ1[b][h]·x_b[d] / bsz)             (Eqs.12-13; SIMT GEMM tile)
// all in fp32 FMA (no tensor cores: fp32 parity with the fp32 oracle, max-abs 1e-4).
// The epoch's 4·steps launches are captured once into a CUDA graph and replayed.
#include <cstdio>
#include <cuda_runtime.h>
#include "pnn.h"
#include "pnn_internal.h"
#include "pnn_device.cuh"

struct Mb32State {
    int K_local, B;
    float *A1 = nullptr, *A1P = nullptr, *D1 = nullptr, *D2 = nullptr;
    cudaStream_t cap = nullptr;
    struct G {
        cudaGraphExec_t exec = nullptr;
        const void *children = nullptr, *x = nullptr, *y = nullptr;
        long long n = -1;
        int first = -1, count = -1;
        float lr = 0.f;
        unsigned long long used = 0;
    } g[8];
    unsigned long long tick = 0;
};

namespace {

constexpr int BMAX = 64;      // batch rows per step (one tile)
constexpr int OMAX = 16;
constexpr int UT = 64;        // upd1: 64 h × 64 d per CTA (256 threads, 4 × 4 each)

__device__ __forceinline__ long long batch_rows(long long n_local, int K_local, int z, int step, int B,
                                                long long* row0) {
    long long st, cnt;
    shard_of(n_local, K_local, z, &st, &cnt);
    long long b = cnt - (long long)step * B;
    b = b < 0 ? 0 : (b > B ? B : b);
    *row0 = st + (long long)step * B;
    return b;
}

// fwd1: a 64 (hidden) × 32 (batch) tile of one K-split's partial Z1 per CTA, 256 threads ×
// (4 h × 2 b), k-tiles of 32 staged transposed in shared memory (W1 as [k][h], x as [k][b])
// and prefetched into registers one tile ahead: 8 FMA per 2 shared loads.  The input
// dimension is split KS ways (grid.y = batch tile × KS) so a step fills the GPU; the
// partials go to A1P[ks] and f32_out sums them in a fixed order.
constexpr int GH = 64, GB = 32, GK = 32, KS = 4;
__global__ void __launch_bounds__(256) f32_fwd1(const float* __restrict__ children, const float* __restrict__ X,
                                                float* __restrict__ A1P, NetDesc d, long long n_local,
                                                int K_local, int z0, int step, int B) {
    __shared__ __align__(16) float ws[GK][GH + 4];
    __shared__ __align__(16) float xs[GK][GB + 4];
    const int nbt = (B + GB - 1) / GB, ks = blockIdx.y / nbt;
    const int z = z0 + blockIdx.z, h0 = blockIdx.x * GH, b0 = (blockIdx.y - ks * nbt) * GB;
    const int D = d.n[0], H = d.n[1];
    const int chunk = (((D + KS - 1) / KS) + GK - 1) / GK * GK;
    const int kb = ks * chunk, ke = min(D, kb + chunk);
    long long row0;
    const long long bsz = batch_rows(n_local, K_local, z, step, B, &row0);
    const float* W1 = children + (long long)z * d.P + d.woff[1];
    const int tid = threadIdx.x, hg = tid >> 4, bg = tid & 15;
    float acc[4][2] = {};
    // staging: W1 tile = 64 rows × 32 k = 512 float4-equivalents (2 per thread, as float2 pairs:
    // the CN slab is only 8-byte aligned); x tile = 32 rows × 32 k = 256 float4 (1 per thread)
    float2 wr[4];
    float4 xr;
    auto load_tile = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int slot = tid + 256 * q;                 // 0..511: row = slot >> 3, k = 4·(slot & 7)
            const int r = slot >> 3, kk = k0 + 4 * (slot & 7);
            const bool ok = h0 + r < H && kk < ke;
            const float2* src = reinterpret_cast<const float2*>(W1 + (long long)(h0 + r) * D + kk);
            wr[2 * q] = ok ? src[0] : make_float2(0.f, 0.f);
            wr[2 * q + 1] = ok ? src[1] : make_float2(0.f, 0.f);
        }
        {
            const int r = tid >> 3, kk = k0 + 4 * (tid & 7);
            const bool ok = b0 + r < bsz && kk < ke;
            xr = ok ? *reinterpret_cast<const float4*>(X + (row0 + b0 + r) * D + kk) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store_tile = [&]() {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int slot = tid + 256 * q;
            const int r = slot >> 3, kk = 4 * (slot & 7);
            ws[kk][r] = wr[2 * q].x; ws[kk + 1][r] = wr[2 * q].y;
            ws[kk + 2][r] = wr[2 * q + 1].x; ws[kk + 3][r] = wr[2 * q + 1].y;
        }
        const int r = tid >> 3, kk = 4 * (tid & 7);
        xs[kk][r] = xr.x; xs[kk + 1][r] = xr.y; xs[kk + 2][r] = xr.z; xs[kk + 3][r] = xr.w;
    };
    load_tile(kb);
    store_tile();
    __syncthreads();
    for (int k0 = kb; k0 < ke; k0 += GK) {
        const bool more = k0 + GK < ke;
        if (more) load_tile(k0 + GK);
        const int kn = (ke - k0) < GK ? (ke - k0) : GK;
#pragma unroll 8
        for (int k = 0; k < kn; ++k) {
            const float4 w4 = *reinterpret_cast<const float4*>(&ws[k][4 * hg]);
            const float2 x2 = *reinterpret_cast<const float2*>(&xs[k][2 * bg]);
            acc[0][0] = fmaf(w4.x, x2.x, acc[0][0]); acc[0][1] = fmaf(w4.x, x2.y, acc[0][1]);
            acc[1][0] = fmaf(w4.y, x2.x, acc[1][0]); acc[1][1] = fmaf(w4.y, x2.y, acc[1][1]);
            acc[2][0] = fmaf(w4.z, x2.x, acc[2][0]); acc[2][1] = fmaf(w4.z, x2.y, acc[2][1]);
            acc[3][0] = fmaf(w4.w, x2.x, acc[3][0]); acc[3][1] = fmaf(w4.w, x2.y, acc[3][1]);
        }
        __syncthreads();
        if (more) {
            store_tile();
            __syncthreads();
        }
    }
    const long long zoff = ((long long)ks * K_local + z) * BMAX;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int b = b0 + 2 * bg + j;
        if (b >= B) continue;
        float* dst = A1P + (zoff + b) * H;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int h = h0 + 4 * hg + i;
            if (h < H) dst[h] = acc[i][j];
        }
    }
}

// a1 = φ1(Σ_ks partials + b1) (fixed order), then the output layer + δ2: one warp per batch row
template <int A1, int A2>
__global__ void __launch_bounds__(256) f32_out(const float* __restrict__ children, const int32_t* __restrict__ Y,
                                               const float* __restrict__ A1P, float* __restrict__ A1buf,
                                               float* __restrict__ D2buf,
                                               NetDesc d, long long n_local, int K_local, int z0, int step, int B) {
    extern __shared__ float w2s[];                 // [O][H]: W2 staged once per CTA
    const int z = z0 + blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int H = d.n[1], O = d.n[2];
    const float* W2 = children + (long long)z * d.P + d.woff[2];
    for (int i = threadIdx.x; i < O * H; i += blockDim.x) w2s[i] = W2[i];
    __syncthreads();
    const int b = blockIdx.x * 8 + warp;
    if (b >= B) return;
    long long row0;
    const long long bsz = batch_rows(n_local, K_local, z, step, B, &row0);
    const float* b2 = W2 + (long long)O * H;
    const float* b1 = children + (long long)z * d.P + d.woff[1] + (long long)H * d.n[0];
    float* a1 = A1buf + ((long long)z * BMAX + b) * H;
    const long long pstride = (long long)K_local * BMAX * H;
    const float* p0 = A1P + ((long long)z * BMAX + b) * H;
    float acc[OMAX];
#pragma unroll
    for (int o = 0; o < OMAX; ++o) acc[o] = 0.f;
    for (int h = lane; h < H; h += 32) {
        float zs = p0[h];
#pragma unroll
        for (int q = 1; q < KS; ++q) zs += p0[q * pstride + h];
        const float a = (b < bsz) ? act_fwd_t<A1>(zs + b1[h]) : 0.f;
        a1[h] = a;
#pragma unroll
        for (int o = 0; o < OMAX; ++o)
            if (o < O) acc[o] = fmaf(w2s[o * H + h], a, acc[o]);
    }
#pragma unroll
    for (int o = 0; o < OMAX; ++o) acc[o] = warp_sum(acc[o]);
    // lane o < O forms output o (one exp per lane instead of O per lane)
    float zmine = acc[0] + b2[0];
#pragma unroll
    for (int o = 1; o < OMAX; ++o)
        if (o < O && lane == o) zmine = acc[o] + b2[o];
    float xmine;
    if constexpr (A2 == PNN_SOFTMAX) {
        float m = -INFINITY;                       // max-subtracted (R4)
#pragma unroll
        for (int o = 0; o < OMAX; ++o)
            if (o < O) m = fmaxf(m, acc[o] + b2[o]);
        const float e = (lane < O) ? expf(zmine - m) : 0.f;
        xmine = e / warp_sum(e);
    } else {
        xmine = act_fwd_t<A2>(zmine);
    }
    const int label = (b < bsz) ? Y[row0 + b] : -1;
    if (lane < O) {
        float dl = 0.f;
        if (b < bsz) {
            const float e = (lane == label) ? 1.f : 0.f;
            dl = (A2 == PNN_SOFTMAX) ? xmine - e : (xmine - e) * act_deriv_t<A2>(xmine);
        }
        D2buf[((long long)z * BMAX + b) * OMAX + lane] = dl;
    }
}

// hidden deltas + output-layer / bias updates: 64 hidden units × 4 batch quarters per CTA
template <int A1>
__global__ void __launch_bounds__(256) f32_hid(float* __restrict__ children, const float* __restrict__ A1buf,
                                               const float* __restrict__ D2buf, float* __restrict__ D1buf,
                                               NetDesc d, long long n_local, int K_local, int z0, int step, int B,
                                               float lr) {
    __shared__ float d2s[BMAX][OMAX];
    __shared__ float part[3][64][OMAX + 1];
    const int z = z0 + blockIdx.y;
    const int H = d.n[1], O = d.n[2];
    long long row0;
    const long long bsz = batch_rows(n_local, K_local, z, step, B, &row0);
    const float fb = bsz > 0 ? (float)bsz : 1.f;
    for (int i = threadIdx.x; i < BMAX * OMAX; i += blockDim.x)
        (&d2s[0][0])[i] = (i / OMAX < B) ? D2buf[(long long)z * BMAX * OMAX + i] : 0.f;
    __syncthreads();
    float* P = children + (long long)z * d.P;
    float* W2 = P + d.woff[2];
    if (blockIdx.x == 0 && threadIdx.x < O) {           // b2 -= η·(Σ_b δ2 / bsz)
        float t = 0.f;
        for (int b = 0; b < B; ++b) t += d2s[b][threadIdx.x];
        W2[(long long)O * H + threadIdx.x] -= lr * (t / fb);
    }
    const int hl = threadIdx.x & 63, g = threadIdx.x >> 6;
    const int h = blockIdx.x * 64 + hl;
    const bool hok = h < H;
    float wold[OMAX], gw[OMAX];
#pragma unroll
    for (int o = 0; o < OMAX; ++o) {
        wold[o] = (hok && o < O) ? W2[(long long)o * H + h] : 0.f;
        gw[o] = 0.f;
    }
    float db = 0.f;
    const int bq = (B + 3) / 4;
    const int b_lo = g * bq, b_hi = (b_lo + bq) < B ? (b_lo + bq) : B;
    if (hok) {
        for (int b = b_lo; b < b_hi; ++b) {
            const float a = A1buf[((long long)z * BMAX + b) * H + h];
            float da = 0.f;
#pragma unroll
            for (int o = 0; o < OMAX; ++o) {
                if (o < O) {
                    gw[o] = fmaf(d2s[b][o], a, gw[o]);
                    da = fmaf(wold[o], d2s[b][o], da);
                }
            }
            const float d1 = da * act_deriv_t<A1>(a);
            D1buf[((long long)z * BMAX + b) * H + h] = d1;
            db += d1;
        }
    }
    if (g > 0) {
#pragma unroll
        for (int o = 0; o < OMAX; ++o) part[g - 1][hl][o] = gw[o];
        part[g - 1][hl][OMAX] = db;
    }
    __syncthreads();
    if (g == 0 && hok) {
        for (int q = 0; q < 3; ++q) {
#pragma unroll
            for (int o = 0; o < OMAX; ++o) gw[o] += part[q][hl][o];
            db += part[q][hl][OMAX];
        }
#pragma unroll
        for (int o = 0; o < OMAX; ++o)
            if (o < O) W2[(long long)o * H + h] -= lr * (gw[o] / fb);
        P[d.woff[1] + (long long)H * d.n[0] + h] -= lr * (db / fb);
    }
}

// W1 −= η·(δ1ᵀ·X / bsz): 64 × 64 tile of W1 per CTA, K = the batch (ascending b per output)
__global__ void __launch_bounds__(256) f32_upd1(float* __restrict__ children, const float* __restrict__ X,
                                                const float* __restrict__ D1buf, NetDesc d, long long n_local,
                                                int K_local, int z0, int step, int B, float lr) {
    __shared__ __align__(16) float ds[BMAX][UT];
    __shared__ __align__(16) float xs[BMAX][UT];
    const int z = z0 + blockIdx.z, h0 = blockIdx.x * UT, d0 = blockIdx.y * UT;
    const int D = d.n[0], H = d.n[1];
    long long row0;
    const long long bsz = batch_rows(n_local, K_local, z, step, B, &row0);
    if (bsz == 0) return;
    // this thread's 4 × 4 W1 values, loaded first so their latency overlaps the staging and
    // the product (scalar: the CN slab need not be 16-B aligned)
    const int th = (threadIdx.x >> 4) * 4, tdd = (threadIdx.x & 15) * 4;
    float* W1 = children + (long long)z * d.P + d.woff[1];
    float wold[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int h = h0 + th + i, dd = d0 + tdd + j;
            wold[i][j] = (h < H && dd < D) ? W1[(long long)h * D + dd] : 0.f;
        }
    for (int slot = threadIdx.x; slot < (int)bsz * (UT / 4); slot += blockDim.x) {
        const int b = slot / (UT / 4), c = (slot % (UT / 4)) * 4;
        float4 dv = make_float4(0.f, 0.f, 0.f, 0.f), xv = dv;
        if (h0 + c < H) dv = *reinterpret_cast<const float4*>(D1buf + ((long long)z * BMAX + b) * H + h0 + c);
        if (d0 + c < D) xv = *reinterpret_cast<const float4*>(X + (row0 + b) * D + d0 + c);
        *reinterpret_cast<float4*>(&ds[b][c]) = dv;
        *reinterpret_cast<float4*>(&xs[b][c]) = xv;
    }
    __syncthreads();
    float acc[4][4] = {};
    for (int b = 0; b < (int)bsz; ++b) {
        const float4 dv = *reinterpret_cast<const float4*>(&ds[b][th]);
        const float4 xv = *reinterpret_cast<const float4*>(&xs[b][tdd]);
        const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(dd[i], xx[j], acc[i][j]);
    }
    const float fb = (float)bsz;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int h = h0 + th + i;
        if (h >= H) continue;
        float* w = W1 + (long long)h * D + d0 + tdd;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (d0 + tdd + j < D) w[j] = wold[i][j] - lr * (acc[i][j] / fb);
    }
}

template <int A1, int A2>
cudaError_t enqueue_step(Mb32State* s, const NetDesc& d, float* children, const float* x, const int32_t* y,
                         long long n_local, int K_local, int z0, int zc, int step, float lr, cudaStream_t st) {
    const int H = d.n[1], D = d.n[0], B = s->B;
    f32_fwd1<<<dim3((unsigned)((H + GH - 1) / GH), (unsigned)(((B + GB - 1) / GB) * KS), (unsigned)zc), 256, 0, st>>>(
        children, x, s->A1P, d, n_local, K_local, z0, step, B);
    f32_out<A1, A2><<<dim3((unsigned)((B + 7) / 8), (unsigned)zc), 256, sizeof(float) * (size_t)d.n[2] * H, st>>>(
        children, y, s->A1P, s->A1, s->D2, d, n_local, K_local, z0, step, B);
    f32_hid<A1><<<dim3((unsigned)((H + 63) / 64), (unsigned)zc), 256, 0, st>>>(children, s->A1, s->D2, s->D1, d,
                                                                               n_local, K_local, z0, step, B, lr);
    f32_upd1<<<dim3((unsigned)((H + UT - 1) / UT), (unsigned)((D + UT - 1) / UT), (unsigned)zc), 256, 0, st>>>(
        children, x, s->D1, d, n_local, K_local, z0, step, B, lr);
    return cudaGetLastError();
}

template <int A1, int A2>
cudaError_t enqueue_epoch_t(Mb32State* s, const NetDesc& d, float* children, const float* x, const int32_t* y,
                            long long n_local, int K_local, int z0, int zc, float lr, cudaStream_t st) {
    long long r0, c0;
    shard_of(n_local, K_local, z0, &r0, &c0);          // the first slice is the longest (R17)
    const long long steps = (c0 + s->B - 1) / s->B;
    for (long long j = 0; j < steps; ++j) {
        cudaError_t e = enqueue_step<A1, A2>(s, d, children, x, y, n_local, K_local, z0, zc, (int)j, lr, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t enqueue_epoch(Mb32State* s, const NetDesc& d, float* children, const float* x, const int32_t* y,
                          long long n_local, int K_local, int z0, int zc, float lr, cudaStream_t st) {
#define PNN_MB32(A1_, A2_)                                                                          \
    if (d.act[0] == A1_ && d.act[1] == A2_)                                                       \
        return enqueue_epoch_t<A1_, A2_>(s, d, children, x, y, n_local, K_local, z0, zc, lr, st);
    PNN_MB32(PNN_RELU, PNN_SOFTMAX)
    PNN_MB32(PNN_LEAKY_RELU, PNN_SOFTMAX)
    PNN_MB32(PNN_TANH, PNN_SOFTMAX)
    PNN_MB32(PNN_SIGMOID, PNN_SOFTMAX)
    PNN_MB32(PNN_SIGMOID, PNN_SIGMOID)
#undef PNN_MB32
    return cudaErrorInvalidValue;
}

}  // namespace

const char* mb32_plan(const NetDesc& d, int batch) {
    if (d.L != 2) return "fp32 mini-batch kernel covers 2-layer nets (D-H-O)";
    if (batch < 2 || batch > BMAX) return "fp32 mini-batch kernel covers batches of 2..64";
    if (d.n[0] % 4 != 0) return "inputs must be a multiple of 4 (16-byte rows)";
    if (d.n[1] % 4 != 0) return "hidden width must be a multiple of 4";
    if (d.n[2] > OMAX) return "at most 16 outputs";
    if ((size_t)d.n[2] * d.n[1] * sizeof(float) > 48 * 1024) return "W2 (outputs × hidden) must fit 48 KB of shared memory";
    const int a1 = d.act[0], a2 = d.act[1];
    const bool built = (a2 == PNN_SOFTMAX && (a1 == PNN_RELU || a1 == PNN_LEAKY_RELU || a1 == PNN_TANH ||
                                              a1 == PNN_SIGMOID)) ||
                       (a1 == PNN_SIGMOID && a2 == PNN_SIGMOID);
    if (!built) return "activation pair not instantiated in the fp32 mini-batch kernel";
    return nullptr;
}

void mb32_destroy(Mb32State* s) {
    if (!s) return;
    cudaFree(s->A1);
    cudaFree(s->A1P);
    cudaFree(s->D1);
    cudaFree(s->D2);
    for (auto& e : s->g)
        if (e.exec) cudaGraphExecDestroy(e.exec);
    if (s->cap) cudaStreamDestroy(s->cap);
    delete s;
}

Mb32State* mb32_create(const NetDesc& d, int K_local, int batch, cudaError_t* err) {
    Mb32State* s = new Mb32State{};
    s->K_local = K_local;
    s->B = batch;
    const size_t Z = (size_t)K_local, H = (size_t)d.n[1];
    *err = cudaMalloc(&s->A1, sizeof(float) * Z * BMAX * H);
    if (*err == cudaSuccess) *err = cudaMalloc(&s->A1P, sizeof(float) * KS * Z * BMAX * H);
    if (*err == cudaSuccess) *err = cudaMalloc(&s->D1, sizeof(float) * Z * BMAX * H);
    if (*err == cudaSuccess) *err = cudaMalloc(&s->D2, sizeof(float) * Z * BMAX * OMAX);
    if (*err == cudaSuccess) *err = cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking);
    if (*err != cudaSuccess) {
        mb32_destroy(s);
        return nullptr;
    }
    return s;
}

cudaError_t launch_minibatch_f32(Mb32State* s, const NetDesc& d, float* children, const float* x,
                                 const int32_t* y, long long n_local, int K_local, int s_first, int s_count,
                                 float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    Mb32State::G* hit = nullptr;
    Mb32State::G* lru = &s->g[0];
    for (auto& e : s->g) {
        if (e.exec && e.children == children && e.x == x && e.y == y && e.n == n_local && e.first == s_first &&
            e.count == s_count && e.lr == lr)
            hit = &e;
        if (e.used < lru->used) lru = &e;
    }
    if (!hit) {
        hit = lru;
        if (hit->exec) { cudaGraphExecDestroy(hit->exec); hit->exec = nullptr; }
        cudaError_t e = cudaStreamBeginCapture(s->cap, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return e;
        cudaError_t eq = enqueue_epoch(s, d, children, x, y, n_local, K_local, s_first, s_count, lr, s->cap);
        cudaGraph_t g = nullptr;
        e = cudaStreamEndCapture(s->cap, &g);
        if (eq != cudaSuccess) { if (g) cudaGraphDestroy(g); return eq; }
        if (e != cudaSuccess) return e;
        e = cudaGraphInstantiate(&hit->exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) { hit->exec = nullptr; return e; }
        hit->children = children; hit->x = x; hit->y = y; hit->n = n_local;
        hit->first = s_first; hit->count = s_count; hit->lr = lr;
    }
    hit->used = ++s->tick;
    return cudaGraphLaunch(hit->exec, st);
}
