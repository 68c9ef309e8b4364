// k_minibatch.cu — the bf16 mini-batch variant (a10) on tcgen05 GEMMs, and a test hook
// for the GEMM alone.  See k_tcgemm.cuh for the GEMM kernel.
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "pnn.h"
#include "pnn_internal.h"
#include "k_tcgemm.cuh"

namespace {

using PFN_encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encode encode_fn() {
    static PFN_encode fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encode>(p);
    }
    return fn;
}

}  // namespace

// A K-major bf16 tensor [Z][rows][K] as a TMA map with a 64 × box_rows box, 128-byte
// swizzle, zero fill out of bounds.  Returns false on failure.
bool make_tmap_kmajor(CUtensorMap* tm, const void* base, int K, int rows, int Z, int box_rows) {
    PFN_encode fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)Z};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)K * rows * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int EPI>
static cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int Z, int M, int N, int K,
                               const tc::Epi& ep, cudaStream_t st) {
    auto kern = tc::gemm_kernel<BN, EPI>;
    const size_t smem = tc::smem_bytes<BN>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((M + tc::BM - 1) / tc::BM), (unsigned)((N + BN - 1) / BN), (unsigned)Z);
    kern<<<grid, 128, smem, st>>>(ta, tb, K, ep);
    return cudaGetLastError();
}

// Test hook (tests/test_gpu_tcgemm.py): C[z][m][n] = Σ_k A[z][m][k]·B[z][n][k], fp32 out.
extern "C" int pnn_debug_tc_gemm(const void* A, const void* B, float* C, int Z, int M, int N, int K, int bn) {
    CUtensorMap ta, tb;
    if (!make_tmap_kmajor(&ta, A, K, M, Z, tc::BM)) return 1;
    if (!make_tmap_kmajor(&tb, B, K, N, Z, bn)) return 2;
    tc::Epi ep{};
    ep.M = M;
    ep.N = N;
    ep.nvalid = N;
    ep.out_f32 = C;
    ep.zs_out = (long long)M * N;
    cudaError_t e;
    switch (bn) {
    case 64: e = launch_gemm<64, tc::EPI_STORE_F32>(ta, tb, Z, M, N, K, ep, 0); break;
    case 128: e = launch_gemm<128, tc::EPI_STORE_F32>(ta, tb, Z, M, N, K, ep, 0); break;
    case 256: e = launch_gemm<256, tc::EPI_STORE_F32>(ta, tb, Z, M, N, K, ep, 0); break;
    default: return 3;
    }
    if (e != cudaSuccess) return 10 + (int)e;
    e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 1000 + (int)e;
}

// =====================================================================================
// The bf16 mini-batch step (a10): 784-H1-H2-O, ReLU, ReLU, softmax + cross entropy
// (C5: 784-1024-1024-10, batch 64; reading R13), per-CN fp32 master weights in the
// canonical slabs, bf16 operand copies, rounding points of reading R25 (as the
// oracle's orc_train_bf16).  Per mini-batch step (the batch's gradients
// are averaged before one update; short last batch averaged over its size, R14):
//   cast     Xs = bf16(x rows of the batch) and its transpose XsT (rows past the slice: 0)
//   F1 (tc)  A1 = bf16(relu(W1b·Xsᵀ + b1))            -> A1 [z][B][H1], A1T [z][H1][B]
//   F2 (tc)  A2 = bf16(relu(W2b·A1ᵀ + b2))            -> A2 [z][B][H2]
//   out_fwd  z3 = A2·W3bᵀ + b3, softmax, δ3 = p - e (0 past the batch), δ3b; b3 update
//   out_bwd  dW3 = δ3bᵀ·A2 -> W3, W3b; dA2 = δ3b·W3b(old); δ2 = dA2 ⊙ [A2 > 0] -> δ2b,
//            δ2bT; b2 update
//   B4 (tc)  dA1ᵀ = W2bT·δ2bᵀ (pre-update W2, R6); δ1 = dA1 ⊙ [A1 > 0] -> δ1T; b1 update
//   B3 (tc)  dW2 = δ2bT·A1Tᵀ -> W2 -= η/B·dW2, W2b, W2bT
//   B5 (tc)  dW1 = δ1T·XsTᵀ  -> W1 -= η/B·dW1, W1b
// =====================================================================================

struct MbState {
    int K_local, D, H1, H2, O, B;
    long long P, woff1, woff2, woff3;
    __nv_bfloat16 *W1b, *W2b, *W2bT, *W3b, *Xs, *XsT, *A1, *A1T, *A2, *d2b, *d2bT, *d1T, *d3b;
    float* d3;
    CUtensorMap tW1b, tXs, tW2b, tA1, tW2bT, td2b, td2bT, tA1T, td1T, tXsT;
};

const char* mb_plan(const NetDesc& d, int batch) {
    if (d.L != 3) return "bf16 mini-batch is built for 3-layer nets (D-H1-H2-O)";
    if (d.act[0] != PNN_RELU || d.act[1] != PNN_RELU || d.act[2] != PNN_SOFTMAX)
        return "bf16 mini-batch is built for ReLU, ReLU, softmax";
    if (batch != 64) return "bf16 mini-batch is built for batch 64";
    if (d.n[0] % 8 != 0 || d.n[0] > 4096) return "inputs must be a multiple of 8 (16-byte TMA rows)";
    if (d.n[1] % 128 != 0 || d.n[2] % 256 != 0 || d.n[1] > 4096 || d.n[2] > 4096)
        return "hidden widths must be multiples of 128 (H1) and 256 (H2)";
    if (d.n[3] > 16) return "at most 16 outputs";
    return nullptr;
}

void mb_destroy(MbState* s) {
    if (!s) return;
    __nv_bfloat16* bufs[] = {s->W1b, s->W2b, s->W2bT, s->W3b, s->Xs, s->XsT, s->A1, s->A1T, s->A2, s->d2b,
                             s->d2bT, s->d1T, s->d3b};
    for (auto* b : bufs) cudaFree(b);
    cudaFree(s->d3);
    delete s;
}

MbState* mb_create(const NetDesc& d, int K_local, int batch, cudaError_t* err) {
    MbState* s = new MbState{};
    s->K_local = K_local;
    s->D = d.n[0]; s->H1 = d.n[1]; s->H2 = d.n[2]; s->O = d.n[3]; s->B = batch;
    s->P = d.P; s->woff1 = d.woff[1]; s->woff2 = d.woff[2]; s->woff3 = d.woff[3];
    const long long Z = K_local, D = s->D, H1 = s->H1, H2 = s->H2, B = s->B;
    struct { __nv_bfloat16** p; long long n; } al[] = {
        {&s->W1b, Z * H1 * D}, {&s->W2b, Z * H2 * H1}, {&s->W2bT, Z * H1 * H2}, {&s->W3b, Z * 16 * H2},
        {&s->Xs, Z * B * D}, {&s->XsT, Z * D * B}, {&s->A1, Z * B * H1}, {&s->A1T, Z * H1 * B},
        {&s->A2, Z * B * H2}, {&s->d2b, Z * B * H2}, {&s->d2bT, Z * H2 * B}, {&s->d1T, Z * H1 * B},
        {&s->d3b, Z * B * 16}};
    *err = cudaSuccess;
    for (auto& a : al)
        if (*err == cudaSuccess) *err = cudaMalloc(a.p, sizeof(__nv_bfloat16) * (size_t)a.n);
    if (*err == cudaSuccess) *err = cudaMalloc(&s->d3, sizeof(float) * (size_t)(Z * B * 16));
    if (*err == cudaSuccess) cudaMemset(s->W3b, 0, sizeof(__nv_bfloat16) * (size_t)(Z * 16 * H2));
    bool ok = *err == cudaSuccess;
    const int iZ = (int)Z;
    ok = ok && make_tmap_kmajor(&s->tW1b, s->W1b, (int)D, (int)H1, iZ, tc::BM);
    ok = ok && make_tmap_kmajor(&s->tXs, s->Xs, (int)D, (int)B, iZ, (int)B);
    ok = ok && make_tmap_kmajor(&s->tW2b, s->W2b, (int)H1, (int)H2, iZ, tc::BM);
    ok = ok && make_tmap_kmajor(&s->tA1, s->A1, (int)H1, (int)B, iZ, (int)B);
    ok = ok && make_tmap_kmajor(&s->tW2bT, s->W2bT, (int)H2, (int)H1, iZ, tc::BM);
    ok = ok && make_tmap_kmajor(&s->td2b, s->d2b, (int)H2, (int)B, iZ, (int)B);
    ok = ok && make_tmap_kmajor(&s->td2bT, s->d2bT, (int)B, (int)H2, iZ, tc::BM);
    ok = ok && make_tmap_kmajor(&s->tA1T, s->A1T, (int)B, (int)H1, iZ, 256);
    ok = ok && make_tmap_kmajor(&s->td1T, s->d1T, (int)B, (int)H1, iZ, tc::BM);
    ok = ok && make_tmap_kmajor(&s->tXsT, s->XsT, (int)B, (int)D, iZ, 256);
    if (!ok) {
        if (*err == cudaSuccess) *err = cudaErrorInvalidValue;
        mb_destroy(s);
        return nullptr;
    }
    return s;
}

namespace {

__device__ __forceinline__ long long slice_rows(long long n_local, int K_local, int z, long long* start) {
    long long st, cnt;
    shard_of(n_local, K_local, z, &st, &cnt);
    *start = st;
    return cnt;
}

// bf16 operand copies of the fp32 master weights of CNs [z0, z0 + zc)
__global__ void mb_cast_w(const float* __restrict__ children, MbState s, int z0, int zc) {
    const long long per = (long long)s.H1 * s.D + (long long)s.H2 * s.H1 + 16LL * s.H2;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per * zc;
         i += (long long)gridDim.x * blockDim.x) {
        const int z = z0 + (int)(i / per);
        long long r = i % per;
        const float* P = children + (long long)z * s.P;
        if (r < (long long)s.H1 * s.D) {
            s.W1b[(long long)z * s.H1 * s.D + r] = __float2bfloat16_rn(P[s.woff1 + r]);
            continue;
        }
        r -= (long long)s.H1 * s.D;
        if (r < (long long)s.H2 * s.H1) {
            const int o = (int)(r / s.H1), j = (int)(r % s.H1);
            const __nv_bfloat16 v = __float2bfloat16_rn(P[s.woff2 + r]);
            s.W2b[(long long)z * s.H2 * s.H1 + r] = v;
            s.W2bT[(long long)z * s.H1 * s.H2 + (long long)j * s.H2 + o] = v;
            continue;
        }
        r -= (long long)s.H2 * s.H1;
        const int o = (int)(r / s.H2), j = (int)(r % s.H2);
        s.W3b[(long long)z * 16 * s.H2 + r] = (o < s.O) ? __float2bfloat16_rn(P[s.woff3 + (long long)o * s.H2 + j])
                                                        : __float2bfloat16_rn(0.f);
    }
}

// Xs[z][b][d] = bf16(x[row]) and XsT[z][d][b], row = start(z) + step·B + b (0 past the slice)
__global__ void mb_cast_x(const float* __restrict__ X, MbState s, long long n_local, int K_local, int z0, int step) {
    const int z = z0 + blockIdx.y;
    long long st;
    const long long cnt = slice_rows(n_local, K_local, z, &st);
    const int b = blockIdx.x;                      // one CTA per batch row
    const long long t = (long long)step * s.B + b;
    const bool live = t < cnt;
    const float* xr = X + (st + t) * s.D;
    for (int dcol = threadIdx.x; dcol < s.D; dcol += blockDim.x) {
        const __nv_bfloat16 v = __float2bfloat16_rn(live ? xr[dcol] : 0.f);
        s.Xs[((long long)z * s.B + b) * s.D + dcol] = v;
        s.XsT[((long long)z * s.D + dcol) * s.B + b] = v;
    }
}

// Output layer forward + δ3 (one CTA of 8 warps per CN; warp w: batch rows w, w+8, ...)
__global__ void __launch_bounds__(256) mb_out_fwd(float* __restrict__ children, const int32_t* __restrict__ Y,
                                                  MbState s, long long n_local, int K_local, int z0, int step,
                                                  float lr) {
    extern __shared__ float w3s[];                 // [O][H2] fp32 copy of W3b
    __shared__ float dsum[16][8];
    const int z = z0 + blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long st;
    const long long cnt = slice_rows(n_local, K_local, z, &st);
    long long bsz = cnt - (long long)step * s.B;
    bsz = bsz < 0 ? 0 : (bsz > s.B ? s.B : bsz);
    float* P = children + (long long)z * s.P;
    const float* b3 = P + s.woff3 + (long long)s.O * s.H2;
    for (int i = threadIdx.x; i < s.O * s.H2; i += blockDim.x)
        w3s[i] = __bfloat162float(s.W3b[(long long)z * 16 * s.H2 + i]);
    __syncthreads();
    float dacc[16];
#pragma unroll
    for (int o = 0; o < 16; ++o) dacc[o] = 0.f;
    for (int b = warp; b < s.B; b += 8) {
        const __nv_bfloat16* a2 = s.A2 + ((long long)z * s.B + b) * s.H2;
        float acc[16];
#pragma unroll
        for (int o = 0; o < 16; ++o) acc[o] = 0.f;
        for (int j = lane; j < s.H2; j += 32) {
            const float a = __bfloat162float(a2[j]);
#pragma unroll
            for (int o = 0; o < 16; ++o)
                if (o < s.O) acc[o] = fmaf(a, w3s[o * s.H2 + j], acc[o]);
        }
#pragma unroll
        for (int o = 0; o < 16; ++o)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], off);
        // softmax (max-subtracted, R4) and δ3 = p - e (Eq.10); rows past the slice: 0
        float m = -INFINITY;
#pragma unroll
        for (int o = 0; o < 16; ++o)
            if (o < s.O) { acc[o] += b3[o]; m = fmaxf(m, acc[o]); }
        float sum = 0.f;
#pragma unroll
        for (int o = 0; o < 16; ++o)
            if (o < s.O) { acc[o] = expf(acc[o] - m); sum += acc[o]; }
        const int label = (b < bsz) ? Y[st + (long long)step * s.B + b] : -1;
#pragma unroll
        for (int o = 0; o < 16; ++o) {
            float dl = 0.f;
            if (o < s.O && b < bsz) dl = acc[o] / sum - ((o == label) ? 1.f : 0.f);
            dacc[o] += dl;
            if (lane == o) {
                s.d3[((long long)z * s.B + b) * 16 + o] = dl;
                s.d3b[((long long)z * s.B + b) * 16 + o] = __float2bfloat16_rn(dl);
            }
        }
    }
    if (lane == 0)
#pragma unroll
        for (int o = 0; o < 16; ++o) dsum[o][warp] = dacc[o];
    __syncthreads();
    if (threadIdx.x < s.O && bsz > 0) {            // b3 -= η·(Σ_b δ3 / B)
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += dsum[threadIdx.x][w];
        P[s.woff3 + (long long)s.O * s.H2 + threadIdx.x] -= (lr / (float)bsz) * t;
    }
}

// Output layer backward, one thread per hidden unit j of layer 2
__global__ void __launch_bounds__(128) mb_out_bwd(float* __restrict__ children, MbState s, long long n_local,
                                                  int K_local, int z0, int step, float lr) {
    __shared__ float d3s[64][16];
    const int z = z0 + blockIdx.y;
    long long st;
    const long long cnt = slice_rows(n_local, K_local, z, &st);
    long long bsz = cnt - (long long)step * s.B;
    bsz = bsz < 0 ? 0 : (bsz > s.B ? s.B : bsz);
    const float scale = bsz > 0 ? lr / (float)bsz : 0.f;
    for (int i = threadIdx.x; i < s.B * 16; i += blockDim.x)
        (&d3s[0][0])[i] = __bfloat162float(s.d3b[(long long)z * s.B * 16 + i]);
    __syncthreads();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= s.H2) return;
    float* P = children + (long long)z * s.P;
    float* W3 = P + s.woff3;
    float* b2 = P + s.woff2 + (long long)s.H2 * s.H1;
    __nv_bfloat16* w3b = s.W3b + (long long)z * 16 * s.H2;
    float wold[16], gw[16];
#pragma unroll
    for (int o = 0; o < 16; ++o) {
        wold[o] = (o < s.O) ? __bfloat162float(w3b[(long long)o * s.H2 + j]) : 0.f;
        gw[o] = 0.f;
    }
    float db = 0.f;
    const __nv_bfloat16* a2 = s.A2 + (long long)z * s.B * s.H2 + j;
    __nv_bfloat16* d2b = s.d2b + (long long)z * s.B * s.H2 + j;
    __nv_bfloat16* d2bT = s.d2bT + ((long long)z * s.H2 + j) * s.B;
    for (int b = 0; b < s.B; ++b) {
        const float a = __bfloat162float(a2[(long long)b * s.H2]);
        float da = 0.f;                            // (W3bᵀ δ3b)_j with the pre-update W3 (R6)
#pragma unroll
        for (int o = 0; o < 16; ++o) {
            if (o < s.O) {
                gw[o] = fmaf(d3s[b][o], a, gw[o]);             // dW3[o][j] = Σ_b δ3b·A2
                da = fmaf(wold[o], d3s[b][o], da);
            }
        }
        const float d2 = (a > 0.f) ? da : 0.f;                 // ⊙ ReLU'(z2) (R9)
        const __nv_bfloat16 d2h = __float2bfloat16_rn(d2);
        d2b[(long long)b * s.H2] = d2h;
        d2bT[b] = d2h;
        db += d2;
    }
#pragma unroll
    for (int o = 0; o < 16; ++o) {
        if (o < s.O) {
            const float w = fmaf(-scale, gw[o], W3[(long long)o * s.H2 + j]);
            W3[(long long)o * s.H2 + j] = w;
            w3b[(long long)o * s.H2 + j] = __float2bfloat16_rn(w);
        }
    }
    b2[j] -= scale * db;
}

}  // namespace

cudaError_t launch_minibatch_bf16(MbState* s, const NetDesc& d, float* children, const float* x,
                                  const int32_t* y, long long n_local, int K_local, int s_first, int s_count,
                                  float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    const int B = s->B;
    long long st0, cnt0;
    shard_of(n_local, K_local, s_first, &st0, &cnt0);
    const long long steps = (cnt0 + B - 1) / B;    // the first slice is the longest (R17)
    mb_cast_w<<<1184, 256, 0, st>>>(children, *s, s_first, s_count);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t out_smem = sizeof(float) * (size_t)s->O * s->H2;
    e = cudaFuncSetAttribute(mb_out_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out_smem);
    if (e != cudaSuccess) return e;
    tc::Epi base{};
    base.zoff = s_first;
    base.lr = lr;
    base.n_local = n_local;
    base.K_local = K_local;
    base.batch = B;
    for (long long j = 0; j < steps; ++j) {
        base.step = (int)j;
        mb_cast_x<<<dim3((unsigned)B, (unsigned)s_count), 256, 0, st>>>(x, *s, n_local, K_local, s_first, (int)j);
        // F1: A1 = relu(W1b·Xsᵀ + b1)
        tc::Epi f1 = base;
        f1.M = s->H1; f1.N = B; f1.nvalid = B;
        f1.bias = children + s->woff1 + (long long)s->H1 * s->D; f1.zs_bias = s->P;
        f1.out_bm = s->A1; f1.out_mb = s->A1T; f1.zs_act = (long long)s->H1 * B;
        if ((e = launch_gemm<64, tc::EPI_FWD>(s->tW1b, s->tXs, s_count, s->H1, B, s->D, f1, st))) return e;
        // F2: A2 = relu(W2b·A1ᵀ + b2)
        tc::Epi f2 = base;
        f2.M = s->H2; f2.N = B; f2.nvalid = B;
        f2.bias = children + s->woff2 + (long long)s->H2 * s->H1; f2.zs_bias = s->P;
        f2.out_bm = s->A2; f2.out_mb = nullptr; f2.zs_act = (long long)s->H2 * B;
        if ((e = launch_gemm<64, tc::EPI_FWD>(s->tW2b, s->tA1, s_count, s->H2, B, s->H1, f2, st))) return e;
        // output layer (CUDA cores: N = 10 / K = 10 are not dense contractions)
        mb_out_fwd<<<s_count, 256, out_smem, st>>>(children, y, *s, n_local, K_local, s_first, (int)j, lr);
        mb_out_bwd<<<dim3((unsigned)((s->H2 + 127) / 128), (unsigned)s_count), 128, 0, st>>>(
            children, *s, n_local, K_local, s_first, (int)j, lr);
        // B4: δ1 = (W2bᵀ·δ2b) ⊙ [A1 > 0]; b1 update (pre-update W2: before B3)
        tc::Epi b4 = base;
        b4.M = s->H1; b4.N = B; b4.nvalid = B;
        b4.mask = s->A1; b4.out_mb = s->d1T; b4.zs_act = (long long)s->H1 * B;
        b4.bias_upd = children + s->woff1 + (long long)s->H1 * s->D; b4.zs_bias = s->P;
        if ((e = launch_gemm<64, tc::EPI_BWD>(s->tW2bT, s->td2b, s_count, s->H1, B, s->H2, b4, st))) return e;
        // B3: W2 -= η/B · δ2bᵀ·A1
        tc::Epi b3 = base;
        b3.M = s->H2; b3.N = s->H1; b3.nvalid = s->H1;
        b3.master = children + s->woff2; b3.zs_master = s->P;
        b3.wb = s->W2b; b3.wbt = s->W2bT; b3.zs_w = (long long)s->H2 * s->H1;
        if ((e = launch_gemm<256, tc::EPI_UPD>(s->td2bT, s->tA1T, s_count, s->H2, s->H1, B, b3, st))) return e;
        // B5: W1 -= η/B · δ1ᵀ·Xs
        tc::Epi b5 = base;
        b5.M = s->H1; b5.N = s->D; b5.nvalid = s->D;
        b5.master = children + s->woff1; b5.zs_master = s->P;
        b5.wb = s->W1b; b5.wbt = nullptr; b5.zs_w = (long long)s->H1 * s->D;
        if ((e = launch_gemm<256, tc::EPI_UPD>(s->td1T, s->tXsT, s_count, s->H1, s->D, B, b5, st))) return e;
    }
    return cudaGetLastError();
}
