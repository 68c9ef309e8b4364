// Microbenchmarks for the resident-kernel design (B200, sm_100a):
//   FFMA (3 register operands) and FFMA2 (fma.rn.f32x2) throughput per SM vs warps/SM,
//   LDS.32 bandwidth, and the pass-loop mix (1 LDS : 8 FFMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu && ./ubench
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_ffma(float* out, int iters, float s) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
    float b = s, c = s * 0.5f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
        b += 1e-7f;
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) r += a[i];
    if (r == 1234.5f) out[threadIdx.x] = r;
}

__global__ void k_ffma_w(float* out, int iters, float s) {   // pass-like: w = fma(-g, xo, w); acc = fma(w, xn, acc)
    float w[4][8], acc[4] = {0, 0, 0, 0};
    float g[4] = {s, s * 2, s * 3, s * 4};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int m = 0; m < 8; ++m) w[r][m] = r + m * 0.1f + threadIdx.x;
    float xo[8], xn[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) { xo[m] = m * s; xn[m] = m + s; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                w[r][m] = fmaf(-g[r], xo[m], w[r][m]);
                acc[r] = fmaf(w[r][m], xn[m], acc[r]);
            }
#pragma unroll
        for (int m = 0; m < 8; ++m) { float t = xo[m]; xo[m] = xn[m]; xn[m] = t; }
    }
    float r = acc[0] + acc[1] + acc[2] + acc[3];
    if (r == 1234.5f) out[threadIdx.x] = r + w[0][0] + w[3][7];
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

__global__ void k_ffma2(float* out, int iters, float s) {
    unsigned long long a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 v = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
        a[i] = *reinterpret_cast<unsigned long long*>(&v);
    }
    float2 bv = make_float2(s, s), cv = make_float2(s * 0.5f, s * 0.25f);
    unsigned long long b = *reinterpret_cast<unsigned long long*>(&bv);
    unsigned long long c = *reinterpret_cast<unsigned long long*>(&cv);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], b, c);
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&a[i]); r += v.x + v.y; }
    if (r == 1234.5f) out[threadIdx.x] = r;
}

__global__ void k_lds(float* out, int iters) {
    __shared__ float sm[32 * 64];
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) sm[i] = i;
    __syncthreads();
    float acc = 0;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 16; ++m) acc += sm[lane + 32 * ((m + it) & 63)];
    }
    if (acc == 1234.5f) out[threadIdx.x] = acc;
}

__global__ void k_mix(float* out, int iters, float s) {   // per 8 FFMA: 1 LDS (the pass mix with x from SMEM)
    __shared__ float sm[32 * 32];
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) sm[i] = i * 1e-3f;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float w[4][8], acc[4] = {0, 0, 0, 0};
    float g[4] = {s, s * 2, s * 3, s * 4};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int m = 0; m < 8; ++m) w[r][m] = r + m * 0.1f + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            float xn = sm[lane + 32 * ((m + it) & 31)];
            float xo = sm[lane + 32 * ((m + it + 7) & 31)];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                w[r][m] = fmaf(-g[r], xo, w[r][m]);
                acc[r] = fmaf(w[r][m], xn, acc[r]);
            }
        }
    }
    float r = acc[0] + acc[1] + acc[2] + acc[3];
    if (r == 1234.5f) out[threadIdx.x] = r + w[0][0] + w[3][7];
}


__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d)
                 : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
                   "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return *reinterpret_cast<float2*>(&d);
}

// pass-like with FFMA2: w pair -= g * xo pair; acc pair += w pair * xn pair (8 rows x 4 pairs per iter)
__global__ void k_pass2(float* out, int iters, float s) {
    __shared__ float2 sm[32 * 32];
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) sm[i] = make_float2(i * 1e-3f, i * 2e-3f);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float2 w[8][4], acc[8];
    float g[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        g[r] = s * (r + 1);
        acc[r] = make_float2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < 4; ++m) w[r][m] = make_float2(r + m * 0.1f + threadIdx.x, r - m);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            float2 xn = sm[lane + 32 * ((m + it) & 31)];
            float2 xo = sm[lane + 32 * ((m + it + 7) & 31)];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                w[r][m] = f2fma(make_float2(-g[r], -g[r]), xo, w[r][m]);
                acc[r] = f2fma(w[r][m], xn, acc[r]);
            }
        }
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += acc[i].x + acc[i].y + w[i][0].x;
    if (r == 1234.5f) out[threadIdx.x] = r;
}

// scalar pass with R=8 rows and x from SMEM (the resident kernel's current inner loop)
__global__ void k_pass1(float* out, int iters, float s) {
    __shared__ float sm[32 * 32];
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) sm[i] = i * 1e-3f;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float w[8][8], acc[8], g[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        g[r] = s * (r + 1); acc[r] = 0.f;
#pragma unroll
        for (int m = 0; m < 8; ++m) w[r][m] = r + m * 0.1f + threadIdx.x;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            float xn = sm[lane + 32 * ((m + it) & 31)];
            float xo = sm[lane + 32 * ((m + it + 7) & 31)];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                w[r][m] = fmaf(-g[r], xo, w[r][m]);
                acc[r] = fmaf(w[r][m], xn, acc[r]);
            }
        }
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += acc[i] + w[i][0];
    if (r == 1234.5f) out[threadIdx.x] = r;
}


// Arbiter test: warp `chain_w` runs a dependent FFMA chain (latency-bound), the other warps
// (if spam) run independent FFMAs.  Returns cycles per chain step.
__global__ void k_arb(float* out, long long* cyc, int chain_w, int spam, int iters) {
    const int w = threadIdx.x >> 5;
    if (w == chain_w) {
        float a = threadIdx.x * 1e-3f;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            a = fmaf(a, 1.0001f, 0.5f);
            a = __shfl_xor_sync(0xffffffffu, a, 1);
        }
        long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) cyc[blockIdx.x] = t1 - t0;
        if (a == 1234.5f) out[0] = a;
    } else if (spam) {
        float a[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
        for (int it = 0; it < iters / 2; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], 1.0001f, 0.5f);
        }
        float r = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) r += a[i];
        if (r == 1234.5f) out[threadIdx.x] = r;
    }
}

template <typename F>
double run(F f, int blocks, int threads, double ops_per_thread_iter, int iters, float* out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f<<<blocks, threads>>>(out, iters, 1.0001f);
    cudaEventRecord(a);
    f<<<blocks, threads>>>(out, iters, 1.0001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ops_per_thread_iter * iters * (double)blocks * threads / (ms * 1e-3);
}

int main() {
    float* out; CK(cudaMalloc(&out, 1 << 20));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double hz = clk * 1e3;
    printf("SMs %d, clock attr %.0f MHz\n", sms, clk / 1e3);
    int iters = 20000;
    for (int w : {2, 4, 8, 16, 32}) {
        double r = run(k_ffma, sms, 32 * w, 16, iters, out);
        double r2 = run(k_ffma2, sms, 32 * w, 16, iters, out);
        double r3 = run(k_ffma_w, sms, 32 * w, 64, iters / 4, out);
        printf("warps/SM %2d: FFMA %.1f FMA/clk/SM | FFMA2 %.1f FMA/clk/SM | pass-like FFMA %.1f FMA/clk/SM  (at %.0f MHz)\n",
               w, r / sms / hz, r2 / sms / hz, r3 / sms / hz, hz / 1e6);
    }
    for (int w : {2, 4, 8, 16}) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        k_lds<<<sms, 32 * w>>>(out, 2000);
        cudaEventRecord(a);
        k_lds<<<sms, 32 * w>>>(out, 20000);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bytes = 16.0 * 20000 * 4 * 32 * w * sms;
        printf("warps/SM %2d: LDS.32 %.1f B/clk/SM\n", w, bytes / (ms * 1e-3) / sms / hz);
        double r = run(k_mix, sms, 32 * w, 64, iters / 4, out);
        printf("            mix (2 LDS : 8 FFMA per lane) %.1f FMA/clk/SM\n", r / sms / hz);
    }
    {
        long long* cyc; cudaMalloc(&cyc, 8 * 148);
        int iters = 4096;
        for (int nw : {8, 32}) {
            for (int cw : {0, nw - 1}) {
                for (int spam : {0, 1}) {
                    k_arb<<<sms, 32 * nw>>>(out, cyc, cw, spam, iters);
                    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
                    printf("arbiter: %2d warps, chain warp %2d, spam %d: %.1f cycles per (FFMA+SHFL) step\n",
                           nw, cw, spam, (double)h / iters);
                }
            }
        }
    }
    for (int w : {4, 8}) {
        double r1 = run(k_pass1, sms, 32 * w, 128, iters / 8, out);
        double r2 = run(k_pass2, sms, 32 * w, 128, iters / 8, out);
        printf("warps/SM %2d: resident pass (R=8, 1 LDS.32 x2 per 16 FFMA) %.1f FMA/clk/SM | FFMA2 + LDS.64 %.1f FMA/clk/SM\n",
               w, r1 / sms / hz, r2 / sms / hz);
    }
    return 0;
}
