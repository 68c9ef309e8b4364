// Microbenchmark of the 2-SM-cluster pass design (resident v4):
// 8 warps per SM, each lane holding 8 W1 rows x 25 columns (12 column pairs +
// 1 single column) in registers; per step: w -= g(t-2) x(t-2), acc += w x(t)
// with x from a shared-memory ring, then the 8 row sums reduced over the warp.
// Reports FMA/clk/SM (algorithmic: 400 FMA per lane per step).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xptxas -v -o pass2sm pass2sm.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t f2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void uf2(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

constexpr int R = 8, NP = 12, SLOTS = 8, DP = 800;

template <bool PAIRS, bool REDUCE>
__global__ void __launch_bounds__(256, 1) k_pass(float* out, int steps, float s, long long* cyc) {
    __shared__ __align__(16) float xr[SLOTS * DP];
    __shared__ __align__(16) float gs[2][64];
    __shared__ float accs[2][64];
    for (int i = threadIdx.x; i < SLOTS * DP; i += blockDim.x) xr[i] = (i % 97) * 1e-2f;
    for (int i = threadIdx.x; i < 128; i += blockDim.x) (&gs[0][0])[i] = s * 1e-3f * (i % 7);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long t0 = clock64();
    float accsum = 0.f;
    if constexpr (PAIRS) {
        uint64_t w[R][NP];
        float ws[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ws[r] = r * 0.01f + lane;
#pragma unroll
            for (int m = 0; m < NP; ++m) w[r][m] = f2(r + m * 0.1f, lane * 0.01f - m);
        }
        for (int t = 0; t < steps; ++t) {
            const float* xn = xr + (t % SLOTS) * DP;
            const float* xo = xr + ((t + SLOTS - 2) % SLOTS) * DP;
            uint64_t g2[R];
            float g1[R];
            const float4* gv = reinterpret_cast<const float4*>(&gs[t & 1][warp * 8]);
            float4 ga = gv[0], gb = gv[1];
            g1[0] = -ga.x; g1[1] = -ga.y; g1[2] = -ga.z; g1[3] = -ga.w;
            g1[4] = -gb.x; g1[5] = -gb.y; g1[6] = -gb.z; g1[7] = -gb.w;
#pragma unroll
            for (int r = 0; r < R; ++r) g2[r] = f2(g1[r], g1[r]);
            uint64_t acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0ull;
#pragma unroll
            for (int m = 0; m < NP; ++m) {
                const uint64_t xo2 = *reinterpret_cast<const uint64_t*>(xo + 2 * lane + 64 * m);
                const uint64_t xn2 = *reinterpret_cast<const uint64_t*>(xn + 2 * lane + 64 * m);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    w[r][m] = ffma2(g2[r], xo2, w[r][m]);
                    acc[r] = ffma2(w[r][m], xn2, acc[r]);
                }
            }
            float a[R];
            {
                const float xos = xo[768 + (lane & 15)], xns = xn[768 + (lane & 15)];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    ws[r] = fmaf(g1[r], xos, ws[r]);
                    float lo, hi;
                    uf2(acc[r], lo, hi);
                    a[r] = fmaf(ws[r], xns, lo + hi);
                }
            }
            if constexpr (REDUCE) {
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                float u4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    u4[i] = (b4 ? a[i + 4] : a[i]) + __shfl_xor_sync(0xffffffffu, b4 ? a[i] : a[i + 4], 16);
                float u2[2];
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    u2[i] = (b3 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b3 ? u4[i] : u4[i + 2], 8);
                float v = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                if ((lane & 3) == 0) accs[t & 1][warp * 8 + (lane >> 2)] = v;
                accsum += v;
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) accsum += a[r];
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float lo, hi;
            uf2(w[r][0], lo, hi);
            accsum += lo + hi + ws[r];
        }
    } else {
        float w[R][2 * NP + 1];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int m = 0; m < 2 * NP + 1; ++m) w[r][m] = r + m * 0.1f + lane;
        for (int t = 0; t < steps; ++t) {
            const float* xn = xr + (t % SLOTS) * DP + lane;
            const float* xo = xr + ((t + SLOTS - 2) % SLOTS) * DP + lane;
            float g[R];
            const float4* gv = reinterpret_cast<const float4*>(&gs[t & 1][warp * 8]);
            float4 ga = gv[0], gb = gv[1];
            g[0] = ga.x; g[1] = ga.y; g[2] = ga.z; g[3] = ga.w;
            g[4] = gb.x; g[5] = gb.y; g[6] = gb.z; g[7] = gb.w;
            float acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0.f;
#pragma unroll
            for (int m = 0; m < 2 * NP + 1; ++m) {
                const float xom = xo[32 * m], xnm = xn[32 * m];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    w[r][m] = fmaf(-g[r], xom, w[r][m]);
                    acc[r] = fmaf(w[r][m], xnm, acc[r]);
                }
            }
            if constexpr (REDUCE) {
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                float u4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    u4[i] = (b4 ? acc[i + 4] : acc[i]) + __shfl_xor_sync(0xffffffffu, b4 ? acc[i] : acc[i + 4], 16);
                float u2[2];
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    u2[i] = (b3 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b3 ? u4[i] : u4[i + 2], 8);
                float v = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                if ((lane & 3) == 0) accs[t & 1][warp * 8 + (lane >> 2)] = v;
                accsum += v;
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) accsum += acc[r];
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) accsum += w[r][0] + w[r][2 * NP];
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (accsum == 1234.5f) out[threadIdx.x] = accsum;
}

template <typename K>
void run(const char* name, K kern, int threads, int sms, float* out, long long* cyc) {
    const int steps = 4000;
    kern<<<sms, threads>>>(out, 100, 1.0f, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<sms, threads>>>(out, steps, 1.0f, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h[148]; cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < sms; ++i) mean += h[i]; mean /= sms;
    const double fma = 400.0 * threads;   // per SM per step
    printf("%-34s warps/SM %d: %.0f cyc/step, %.1f FMA/clk/SM (clock64); %.3f ms -> %.2f TFLOP/s\n", name,
           threads / 32, mean / steps, fma * steps / mean, ms, 2 * fma * steps * sms / (ms * 1e-3) / 1e12);
}

int main() {
    float* out; CK(cudaMalloc(&out, 1 << 20));
    long long* cyc; CK(cudaMalloc(&cyc, 8 * 160));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int th : {128, 256}) {
        run("FFMA2 pairs, no reduce", k_pass<true, false>, th, sms, out, cyc);
        run("FFMA2 pairs + reduce", k_pass<true, true>, th, sms, out, cyc);
        run("FFMA scalar, no reduce", k_pass<false, false>, th, sms, out, cyc);
        run("FFMA scalar + reduce", k_pass<false, true>, th, sms, out, cyc);
    }
    return 0;
}
