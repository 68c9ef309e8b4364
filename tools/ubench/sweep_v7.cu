// Microbenchmark of the resident kernel's W1 sweeps in isolation (8 warps/SM, 8 rows x 6
// column quads per lane, x from a shared-memory ring), no tail, no synchronisation:
//   mode 0: F (forward, 1 LDS.128 : 16 FFMA2) then U (update, scalar-broadcast FFMA2)
//   mode 1: fused per quad: w -= g·xo; acc += w·xn (2 LDS.128 : 16 FFMA2)
// Reports cycles per step and FMA/clk/SM (algorithmic: 2·8·24 FMA per lane per step).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xptxas -v -o sweep_v7 sweep_v7.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int R = 8, NQ = 6, DP = 800, S = 12;

__device__ __forceinline__ uint64_t pk(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ void lds4(const float* p, uint64_t& a, uint64_t& b) {
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
    a = v.x;
    b = v.y;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(float* out, int steps, long long* cyc) {
    __shared__ __align__(16) float xr[S * DP];
    __shared__ __align__(16) float gw[2][8][R];
    for (int i = threadIdx.x; i < S * DP; i += blockDim.x) xr[i] = (i % 97) * 1e-2f;
    for (int i = threadIdx.x; i < 2 * 8 * R; i += blockDim.x) (&gw[0][0][0])[i] = 1e-4f * (i % 13);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t w[R][2 * NQ];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < 2 * NQ; ++m) w[r][m] = pk(r + m * 0.1f, lane * 0.01f - m);
    float sink = 0.f;
    long long t0 = clock64();
    int sx = 0;
    for (int t = 0; t < steps; ++t) {
        const int s2 = (sx >= 2) ? sx - 2 : sx + S - 2;
        const float* xn = xr + sx * DP + 4 * lane;
        const float* xo = xr + s2 * DP + 4 * lane;
        const float4* gv = reinterpret_cast<const float4*>(&gw[t & 1][warp][0]);
        const float4 g0 = gv[0], g1 = gv[1];
        const float gp[R] = {-g0.x, -g0.y, -g0.z, -g0.w, -g1.x, -g1.y, -g1.z, -g1.w};
        uint64_t acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0ull;
        if constexpr (MODE == 0) {
            uint64_t xa, xb;
            lds4(xn, xa, xb);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint64_t na = 0, nb = 0;
                if (q + 1 < NQ) lds4(xn + 128 * (q + 1), na, nb);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    acc[r] = ffma2(w[r][2 * q], xa, acc[r]);
                    acc[r] = ffma2(w[r][2 * q + 1], xb, acc[r]);
                }
                xa = na; xb = nb;
            }
            lds4(xo, xa, xb);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint64_t na = 0, nb = 0;
                if (q + 1 < NQ) lds4(xo + 128 * (q + 1), na, nb);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    w[r][2 * q] = ffma2(pk(gp[r], gp[r]), xa, w[r][2 * q]);
                    w[r][2 * q + 1] = ffma2(pk(gp[r], gp[r]), xb, w[r][2 * q + 1]);
                }
                xa = na; xb = nb;
            }
        } else {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint64_t oa, ob, na, nb;
                lds4(xo + 128 * q, oa, ob);
                lds4(xn + 128 * q, na, nb);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    w[r][2 * q] = ffma2(pk(gp[r], gp[r]), oa, w[r][2 * q]);
                    acc[r] = ffma2(w[r][2 * q], na, acc[r]);
                    w[r][2 * q + 1] = ffma2(pk(gp[r], gp[r]), ob, w[r][2 * q + 1]);
                    acc[r] = ffma2(w[r][2 * q + 1], nb, acc[r]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float lo, hi;
            upk(acc[r], lo, hi);
            sink += lo + hi;
        }
        if (++sx == S) sx = 0;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        float lo, hi;
        upk(w[r][0], lo, hi);
        sink += lo + hi;
    }
    if (sink == 1234.5f) out[threadIdx.x] = sink;
}

template <typename K>
void run(const char* name, K kern, int threads, int sms, float* out, long long* cyc) {
    const int steps = 4000;
    kern<<<sms, threads>>>(out, 50, cyc);
    kern<<<sms, threads>>>(out, steps, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += h[i];
    mean /= sms;
    const double fma = 2.0 * 8 * 24 * threads;    // per SM per step (update + forward, 8 rows x 24 cols)
    printf("%-28s warps/SM %d: %.0f cyc/step, %.1f FMA/clk/SM\n", name, threads / 32, mean / steps,
           fma * steps / mean);
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 8 * 160);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int th : {128, 256}) {
        run("F then U (v7)", k<0>, th, sms, out, cyc);
        run("fused per quad", k<1>, th, sms, out, cyc);
    }
    return 0;
}
