// TMEM as a second weight store: tcgen05.ld / tcgen05.st bandwidth and latency per SM,
// alone and beside FFMA2 sweeps (B200, sm_100a).  Answers VERDICT r1 "next" 2: can the
// per-sample resident kernel keep half of a 128-unit W1 in TMEM and stream it through
// registers every sample?
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem tmem.cu && ./tmem
//
// Tests (one CTA per SM, 148 CTAs, 512 TMEM columns per CTA):
//   ld<X>   : each warp loops tcgen05.ld.32x32b.x<X> over its lane quadrant, wait::ld,
//             folds the values into an accumulator (FADD) -> TMEM read B/clk/SM
//   st<X>   : tcgen05.st.32x32b.x<X> + wait::st                 -> TMEM write B/clk/SM
//   lat     : dependent ld -> wait chain (one warp)              -> latency in cycles
//   fpass R,T / upass R,T : the planned F (two samples' dot products) and U (rank-2 update)
//             passes over R register rows + T TMEM rows per warp, x quads from shared memory
//             -> FMA/clk/SM (peak 128)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#define R4(a, i) "=r"(a[i]), "=r"(a[i + 1]), "=r"(a[i + 2]), "=r"(a[i + 3])
#define W4(a, i) "r"(a[i]), "r"(a[i + 1]), "r"(a[i + 2]), "r"(a[i + 3])
__device__ __forceinline__ void ld4(uint32_t t, uint32_t (&a)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : R4(a, 0) : "r"(t));
}
__device__ __forceinline__ void ld8(uint32_t t, uint32_t* a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : R4(a, 0), R4(a, 4) : "r"(t));
}
__device__ __forceinline__ void ld16(uint32_t t, uint32_t* a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : R4(a, 0), R4(a, 4), R4(a, 8), R4(a, 12) : "r"(t));
}
__device__ __forceinline__ void ld32(uint32_t t, uint32_t* a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : R4(a, 0), R4(a, 4), R4(a, 8), R4(a, 12), R4(a, 16), R4(a, 20), R4(a, 24), R4(a, 28) : "r"(t));
}
__device__ __forceinline__ void st8(uint32_t t, const uint32_t* a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(t), W4(a, 0), W4(a, 4) : "memory");
}
__device__ __forceinline__ void st16(uint32_t t, const uint32_t* a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(t), W4(a, 0), W4(a, 4), W4(a, 8), W4(a, 12) : "memory");
}
__device__ __forceinline__ void st32(uint32_t t, const uint32_t* a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(t), W4(a, 0), W4(a, 4), W4(a, 8), W4(a, 12), W4(a, 16), W4(a, 20), W4(a, 24), W4(a, 28) : "memory");
}

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}

struct Res { long long cyc; float sink; };

// ---- bandwidth: ld / st of X columns per instruction, NW warps per CTA ----------------
template <int X, bool ST>
__global__ void k_bw(Res* out, int iters) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&tbase, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t quad = warp & 3, half = (warp >> 2) & 1;
    const uint32_t t0 = tbase + ((quad * 32u) << 16) + half * 256u;
    uint32_t a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = threadIdx.x + i;
    float acc = 0.f;
    __syncthreads();
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 256; c += X) {
            if (ST) {
                if (X == 8) st8(t0 + c, a);
                if (X == 16) st16(t0 + c, a);
                if (X == 32) st32(t0 + c, a);
            } else {
                if (X == 8) ld8(t0 + c, a);
                if (X == 16) ld16(t0 + c, a);
                if (X == 32) ld32(t0 + c, a);
            }
        }
        if (ST) wait_st(); else wait_ld();
        if (!ST) {
#pragma unroll
            for (int i = 0; i < X; ++i) acc += __uint_as_float(a[i]);
        } else {
            a[0] += 1;
        }
    }
    long long c1 = clock64();
    fence_before();
    __syncthreads();
    if (threadIdx.x == 0) { out[blockIdx.x].cyc = c1 - c0; out[blockIdx.x].sink = acc + a[0]; }
    if (warp == 0) tmem_dealloc(tbase, 512);
}

// ---- latency: dependent chain ld -> wait -> address from value ------------------------
__global__ void k_lat(Res* out, int iters) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&tbase, 512);
    fence_before();
    __syncthreads();
    fence_after();
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (warp == 0) { st8(tbase, z); st8(tbase + 8, z); wait_st(); }
    uint32_t a[8];
    uint32_t off = 0;
    long long c0 = clock64();
    if (warp == 0) {
        for (int it = 0; it < iters; ++it) {
            ld8(tbase + off, a);
            wait_ld();
            off = a[0] & 8;   // always 0, but a true dependency
        }
    }
    long long c1 = clock64();
    fence_before();
    __syncthreads();
    if (threadIdx.x == 0) { out[blockIdx.x].cyc = c1 - c0; out[blockIdx.x].sink = (float)off; }
    if (warp == 0) tmem_dealloc(tbase, 512);
}

// ---- the planned passes: R register rows + T TMEM rows per warp, 8 warps ---------------
// Lane l holds columns 4l + 128q .. +3 (q < 6) of every row.  x rows (4: a, b for F; c, d
// for U) live in shared memory.  TMEM layout: column = half*256 + q*(4T) + 4t + j.
// F pass: acc_a[r] += w.x_a, acc_b[r] += w.x_b  (4 FFMA2 per row-quad)
// U pass: w -= g_c x_c + g_d x_d                (4 FFMA2 per row-quad), TMEM rows stored back
template <int R, int T, bool U>
__global__ void __launch_bounds__(256, 1) k_pass(Res* out, int iters, float s) {
    __shared__ __align__(16) float xs[4][784];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4 * 784; i += 256) (&xs[0][0])[i] = (i % 97) * 1e-3f;
    if (warp == 0) tmem_alloc(&tbase, 512);
    fence_before();
    __syncthreads();
    fence_after();
    __syncthreads();
    const uint32_t tq = tbase + (((warp & 3) * 32u) << 16) + ((warp >> 2) & 1) * 256u;
    float2 w[R > 0 ? R : 1][12];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < 12; ++k) w[r][k] = make_float2(xs[0][lane + r * 12 + k], xs[1][lane + 2 * k + r]);
    // initialise the TMEM rows
    {
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(0.001f * i);
        for (int c = 0; c < 6 * 4 * T; c += 8) st8(tq + c, z);
        wait_st();
    }
    float2 acc[R + T][2];
    float2 g[R + T][2];
#pragma unroll
    for (int r = 0; r < R + T; ++r) {
        acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
        g[r][0] = make_float2(s * r, s * r);
        g[r][1] = make_float2(-s * r, -s * r);
    }
    __syncthreads();
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            // issue the TMEM loads of this quad's T rows first (latency hidden by the R rows)
            uint32_t tv[T > 0 ? 4 * T : 1];
            if (T > 0) {
#pragma unroll
                for (int t = 0; t + 4 <= T; t += 4) ld16(tq + q * 4 * T + 4 * t, &tv[4 * t]);
                if (T % 4 >= 2) ld8(tq + q * 4 * T + 4 * (T & ~3), &tv[4 * (T & ~3)]);
            }
            const float4 xa = *reinterpret_cast<const float4*>(&xs[U ? 2 : 0][4 * lane + 128 * q]);
            const float4 xb = *reinterpret_cast<const float4*>(&xs[U ? 3 : 1][4 * lane + 128 * q]);
            const float2 a0 = make_float2(xa.x, xa.y), a1 = make_float2(xa.z, xa.w);
            const float2 b0 = make_float2(xb.x, xb.y), b1 = make_float2(xb.z, xb.w);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2& w0 = w[r][2 * q];
                float2& w1 = w[r][2 * q + 1];
                if (U) {
                    w0 = fma2(g[r][0], a0, w0); w0 = fma2(g[r][1], b0, w0);
                    w1 = fma2(g[r][0], a1, w1); w1 = fma2(g[r][1], b1, w1);
                } else {
                    acc[r][0] = fma2(w0, a0, acc[r][0]); acc[r][0] = fma2(w1, a1, acc[r][0]);
                    acc[r][1] = fma2(w0, b0, acc[r][1]); acc[r][1] = fma2(w1, b1, acc[r][1]);
                }
            }
            if (T > 0) {
                wait_ld();
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    float2 w0 = make_float2(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1]));
                    float2 w1 = make_float2(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3]));
                    const int r = R + t;
                    if (U) {
                        w0 = fma2(g[r][0], a0, w0); w0 = fma2(g[r][1], b0, w0);
                        w1 = fma2(g[r][0], a1, w1); w1 = fma2(g[r][1], b1, w1);
                        tv[4 * t] = __float_as_uint(w0.x); tv[4 * t + 1] = __float_as_uint(w0.y);
                        tv[4 * t + 2] = __float_as_uint(w1.x); tv[4 * t + 3] = __float_as_uint(w1.y);
                    } else {
                        acc[r][0] = fma2(w0, a0, acc[r][0]); acc[r][0] = fma2(w1, a1, acc[r][0]);
                        acc[r][1] = fma2(w0, b0, acc[r][1]); acc[r][1] = fma2(w1, b1, acc[r][1]);
                    }
                }
                if (U) {
#pragma unroll
                    for (int t = 0; t + 4 <= T; t += 4) st16(tq + q * 4 * T + 4 * t, &tv[4 * t]);
                    if (T % 4 >= 2) st8(tq + q * 4 * T + 4 * (T & ~3), &tv[4 * (T & ~3)]);
                }
            }
        }
        if (U && T > 0) wait_st();
    }
    long long c1 = clock64();
    float sink = 0.f;
#pragma unroll
    for (int r = 0; r < R + T; ++r) sink += acc[r][0].x + acc[r][0].y + acc[r][1].x + acc[r][1].y;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < 12; ++k) sink += w[r][k].x + w[r][k].y;
    fence_before();
    __syncthreads();
    if (threadIdx.x == 0) { out[blockIdx.x].cyc = c1 - c0; out[blockIdx.x].sink = sink; }
    if (warp == 0) tmem_dealloc(tbase, 512);
}

template <typename K>
static int run(const char* name, K kern, int threads, int iters, double units_per_iter, const char* unit, float s = 1e-3f,
               bool pass = false) {
    Res* d;
    CK(cudaMalloc(&d, 148 * sizeof(Res)));
    Res h[148];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (pass) ((void (*)(Res*, int, float))kern)<<<148, threads>>>(d, iters, s);
        else ((void (*)(Res*, int))kern)<<<148, threads>>>(d, iters);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i].cyc > mx ? h[i].cyc : mx;
    double per_iter = (double)mx / iters;
    printf("%-14s cycles/iter %9.1f  %8.2f %s/clk/SM   (kernel %.3f ms, sink %g)\n", name, per_iter,
           units_per_iter / per_iter, unit, ms, (double)h[0].sink);
    cudaFree(d);
    return 0;
}

int main() {
    const int it = 2000;
    // bytes per iteration per CTA: warps * 32 lanes * 256 cols * 4 B
    for (int nw : {4, 8}) {
        double b = nw * 32.0 * 256 * 4;
        printf("-- %d warps/SM\n", nw);
        run("ld x8", k_bw<8, false>, nw * 32, it, b, "B");
        run("ld x16", k_bw<16, false>, nw * 32, it, b, "B");
        run("ld x32", k_bw<32, false>, nw * 32, it, b, "B");
        run("st x8", k_bw<8, true>, nw * 32, it, b, "B");
        run("st x16", k_bw<16, true>, nw * 32, it, b, "B");
        run("st x32", k_bw<32, true>, nw * 32, it, b, "B");
    }
    run("lat ld8", k_lat, 256, 20000, 1.0, "ld");
    // passes: FMA per iter per SM = 8 warps * 32 lanes * (R+T) rows * 6 quads * 4 FFMA2 * 2
    const int pit = 400;
#define PASS(R, T)                                                                                          \
    run("fpass " #R "," #T, k_pass<R, T, false>, 256, pit, 8.0 * 32 * (R + T) * 6 * 8, "FMA", 1e-3f, true); \
    run("upass " #R "," #T, k_pass<R, T, true>, 256, pit, 8.0 * 32 * (R + T) * 6 * 8, "FMA", 1e-3f, true);
    PASS(8, 0)
    PASS(6, 0)
    PASS(6, 10)
    PASS(8, 8)
    PASS(0, 10)
    PASS(8, 4)
    return 0;
}
