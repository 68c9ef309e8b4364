// Latency / throughput probes for the deep kernel's chain: dependent SHFL, FFMA, LDS,
// MUFU chains in one warp, and SHFL with 1..8 warps active.  nvcc -arch=sm_100a lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(long long* out, float* buf, int nw_active) {
    __shared__ float sm[1024];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0f + i * 1e-7f;
    __syncthreads();
    float v = buf[threadIdx.x];
    long long t0, t1;
    if (warp < nw_active) {
        // 1. dependent SHFL.BFLY chain (100)
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1 + (i & 15));
        t1 = clock64();
        if (lane == 0) out[warp * 16 + 0] = t1 - t0;
        // 2. five independent SHFL chains (x 20)
        float a = v, b = v + 1, c = v + 2, d = v + 3, e = v + 4;
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 20; ++i) {
            a = __shfl_xor_sync(0xffffffffu, a, 1); b = __shfl_xor_sync(0xffffffffu, b, 2);
            c = __shfl_xor_sync(0xffffffffu, c, 4); d = __shfl_xor_sync(0xffffffffu, d, 8);
            e = __shfl_xor_sync(0xffffffffu, e, 16);
        }
        t1 = clock64();
        v = a + b + c + d + e;
        if (lane == 0) out[warp * 16 + 1] = t1 - t0;
        // 3. dependent FFMA chain (100)
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) v = fmaf(v, 0.999f, 1e-3f);
        t1 = clock64();
        if (lane == 0) out[warp * 16 + 2] = t1 - t0;
        // 4. dependent LDS chain (100)
        int idx = lane;
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) idx = (int)sm[idx] & 1023;
        t1 = clock64();
        v += idx;
        if (lane == 0) out[warp * 16 + 3] = t1 - t0;
        // 5. dependent __expf chain (100)
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) v = __expf(v * 1e-3f);
        t1 = clock64();
        if (lane == 0) out[warp * 16 + 4] = t1 - t0;
        // 6. dependent tanhf chain (100)
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) v = tanhf(v);
        t1 = clock64();
        if (lane == 0) out[warp * 16 + 5] = t1 - t0;
        // 7. dependent __fdividef chain
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) v = __fdividef(1.f, v + 2.f);
        t1 = clock64();
        if (lane == 0) out[warp * 16 + 6] = t1 - t0;
        // 8. dependent IEEE division chain
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) v = 1.f / (v + 2.f);
        t1 = clock64();
        if (lane == 0) out[warp * 16 + 7] = t1 - t0;
        // 9. SHFL.IDX chain
        t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 100; ++i) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31);
        t1 = clock64();
        if (lane == 0) out[warp * 16 + 8] = t1 - t0;
    }
    buf[threadIdx.x] = v;
}

int main() {
    long long* d_out; float* d_buf;
    cudaMalloc(&d_out, 16 * 8 * sizeof(long long));
    cudaMalloc(&d_buf, 256 * sizeof(float));
    cudaMemset(d_buf, 0, 256 * sizeof(float));
    const char* names[] = {"shfl.bfly dep x100", "5 indep shfl chains x20", "ffma dep x100", "lds dep x100",
                           "__expf dep x100", "tanhf dep x100", "__fdividef dep x100", "ieee div dep x100",
                           "shfl.idx dep x100"};
    for (int nw : {1, 3, 8}) {
        for (int rep = 0; rep < 2; ++rep) probe<<<1, 256>>>(d_out, d_buf, nw);
        cudaDeviceSynchronize();
        long long h[128];
        cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
        printf("active warps %d (warp 0):\n", nw);
        for (int k = 0; k < 9; ++k) printf("  %-26s %lld cycles\n", names[k], h[k]);
    }
    return 0;
}
