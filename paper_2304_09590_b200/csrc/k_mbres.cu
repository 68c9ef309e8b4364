// k_mbres.cu — fp32 mini-batch GD for D-H-O nets as ONE persistent launch per epoch:
// W¹ register-resident across a cluster of C = ⌈H/32⌉ CTAs (the paper's
// own workload 784-256-10 ReLU + softmax/CE, batch 50; "the gradients of all
// instances are averaged before the updates", :277-279, 336-337; R14 short last batch).
//
// One cluster trains one child network over all its mini-batch steps.  CTA r owns hidden
// units [32r, 32r + 32): warp w keeps W¹ rows 4w..4w+3 in registers (lane l: columns
// 4l + 128q .. +3, q < 6, as f32x2 pairs; columns 768..783 in shared memory), plus the
// matching W² columns, b¹ and (replicated) b².  Per step t (weights fixed over the batch):
//   P1  z1 = W¹x_b + b1, h_b = φ1(z1) for every row b of the batch        (Eqs.2-3)
//   P2  the CTA's partial logits W²[:, own]·h_b → every CTA (16-byte st.async, zfull)
//   P3  z2 = b2 + Σ_cta partials (fixed order), softmax / φ2, δ2_b           (Eqs.4-5, 9-10)
//   P4  δ1_b = (W²ᵀδ2_b) ⊙ φ1'(h_b) with the pre-update W² (R6); then
//       W² −= η·Σ_b δ2_b h_bᵀ / bsz, b2 −= η·Σ_b δ2_b / bsz, b1 −= η·Σ_b δ1_b / bsz
//   P5  W¹ −= η·(Σ_b δ1_b x_bᵀ) / bsz: the sum accumulates in tensor memory in ascending
//       batch order (the oracle's association), then one scaled update per weight
// x rows stream HBM/L2 → shared memory twice per step (P1 and P5) through a 16-slot ring of
// 1-D bulk copies (cp.async.bulk + mbarrier complete_tx; slots released by an 8-warp
// mbarrier).  No launches per step: the step loop lives in the kernel.
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"
#include "pnn_tmem.cuh"

extern long long* g_trace;   // debug timeline (k_resident.cu; tools/trace_mbres.py)

namespace {

using namespace ptx;

constexpr int R = 4;                  // W¹ rows per warp
constexpr int NW = 8;
constexpr int UC = R * NW;            // hidden units per CTA
constexpr int NQ = 6, NP = 2 * NQ;
constexpr int XC = 768;
constexpr int DP = 800;               // ring slot stride (floats)
constexpr int S = 32;                 // ring slots
constexpr int G = 4;                  // rows per ring group (one full / one empty barrier each)
constexpr int NG = S / G;             // ring groups
constexpr int GA = 6;                 // groups issued ahead of the one being consumed (24 rows in flight)
constexpr int BMX = 64;               // batch rows
constexpr int OM = 16;                // outputs (padded)
constexpr int CM = 8;                 // cluster size

struct __align__(16) MSmem {
    uint64_t xfull[NG];               // count 1 + tx (the group's rows)
    uint64_t xempty[NG];              // count NW
    uint64_t zfull[2];                // [step & 1], count 1 + tx
    float pz[2][CM][BMX][OM];         // [par][cta][b][o] partial logits
    float hs[BMX][UC];                // h of the CTA's units
    float d1[BMX][UC];                // δ1 of the CTA's units
    float d2[BMX][OM];                // δ2
    float w2c[OM][UC];                // W²[o][k0 + k]
    float b1s[UC];
    float b2s[OM];
    int lab[BMX];                     // labels of the step's batch
    uint32_t tbase;                   // TMEM: the W¹ gradient sums of the step
};
constexpr size_t kHead = ((sizeof(MSmem) + 127) / 128) * 128;
constexpr size_t kSmem = kHead + sizeof(float) * (size_t)S * DP;

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
__device__ __forceinline__ int pcol(int l, int j) { return 4 * l + 128 * (j >> 1) + 2 * (j & 1); }
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, float4 v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     remote_addr),
                 "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                 "r"(__float_as_uint(v.w)), "r"(remote_bar)
                 : "memory");
}
template <typename T> __device__ __forceinline__ T* opaque(T* p) {
    asm volatile("mov.b64 %0, %0;" : "+l"(p));
    return p;
}

template <int C, int A1, int A2>
__global__ void __launch_bounds__(NW * 32, 1)
mbres_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X, const int32_t* __restrict__ Y,
             long long n_local, int K_local, int s_first, int B, float lr, long long* __restrict__ trace) {
    extern __shared__ __align__(128) unsigned char smraw[];
    MSmem& sm = *reinterpret_cast<MSmem*>(smraw);
    float* ring = reinterpret_cast<float*>(smraw + kHead);
    const int D = d.n[0], H = d.n[1], O = d.n[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int crank = (C > 1) ? (int)cluster_rank() : 0;
    const int cn = s_first + (int)(blockIdx.x / C);
    const int k0 = crank * UC, own = max(0, min(UC, H - k0));
    long long row0, T64;
    shard_of(n_local, K_local, cn, &row0, &T64);
    const int T = (int)T64;
    const int steps = (T + B - 1) / B;
    float* P = children + (long long)cn * d.P;
    float* W1 = P;
    float* b1g = W1 + (long long)H * D;
    float* W2 = b1g + H;
    float* b2g = W2 + (long long)O * H;
    const float* Xc = X + row0 * (long long)D;
    const uint32_t xbytes = (uint32_t)D * 4u;

    if (warp == 0) tmem::alloc(&sm.tbase, 256);
    if (tid == 32) {
        for (int i = 0; i < NG; ++i) {
            mbar_init(&sm.xfull[i], 1);
            mbar_init(&sm.xempty[i], NW);
        }
        mbar_init(&sm.zfull[0], 1);
        mbar_init(&sm.zfull[1], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < S * DP; i += blockDim.x) ring[i] = 0.f;   // columns >= D stay 0
    for (int i = tid; i < OM * UC; i += blockDim.x) {
        const int o = i / UC, k = i - o * UC;
        sm.w2c[o][k] = (o < O && k < own) ? W2[(long long)o * H + k0 + k] : 0.f;
    }
    for (int i = tid; i < UC; i += blockDim.x) sm.b1s[i] = (i < own) ? b1g[k0 + i] : 0.f;
    for (int i = tid; i < OM; i += blockDim.x) sm.b2s[i] = (i < O) ? b2g[i] : 0.f;
    for (int i = tid; i < BMX * OM; i += blockDim.x) (&sm.d2[0][0])[i] = 0.f;
    fence_proxy_async_smem();
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    if constexpr (C > 1) cluster_sync_all();
    // this warp's TMEM columns: lane quadrant warp & 3, columns 128·(warp >> 2) .. +104
    const uint32_t tg = sm.tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 128u * (uint32_t)(warp >> 2);

    // ---- the x stream in groups of G = 4 batch rows: per step, pass 0 (P1) then pass 1 (P5)
    //      each stream ⌈bsz/4⌉ groups (the last group's missing rows repeat the batch's last
    //      row and are masked).  Group u lives in ring group u % NG; the lane 0 of warp
    //      u % NW issues group u + GA when it starts group u. ----
    const int gps = 2 * ((B + G - 1) / G);         // groups of a full step
    const int last = T - (steps - 1) * B;
    const int gtotal = (steps - 1) * gps + 2 * ((last + G - 1) / G);
    auto issue_group = [&](int u) {
        const int j = u / gps, rem = u - j * gps;
        const int bsz = min(B, T - j * B), nb4 = (bsz + G - 1) / G;
        const int i = rem % nb4;                   // (pass = rem / nb4)
        const int gs = u % NG;
        if (u >= NG) mbar_wait(&sm.xempty[gs], (uint32_t)(((u - NG) / NG) & 1));   // group u - NG consumed
        uint64_t* bar = &sm.xfull[gs];
        mbar_arrive_expect_tx(bar, xbytes * (uint32_t)G);
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const int b = min(G * i + k, bsz - 1);
            bulk_g2s(ring + (gs * G + k) * DP, Xc + ((long long)j * B + b) * D, xbytes, bar);
        }
    };
    if (tid == 0)
        for (int u = 0; u < GA && u < gtotal; ++u) issue_group(u);
    int u = 0;                                     // next group to consume
    auto consume = [&]() -> const float* {
        if (lane == 0 && warp == u % NW && u + GA < gtotal) issue_group(u + GA);
        __syncwarp();
        mbar_wait(&sm.xfull[u % NG], (uint32_t)((u / NG) & 1));
        return ring + (u % NG) * G * DP;
    };
    auto release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.xempty[u % NG]);
        ++u;
    };

    // ---- this warp's W¹ rows: columns < 768 in registers (lane l: 4l + 128q .. +3) ----
    const int kr0 = warp * R;
    uint64_t w[R][NP];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const bool live = kr0 + r < own;
        const float* src = W1 + (long long)(k0 + kr0 + r) * D;
#pragma unroll
        for (int m = 0; m < NP; ++m) w[r][m] = live ? *reinterpret_cast<const uint64_t*>(src + pcol(lane, m)) : 0ull;
    }
    // columns 768..783: lane l = (row rt, sample st, half hf) holds row rt's columns 768 + 8hf .. +7
    // (the four st lanes keep identical copies); it also forms that row × sample's tail product
    const int rt = lane >> 3, st = (lane >> 1) & 3, hf = lane & 1;
    const int tcol = XC + 8 * hf;
    const bool tlive = kr0 + rt < own;
    float wt[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
        wt[c] = (tlive && tcol + c < D) ? W1[(long long)(k0 + kr0 + rt) * D + tcol + c] : 0.f;

    long long* trw = (trace && blockIdx.x == 0 && lane == 0) ? trace + warp * 16 * 16 : nullptr;
#define MTR(pt)                                                                                    \
    do {                                                                                           \
        if (trw && j < 16) trw[j * 16 + (pt)] = ptx::clock64();                                    \
    } while (0)
    for (int j = 0; j < steps; ++j) {
        MTR(0);
        const int bsz = min(B, T - j * B), nb4 = (bsz + G - 1) / G;
        const int par = j & 1;
        const float invb = 1.f / (float)bsz;
        const int ng = (O + 3) >> 2;               // 16-byte groups of a logit vector
        if (tid == 0) mbar_arrive_expect_tx(&sm.zfull[par], 16u * (uint32_t)(C * bsz * ng));
        if (tid < bsz) sm.lab[tid] = Y[row0 + (long long)j * B + tid];
        // ---------------- P1: h_b for the CTA's units, 4 batch rows per group ----------------
        for (int i = 0; i < nb4; ++i) {
            const float* xg = consume();
            uint64_t acc[R][G];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int s2 = 0; s2 < G; ++s2) acc[r][s2] = 0ull;
            uint64_t xa[G], xb[G];
#pragma unroll
            for (int s2 = 0; s2 < G; ++s2) lds4(xg + s2 * DP + 4 * lane, xa[s2], xb[s2]);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint64_t na[G], nb[G];
#pragma unroll
                for (int s2 = 0; s2 < G; ++s2) {
                    na[s2] = 0ull; nb[s2] = 0ull;
                    if (q + 1 < NQ) lds4(xg + s2 * DP + 4 * lane + 128 * (q + 1), na[s2], nb[s2]);
                }
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int s2 = 0; s2 < G; ++s2) {
                        acc[r][s2] = ffma2(w[r][2 * q], xa[s2], acc[r][s2]);
                        acc[r][s2] = ffma2(w[r][2 * q + 1], xb[s2], acc[r][s2]);
                    }
#pragma unroll
                for (int s2 = 0; s2 < G; ++s2) { xa[s2] = na[s2]; xb[s2] = nb[s2]; }
            }
            float px;
            {
                const float4 x0 = *reinterpret_cast<const float4*>(xg + st * DP + tcol);
                const float4 x1 = *reinterpret_cast<const float4*>(xg + st * DP + tcol + 4);
                px = wt[0] * x0.x;
                px = fmaf(wt[1], x0.y, px); px = fmaf(wt[2], x0.z, px); px = fmaf(wt[3], x0.w, px);
                px = fmaf(wt[4], x1.x, px); px = fmaf(wt[5], x1.y, px); px = fmaf(wt[6], x1.z, px);
                px = fmaf(wt[7], x1.w, px);
            }
            release();
            float v[16];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int s2 = 0; s2 < G; ++s2) {
                    float lo, hi;
                    upk(acc[r][s2], lo, hi);
                    v[r * G + s2] = lo + hi;
                }
            // transpose-reduce 16 values: lane l ends with v[l >> 1] = (row l >> 3, sample (l >> 1) & 3)
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
            float u8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                u8[k] = (b4 ? v[k + 8] : v[k]) + __shfl_xor_sync(0xffffffffu, b4 ? v[k] : v[k + 8], 16);
            float u4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                u4[k] = (b3 ? u8[k + 4] : u8[k]) + __shfl_xor_sync(0xffffffffu, b3 ? u8[k] : u8[k + 4], 8);
            float u2[2];
#pragma unroll
            for (int k = 0; k < 2; ++k)
                u2[k] = (b2 ? u4[k + 2] : u4[k]) + __shfl_xor_sync(0xffffffffu, b2 ? u4[k] : u4[k + 2], 4);
            float z = (b1 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? u2[0] : u2[1], 2) + px;
            z += __shfl_xor_sync(0xffffffffu, z, 1);
            const int b = G * i + st, k = kr0 + rt;
            if (hf == 0 && b < bsz) sm.hs[b][k] = (k < own) ? act_fwd_t<A1>(z + sm.b1s[k]) : 0.f;
        }
        MTR(1);
        __syncthreads();
        MTR(2);
        // ---------------- P2: partial logits of the CTA's units → every CTA ----------------
        if (tid < bsz * ng) {
            const int b = tid / ng, g = tid - b * ng;
            float p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < UC; k += 4) {
                const float4 h4 = *reinterpret_cast<const float4*>(&sm.hs[b][k]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float4 w4 = *reinterpret_cast<const float4*>(&sm.w2c[4 * g + i][k]);
                    p[i] = fmaf(w4.w, h4.w, fmaf(w4.z, h4.z, fmaf(w4.y, h4.y, fmaf(w4.x, h4.x, p[i]))));
                }
            }
            const float4 pv = make_float4(p[0], p[1], p[2], p[3]);
            const uint32_t dst = smem_u32(&sm.pz[par][crank][b][4 * g]), bar = smem_u32(&sm.zfull[par]);
#pragma unroll
            for (int q = 0; q < C; ++q) {
                if constexpr (C > 1) st_async_v4(mapa(dst, (uint32_t)q), pv, mapa(bar, (uint32_t)q));
                else st_async_v4(dst, pv, bar);
            }
        }
        MTR(3);
        // ---------------- P3: z2, δ2 (warp per batch row, lane per output) ----------------
        mbar_wait(&sm.zfull[par], (uint32_t)((j >> 1) & 1));
        MTR(4);
        for (int b = warp + NW * (lane >> 4); b - (lane >> 4) * NW < bsz; b += 2 * NW) {   // half-warp per row
            const int o = lane & 15;
            const bool live = o < O && b < bsz;
            const int bb = min(b, BMX - 1);
            float z = sm.b2s[o];
#pragma unroll
            for (int q = 0; q < C; ++q) z += sm.pz[par][q][bb][o];
            const int label = sm.lab[bb];
            float dl;
            if constexpr (A2 == PNN_SOFTMAX) {
                float m = live ? z : -INFINITY;    // max-subtracted (R4)
#pragma unroll
                for (int k = 8; k > 0; k >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, k));
                const float e = live ? expf(z - m) : 0.f;
                float sum = e;
#pragma unroll
                for (int k = 8; k > 0; k >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, k);
                dl = e / sum - ((o == label) ? 1.f : 0.f);
            } else {
                const float x2 = act_fwd_t<A2>(z);
                dl = (x2 - ((o == label) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
            }
            if (b < bsz) sm.d2[b][o] = live ? dl : 0.f;
        }
        MTR(5);
        __syncthreads();
        MTR(6);
        // ---------------- P4: δ1 (pre-update W², R6), then the W², b1, b2 updates ----------------
        {
            const int k = tid & (UC - 1);
            for (int b = tid / UC; b < bsz; b += NW) {
                float s1 = 0.f;
#pragma unroll
                for (int o = 0; o < OM; ++o) s1 = fmaf(sm.w2c[o][k], sm.d2[b][o], s1);   // padded o: 0
                sm.d1[b][k] = s1 * act_deriv_t<A1>(sm.hs[b][k]);
            }
        }
        __syncthreads();
        for (int e = tid; e < O * UC; e += blockDim.x) {      // W² rows o < O
            const int o = e / UC, k = e - o * UC;
            float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
            int b = 0;
            for (; b + 3 < bsz; b += 4) {
                g0 = fmaf(sm.d2[b][o], sm.hs[b][k], g0);
                g1 = fmaf(sm.d2[b + 1][o], sm.hs[b + 1][k], g1);
                g2 = fmaf(sm.d2[b + 2][o], sm.hs[b + 2][k], g2);
                g3 = fmaf(sm.d2[b + 3][o], sm.hs[b + 3][k], g3);
            }
            for (; b < bsz; ++b) g0 = fmaf(sm.d2[b][o], sm.hs[b][k], g0);
            sm.w2c[o][k] -= lr * (((g0 + g1) + (g2 + g3)) * invb);
        }
        if (tid >= 256 - UC) {                                // b1 (the last warp)
            const int k = tid - (256 - UC);
            float g0 = 0.f, g1 = 0.f;
            int b = 0;
            for (; b + 1 < bsz; b += 2) { g0 += sm.d1[b][k]; g1 += sm.d1[b + 1][k]; }
            if (b < bsz) g0 += sm.d1[b][k];
            sm.b1s[k] -= lr * ((g0 + g1) * invb);
        } else if (tid >= 256 - UC - OM && tid < 256 - UC) {  // b2
            const int o = tid - (256 - UC - OM);
            float g0 = 0.f, g1 = 0.f;
            int b = 0;
            for (; b + 1 < bsz; b += 2) { g0 += sm.d2[b][o]; g1 += sm.d2[b + 1][o]; }
            if (b < bsz) g0 += sm.d2[b][o];
            sm.b2s[o] -= lr * ((g0 + g1) * invb);
        }
        MTR(7);
        // ---------------- P5: W¹ −= η · (Σ_b δ1_b x_bᵀ) / bsz: the batch sum first ----------------
        // The gradient sum accumulates in tensor memory (this warp's 4 rows: quad q at
        // columns 16q + 4r, the tail lane's 8 columns at 96), in ascending batch order, then
        // one scaled update per weight ("the gradients … are averaged before the
        // updates"; the oracle's association order, R14).
        {
            uint32_t z[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) z[c] = 0u;
#pragma unroll
            for (int q = 0; q < NQ; ++q) tmem::st16(tg + 16 * q, z);
            tmem::st8(tg + 96, z);
            tmem::wait_st();
        }
        for (int i = 0; i < nb4; ++i) {
            const float* xg = consume();
            float cr[G][R];                        // δ1[b][row] (0 for masked rows)
#pragma unroll
            for (int s2 = 0; s2 < G; ++s2) {
                const int b = G * i + s2;
                float4 dv = make_float4(0.f, 0.f, 0.f, 0.f);
                if (b < bsz) dv = *reinterpret_cast<const float4*>(&sm.d1[b][kr0]);
                cr[s2][0] = dv.x; cr[s2][1] = dv.y; cr[s2][2] = dv.z; cr[s2][3] = dv.w;
            }
            uint64_t xa[G], xb[G];
#pragma unroll
            for (int s2 = 0; s2 < G; ++s2) lds4(xg + s2 * DP + 4 * lane, xa[s2], xb[s2]);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint32_t ta[16];
                tmem::ld16(tg + 16 * q, ta);
                uint64_t na[G], nb[G];
#pragma unroll
                for (int s2 = 0; s2 < G; ++s2) {
                    na[s2] = 0ull; nb[s2] = 0ull;
                    if (q + 1 < NQ) lds4(xg + s2 * DP + 4 * lane + 128 * (q + 1), na[s2], nb[s2]);
                }
                tmem::wait_ld_regs<16>(ta);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    uint64_t ga = pk(__uint_as_float(ta[4 * r]), __uint_as_float(ta[4 * r + 1]));
                    uint64_t gb = pk(__uint_as_float(ta[4 * r + 2]), __uint_as_float(ta[4 * r + 3]));
#pragma unroll
                    for (int s2 = 0; s2 < G; ++s2) {
                        ga = ffma2(pk(cr[s2][r], cr[s2][r]), xa[s2], ga);
                        gb = ffma2(pk(cr[s2][r], cr[s2][r]), xb[s2], gb);
                    }
                    float a0, a1, b0, b1;
                    upk(ga, a0, a1);
                    upk(gb, b0, b1);
                    ta[4 * r] = __float_as_uint(a0); ta[4 * r + 1] = __float_as_uint(a1);
                    ta[4 * r + 2] = __float_as_uint(b0); ta[4 * r + 3] = __float_as_uint(b1);
                }
                tmem::st16(tg + 16 * q, ta);
#pragma unroll
                for (int s2 = 0; s2 < G; ++s2) { xa[s2] = na[s2]; xb[s2] = nb[s2]; }
            }
            {
                uint32_t tt[8];
                tmem::ld8(tg + 96, tt);
                tmem::wait_ld_regs<8>(tt);
#pragma unroll
                for (int s2 = 0; s2 < G; ++s2) {
                    const float ct = (rt == 0) ? cr[s2][0] : (rt == 1) ? cr[s2][1] : (rt == 2) ? cr[s2][2] : cr[s2][3];
                    const float4 x0 = *reinterpret_cast<const float4*>(xg + s2 * DP + tcol);
                    const float4 x1 = *reinterpret_cast<const float4*>(xg + s2 * DP + tcol + 4);
                    const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                    for (int c = 0; c < 8; ++c) tt[c] = __float_as_uint(fmaf(ct, xv[c], __uint_as_float(tt[c])));
                }
                tmem::st8(tg + 96, tt);
            }
            release();
        }
        tmem::wait_st();
        {
            const float nl = -lr * invb;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint32_t ta[16];
                tmem::ld16(tg + 16 * q, ta);
                tmem::wait_ld_regs<16>(ta);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    w[r][2 * q] = ffma2(pk(nl, nl), pk(__uint_as_float(ta[4 * r]), __uint_as_float(ta[4 * r + 1])),
                                        w[r][2 * q]);
                    w[r][2 * q + 1] = ffma2(pk(nl, nl), pk(__uint_as_float(ta[4 * r + 2]), __uint_as_float(ta[4 * r + 3])),
                                            w[r][2 * q + 1]);
                }
            }
            uint32_t tt[8];
            tmem::ld8(tg + 96, tt);
            tmem::wait_ld_regs<8>(tt);
#pragma unroll
            for (int c = 0; c < 8; ++c) wt[c] = fmaf(nl, __uint_as_float(tt[c]), wt[c]);
        }
        MTR(8);
        __syncthreads();                           // W², b updates visible to the next step's P2/P1
        MTR(9);
    }
#undef MTR

    // ---- write back ----
    float* W1o = opaque(W1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (kr0 + r < own) {
            float* dst = W1o + (long long)(k0 + kr0 + r) * D;
#pragma unroll
            for (int m = 0; m < NP; ++m) *reinterpret_cast<uint64_t*>(dst + pcol(lane, m)) = w[r][m];
        }
    }
    if (tlive && st == 0) {
        float* dst = W1o + (long long)(k0 + kr0 + rt) * D;
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (tcol + c < D) dst[tcol + c] = wt[c];
    }
    for (int i = tid; i < O * own; i += blockDim.x) {
        const int o = i / own, k = i - o * own;
        opaque(W2)[(long long)o * H + k0 + k] = sm.w2c[o][k];
    }
    for (int i = tid; i < own; i += blockDim.x) opaque(b1g)[k0 + i] = sm.b1s[i];
    if (crank == 0 && tid < O) opaque(b2g)[tid] = sm.b2s[tid];
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    if (warp == 0) tmem::dealloc(sm.tbase, 256);
    if constexpr (C > 1) cluster_sync_all();       // no CTA leaves while a peer may still st.async into it
}

#define PNN_MBRES_ACTS(X_)                                                                         \
    X_(PNN_RELU, PNN_SOFTMAX)                                                                      \
    X_(PNN_LEAKY_RELU, PNN_SOFTMAX)                                                                \
    X_(PNN_TANH, PNN_SOFTMAX)                                                                      \
    X_(PNN_SIGMOID, PNN_SOFTMAX)                                                                   \
    X_(PNN_SIGMOID, PNN_SIGMOID)

template <int C, int A1, int A2>
cudaError_t launch_one(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                       int K_local, int s_first, int s_count, int B, float lr, cudaStream_t st) {
    auto kern = mbres_kernel<C, A1, A2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(s_count * C));
    cfg.blockDim = dim3((unsigned)(NW * 32));
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, d, children, x, y, n_local, K_local, s_first, B, lr, g_trace);
}

template <int C>
cudaError_t launch_c(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                     int K_local, int s_first, int s_count, int B, float lr, cudaStream_t st) {
#define PNN_CASE(A1_, A2_)                                                                         \
    if (d.act[0] == A1_ && d.act[1] == A2_)                                                        \
        return launch_one<C, A1_, A2_>(d, children, x, y, n_local, K_local, s_first, s_count, B, lr, st);
    PNN_MBRES_ACTS(PNN_CASE)
#undef PNN_CASE
    return cudaErrorInvalidValue;
}

}  // namespace

const char* mbres_plan(const NetDesc& d, int batch) {
    if (d.L != 2) return "2-layer nets only";
    if (batch < 2 || batch > BMX) return "batches of 2..64";
    const int D = d.n[0];
    if (D % 4 != 0 || D <= XC || D > XC + 16) return "built for 768 < inputs <= 784, a multiple of 4";
    if (d.n[1] > CM * UC) return "hidden layer wider than 256";
    if (d.n[2] > OM) return "more than 16 outputs";
    if (d.P % 2 != 0) return "odd parameter count (W1 rows are moved as 8-byte pairs)";
    bool built = false;
#define PNN_CASE(A1_, A2_) built = built || (d.act[0] == A1_ && d.act[1] == A2_);
    PNN_MBRES_ACTS(PNN_CASE)
#undef PNN_CASE
    if (!built) return "activation pair not instantiated in the resident mini-batch kernel";
    return nullptr;
}

int mbres_cluster(const NetDesc& d) {
    const int c = (d.n[1] + UC - 1) / UC;
    return c <= 1 ? 1 : c <= 2 ? 2 : c <= 4 ? 4 : 8;
}

cudaError_t launch_mbres(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                         int K_local, int s_first, int s_count, int B, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    switch (mbres_cluster(d)) {
    case 1: return launch_c<1>(d, children, x, y, n_local, K_local, s_first, s_count, B, lr, st);
    case 2: return launch_c<2>(d, children, x, y, n_local, K_local, s_first, s_count, B, lr, st);
    case 4: return launch_c<4>(d, children, x, y, n_local, K_local, s_first, s_count, B, lr, st);
    case 8: return launch_c<8>(d, children, x, y, n_local, K_local, s_first, s_count, B, lr, st);
    default: return cudaErrorInvalidValue;
    }
}
