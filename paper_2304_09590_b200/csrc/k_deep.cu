// k_deep.cu — persistent per-sample SGD for 3-layer nets D-H1-H2-O (the C3 shape
// 784-300-100-10), W¹ register-resident across a cluster of C CTAs.
//
// One cluster of C ∈ {4, 8} CTAs trains one child network over its whole slice
// (PAPER.md:168).  CTA r owns units [r·R1, r·R1 + R1) of layer 1 and [r·R2, r·R2 + R2)
// of layer 2 (R_l = ⌈n_l / C⌉); the output layer (O <= 16) is split by columns: CTA r
// keeps W³[:, its layer-2 units].  Per sample, in the paper's sequential order
// (§3, Eqs.2-13; δ with the pre-update weights, R6):
//   h1 = φ1(W¹x + b1), h2 = φ2(W²h1 + b2), x3 = φ3(W³h2 + b3)           (Eqs.2-5)
//   δ3 = x3 - e (softmax+CE, Eq.10) or (x3 - e)⊙φ3'(x3) (R11)
//   δ2 = (W³ᵀδ3)⊙φ2'(h2), δ1 = (W²ᵀδ2)⊙φ1'(h1)                         (Eq.11)
//   W -= η δ (input)ᵀ, b -= η δ                                          (Eqs.12-13)
//
// Warps 0..4 ("sweeps") hold 8 W¹ rows each in registers and run the R27 lookahead of
// k_resident.cu unchanged: F(s) = W¹(s-L)·x(s) as f32x2 FMAs, U(s): W¹ -= g(s-L)·x(s-L)ᵀ,
// the Gram records from the same pre-pass (launch_gram) carried with x(s) in the ring.
// Warps 5..7 ("chain") run the per-sample chain for the CTA's units with W² (own rows),
// W³ (own columns), the biases and the g history in shared memory.  The chain has no
// CTA barrier at all: every cross-warp / cross-CTA value travels by st.async into the
// receiving CTA's buffer (the sender's own CTA included) and is consumed after an
// mbarrier wait on its byte count:
//   h1full  all H1 values of h1(c)            (each CTA's layer-1 units → every CTA)
//   zfull   3C partial logit vectors          (each chain warp's W³[:, its rows]·h2)
//   d1full  3C partial (W²ᵀδ2) per own unit   (each chain warp's rows → the owner CTA)
// Each chain warp owns layer-2 rows cw, cw+3, … of its CTA and does everything for
// them in registers (z2, h2, its partial logits, the softmax redundantly, δ2, the fused
// δ1-partial / W² update pass, the W³ / b2 updates); threads 0..R1-1 of the chain
// own the CTA's layer-1 units (z1 by the lookahead correction, g = η δ1, b1).
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"
#include "pnn_tmem.cuh"

extern long long* g_trace;   // debug timeline (k_resident.cu; tools/trace_deep.py)

namespace {

using namespace ptx;

constexpr int NSW = 5;                // sweep warps
constexpr int NCW = 3;                // chain warps
constexpr int NW = NSW + NCW;
// Per cluster size: W¹ rows per sweep warp in registers (RR) and in tensor memory (TRW), and
// layer-2 rows per chain warp (RW2).  C = 8: 40 register rows per CTA (the C3 shape in 3 waves
// of at most 15 co-resident 8-CTA clusters); C = 4: 30 register + 50 TMEM rows per CTA, so the
// C3 shape fits 4-CTA clusters and all 32 of its CNs run at once (33 co-resident).
template <int C> struct DeepShape;
template <> struct DeepShape<8> { static constexpr int RR = 8, TRW = 0, RW2 = 5; };
template <> struct DeepShape<4> { static constexpr int RR = 6, TRW = 10, RW2 = 9; };
constexpr int RPWMAX = 16;            // W¹ rows per sweep warp (max over C)
constexpr int R1MAX = RPWMAX * NSW;   // layer-1 units per CTA (max)
constexpr int RW2MAX = 9;
constexpr int R2MAX = RW2MAX * NCW;   // layer-2 units per CTA (max)
template <int C> constexpr int r1cap() { return (DeepShape<C>::RR + DeepShape<C>::TRW) * NSW; }
template <int C> constexpr int r2cap() { return DeepShape<C>::RW2 * NCW; }
constexpr int H1MAX = 384;            // W² row stride in shared memory (h1 padded with zeros)
constexpr int NJ4 = H1MAX / 128;      // 16-byte column groups per lane
constexpr int OMAX = 16;
constexpr int CMAX = 8;
constexpr int NGMAX = NCW * CMAX;     // partial sources (chain warps of the cluster)
constexpr int NQ = 6;
constexpr int NP = 2 * NQ;
constexpr int XC = 768;
constexpr int GOFF = 784;
constexpr int DP = 800;
constexpr int LAG = 4;
constexpr int S = 16;
constexpr int PF = 8;                 // x(c+PF) is issued at chain step c: PF <= S - LAG - 1
constexpr int AR = 8;
constexpr int GR = 8;
static_assert(AR > LAG + 1 && GR > LAG && PF <= S - LAG - 1, "ring sizes");
#ifdef PNN_DEEP_EXP_NO_SWEEP
constexpr bool kNoSweep = true;    // timing experiment only: the sweeps skip their FMAs (wrong results)
#else
constexpr bool kNoSweep = false;
#endif

struct __align__(16) DSmem {
    uint64_t xfull[S];
    uint64_t aready[AR];               // count NSW
    uint64_t gready[GR];               // count NCW
    uint64_t h1full[2], zfull[2], d1full[2];   // [c & 1], count 1 + tx
    float asum[AR][R1MAX][4];
    float gbuf[GR][R1MAX];
    float b1s[R1MAX];
    float wx[NSW][RPWMAX][16];
    float h1buf[2][H1MAX];
    float zbuf[2][NGMAX][OMAX];
    float p1buf[2][NGMAX][R1MAX];
    float b2s[R2MAX + 1];
    float w3s[OMAX][R2MAX + 1];        // W³[o][r·R2 + i]
    uint32_t tbase;                    // TMEM base (C = 4: the sweeps' TMEM rows)
};
constexpr size_t kHead = ((sizeof(DSmem) + 127) / 128) * 128;
constexpr size_t kSmem = kHead + sizeof(float) * ((size_t)R2MAX * H1MAX + (size_t)S * DP);

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
// the chain's waits: try_wait (hardware sleep, ~60-cycle wake-up) or, PNN_DEEP_SPIN=1, test_wait polling
#ifndef PNN_DEEP_SPIN
#define PNN_DEEP_SPIN 0
#endif
__device__ __forceinline__ void chain_wait(uint64_t* b, uint32_t parity) {
#if PNN_DEEP_SPIN && !defined(PNN_DEBUG_WAIT)
    mbar_wait_spin(b, parity);
#else
    mbar_wait(b, parity);
#endif
}
// φ on the chain's critical path (R32): tanh(z) = 1 - 2/(1 + e^{2z}) and
// sigmoid(z) = 1/(1 + e^{-z}) with ex2.approx / rcp.approx (absolute error ~1e-7; libdevice
// tanhf costs ~120 dependent cycles per call here); ReLU / leaky ReLU exact.
template <int A> __device__ __forceinline__ float act_fast(float z) {
    if constexpr (A == PNN_TANH) return 1.f - __fdividef(2.f, 1.f + __expf(2.f * z));
    else if constexpr (A == PNN_SIGMOID) return __fdividef(1.f, 1.f + __expf(-z));
    else return act_fwd_t<A>(z);
}
template <typename T> __device__ __forceinline__ T* opaque(T* p) {
    asm volatile("mov.b64 %0, %0;" : "+l"(p));
    return p;
}

template <int C, int A1, int A2, int A3>
__global__ void __launch_bounds__(NW * 32, 1)
sgd_deep_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                const float4* __restrict__ rec, long long n_local, int K_local, int s_first, float lr,
                long long* __restrict__ trace) {
    extern __shared__ __align__(128) unsigned char smraw[];
    DSmem& sm = *reinterpret_cast<DSmem*>(smraw);
    float* w2s = reinterpret_cast<float*>(smraw + kHead);   // [R2MAX][H1MAX] own rows of W²
    float* xring = w2s + R2MAX * H1MAX;
    const int D = d.n[0], H1 = d.n[1], H2 = d.n[2], O = d.n[3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int crank = (int)cluster_rank();
    const int cn = s_first + (int)(blockIdx.x / C);
    constexpr int R = DeepShape<C>::RR;            // W¹ rows per sweep warp in registers
    constexpr int TRW = DeepShape<C>::TRW;         // … and in tensor memory
    constexpr int RW2 = DeepShape<C>::RW2;         // layer-2 rows per chain warp
    const int R1 = (((H1 + C - 1) / C) + 3) & ~3, k0 = crank * R1, own1 = max(0, min(R1, H1 - k0));
    const int R2 = (H2 + C - 1) / C, k02 = crank * R2, own2 = max(0, min(R2, H2 - k02));

    long long row0, T64;
    shard_of(n_local, K_local, cn, &row0, &T64);
    const int T = (int)T64;
    float* P = children + (long long)cn * d.P;
    float* W1 = P + d.woff[1];
    float* b1g = W1 + (long long)H1 * D;
    float* W2 = P + d.woff[2];
    float* b2g = W2 + (long long)H2 * H1;
    float* W3 = P + d.woff[3];
    float* b3g = W3 + (long long)O * H2;
    const float* Xc = X + row0 * (long long)D;
    const float4* Rc = rec + 2 * row0;
    const uint32_t xbytes = (uint32_t)D * 4u;

    if constexpr (TRW > 0) {
        if (warp == 0) tmem::alloc(&sm.tbase, 512);
    }
    if (threadIdx.x == 32) {
        for (int i = 0; i < S; ++i) mbar_init(&sm.xfull[i], 1);
        for (int i = 0; i < AR; ++i) mbar_init(&sm.aready[i], NSW);
        for (int i = 0; i < GR; ++i) mbar_init(&sm.gready[i], NCW);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.h1full[i], 1);
            mbar_init(&sm.zfull[i], 1);
            mbar_init(&sm.d1full[i], 1);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < S * DP; i += blockDim.x) xring[i] = 0.f;
    for (int i = threadIdx.x; i < GR * R1MAX; i += blockDim.x) (&sm.gbuf[0][0])[i] = 0.f;
    for (int i = threadIdx.x; i < 2 * H1MAX; i += blockDim.x) (&sm.h1buf[0][0])[i] = 0.f;   // pad: 0
    for (int i = threadIdx.x; i < R1MAX; i += blockDim.x) sm.b1s[i] = (i < own1) ? b1g[k0 + i] : 0.f;
    for (int i = threadIdx.x; i < R2MAX * H1MAX; i += blockDim.x) {
        const int r = i / H1MAX, j = i - r * H1MAX;
        w2s[i] = (r < own2 && j < H1) ? W2[(long long)(k02 + r) * H1 + j] : 0.f;
    }
    for (int i = threadIdx.x; i < R2MAX + 1; i += blockDim.x) sm.b2s[i] = (i < own2) ? b2g[k02 + i] : 0.f;
    for (int i = threadIdx.x; i < OMAX * (R2MAX + 1); i += blockDim.x) {
        const int o = i / (R2MAX + 1), r = i - o * (R2MAX + 1);
        sm.w3s[o][r] = (o < O && r < own2) ? W3[(long long)o * H2 + k02 + r] : 0.f;
    }
    for (int i = threadIdx.x; i < AR * R1MAX * 4; i += blockDim.x) (&sm.asum[0][0][0])[i] = 0.f;
    fence_proxy_async_smem();
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    cluster_sync_all();                            // peers' barriers exist before any st.async
    auto issue_x = [&](int u, int slot) {
        uint64_t* bar = &sm.xfull[slot];
        mbar_arrive_expect_tx(bar, xbytes + 32u);
        bulk_g2s(xring + slot * DP, Xc + (long long)u * D, xbytes, bar);
        bulk_g2s(xring + slot * DP + GOFF, Rc + 2 * u, 32u, bar);
    };
    if (threadIdx.x == (NSW + 2) * 32)
        for (int u = 0; u < PF && u < T; ++u) issue_x(u, u);   // chain step c issues x(c+PF)

    if (warp < NSW) {
        if constexpr (TRW == 0) {
            // ======================= sweeps: this warp's W¹ rows =======================
            const int kr0 = warp * R;
            uint64_t w[R][NP];
    #pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool live = kr0 + r < own1;
                const float* src = W1 + (long long)(k0 + kr0 + r) * D;
    #pragma unroll
                for (int m = 0; m < NP; ++m)
                    w[r][m] = live ? *reinterpret_cast<const uint64_t*>(src + pcol(lane, m)) : 0ull;
            }
            const int tr = lane >> 2, tq = lane & 3;
            const int nx = D - XC - 4 * tq;
            const bool xlive = kr0 + tr < own1;
            float* wxp = &sm.wx[warp][tr][4 * tq];
            {
                float4 w4 = make_float4(0.f, 0.f, 0.f, 0.f);
                const float* src = W1 + (long long)(k0 + kr0 + tr) * D + XC + 4 * tq;
                if (xlive) {
                    if (nx > 0) w4.x = src[0];
                    if (nx > 1) w4.y = src[1];
                    if (nx > 2) w4.z = src[2];
                    if (nx > 3) w4.w = src[3];
                }
                *reinterpret_cast<float4*>(wxp) = w4;
            }
            __syncwarp();
            int sx = 0;
            for (int s = 0; s < T + LAG; ++s) {
                if (s < T) {
                    mbar_wait(&sm.xfull[sx], (uint32_t)((s / S) & 1));
                    // F(s): acc = W¹(s-L)·x(s)
                    const float* xn = xring + sx * DP + 4 * lane;
                    uint64_t acc[R];
    #pragma unroll
                    for (int r = 0; r < R; ++r) acc[r] = 0ull;
                    uint64_t xa, xb;
                    lds4(xn, xa, xb);
    #pragma unroll
                    for (int q = 0; q < (kNoSweep ? 0 : NQ); ++q) {
                        uint64_t na = 0ull, nb = 0ull;
                        if (q + 1 < NQ) lds4(xn + 128 * (q + 1), na, nb);
    #pragma unroll
                        for (int r = 0; r < R; ++r) {
                            acc[r] = ffma2(w[r][2 * q], xa, acc[r]);
                            acc[r] = ffma2(w[r][2 * q + 1], xb, acc[r]);
                        }
                        xa = na;
                        xb = nb;
                    }
                    float px;
                    {
                        const float4 w4 = *reinterpret_cast<const float4*>(wxp);
                        const float4 x4 = *reinterpret_cast<const float4*>(xring + sx * DP + XC + 4 * tq);
                        px = fmaf(w4.w, x4.w, fmaf(w4.z, x4.z, fmaf(w4.y, x4.y, w4.x * x4.x)));
                    }
                    float v[R];
    #pragma unroll
                    for (int r = 0; r < R; ++r) {
                        float lo, hi;
                        upk(acc[r], lo, hi);
                        v[r] = lo + hi;
                    }
                    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                    float u4[4];
    #pragma unroll
                    for (int i = 0; i < 4; ++i)
                        u4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, b4 ? v[i] : v[i + 4], 16);
                    float u2[2];
    #pragma unroll
                    for (int i = 0; i < 2; ++i)
                        u2[i] = (b3 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b3 ? u4[i] : u4[i + 2], 8);
                    const float part = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4) + px;
                    sm.asum[s % AR][kr0 + tr][tq] = part;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.aready[s % AR]);
                }
                if (s >= LAG) {
                    // U(s): W¹ -= g(s-L)·x(s-L)ᵀ
                    const int u = s - LAG;
                    mbar_wait(&sm.gready[u % GR], (uint32_t)((u / GR) & 1));
                    const int su = (sx >= LAG) ? sx - LAG : sx + S - LAG;
                    const float* xo = xring + su * DP + 4 * lane;
                    const float4* gv = reinterpret_cast<const float4*>(&sm.gbuf[u % GR][kr0]);
                    const float4 g0 = gv[0], g1 = gv[1];
                    const float gp[R] = {-g0.x, -g0.y, -g0.z, -g0.w, -g1.x, -g1.y, -g1.z, -g1.w};
                    uint64_t xa, xb;
                    lds4(xo, xa, xb);
    #pragma unroll
                    for (int q = 0; q < (kNoSweep ? 0 : NQ); ++q) {
                        uint64_t na = 0ull, nb = 0ull;
                        if (q + 1 < NQ) lds4(xo + 128 * (q + 1), na, nb);
    #pragma unroll
                        for (int r = 0; r < R; ++r) {
                            w[r][2 * q] = ffma2(pk(gp[r], gp[r]), xa, w[r][2 * q]);
                            w[r][2 * q + 1] = ffma2(pk(gp[r], gp[r]), xb, w[r][2 * q + 1]);
                        }
                        xa = na;
                        xb = nb;
                    }
                    float4 w4 = *reinterpret_cast<const float4*>(wxp);
                    const float4 x4 = *reinterpret_cast<const float4*>(xring + su * DP + XC + 4 * tq);
                    const float gq = -sm.gbuf[u % GR][kr0 + tr];
                    w4.x = fmaf(gq, x4.x, w4.x); w4.y = fmaf(gq, x4.y, w4.y);
                    w4.z = fmaf(gq, x4.z, w4.z); w4.w = fmaf(gq, x4.w, w4.w);
                    *reinterpret_cast<float4*>(wxp) = w4;
                }
                if (++sx == S) sx = 0;
            }
            float* W1o = opaque(W1);
    #pragma unroll
            for (int r = 0; r < R; ++r) {
                if (kr0 + r < own1) {
                    float* dst = W1o + (long long)(k0 + kr0 + r) * D;
    #pragma unroll
                    for (int m = 0; m < NP; ++m) *reinterpret_cast<uint64_t*>(dst + pcol(lane, m)) = w[r][m];
                }
            }
            if (xlive) {
                const float4 w4 = *reinterpret_cast<const float4*>(wxp);
                float* dst = W1o + (long long)(k0 + kr0 + tr) * D + XC + 4 * tq;
                if (nx > 0) dst[0] = w4.x;
                if (nx > 1) dst[1] = w4.y;
                if (nx > 2) dst[2] = w4.z;
                if (nx > 3) dst[3] = w4.w;
            }
        } else {
        // ============= sweeps with TMEM rows (C = 4): RR register + TRW tensor-memory rows =============
        // TMEM: lane quadrant warp & 3, columns 256·(warp >> 2); quad q of TMEM row t at q·40 + 4t
        constexpr int RPW = R + TRW;
        constexpr int TQC = 4 * TRW;
        static_assert(RPW == 16 && TRW == 10, "the 16-row sweep (treduce over 16 rows, x32 + x8 TMEM loads)");
        const uint32_t tq = sm.tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2);
        const int kr0 = warp * RPW;
        uint64_t w[R][NP];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool live = kr0 + r < own1;
            const float* src = W1 + (long long)(k0 + kr0 + r) * D;
#pragma unroll
            for (int m = 0; m < NP; ++m)
                w[r][m] = live ? *reinterpret_cast<const uint64_t*>(src + pcol(lane, m)) : 0ull;
        }
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            uint32_t tv[TQC];
#pragma unroll
            for (int t = 0; t < TRW; ++t) {
                const bool live = kr0 + R + t < own1;
                const float* src = W1 + (long long)(k0 + kr0 + R + t) * D + 4 * lane + 128 * q;
                // (slabs are 8-byte aligned only: P is even)
                const float2 a = live ? *reinterpret_cast<const float2*>(src) : make_float2(0.f, 0.f);
                const float2 b = live ? *reinterpret_cast<const float2*>(src + 2) : make_float2(0.f, 0.f);
                tv[4 * t] = __float_as_uint(a.x); tv[4 * t + 1] = __float_as_uint(a.y);
                tv[4 * t + 2] = __float_as_uint(b.x); tv[4 * t + 3] = __float_as_uint(b.y);
            }
            tmem::st32(tq + q * TQC, tv);
            tmem::st8(tq + q * TQC + 32, tv + 32);
        }
        tmem::wait_st();
        const int trow = lane >> 1, th8 = lane & 1;   // tail: row kr0 + trow, columns 768 + 8·th8 .. +7
        const bool xlive = kr0 + trow < own1;
        float* wxp = &sm.wx[warp][trow][8 * th8];
        {
            const float* src = W1 + (long long)(k0 + kr0 + trow) * D + XC + 8 * th8;
#pragma unroll
            for (int j = 0; j < 8; ++j) wxp[j] = (xlive && XC + 8 * th8 + j < D) ? src[j] : 0.f;
        }
        __syncwarp();
        int sx = 0;
        for (int s = 0; s < T + LAG; ++s) {
            if (s < T) {
                mbar_wait(&sm.xfull[sx], (uint32_t)((s / S) & 1));
                // F(s): acc = W¹(s-L)·x(s)
                const float* xn = xring + sx * DP + 4 * lane;
                uint64_t acc[RPW];
#pragma unroll
                for (int r = 0; r < RPW; ++r) acc[r] = 0ull;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    uint32_t tv[TQC];
                    tmem::ld32(tq + q * TQC, tv);
                    tmem::ld8(tq + q * TQC + 32, tv + 32);
                    uint64_t xa, xb;
                    lds4(xn + 128 * q, xa, xb);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        acc[r] = ffma2(w[r][2 * q], xa, acc[r]);
                        acc[r] = ffma2(w[r][2 * q + 1], xb, acc[r]);
                    }
                    tmem::wait_ld_regs<TQC>(tv);
#pragma unroll
                    for (int t = 0; t < TRW; ++t) {
                        acc[R + t] = ffma2(pk(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1])), xa, acc[R + t]);
                        acc[R + t] = ffma2(pk(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3])), xb,
                                           acc[R + t]);
                    }
                }
                float px;
                {
                    const float4 w0 = *reinterpret_cast<const float4*>(wxp), w1 = *reinterpret_cast<const float4*>(wxp + 4);
                    const float* xt = xring + sx * DP + XC + 8 * th8;
                    const float4 x0 = *reinterpret_cast<const float4*>(xt), x1 = *reinterpret_cast<const float4*>(xt + 4);
                    px = w0.x * x0.x;
                    px = fmaf(w0.y, x0.y, px); px = fmaf(w0.z, x0.z, px); px = fmaf(w0.w, x0.w, px);
                    px = fmaf(w1.x, x1.x, px); px = fmaf(w1.y, x1.y, px); px = fmaf(w1.z, x1.z, px);
                    px = fmaf(w1.w, x1.w, px);
                }
                float v[RPW];
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
                    float lo, hi;
                    upk(acc[r], lo, hi);
                    v[r] = lo + hi;
                }
                // transpose-reduce 16 row sums: lane l ends with row l >> 1, part l & 1
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
                float u8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    u8[i] = (b4 ? v[i + 8] : v[i]) + __shfl_xor_sync(0xffffffffu, b4 ? v[i] : v[i + 8], 16);
                float u4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    u4[i] = (b3 ? u8[i + 4] : u8[i]) + __shfl_xor_sync(0xffffffffu, b3 ? u8[i] : u8[i + 4], 8);
                float u2[2];
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    u2[i] = (b2 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b2 ? u4[i] : u4[i + 2], 4);
                const float part = (b1 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? u2[0] : u2[1], 2) + px;
                sm.asum[s % AR][kr0 + trow][th8] = part;   // (parts 2, 3 stay 0)
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.aready[s % AR]);
            }
            if (s >= LAG) {
                // U(s): W¹ -= g(s-L)·x(s-L)ᵀ
                const int u = s - LAG;
                mbar_wait(&sm.gready[u % GR], (uint32_t)((u / GR) & 1));
                const int su = (sx >= LAG) ? sx - LAG : sx + S - LAG;
                const float* xo = xring + su * DP + 4 * lane;
                float gp[RPW];
                {
                    const float4* gv = reinterpret_cast<const float4*>(&sm.gbuf[u % GR][kr0]);
#pragma unroll
                    for (int i = 0; i < RPW / 4; ++i) {
                        const float4 a = gv[i];
                        gp[4 * i] = -a.x; gp[4 * i + 1] = -a.y; gp[4 * i + 2] = -a.z; gp[4 * i + 3] = -a.w;
                    }
                }
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    uint32_t tv[TQC];
                    tmem::ld32(tq + q * TQC, tv);
                    tmem::ld8(tq + q * TQC + 32, tv + 32);
                    uint64_t xa, xb;
                    lds4(xo + 128 * q, xa, xb);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        w[r][2 * q] = ffma2(pk(gp[r], gp[r]), xa, w[r][2 * q]);
                        w[r][2 * q + 1] = ffma2(pk(gp[r], gp[r]), xb, w[r][2 * q + 1]);
                    }
                    tmem::wait_ld_regs<TQC>(tv);
#pragma unroll
                    for (int t = 0; t < TRW; ++t) {
                        const uint64_t gg = pk(gp[R + t], gp[R + t]);
                        const uint64_t a = ffma2(gg, xa, pk(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1])));
                        const uint64_t b = ffma2(gg, xb, pk(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3])));
                        float a0, a1, b0, b1;
                        upk(a, a0, a1);
                        upk(b, b0, b1);
                        tv[4 * t] = __float_as_uint(a0); tv[4 * t + 1] = __float_as_uint(a1);
                        tv[4 * t + 2] = __float_as_uint(b0); tv[4 * t + 3] = __float_as_uint(b1);
                    }
                    tmem::st32(tq + q * TQC, tv);
                    tmem::st8(tq + q * TQC + 32, tv + 32);
                }
                {
                    const float gq = -sm.gbuf[u % GR][kr0 + trow];
                    const float* xt = xring + su * DP + XC + 8 * th8;
                    const float4 x0 = *reinterpret_cast<const float4*>(xt), x1 = *reinterpret_cast<const float4*>(xt + 4);
                    float4 w0 = *reinterpret_cast<const float4*>(wxp), w1 = *reinterpret_cast<const float4*>(wxp + 4);
                    w0.x = fmaf(gq, x0.x, w0.x); w0.y = fmaf(gq, x0.y, w0.y); w0.z = fmaf(gq, x0.z, w0.z);
                    w0.w = fmaf(gq, x0.w, w0.w); w1.x = fmaf(gq, x1.x, w1.x); w1.y = fmaf(gq, x1.y, w1.y);
                    w1.z = fmaf(gq, x1.z, w1.z); w1.w = fmaf(gq, x1.w, w1.w);
                    *reinterpret_cast<float4*>(wxp) = w0;
                    *reinterpret_cast<float4*>(wxp + 4) = w1;
                }
                tmem::wait_st();
            }
            if (++sx == S) sx = 0;
        }
        float* W1o = opaque(W1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (kr0 + r < own1) {
                float* dst = W1o + (long long)(k0 + kr0 + r) * D;
#pragma unroll
                for (int m = 0; m < NP; ++m) *reinterpret_cast<uint64_t*>(dst + pcol(lane, m)) = w[r][m];
            }
        }
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            uint32_t tv[TQC];
            tmem::ld32(tq + q * TQC, tv);
            tmem::ld8(tq + q * TQC + 32, tv + 32);
            tmem::wait_ld_regs<TQC>(tv);
#pragma unroll
            for (int t = 0; t < TRW; ++t) {
                if (kr0 + R + t < own1) {
                    float* dst = W1o + (long long)(k0 + kr0 + R + t) * D + 4 * lane + 128 * q;
                    *reinterpret_cast<float2*>(dst) = make_float2(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1]));
                    *reinterpret_cast<float2*>(dst + 2) =
                        make_float2(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3]));
                }
            }
        }
        if (xlive) {
            float* dst = W1o + (long long)(k0 + kr0 + trow) * D + XC + 8 * th8;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (XC + 8 * th8 + j < D) dst[j] = wxp[j];
        }
        }
    } else {
        // ======================= the chain =======================
        const int cw = warp - NSW;                 // this warp's layer-2 rows: cw + 3m, m < RW2
        const int ct = threadIdx.x - NSW * 32;     // chain thread: layer-1 unit ct (< own1)
        const int gw = crank * NCW + cw;           // this warp's partial-source index
        const int t4 = lane & 3, l4 = lane & ~3;   // 16-byte groups: lane 4i + t sends to ranks ≡ t (mod 4)
        const uint32_t sbase = smem_u32(smraw);
        auto off = [&](const void* p) { return smem_u32(p) - sbase; };
        float b3r = (lane < O) ? b3g[lane] : 0.f;  // b³ (every chain warp keeps an identical copy)
        bool rv[RW2];
#pragma unroll
        for (int m = 0; m < RW2; ++m) rv[m] = cw + NCW * m < own2;
        const int g1own = (own1 + 3) >> 2;         // 16-byte groups of the CTA's layer-1 units
        uint32_t h1bytes = 0;                      // every CTA's groups of h1
        for (int q = 0; q < C; ++q) h1bytes += 16u * (uint32_t)((max(0, min(R1, H1 - q * R1)) + 3) >> 2);
        const int og = (O + 3) >> 2;               // 16-byte groups of a partial-logit vector
        // fused pass: the owner CTA of this lane's h1 groups and the DSMEM addresses there
        uint32_t p1dst[NJ4], p1bar[NJ4];
#pragma unroll
        for (int k = 0; k < NJ4; ++k) {
            const int j0 = 4 * lane + 128 * k;
            const int q = min(j0 / R1, C - 1), jj = j0 - q * R1;
            p1dst[k] = mapa(sbase + off(&sm.p1buf[0][gw][0]) + 4u * (uint32_t)jj, (uint32_t)q);
            p1bar[k] = mapa(sbase + off(&sm.d1full[0]), (uint32_t)q);
        }
        constexpr uint32_t kP1Par = sizeof(float) * NGMAX * R1MAX;   // p1buf[1] - p1buf[0]
        int cs = 0;                                // ring slot of x(c)
        // debug timeline: [cta < C][chain warp][c < 64][point], clock64 of lane 0
        long long* trw = (trace && blockIdx.x < C && lane == 0) ? trace + (long long)(blockIdx.x * NCW + cw) * 64 * 16
                                                                  : nullptr;
#define DTR(pt)                                                                                    \
    do {                                                                                           \
        if (trw && c < 64) trw[c * 16 + (pt)] = ptx::clock64();                                    \
    } while (0)
        for (int c = 0; c < T; ++c) {
            DTR(0);
            const int par = c & 1;
            const uint32_t ph = (uint32_t)((c >> 1) & 1);
            // the chain warp without layer-1 units posts this sample's byte counts and the
            // x prefetch (off the critical path).  Safe: it has passed h1full(c-1), so every
            // CTA has finished δ1(c-2) and the [par] barriers' previous phases are complete.
            if (ct == 2 * 32) {
                mbar_arrive_expect_tx(&sm.h1full[par], h1bytes);
                mbar_arrive_expect_tx(&sm.zfull[par], 16u * (uint32_t)(og * NCW * C));
                mbar_arrive_expect_tx(&sm.d1full[par], 16u * (uint32_t)(g1own * NCW * C));
            }
            mbar_wait(&sm.aready[c % AR], (uint32_t)((c / AR) & 1));   // every sweep's F(c)
            // x(c) and its Gram record are visible through aready(c): every sweep waited xfull
            // for x(c) before its F(c) (acquire) and arrived aready(c) after it (release)
            // every sweep has passed U(c-1): the slot of x(c-1-L) is free for x(c+PF)
            if (ct == 2 * 32 && c + PF < T) issue_x(c + PF, (cs + PF) % S);
            const float4 G = *reinterpret_cast<const float4*>(xring + cs * DP + GOFF);
            const int label = __float_as_int(xring[cs * DP + GOFF + 4]);
            DTR(1);
            // ---- z1(c) = acc - Σ_k g(c-k) G(c-k,c) + b1(c), h1 of unit ct → every CTA ----
            float h1u = 0.f;
            if (ct < own1) {
                const float4 pa = *reinterpret_cast<const float4*>(&sm.asum[c % AR][ct][0]);
                float z = (pa.x + pa.y) + (pa.z + pa.w);
                z = fmaf(-sm.gbuf[(c + GR - 4) % GR][ct], G.x, z);
                z = fmaf(-sm.gbuf[(c + GR - 3) % GR][ct], G.y, z);
                z = fmaf(-sm.gbuf[(c + GR - 2) % GR][ct], G.z, z);
                z = fmaf(-sm.gbuf[(c + GR - 1) % GR][ct], G.w, z);
                z += sm.b1s[ct];
                h1u = act_fast<A1>(z);
            }
            if (cw * 32 < own1) {                      // the chain threads that own layer-1 units
                float4 v;
                v.x = __shfl_sync(0xffffffffu, h1u, l4);
                v.y = __shfl_sync(0xffffffffu, h1u, l4 + 1);
                v.z = __shfl_sync(0xffffffffu, h1u, l4 + 2);
                v.w = __shfl_sync(0xffffffffu, h1u, l4 + 3);
                if ((ct >> 2) < g1own) {
                    const uint32_t dst = sbase + off(&sm.h1buf[par][k0 + (ct & ~3)]);
                    const uint32_t bar = sbase + off(&sm.h1full[par]);
                    for (int q = t4; q < C; q += 4) st_async_v4(mapa(dst, (uint32_t)q), v, mapa(bar, (uint32_t)q));
                }
            }
            DTR(2);
            // ---- z2, h2 of this warp's rows: lane covers h1 units 4·lane + 128k + (0..3) ----
            chain_wait(&sm.h1full[par], ph);
            DTR(3);
            float4 hv[NJ4];
#pragma unroll
            for (int k = 0; k < NJ4; ++k) hv[k] = *reinterpret_cast<const float4*>(&sm.h1buf[par][4 * lane + 128 * k]);
            float a2[RW2];
#pragma unroll
            for (int m = 0; m < RW2; ++m) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < NJ4; ++k) {
                    const float4 w4 = *reinterpret_cast<const float4*>(w2s + (cw + NCW * m) * H1MAX + 4 * lane + 128 * k);
                    acc = fmaf(w4.x, hv[k].x, acc);
                    acc = fmaf(w4.y, hv[k].y, acc);
                    acc = fmaf(w4.z, hv[k].z, acc);
                    acc = fmaf(w4.w, hv[k].w, acc);
                }
                a2[m] = acc;
            }
            DTR(10);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int m = 0; m < RW2; ++m) a2[m] += __shfl_xor_sync(0xffffffffu, a2[m], o);
            DTR(11);
            float h2v[RW2];
            {                                       // branch-free: the RW2 activations interleave
                float bz[RW2];
#pragma unroll
                for (int m = 0; m < RW2; ++m) bz[m] = sm.b2s[cw + NCW * m];   // (rows past own2: unused)
#pragma unroll
                for (int m = 0; m < RW2; ++m) {
                    const float t = act_fast<A2>(a2[m] + bz[m]);
                    h2v[m] = rv[m] ? t : 0.f;
                }
            }
            DTR(12);
            // ---- this warp's partial logits W³[:, rows]·h2 → every CTA ----
            {
                float pz = 0.f;
                if (lane < O) {
#pragma unroll
                    for (int m = 0; m < RW2; ++m) pz = fmaf(sm.w3s[lane][cw + NCW * m], h2v[m], pz);
                }
                float4 v;
                v.x = __shfl_sync(0xffffffffu, pz, l4);
                v.y = __shfl_sync(0xffffffffu, pz, l4 + 1);
                v.z = __shfl_sync(0xffffffffu, pz, l4 + 2);
                v.w = __shfl_sync(0xffffffffu, pz, l4 + 3);
                DTR(13);
                if ((lane >> 2) < og) {
                    const uint32_t dst = sbase + off(&sm.zbuf[par][gw][l4]), bar = sbase + off(&sm.zfull[par]);
                    for (int q = t4; q < C; q += 4) st_async_v4(mapa(dst, (uint32_t)q), v, mapa(bar, (uint32_t)q));
                }
            }
            DTR(4);
            // ---- δ3 (every chain warp, identically): z3 = b3 + Σ partials in a fixed order ----
            chain_wait(&sm.zfull[par], ph);
            DTR(5);
            float d3 = 0.f;
            {
                float z3 = b3r;
                if (lane < O) {
                    float zs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int g = 0; g < NCW * C; ++g) zs[g & 3] += sm.zbuf[par][g][lane];
                    z3 += (zs[0] + zs[1]) + (zs[2] + zs[3]);
                }
                DTR(14);
                if constexpr (A3 == PNN_SOFTMAX) {
                    float m = (lane < O) ? z3 : -INFINITY;
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                    float e = (lane < O) ? __expf(z3 - m) : 0.f;   // R28
                    float sum = e;
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    if (lane < O) d3 = __fdividef(e, sum) - ((lane == label) ? 1.f : 0.f);
                } else {
                    if (lane < O) {
                        const float x3 = act_fast<A3>(z3);
                        d3 = (x3 - ((lane == label) ? 1.f : 0.f)) * act_deriv_t<A3>(x3);
                    }
                }
                DTR(15);
                b3r = fmaf(-lr, d3, b3r);
            }
            // ---- δ2 of this warp's rows (pre-update W³, R6); W³, b2 updates ----
            float d2[RW2];
            {                                       // branch-free loads, predicated stores
                const int ol = lane < O ? lane : 0;
                float w3v[RW2];
#pragma unroll
                for (int m = 0; m < RW2; ++m) w3v[m] = sm.w3s[ol][cw + NCW * m];
                const float e3 = -lr * d3;          // d3 = 0 for lanes >= O
#pragma unroll
                for (int m = 0; m < RW2; ++m) {
                    d2[m] = w3v[m] * d3;
                    if (lane < O) sm.w3s[lane][cw + NCW * m] = fmaf(e3, h2v[m], w3v[m]);   // invalid rows: h2 = 0
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int m = 0; m < RW2; ++m) d2[m] += __shfl_xor_sync(0xffffffffu, d2[m], o);
            {                                       // lane m < RW2 updates b2 of row m (one store per lane)
                float dsel = 0.f;
#pragma unroll
                for (int m = 0; m < RW2; ++m) {
                    d2[m] = rv[m] ? d2[m] * act_deriv_t<A2>(h2v[m]) : 0.f;
                    dsel = (lane == m) ? d2[m] : dsel;
                }
                if (lane < RW2 && cw + NCW * lane < own2) sm.b2s[cw + NCW * lane] -= lr * dsel;
            }
            DTR(6);
            // ---- fused: partial (W²ᵀδ2)_j over this warp's rows (pre-update, R6) → unit j's
            //      owner CTA (R1 is a multiple of 4: a group has one owner), and
            //      W² -= η δ2 h1ᵀ on the same elements ----
            {
#pragma unroll
                for (int k = 0; k < NJ4; ++k) {
                    const int j0 = 4 * lane + 128 * k;
                    if (j0 < H1) {
                        float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int m = 0; m < RW2; ++m) {
                            float4* wp = reinterpret_cast<float4*>(w2s + (cw + NCW * m) * H1MAX + j0);
                            float4 w4 = *wp;
                            p.x = fmaf(w4.x, d2[m], p.x); p.y = fmaf(w4.y, d2[m], p.y);
                            p.z = fmaf(w4.z, d2[m], p.z); p.w = fmaf(w4.w, d2[m], p.w);
                            const float e = -lr * d2[m];
                            w4.x = fmaf(e, hv[k].x, w4.x); w4.y = fmaf(e, hv[k].y, w4.y);
                            w4.z = fmaf(e, hv[k].z, w4.z); w4.w = fmaf(e, hv[k].w, w4.w);
                            *wp = w4;
                        }
                        st_async_v4(p1dst[k] + par * kP1Par, p, p1bar[k] + par * 8u);
                    }
                }
            }
            DTR(7);
            // ---- δ1, g = η δ1 and b1 of unit ct ----
            if (ct < own1) {
                chain_wait(&sm.d1full[par], ph);
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int g = 0; g < NCW * C; ++g) ps[g & 3] += sm.p1buf[par][g][ct];
                const float s1 = (ps[0] + ps[1]) + (ps[2] + ps[3]);
                const float gu = lr * (s1 * act_deriv_t<A1>(h1u));
                sm.gbuf[c % GR][ct] = gu;
                sm.b1s[ct] -= gu;
            }
            DTR(8);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.gready[c % GR]);
            DTR(9);
            if (++cs == S) cs = 0;
        }
#undef DTR
        // ---- write back the chain's parameters ----
        for (int i = ct; i < own1; i += NCW * 32) opaque(b1g)[k0 + i] = sm.b1s[i];
        __syncwarp();
        for (int m = 0; m < RW2; ++m) {
            if (!rv[m]) continue;
            const int i = cw + NCW * m;
            float* dst = opaque(W2) + (long long)(k02 + i) * H1;
            for (int j = lane; j < H1; j += 32) dst[j] = w2s[i * H1MAX + j];
            if (lane == 0) opaque(b2g)[k02 + i] = sm.b2s[i];
            if (lane < O) opaque(W3)[(long long)lane * H2 + k02 + i] = sm.w3s[lane][i];
        }
        if (crank == 0 && cw == 0 && lane < O) opaque(b3g)[lane] = b3r;
    }
    if constexpr (TRW > 0) {
        tmem::fence_before();
        __syncthreads();
        tmem::fence_after();
        if (warp == 0) tmem::dealloc(sm.tbase, 512);
    }
    cluster_sync_all();                            // no CTA leaves while a peer may still st.async into it
}

template <int C, int A1, int A2, int A3>
cudaError_t launch_one(const NetDesc& d, float* children, const float* x, const float4* rec, long long n_local,
                       int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    auto kern = sgd_deep_kernel<C, A1, A2, A3>;
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
    return cudaLaunchKernelEx(&cfg, kern, d, children, x, rec, n_local, K_local, s_first, lr, g_trace);
}

#define PNN_DEEP_ACTS(X_)                                                                          \
    X_(PNN_TANH, PNN_TANH, PNN_SOFTMAX)                                                            \
    X_(PNN_RELU, PNN_RELU, PNN_SOFTMAX)                                                            \
    X_(PNN_SIGMOID, PNN_SIGMOID, PNN_SOFTMAX)                                                      \
    X_(PNN_SIGMOID, PNN_SIGMOID, PNN_SIGMOID)                                                      \
    X_(PNN_LEAKY_RELU, PNN_LEAKY_RELU, PNN_SOFTMAX)

template <int C>
cudaError_t launch_c(const NetDesc& d, float* children, const float* x, const float4* rec, long long n_local,
                     int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
#define PNN_CASE(A1_, A2_, A3_)                                                                    \
    if (d.act[0] == A1_ && d.act[1] == A2_ && d.act[2] == A3_)                                     \
        return launch_one<C, A1_, A2_, A3_>(d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
    PNN_DEEP_ACTS(PNN_CASE)
#undef PNN_CASE
    return cudaErrorInvalidValue;
}

int deep_cluster(const NetDesc& d) {
    // the smallest cluster whose CTAs hold the layers (R1 rounded to a multiple of 4, as the
    // kernel does): fewer SMs per CN, more CNs at once
    auto r1 = [&](int c) { return (((d.n[1] + c - 1) / c) + 3) & ~3; };
    if (r1(4) <= r1cap<4>() && (d.n[2] + 3) / 4 <= r2cap<4>()) return 4;
    if (r1(8) <= r1cap<8>() && (d.n[2] + 7) / 8 <= r2cap<8>()) return 8;
    return 0;
}

}  // namespace

const char* deep_plan(const NetDesc& d, int batch) {
    if (batch != 1) return "per-sample SGD only";
    if (d.L != 3) return "3-layer nets only";
    const int D = d.n[0];
    if (D % 4 != 0 || D <= XC || D > XC + 16) return "built for 768 < inputs <= 784, a multiple of 4";
    if (d.n[1] > 320) return "first hidden layer wider than 320";
    if (d.n[3] > OMAX) return "more than 16 outputs";
    if (d.P % 2 != 0) return "odd parameter count (W1 rows are moved as 8-byte pairs)";
    if (!deep_cluster(d)) return "hidden layers too wide for 8 CTAs";
    bool built = false;
#define PNN_CASE(A1_, A2_, A3_) built = built || (d.act[0] == A1_ && d.act[1] == A2_ && d.act[2] == A3_);
    PNN_DEEP_ACTS(PNN_CASE)
#undef PNN_CASE
    if (!built) return "activation triple not instantiated in the deep kernel";
    return nullptr;
}

int deep_cluster_size(const NetDesc& d) { return deep_cluster(d); }

cudaError_t launch_sgd_deep(const NetDesc& d, float* children, const float* x, const int32_t* labels,
                            float4* rec, long long n_local, int K_local, int s_first, int s_count, float lr,
                            cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    cudaError_t e = launch_gram(x, labels, d.n[0], n_local, K_local, s_first, s_count, rec, st);
    if (e != cudaSuccess) return e;
    switch (deep_cluster(d)) {
    case 4: return launch_c<4>(d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
    case 8: return launch_c<8>(d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
    default: return cudaErrorInvalidValue;
    }
}

// Debug: how many clusters of the deep kernel (C = 4 or 8, tanh/tanh/softmax instance) can be
// co-resident on this GPU (cudaOccupancyMaxActiveClusters).
extern "C" int pnn_debug_deep_max_clusters(int C) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(C * 64));
    cfg.blockDim = dim3((unsigned)(NW * 32));
    cfg.dynamicSmemBytes = kSmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e;
    auto q = [&](auto k) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    };
    switch (C) {
    case 4: e = q(sgd_deep_kernel<4, PNN_TANH, PNN_TANH, PNN_SOFTMAX>); break;
    case 8: e = q(sgd_deep_kernel<8, PNN_TANH, PNN_TANH, PNN_SOFTMAX>); break;
    default: return -1;
    }
    return e == cudaSuccess ? n : -(int)e;
}
