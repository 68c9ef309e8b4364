// k_resident.cu — persistent per-sample SGD with register-resident weights (v7).
//
// A thread-block cluster of C CTAs trains NG child networks (CNs) over their
// whole slices ("Each child-network learns only a slice").  Each
// CN's hidden layer is split across the C SMs (CTA c owns units [c·U, c·U+U)),
// and in every CTA the CN is served by NWG warps of 8 W¹ rows each; the rows
// live in REGISTERS for the whole slice (loaded once, written back once).
// C4 shape (784-128-10): C = 2, NG = 1, 8 warps per CTA; or C = 4, NG = 2,
// 2 × 4 warps per CTA (every SM sub-partition then hosts one warp of each of
// two independent CNs, so one CN's serial tail overlaps the other's sweep).
// Scope: 2-layer nets D-H-O, 768 < D <= 784, O = 10, H <= 64·C/NG, per-sample SGD.
//
// Per sample, in the paper's sequential order (§3, Eqs.2-13):
//   z1 = W1 x + b1, h = φ1(z1); z2 = W2 h + b2, x2 = φ2(z2)         (Eqs.2-5)
//   δ2 = x2 - e (softmax+CE, Eq.10) or (x2 - e)⊙φ2'(x2) (R11)       (Eqs.9-10)
//   δ1 = (W2ᵀ δ2) ⊙ φ1'(h), with the pre-update W2 (R6)              (Eq.11)
//   W -= η δ xᵀ, b -= η δ                                             (Eqs.12-13)
//
// Two-step lookahead.  With W¹(t) the weights before sample t's update and
// g(s) = η δ1(s), W¹(t) = W¹(t-2) - g(t-2)x(t-2)ᵀ - g(t-1)x(t-1)ᵀ, so
//     z1(t) = W¹(t-2)x(t) - g(t-2)·G(t-2,t) - g(t-1)·G(t-1,t) + b1(t),
// G(s,t) = x(s)·x(t): the paper's pre-activation in real arithmetic (DESIGN.md
// R27; only the rounding differs).  The Gram terms depend on the data only;
// gram_kernel computes them for every row before training and they travel
// with x(t) through the shared-memory ring.  Step t of every warp:
//   F(t)   acc = W¹(t-2)·x(t): lane l holds columns 4l+128q .. +3 (q < 6) as
//          f32x2 pairs, one LDS.128 feeds 16 fma.rn.f32x2; columns 768..783
//          live in shared memory (4 per lane); row sums by a transpose-reduce;
//   U(t)   W¹ -= g(t-2)·x(t-2)ᵀ (g(t-2) is two steps old: no wait);
//   tail   wait for the partial logits of sample t-1 from every warp of the
//          cluster (mbarrier zfull, st.async from the peers); z2, softmax /
//          φ2 and δ2(t-1) in every lane; δ1 and g(t-1) of the warp's units,
//          their W² columns, b1, b2; then z1(t) by the correction above, h(t)
//          and the partial logits of the warp's units, published to every CTA.
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"

long long* g_trace = nullptr;   // debug: clock64 timeline (tools/trace_resident.py)
extern "C" void pnn_debug_set_trace(long long* dev_buf) { g_trace = dev_buf; }

namespace {

using namespace ptx;

constexpr int R = 8;          // W1 rows per warp
constexpr int NQ = 6;         // column quads per lane: columns [0, 768)
constexpr int NP = 2 * NQ;    // f32x2 pairs per lane
constexpr int XC = 768;       // first shared-memory column
constexpr int GOFF = 784;     // Gram terms of sample u sit at its x ring slot + GOFF
constexpr int DP = 800;       // x ring slot stride (floats)
constexpr int S = 12;         // x ring slots per CN group
constexpr int PF = S - 3;     // prefetch distance
constexpr int O = 10;         // outputs
constexpr int ZS = 4;         // partial-logit ring slots
constexpr int CMAX = 4;       // cluster size
constexpr int NWMAX = 8;      // warps per CTA
constexpr int NGMAX = 2;      // CN groups per CTA
constexpr int kTraceT = 64, kTraceP = 8;   // debug timeline: [cta][warp][t][point]

struct __align__(16) GroupSmem {
    uint64_t xfull[S];                    // x(u) and its Gram terms landed
    uint64_t zfull[ZS];                   // partial logits of sample t from every warp of the CN
    float zbuf[ZS][CMAX * NWMAX][16];     // [t % ZS][cta·NWG + warp][o]
    float gw[2][NWMAX][R];                // [s & 1][warp][row] g(s) of the warp's rows
};
struct __align__(16) Smem {
    GroupSmem grp[NGMAX];
    float wx[NWMAX][R][16];               // W1 columns 768..783 of each warp's rows
    float zg[NWMAX][16];                  // per-warp all-gather of z2
    float b2s[NWMAX][16];                 // per-warp copy of b2 (identical in every warp)
    int32_t ylab[NWMAX][64];              // per-warp label ring: [warp][u & 63] = y(u)
};
constexpr size_t kSmemHead = ((sizeof(Smem) + 127) / 128) * 128;

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
// column of pair j (0 <= j < NP) for lane l
__device__ __forceinline__ int pcol(int l, int j) { return 4 * l + 128 * (j >> 1) + 2 * (j & 1); }
// An opaque copy of a pointer: keeps addresses computed before the slice loop from
// staying alive across it (they would occupy registers the weights need).
template <typename T> __device__ __forceinline__ T* opaque(T* p) {
    asm volatile("mov.b64 %0, %0;" : "+l"(p));
    return p;
}
// v[base + q] for a lane-dependent q in 0..3, without local memory
__device__ __forceinline__ float pick4(const float* v, int base, int q) {
    const float a = v[base], b = v[base + 1], c = v[base + 2], d = v[base + 3];
    return q == 0 ? a : q == 1 ? b : q == 2 ? c : d;
}

// Gram terms of every row of CNs [s_first, s_first + s_count) (shard-local index u):
// gram[row] = {x(u-2)·x(u), x(u-1)·x(u), 0, 0}, terms before the slice start = 0.
// One warp per row; X is read once from HBM (the two previous rows hit in cache).
__global__ void __launch_bounds__(256)
gram_kernel(const float* __restrict__ X, int D, long long n_local, int K_local, int s_first,
            int s_count, float4* __restrict__ gram) {
    long long r0, c0, r1, c1;
    shard_of(n_local, K_local, s_first, &r0, &c0);
    shard_of(n_local, K_local, s_first + s_count - 1, &r1, &c1);
    const long long rows = r1 + c1 - r0;
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    const long long base = n_local / K_local, rem = n_local % K_local;
    for (long long i = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += nwarps) {
        const long long row = r0 + i;
        // the CN owning this row (R17: the first rem slices are one row longer)
        const long long s = (row < rem * (base + 1)) ? row / (base + 1)
                                                     : rem + (row - rem * (base + 1)) / base;
        long long st, cnt;
        shard_of(n_local, K_local, (int)s, &st, &cnt);
        const long long u = row - st;
        const float* xc = X + row * (long long)D;
        float g0 = 0.f, g1 = 0.f;
        for (int j = lane * 4; j < D; j += 128) {
            const float4 c = *reinterpret_cast<const float4*>(xc + j);
            if (u >= 1) {
                const float4 b = *reinterpret_cast<const float4*>(xc - D + j);
                g1 = fmaf(b.w, c.w, fmaf(b.z, c.z, fmaf(b.y, c.y, fmaf(b.x, c.x, g1))));
            }
            if (u >= 2) {
                const float4 a = *reinterpret_cast<const float4*>(xc - 2 * D + j);
                g0 = fmaf(a.w, c.w, fmaf(a.z, c.z, fmaf(a.y, c.y, fmaf(a.x, c.x, g0))));
            }
        }
        g0 = warp_sum(g0);
        g1 = warp_sum(g1);
        if (lane == 0) gram[row] = make_float4(g0, g1, 0.f, 0.f);
    }
}

template <int C, int NG, int A1, int A2, bool TRACE>
__global__ void __launch_bounds__(NWMAX * 32, 1)
sgd_resident_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                    const int32_t* __restrict__ Y, const float4* __restrict__ gram, long long n_local,
                    int K_local, int s_first, int s_count, float lr, long long* __restrict__ trace) {
    extern __shared__ __align__(128) unsigned char smraw[];
    Smem& sm = *reinterpret_cast<Smem*>(smraw);
    const int D = d.n[0], H = d.n[1];
    constexpr int NWG = NWMAX / NG;                // warps per CN group
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = warp / NWG, wl = warp % NWG;     // CN group, warp within the group
    GroupSmem& gs = sm.grp[g];
    float* xring = reinterpret_cast<float*>(smraw + kSmemHead) + g * (S + 1) * DP;
    const int crank = (C > 1) ? (int)cluster_rank() : 0;
    const int cidx = s_first + (int)(blockIdx.x / C) * NG + g;   // this group's CN
    const bool active = cidx < s_first + s_count;
    const int U = (H + C - 1) / C;                 // units per CTA
    const int k0 = crank * U;
    const int Uown = max(0, min(U, H - k0));

    long long row0 = 0, T64 = 0;
    if (active) shard_of(n_local, K_local, cidx, &row0, &T64);
    const int T = (int)T64;
    float* P = children + (long long)(active ? cidx : s_first) * d.P;
    float* W1 = P;
    float* b1g = P + (long long)H * D;
    float* W2 = b1g + H;
    float* b2g = W2 + (long long)O * H;
    const float* Xc = X + row0 * (long long)D;
    const int32_t* Yc = Y + row0;
    const float4* Gc = gram + row0;

    if (threadIdx.x == 0) {
        for (int q = 0; q < NG; ++q) {
            for (int i = 0; i < S; ++i) mbar_init(&sm.grp[q].xfull[i], 1);
            for (int i = 0; i < ZS; ++i) mbar_init(&sm.grp[q].zfull[i], NWG);
        }
        fence_mbar_init();
    }
    {
        float* ring0 = reinterpret_cast<float*>(smraw + kSmemHead);
        for (int i = threadIdx.x; i < NG * (S + 1) * DP; i += blockDim.x) ring0[i] = 0.f;
        for (int q = 0; q < NG; ++q)
            for (int i = threadIdx.x; i < 2 * NWMAX * R; i += blockDim.x) (&sm.grp[q].gw[0][0][0])[i] = 0.f;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if constexpr (C > 1) cluster_sync_all();       // peers' barriers exist before any st.async
    const uint32_t xbytes = (uint32_t)D * 4u;
    if (active && wl == 0 && lane == 0)
        for (int u = 0; u <= PF && u < T; ++u) {   // steps t >= 1 issue x(t + PF)
            uint64_t* bar = &gs.xfull[u];
            mbar_arrive_expect_tx(bar, xbytes + 16u);
            bulk_g2s(xring + u * DP, Xc + (long long)u * D, xbytes, bar);
            bulk_g2s(xring + u * DP + GOFF, Gc + u, 16u, bar);
        }

#define TR(pt)                                                                                   \
    do {                                                                                         \
        if constexpr (TRACE) {                                                                   \
            if (blockIdx.x < 2 && t < kTraceT && lane == 0)                                      \
                trace[(((int)blockIdx.x * NWMAX + warp) * kTraceT + t) * kTraceP + (pt)] =       \
                    ptx::clock64();                                                              \
        }                                                                                        \
    } while (0)

    // ---- this warp's W1 rows ----
    const int kr0 = wl * R;                        // first row (CTA-local)
    uint64_t w[R][NP];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const bool live = active && kr0 + r < Uown;
        const float* src = W1 + (long long)(k0 + kr0 + r) * D;
#pragma unroll
        for (int m = 0; m < NP; ++m)
            w[r][m] = live ? *reinterpret_cast<const uint64_t*>(src + pcol(lane, m)) : 0ull;
    }
    // ---- tail state: lane = 4·r + q holds unit r: W2[o][·] for o = q, q+4, q+8 and the
    //      W1 columns 768+4q .. 768+4q+3 (in shared memory) ----
    const int tr = lane >> 2, tq = lane & 3;
    const bool tlive = active && kr0 + tr < Uown;
    const int ku = k0 + kr0 + tr;                  // global hidden unit of this lane
    const int nx = D - XC - 4 * tq;                // valid extra columns of this lane's quad
    float* wxp = &sm.wx[warp][tr][4 * tq];
    {
        float4 w4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float* src = W1 + (long long)ku * D + XC + 4 * tq;
        if (tlive) {
            if (nx > 0) w4.x = src[0];
            if (nx > 1) w4.y = src[1];
            if (nx > 2) w4.z = src[2];
            if (nx > 3) w4.w = src[3];
        }
        *reinterpret_cast<float4*>(wxp) = w4;
    }
    float w2[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int o = tq + 4 * i;
        w2[i] = (tlive && o < O) ? W2[(long long)o * H + ku] : 0.f;
    }
    float b1 = tlive ? b1g[ku] : 0.f;
    if (lane < 16) sm.b2s[warp][lane] = (active && lane < O) ? b2g[lane] : 0.f;
    float hprev = 0.f, gm1 = 0.f, gm2 = 0.f;       // h(t-1), g(t-1), g(t-2) of this lane's unit
    if (lane < T) cp_async4(&sm.ylab[warp][lane], Yc + lane);
    if (32 + lane < T) cp_async4(&sm.ylab[warp][32 + lane], Yc + 32 + lane);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();

    // DSMEM address of zbuf[0][crank·NWG + wl][0] in each peer (its zfull[0] is at a fixed offset)
    uint32_t rz[C > 1 ? C - 1 : 1];
    if constexpr (C > 1) {
#pragma unroll
        for (int p = 1; p < C; ++p)
            rz[p - 1] = mapa(smem_u32(&gs.zbuf[0][crank * NWG + wl][0]), (uint32_t)((crank + p) % C));
    }
    constexpr uint32_t kZStride = CMAX * NWMAX * 16 * 4;
    constexpr uint32_t kZfullOff = (uint32_t)offsetof(GroupSmem, zfull) - (uint32_t)offsetof(GroupSmem, zbuf);

    float a = 0.f;                                 // acc(t) of row tr (after the reduction)
    int sx = 0;                                    // ring slot of x(t) = t % S
    uint32_t xpar = 0;                             // phase parity of x(t)'s slot = (t / S) & 1
    int sz = 0, pz = ZS - 1;                       // zbuf slots of samples t and t-1
    uint32_t zpar = 0, ppar = 1;                   // phase parities of zfull(t), zfull(t-1)
    for (int t = 0; active && t <= T + 1; ++t) {
        TR(0);
        if (t < T) {
            // x(t) is certified by zfull(t-2) (waited in step t-1); the first two wait here
            if (t <= 1) mbar_wait(&gs.xfull[t], 0u);
            // ---------------- F(t): acc = W¹(t-2)·x(t) ----------------
            const float* xn = xring + sx * DP + 4 * lane;
            uint64_t acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0ull;
            uint64_t xa, xb;
            lds4(xn, xa, xb);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint64_t na = 0ull, nb = 0ull;
                if (q + 1 < NQ) lds4(xn + 128 * (q + 1), na, nb);   // one quad ahead
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    acc[r] = ffma2(w[r][2 * q], xa, acc[r]);
                    acc[r] = ffma2(w[r][2 * q + 1], xb, acc[r]);
                }
                xa = na;
                xb = nb;
            }
            float px;                              // columns 768..783 of row tr
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
            // transpose-reduce 8 row sums over 32 lanes; row (lane >> 2) ends in its 4 lanes
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
            float u4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                u4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, b4 ? v[i] : v[i + 4], 16);
            float u2[2];
#pragma unroll
            for (int i = 0; i < 2; ++i)
                u2[i] = (b3 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b3 ? u4[i] : u4[i + 2], 8);
            a = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4) + px;
            a += __shfl_xor_sync(0xffffffffu, a, 2);
            a += __shfl_xor_sync(0xffffffffu, a, 1);
        }
        TR(1);
        if (t >= 2) {
            // ---------------- U(t): W¹ -= g(t-2)·x(t-2)ᵀ ----------------
            const int s2 = (sx >= 2) ? sx - 2 : sx + S - 2;
            const float* xo = xring + s2 * DP + 4 * lane;
            const float4* gv = reinterpret_cast<const float4*>(&gs.gw[t & 1][wl][0]);
            const float4 g0 = gv[0], g1 = gv[1];
            const float gp[R] = {-g0.x, -g0.y, -g0.z, -g0.w, -g1.x, -g1.y, -g1.z, -g1.w};
            uint64_t xa, xb;
            lds4(xo, xa, xb);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
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
            const float4 x4 = *reinterpret_cast<const float4*>(xring + s2 * DP + XC + 4 * tq);
            const float gq = -gs.gw[t & 1][wl][tr];
            w4.x = fmaf(gq, x4.x, w4.x); w4.y = fmaf(gq, x4.y, w4.y);
            w4.z = fmaf(gq, x4.z, w4.z); w4.w = fmaf(gq, x4.w, w4.w);
            *reinterpret_cast<float4*>(wxp) = w4;
        }
        TR(2);
        if (t > T) break;

        // ================= tail: finish sample t-1, start sample t =================
        if (t >= 33 && ((t - 1) & 31) == 0) {      // refill the half of the label ring used 32 ago
            if (t + 31 + lane < T) cp_async4(&sm.ylab[warp][(t + 31 + lane) & 63], Yc + t + 31 + lane);
            cp_async_commit();
        }
        if (t >= 49 && ((t - 1) & 31) == 16) {
            cp_async_wait_all();
            __syncwarp();
        }
        // δ2(t-1)[o] in lanes o and o+16 (o < 10; δ2(-1) := 0), lane-parallel softmax
        float dl = 0.f;
        if (t >= 1) {
            mbar_wait(&gs.zfull[pz], ppar);
            TR(3);
            // every local warp has passed step t-1: the slot of x(t-3) is free for x(t+PF)
            if (wl == 0 && lane == 0 && t + PF < T) {
                const int u = t + PF, su = (sx + PF >= S) ? sx + PF - S : sx + PF;
                uint64_t* bar = &gs.xfull[su];
                mbar_arrive_expect_tx(bar, xbytes + 16u);
                bulk_g2s(xring + su * DP, Xc + (long long)u * D, xbytes, bar);
                bulk_g2s(xring + su * DP + GOFF, Gc + u, 16u, bar);
            }
            const int o16 = lane & 15, hf = lane >> 4;
            const bool valid = o16 < O;
            float zsum = 0.f;
#pragma unroll
            for (int i = 0; i < C * NWG / 2; ++i) zsum += gs.zbuf[pz][2 * i + hf][o16];
            zsum += __shfl_xor_sync(0xffffffffu, zsum, 16);
            const float b2o = sm.b2s[warp][o16];  // b2(t-1) (pad entries are 0)
            const float z2 = zsum + b2o;           // z2 = W2 h + b2 (Eq.2)
            const int label = sm.ylab[warp][(t + 63) & 63];         // y(t-1)
            if constexpr (A2 == PNN_SOFTMAX) {
                float m = valid ? z2 : -INFINITY;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                const float e = valid ? __expf(z2 - m) : 0.f;
                float sum = e;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                float inv;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(sum));
                dl = e * inv - ((o16 == label) ? 1.f : 0.f);
            } else {
                const float x2 = act_fwd_t<A2>(z2);
                dl = (x2 - ((o16 == label) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
            }
            dl = valid ? dl : 0.f;
            __syncwarp();                          // every lane has read b2s
            if (lane < 16) sm.b2s[warp][lane] = fmaf(-lr, dl, b2o);   // b2(t)
        }
        // ---- δ1, g(t-1) of this lane's unit; W2(t), b1(t) ----
        {
            const float d0 = __shfl_sync(0xffffffffu, dl, tq);
            const float d1 = __shfl_sync(0xffffffffu, dl, tq + 4);
            const float d2 = __shfl_sync(0xffffffffu, dl, tq + 8);     // 0 for o = 10, 11
            float s1 = fmaf(w2[2], d2, fmaf(w2[1], d1, w2[0] * d0));  // (W2ᵀδ2)_k, pre-update W2 (R6)
            s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
            s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
            const float gnew = tlive ? lr * (s1 * act_deriv_t<A1>(hprev)) : 0.f;   // g(t-1) = η δ1
            w2[0] = fmaf(-(lr * d0), hprev, w2[0]);                     // W2(t)
            w2[1] = fmaf(-(lr * d1), hprev, w2[1]);
            w2[2] = fmaf(-(lr * d2), hprev, w2[2]);
            b1 -= gnew;                            // b1(t)
            gm2 = gm1;
            gm1 = gnew;
            if (tq == 0) gs.gw[(t + 1) & 1][wl][tr] = gnew;   // g(t-1), swept in U(t+1)
        }
        TR(4);
        // ---- sample t: z1 = acc - g(t-2)G(t-2,t) - g(t-1)G(t-1,t) + b1(t); h; partial logits ----
        if (t < T) {
            const float2 G = *reinterpret_cast<const float2*>(xring + sx * DP + GOFF);
            const float z1 = fmaf(-gm1, G.y, fmaf(-gm2, G.x, a)) + b1;
            const float h = tlive ? act_fwd_t<A1>(z1) : 0.f;
            hprev = h;
            float pv[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                pv[i] = w2[i] * h;
                pv[i] += __shfl_xor_sync(0xffffffffu, pv[i], 4);
                pv[i] += __shfl_xor_sync(0xffffffffu, pv[i], 8);
                pv[i] += __shfl_xor_sync(0xffffffffu, pv[i], 16);
            }
            const uint32_t zrow = (uint32_t)(crank * NWG + wl);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int o = lane + 4 * i;
                const bool pub = lane < 4 && o < O;
                if (pub) gs.zbuf[sz][zrow][o] = pv[i];
                if constexpr (C > 1) {
#pragma unroll
                    for (int p = 0; p < C - 1; ++p)
                        st_async_f32_if(pub, rz[p] + sz * kZStride + o * 4, pv[i],
                                        rz[p] + kZfullOff - zrow * 64u + sz * 8);
                }
            }
            // certify x(t+2) (and its Gram terms) for step t+2's F through zfull(t)
            if (wl == 0 && t + 2 < T) {
                const int s2 = (sx + 2 >= S) ? sx + 2 - S : sx + 2;
                mbar_wait(&gs.xfull[s2], (sx + 2 >= S) ? (xpar ^ 1u) : xpar);
            }
            __syncwarp();
            if (lane == 0) {
                if constexpr (C > 1) mbar_arrive_expect_tx(&gs.zfull[sz], (uint32_t)((C - 1) * O * 4));
                else mbar_arrive(&gs.zfull[sz]);
            }
        }
        TR(5);
        if (++sx == S) { sx = 0; xpar ^= 1u; }
        pz = sz;
        ppar = zpar;
        if (++sz == ZS) { sz = 0; zpar ^= 1u; }
    }
#undef TR

    // ---- write back ----
    if (active) {
        float* W1o = opaque(W1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (kr0 + r < Uown) {
                float* dst = W1o + (long long)(k0 + kr0 + r) * D;
#pragma unroll
                for (int m = 0; m < NP; ++m) *reinterpret_cast<uint64_t*>(dst + pcol(lane, m)) = w[r][m];
            }
        }
        if (tlive) {
            const float4 w4 = *reinterpret_cast<const float4*>(wxp);
            float* dst = W1o + (long long)ku * D + XC + 4 * tq;
            if (nx > 0) dst[0] = w4.x;
            if (nx > 1) dst[1] = w4.y;
            if (nx > 2) dst[2] = w4.z;
            if (nx > 3) dst[3] = w4.w;
            float* W2o = opaque(W2);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int o = tq + 4 * i;
                if (o < O) W2o[(long long)o * H + ku] = w2[i];
            }
            if (tq == 0) opaque(b1g)[ku] = b1;
        }
        if (crank == 0 && wl == 0 && lane < O) opaque(b2g)[lane] = sm.b2s[warp][lane];
    }
    __syncthreads();
    if constexpr (C > 1) cluster_sync_all();       // no CTA leaves while a peer may still st.async into it
}

template <int C, int NG, int A1, int A2, bool TRACE>
cudaError_t launch_one(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                       const int32_t* labels, float4* gram, long long n_local, int K_local, int s_first,
                       int s_count, float lr, cudaStream_t st) {
    auto kern = sgd_resident_kernel<C, NG, A1, A2, TRACE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    const int clusters = (s_count + NG - 1) / NG;
    cfg.gridDim = dim3((unsigned)(clusters * C));
    cfg.blockDim = dim3((unsigned)p.threads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, d, children, x, labels, (const float4*)gram, n_local, K_local,
                              s_first, s_count, lr, g_trace);
}

template <int C, int NG>
cudaError_t launch_cg(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                      const int32_t* labels, float4* gram, long long n_local, int K_local, int s_first,
                      int s_count, float lr, cudaStream_t st) {
#define PNN_ACTS(A1_, A2_)                                                                        \
    if (d.act[0] == A1_ && d.act[1] == A2_)                                                     \
        return g_trace ? launch_one<C, NG, A1_, A2_, true>(p, d, children, x, labels, gram, n_local, K_local, \
                                                           s_first, s_count, lr, st)              \
                       : launch_one<C, NG, A1_, A2_, false>(p, d, children, x, labels, gram, n_local, K_local, \
                                                            s_first, s_count, lr, st);
    PNN_ACTS(PNN_RELU, PNN_SOFTMAX)
    PNN_ACTS(PNN_TANH, PNN_SOFTMAX)
    PNN_ACTS(PNN_SIGMOID, PNN_SOFTMAX)
    PNN_ACTS(PNN_SIGMOID, PNN_SIGMOID)
    PNN_ACTS(PNN_TANH, PNN_TANH)
    PNN_ACTS(PNN_RELU, PNN_SIGMOID)
#undef PNN_ACTS
    return cudaErrorInvalidValue;
}

}  // namespace

ResidentPlan plan_resident(const NetDesc& d, int batch) {
    ResidentPlan p{};
    auto no = [&](const char* why) {
        p.ok = false;
        snprintf(p.why, sizeof p.why, "%s", why);
        return p;
    };
    if (batch != 1) return no("mini-batch runs on the reference kernel");
    if (d.L != 2) return no("resident kernel covers 2-layer nets (D-H-O)");
    const int D = d.n[0], H = d.n[1], Od = d.n[2];
    if (D % 4 != 0) return no("input width must be a multiple of 4 (16-byte bulk copies)");
    if (D > XC + 16 || D <= XC) return no("built for 768 < inputs <= 784 (6 column quads per lane + 16 columns in shared memory)");
    if (Od != O) return no("built for 10 outputs");
    if (d.P % 2 != 0) return no("odd parameter count (W1 rows are moved as 8-byte pairs)");
    const int a1 = d.act[0], a2 = d.act[1];
    const bool built = (a1 == PNN_RELU && a2 == PNN_SOFTMAX) || (a1 == PNN_TANH && a2 == PNN_SOFTMAX) ||
                       (a1 == PNN_SIGMOID && a2 == PNN_SOFTMAX) || (a1 == PNN_SIGMOID && a2 == PNN_SIGMOID) ||
                       (a1 == PNN_TANH && a2 == PNN_TANH) || (a1 == PNN_RELU && a2 == PNN_SIGMOID);
    if (!built) return no("activation pair not instantiated in the resident kernel");
    // groups per CTA: PNN_RESIDENT_GROUPS=2 puts two CNs on every SM (cluster twice as wide)
    const char* env = getenv("PNN_RESIDENT_GROUPS");
    int ng = (env && atoi(env) == 2) ? 2 : 1;
    int c = 1;
    while (c <= CMAX && (H + c - 1) / c > R * (NWMAX / ng)) c *= 2;
    if (c > CMAX && ng == 2) {                     // too wide for two groups: one group per CTA
        ng = 1;
        c = 1;
        while (c <= CMAX && (H + c - 1) / c > R * NWMAX) c *= 2;
    }
    if (c > CMAX) return no("hidden layer wider than 256");
    const int U = (H + c - 1) / c;
    p.cluster = c;
    p.groups = ng;
    (void)U;
    p.threads = NWMAX * 32;                        // NWMAX/ng warps per group; rows >= U are idle
    p.smem = kSmemHead + sizeof(float) * (size_t)ng * (S + 1) * DP;
    p.variant = 7;
    p.ok = true;
    return p;
}

cudaError_t launch_sgd_resident(const ResidentPlan& p, const NetDesc& d, float* children,
                                const float* x, const int32_t* labels, float4* gram, long long n_local,
                                int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    gram_kernel<<<592, 256, 0, st>>>(x, d.n[0], n_local, K_local, s_first, s_count, gram);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    switch (p.cluster * 10 + p.groups) {
    case 11: return launch_cg<1, 1>(p, d, children, x, labels, gram, n_local, K_local, s_first, s_count, lr, st);
    case 21: return launch_cg<2, 1>(p, d, children, x, labels, gram, n_local, K_local, s_first, s_count, lr, st);
    case 41: return launch_cg<4, 1>(p, d, children, x, labels, gram, n_local, K_local, s_first, s_count, lr, st);
    case 12: return launch_cg<1, 2>(p, d, children, x, labels, gram, n_local, K_local, s_first, s_count, lr, st);
    case 22: return launch_cg<2, 2>(p, d, children, x, labels, gram, n_local, K_local, s_first, s_count, lr, st);
    case 42: return launch_cg<4, 2>(p, d, children, x, labels, gram, n_local, K_local, s_first, s_count, lr, st);
    default: return cudaErrorInvalidValue;
    }
}
