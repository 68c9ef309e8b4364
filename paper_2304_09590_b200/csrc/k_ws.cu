// k_ws.cu — persistent per-sample SGD, one SM per child network, W¹ in registers + tensor
// memory, warp-specialised: the sweeps and the per-sample chain on different warps (variant
// v12).
//
// A CTA trains one child network (CN) over its whole slice ("Each child-network
// learns only a slice").  Scope: 2-layer nets D-H-O, 768 < D <= 784, H <= 128, O = 10,
// per-sample SGD.  Per sample, in the paper's sequential order (§3,
// Eqs.2-13): z1 = W1 x + b1, h = φ1(z1); z2 = W2 h + b2; δ2 (Eq.10 softmax+CE, or Eq.9 / R11);
// δ1 = (W2ᵀδ2) ⊙ φ1'(h) with the pre-update W2 (R6); W -= η δ xᵀ, b -= η δ (Eqs.12-13).
//
// The R27 lookahead: with W¹(t) the weights before sample t's update and
// g(s) = η δ1(s),
//     z1(t) = W¹(t-L) x(t) - Σ_{k=1..L} g(t-k)·G(t-k,t) + b1(t),  G(s,t) = x(s)·x(t),
// the paper's pre-activation in real arithmetic; L = 4 for even and 5 for odd samples (paired
// sweeps).  The Gram terms and labels come from gram_kernel's 32-B records.  W¹'s 128 rows sit
// in the register file and tensor memory of ONE SM, as in v11 (k_tmem.cu); what differs is who
// runs the per-sample chain.  In v11 it runs on a rotating pair of the 8 sweep warps, whose
// sweeps stop for the chain's whole latency (period ~4,300 cycles per sample: sweep time plus
// most of a chain).  Here 12 warps in three warpgroups:
//   warps 0-7  (setmaxnreg ↑ kSweepRegs): sweeps only — paired F(2p), F(2p+1) = W¹(2p-4)·x
//              (row sums to shared memory, arrive aready), then U(2p-4), U(2p-3)
//              (W¹ -= g·xᵀ in sample order, after gready);
//   warps 8-11 (setmaxnreg ↓ kChainRegs): the chain of every sample, one hidden unit per
//              thread (u = 32·(warp-8) + lane) with W2[:, u], b1[u] and g(c-1..c-5)[u] in
//              registers; the four warps' partial logits meet through shared memory and a named
//              barrier; lane o < 10 forms z2_o and δ2_o (softmax by shuffles); g(c) goes to shared
//              memory (arrive gready(c)); the chain warps also issue the x bulk copies.
// The sweeps never run chain code and the chain never waits for a sweep except through
// aready(c) (F(c) ran L samples ahead of the chain's need), so the period is max(sweep, chain)
// instead of their sum (C4 0.542 of FP32 FMA peak for this launch).
#include <cstddef>
#include <cstdio>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"
#include "pnn_tmem.cuh"

#ifdef PNN_WS_TRACE
// experiment builds only: clock64 timeline of CTA 0 (tools/trace_ws.py): [i < 256][point < 8]
#define WS_TR(i, pt) do { if (trace && blockIdx.x == 0 && lane == 0 && (i) < 256) trace[(i) * 8 + (pt)] = ptx::clock64(); } while (0)
#else
#define WS_TR(i, pt) do { } while (0)
#endif
extern long long* g_trace;   // debug: clock64 timeline (k_resident.cu; tools/trace_ws.py, PNN_WS_TRACE builds)
namespace {

using namespace ptx;

constexpr int NSW = 8;          // sweep warps (warpgroups 0, 1)
constexpr int NCW = 4;          // chain warps (warpgroup 2)
constexpr int NT = 32 * (NSW + NCW);
constexpr int RPW = 16;         // W¹ rows per sweep warp (8 per half-warp)
constexpr int RW = 8;           // rows per lane (its half-warp's)
constexpr int RR = 3;           // of which in registers
constexpr int TRW = RW - RR;    // and in TMEM
constexpr int UMAX = NSW * RPW; // 128 hidden units
constexpr int NQ = 12;          // column quads per lane (4 columns each, stride 64): columns [0, 768)
constexpr int NP = 2 * NQ;      // f32x2 pairs per lane per row
constexpr int XC = 768;         // first tail column
constexpr int DP = 800;         // x ring slot stride (floats)
constexpr int GOFF = 784;       // the Gram record of x(u) at its ring slot + GOFF
constexpr int LAG = 4;          // lookahead L
constexpr int S = 16;           // x ring slots (+ one zero row at slot S)
constexpr int PF = 8;           // prefetch distance: x(c+PF) issued after chain c
constexpr int O = 10;           // outputs
constexpr int AR = 8;           // row-sum ring slots (> L)
constexpr int GR = 8;           // g ring slots (> L)
constexpr int GT = 8;           // Gram-term ring slots (> L)
constexpr int TQCOLS = 4 * TRW; // TMEM columns per quad
constexpr int TTAIL = NQ * TQCOLS;
// Register budgets per thread.  The launch gives every thread 168 (384 threads, one CTA per
// SM); setmaxnreg moves them between warpgroups: 2·kSweepRegs + kChainRegs <= 3·168.
#ifndef PNN_WS_SWEEP_REGS
#define PNN_WS_SWEEP_REGS 224
#define PNN_WS_CHAIN_REGS 56
#endif
constexpr int kSweepRegs = PNN_WS_SWEEP_REGS;
constexpr int kChainRegs = PNN_WS_CHAIN_REGS;
static_assert(2 * kSweepRegs + kChainRegs <= 3 * 168, "register pool");
static_assert(TTAIL + 8 <= 256, "TMEM half of a lane quadrant");
static_assert(S >= PF + LAG + 4, "x ring: a refilled slot is no longer read");

struct __align__(16) Smem {
    uint64_t xfull[S];          // x(u) landed (bulk copy complete_tx)
    uint64_t aready[AR];        // F(s) of the 8 sweep warps (count NSW)
    uint64_t gready[GR];        // g(c) of every unit in gbuf (count NCW)
    uint32_t tbase;             // TMEM base address
    uint32_t pad[3];
    float asum[AR][UMAX];       // [s % AR][unit] row sums W¹(s-L)·x(s)
    float gbuf[GR][UMAX];       // [c % GR][unit] g(c) = η δ1(c)
    float zp[2][NCW][16];       // [c & 1][chain warp][o] partial logits
    float b2s[2][12];           // b2 before sample c at [c & 1]
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
template <typename T> __device__ __forceinline__ T* opaque(T* p) {
    asm volatile("mov.b64 %0, %0;" : "+l"(p));
    return p;
}
template <int N> __device__ __forceinline__ void setmaxnreg_inc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N> __device__ __forceinline__ void setmaxnreg_dec() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

// 16 values per lane → lane l holds the sum over the warp of value (l >> 1), halves in
// lanes l and l^1 still to be combined.
__device__ __forceinline__ float treduce16(const float (&v)[16], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    float u8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) u8[i] = (b4 ? v[i + 8] : v[i]) + __shfl_xor_sync(0xffffffffu, b4 ? v[i] : v[i + 8], 16);
    float u4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) u4[i] = (b3 ? u8[i + 4] : u8[i]) + __shfl_xor_sync(0xffffffffu, b3 ? u8[i] : u8[i + 4], 8);
    float u2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) u2[i] = (b2 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b2 ? u4[i] : u4[i + 2], 4);
    return (b1 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? u2[0] : u2[1], 2);
}

// The Gram terms and the label come with x(u) through the ring as the 32-B record of gram_kernel
// (k_resident.cu, launch_gram).  (Forming them in the chain warps instead, one sample ahead, made
// the chain the limit: 12.39 ms per C4 epoch against 10.63 + 0.86 ms.)
template <int A1, int A2>
__global__ void __launch_bounds__(NT, 1)
sgd_ws_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X, const int32_t* __restrict__ Y,
              const float4* __restrict__ rec, long long n_local, int K_local, int s_first, float lr,
              long long* __restrict__ trace) {
    extern __shared__ __align__(128) unsigned char smraw[];
    Smem& sm = *reinterpret_cast<Smem*>(smraw);
    float* xring = reinterpret_cast<float*>(smraw + kSmemHead);
    const int D = d.n[0], H = d.n[1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cn = s_first + (int)blockIdx.x;

    long long row0, T64;
    shard_of(n_local, K_local, cn, &row0, &T64);
    const int T = (int)T64;
    float* P = children + (long long)cn * d.P;
    float* W1 = P;
    float* b1g = P + (long long)H * D;
    float* W2 = b1g + H;
    float* b2g = W2 + (long long)O * H;
    const float* Xc = X + row0 * (long long)D;
    const uint32_t xbytes = (uint32_t)D * 4u;

    if (warp == 0) tmem::alloc(&sm.tbase, 512);
    if (threadIdx.x == 32) {
        for (int i = 0; i < S; ++i) mbar_init(&sm.xfull[i], 1);
        for (int i = 0; i < AR; ++i) mbar_init(&sm.aready[i], NSW);
        for (int i = 0; i < GR; ++i) mbar_init(&sm.gready[i], NCW);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < (S + 1) * DP; i += blockDim.x) xring[i] = 0.f;   // + the zero row
    for (int i = threadIdx.x; i < 24; i += blockDim.x) (&sm.b2s[0][0])[i] = (i < O) ? b2g[i] : 0.f;
    fence_proxy_async_smem();
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();

    if (warp < NSW) {
        // ============================== sweep warps ==============================
        // Half-warp layout: lanes 16·hw .. 16·hw+15 (hw = lane >> 4) hold rows kr0 + 8·hw .. +7 of
        // the warp's 16, lane j = lane & 15 the 48 columns 4j + 64q .. +3 (q < 12) of each: RR rows
        // in registers (f32x2 pairs), TRW in TMEM (20 columns per quad), the 16-column tail in TMEM
        // (lane: row 8·hw + (j >> 1), columns 768 + 8·(j & 1) .. +7).  A row's dot product then sums
        // over 16 lanes (a 16-value transpose-reduce per pair of samples) instead of 32.
        setmaxnreg_inc<kSweepRegs>();
        const uint32_t tq = sm.tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2);
        const int hw = lane >> 4, jl = lane & 15;
        const int kr0 = warp * RPW;                     // the warp's first row
        const int kh = kr0 + RW * hw;                   // this lane's first row
        const int cl = 4 * jl;                          // this lane's first column
        uint64_t w[RR][NP];
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            const bool live = kh + r < H;
            const float* src = W1 + (long long)(kh + r) * D + cl;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                w[r][2 * q] = live ? *reinterpret_cast<const uint64_t*>(src + 64 * q) : 0ull;
                w[r][2 * q + 1] = live ? *reinterpret_cast<const uint64_t*>(src + 64 * q + 2) : 0ull;
            }
        }
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            uint32_t tv[TQCOLS];
#pragma unroll
            for (int t = 0; t < TRW; ++t) {
                const bool live = kh + RR + t < H;
                const float* src = W1 + (long long)(kh + RR + t) * D + cl + 64 * q;
                // (slabs are 8-byte aligned only: P is even, not a multiple of 4)
                const float2 a = live ? *reinterpret_cast<const float2*>(src) : make_float2(0.f, 0.f);
                const float2 b = live ? *reinterpret_cast<const float2*>(src + 2) : make_float2(0.f, 0.f);
                tv[4 * t] = __float_as_uint(a.x); tv[4 * t + 1] = __float_as_uint(a.y);
                tv[4 * t + 2] = __float_as_uint(b.x); tv[4 * t + 3] = __float_as_uint(b.y);
            }
            tmem::st16(tq + q * TQCOLS, tv);
            tmem::st4(tq + q * TQCOLS + 16, tv + 16);
        }
        const int trow = kh + (jl >> 1), th8 = jl & 1;  // tail: row trow, columns 768 + 8·th8 .. +7
        {
            uint32_t tt[8];
            const bool live = trow < H;
            const float* src = W1 + (long long)trow * D + XC + 8 * th8;
#pragma unroll
            for (int j = 0; j < 8; ++j) tt[j] = __float_as_uint((live && XC + 8 * th8 + j < D) ? src[j] : 0.f);
            tmem::st8(tq + TTAIL, tt);
        }
        tmem::wait_st();

        // Paired sweeps: step p runs F for samples 2p, 2p+1 in one pass over W¹ (both x rows per
        // quad, 4 fma.rn.f32x2 per row per quad), then U for samples 2p-4, 2p-3 (in sample order).
        // F(2p), F(2p+1) see W¹(2p-4): sample 2p misses 4 updates, 2p+1 misses 5 (R27; the chain
        // applies 4 / 5 Gram corrections).
        const int npair = (T + 1) >> 1;
        const int trs = lane & 1;                       // F's reduce: lane ends with (row kh + (jl >> 1), sample lane & 1)
        for (int p = 0; p < npair + 2; ++p) {
            if (warp == 0) WS_TR(p, 4);
            if (p < npair) {
                // ---------------- F(2p), F(2p+1): acc = W¹(2p-4)·x ----------------
                const int s0 = 2 * p, s1 = s0 + 1;
                const bool v1 = s1 < T;
                const int sl0 = s0 % S, sl1 = v1 ? s1 % S : S;   // slot S: the zero row
                mbar_wait(&sm.xfull[sl0], (uint32_t)((s0 / S) & 1));   // (x lands early: no sleep hint)
                if (v1) mbar_wait(&sm.xfull[sl1], (uint32_t)((s1 / S) & 1));
                const float* xn0 = xring + sl0 * DP + cl;
                const float* xn1 = xring + sl1 * DP + cl;
                uint64_t acc0[RW], acc1[RW];
#pragma unroll
                for (int r = 0; r < RW; ++r) { acc0[r] = 0ull; acc1[r] = 0ull; }
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    uint32_t tv[TQCOLS];
                    tmem::ld16(tq + q * TQCOLS, tv);
                    tmem::ld4(tq + q * TQCOLS + 16, tv + 16);
                    uint64_t xa, xb, ya, yb;
                    lds4(xn0 + 64 * q, xa, xb);
                    lds4(xn1 + 64 * q, ya, yb);
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        acc0[r] = ffma2(w[r][2 * q], xa, acc0[r]);
                        acc1[r] = ffma2(w[r][2 * q], ya, acc1[r]);
                        acc0[r] = ffma2(w[r][2 * q + 1], xb, acc0[r]);
                        acc1[r] = ffma2(w[r][2 * q + 1], yb, acc1[r]);
                    }
                    tmem::wait_ld_regs<TQCOLS>(tv);
#pragma unroll
                    for (int t = 0; t < TRW; ++t) {
                        const uint64_t wa = pk(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1]));
                        const uint64_t wb = pk(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3]));
                        acc0[RR + t] = ffma2(wa, xa, acc0[RR + t]);
                        acc1[RR + t] = ffma2(wa, ya, acc1[RR + t]);
                        acc0[RR + t] = ffma2(wb, xb, acc0[RR + t]);
                        acc1[RR + t] = ffma2(wb, yb, acc1[RR + t]);
                    }
                }
                // tail partials of both samples (row trow, 8 columns)
                float pt0, pt1;
                {
                    uint32_t tt[8];
                    tmem::ld8(tq + TTAIL, tt);
                    const float* xt0 = xring + sl0 * DP + XC + 8 * th8;
                    const float* xt1 = xring + sl1 * DP + XC + 8 * th8;
                    const float4 a0 = *reinterpret_cast<const float4*>(xt0), a1 = *reinterpret_cast<const float4*>(xt0 + 4);
                    const float4 c0 = *reinterpret_cast<const float4*>(xt1), c1 = *reinterpret_cast<const float4*>(xt1 + 4);
                    tmem::wait_ld_regs<8>(tt);
                    const float wt[8] = {__uint_as_float(tt[0]), __uint_as_float(tt[1]), __uint_as_float(tt[2]),
                                         __uint_as_float(tt[3]), __uint_as_float(tt[4]), __uint_as_float(tt[5]),
                                         __uint_as_float(tt[6]), __uint_as_float(tt[7])};
                    pt0 = wt[0] * a0.x;
                    pt0 = fmaf(wt[1], a0.y, pt0); pt0 = fmaf(wt[2], a0.z, pt0); pt0 = fmaf(wt[3], a0.w, pt0);
                    pt0 = fmaf(wt[4], a1.x, pt0); pt0 = fmaf(wt[5], a1.y, pt0); pt0 = fmaf(wt[6], a1.z, pt0);
                    pt0 = fmaf(wt[7], a1.w, pt0);
                    pt1 = wt[0] * c0.x;
                    pt1 = fmaf(wt[1], c0.y, pt1); pt1 = fmaf(wt[2], c0.z, pt1); pt1 = fmaf(wt[3], c0.w, pt1);
                    pt1 = fmaf(wt[4], c1.x, pt1); pt1 = fmaf(wt[5], c1.y, pt1); pt1 = fmaf(wt[6], c1.z, pt1);
                    pt1 = fmaf(wt[7], c1.w, pt1);
                }
                // transpose-reduce 16 values v[2r + sample] over the half-warp: lane jl ends with value jl
                float v[2 * RW];
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    float lo, hi;
                    upk(acc0[r], lo, hi);
                    v[2 * r] = lo + hi;
                    upk(acc1[r], lo, hi);
                    v[2 * r + 1] = lo + hi;
                }
                float zsum;
                {
                    const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
                    float u8[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        u8[i] = (b3 ? v[i + 8] : v[i]) + __shfl_xor_sync(0xffffffffu, b3 ? v[i] : v[i + 8], 8);
                    float u4[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        u4[i] = (b2 ? u8[i + 4] : u8[i]) + __shfl_xor_sync(0xffffffffu, b2 ? u8[i] : u8[i + 4], 4);
                    float u2[2];
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        u2[i] = (b1 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b1 ? u4[i] : u4[i + 2], 2);
                    zsum = (b0 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b0 ? u2[0] : u2[1], 1);
                    // + the tail of (row trow, sample lane & 1): this lane's half and the partner's
                    const float other = __shfl_xor_sync(0xffffffffu, trs ? pt0 : pt1, 1);
                    zsum += (trs ? pt1 : pt0) + other;
                }
                if (trs == 0 || v1) sm.asum[(trs ? s1 : s0) % AR][trow] = zsum;
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sm.aready[s0 % AR]);
                    if (v1) mbar_arrive(&sm.aready[s1 % AR]);
                }
                if (warp == 0) WS_TR(p, 5);
            }
            // ---------------- U(2p-4), U(2p-3): W¹ -= g(u)·x(u)ᵀ in sample order ----------------
            if (p >= 2 && 2 * (p - 2) < T) {
                const int u0 = 2 * (p - 2), u1 = u0 + 1;
                const bool v1 = u1 < T;
                const int ul = v1 ? u1 : u0;            // chain u1 done ⇒ chain u0 done
                mbar_wait_sleep(&sm.gready[ul % GR], (uint32_t)((ul / GR) & 1));
                if (warp == 0) WS_TR(p, 6);
                const int sl0 = u0 % S, sl1 = v1 ? u1 % S : S;
                const float* xo0 = xring + sl0 * DP + cl;
                const float* xo1 = xring + sl1 * DP + cl;
                float gn0[RW], gn1[RW];                 // -g of each of this lane's rows, samples u0, u1
                {
                    const float4* g0v = reinterpret_cast<const float4*>(&sm.gbuf[u0 % GR][kh]);
                    const float4* g1v = reinterpret_cast<const float4*>(&sm.gbuf[u1 % GR][kh]);
#pragma unroll
                    for (int i = 0; i < RW / 4; ++i) {
                        const float4 a = g0v[i];
                        float4 b = g1v[i];
                        if (!v1) b = make_float4(0.f, 0.f, 0.f, 0.f);
                        gn0[4 * i] = -a.x; gn0[4 * i + 1] = -a.y; gn0[4 * i + 2] = -a.z; gn0[4 * i + 3] = -a.w;
                        gn1[4 * i] = -b.x; gn1[4 * i + 1] = -b.y; gn1[4 * i + 2] = -b.z; gn1[4 * i + 3] = -b.w;
                    }
                }
#define GP0(r) pk(gn0[r], gn0[r])
#define GP1(r) pk(gn1[r], gn1[r])
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    uint32_t tv[TQCOLS];
                    tmem::ld16(tq + q * TQCOLS, tv);
                    tmem::ld4(tq + q * TQCOLS + 16, tv + 16);
                    uint64_t xa, xb, ya, yb;
                    lds4(xo0 + 64 * q, xa, xb);
                    lds4(xo1 + 64 * q, ya, yb);
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        w[r][2 * q] = ffma2(GP1(r), ya, ffma2(GP0(r), xa, w[r][2 * q]));
                        w[r][2 * q + 1] = ffma2(GP1(r), yb, ffma2(GP0(r), xb, w[r][2 * q + 1]));
                    }
                    tmem::wait_ld_regs<TQCOLS>(tv);
#pragma unroll
                    for (int t = 0; t < TRW; ++t) {
                        const uint64_t a = ffma2(GP1(RR + t), ya, ffma2(GP0(RR + t), xa,
                                                 pk(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1]))));
                        const uint64_t b = ffma2(GP1(RR + t), yb, ffma2(GP0(RR + t), xb,
                                                 pk(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3]))));
                        float a0, a1, b0, b1;
                        upk(a, a0, a1);
                        upk(b, b0, b1);
                        tv[4 * t] = __float_as_uint(a0); tv[4 * t + 1] = __float_as_uint(a1);
                        tv[4 * t + 2] = __float_as_uint(b0); tv[4 * t + 3] = __float_as_uint(b1);
                    }
                    tmem::st16(tq + q * TQCOLS, tv);
                    tmem::st4(tq + q * TQCOLS + 16, tv + 16);
                }
                {
                    uint32_t tt[8];
                    tmem::ld8(tq + TTAIL, tt);
                    const float* xt0 = xring + sl0 * DP + XC + 8 * th8;
                    const float* xt1 = xring + sl1 * DP + XC + 8 * th8;
                    const float4 a0 = *reinterpret_cast<const float4*>(xt0), a1 = *reinterpret_cast<const float4*>(xt0 + 4);
                    const float4 c0 = *reinterpret_cast<const float4*>(xt1), c1 = *reinterpret_cast<const float4*>(xt1 + 4);
                    const float ga = -sm.gbuf[u0 % GR][trow];
                    const float gb = v1 ? -sm.gbuf[u1 % GR][trow] : 0.f;
                    tmem::wait_ld_regs<8>(tt);
                    const float xv[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float yv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        tt[j] = __float_as_uint(fmaf(gb, yv[j], fmaf(ga, xv[j], __uint_as_float(tt[j]))));
                    tmem::st8(tq + TTAIL, tt);
                }
                tmem::wait_st();
                if (warp == 0) WS_TR(p, 7);
#undef GP0
#undef GP1
            }
        }

        // ---- write back this lane's W¹ rows (registers, TMEM, tail) ----
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            if (kh + r < H) {
                float* dst = opaque(W1) + (long long)(kh + r) * D + cl;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    *reinterpret_cast<uint64_t*>(dst + 64 * q) = w[r][2 * q];
                    *reinterpret_cast<uint64_t*>(dst + 64 * q + 2) = w[r][2 * q + 1];
                }
            }
        }
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            uint32_t tv[TQCOLS];
            tmem::ld16(tq + q * TQCOLS, tv);
            tmem::ld4(tq + q * TQCOLS + 16, tv + 16);
            tmem::wait_ld_regs<TQCOLS>(tv);
#pragma unroll
            for (int t = 0; t < TRW; ++t) {
                if (kh + RR + t < H) {
                    float* dst = opaque(W1) + (long long)(kh + RR + t) * D + cl + 64 * q;
                    *reinterpret_cast<float2*>(dst) = make_float2(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1]));
                    *reinterpret_cast<float2*>(dst + 2) =
                        make_float2(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3]));
                }
            }
        }
        {
            uint32_t tt[8];
            tmem::ld8(tq + TTAIL, tt);
            tmem::wait_ld_regs<8>(tt);
            if (trow < H) {
                float* dst = opaque(W1) + (long long)trow * D + XC + 8 * th8;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (XC + 8 * th8 + j < D) dst[j] = __uint_as_float(tt[j]);
            }
        }
    } else {
        // ============================== chain warps ==============================
        setmaxnreg_dec<kChainRegs>();
        const int cw = warp - NSW;                  // chain warp 0..3
        const int u = 32 * cw + lane;               // this thread's hidden unit
        const bool lc = u < H;
        const bool leader = threadIdx.x == 32 * NSW;
        float w2[O];                                // W2[:, u]
#pragma unroll
        for (int o = 0; o < O; ++o) w2[o] = lc ? W2[(long long)o * H + u] : 0.f;
        float b1 = lc ? b1g[u] : 0.f;
        float g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f, g5 = 0.f;   // g(c-1) .. g(c-5) of this unit
        const float4* Rc = rec + 2 * row0;
        auto issue_x = [&](int s) {
            uint64_t* bar = &sm.xfull[s % S];
            mbar_arrive_expect_tx(bar, xbytes + 32u);
            bulk_g2s(xring + (s % S) * DP, Xc + (long long)s * D, xbytes, bar);
            bulk_g2s(xring + (s % S) * DP + GOFF, Rc + 2 * s, 32u, bar);
        };
        if (leader)
            for (int s = 0; s < PF && s < T; ++s) issue_x(s);
        for (int c = 0; c < T; ++c) {
            // ---- z1(c) = acc - Σ_k g(c-k) G(c-k,c) + b1(c), h(c) ----
            if (cw == 0) WS_TR(c, 0);
            mbar_wait_sleep(&sm.xfull[c % S], (uint32_t)((c / S) & 1));   // x(c)'s record
            mbar_wait_sleep(&sm.aready[c % AR], (uint32_t)((c / AR) & 1));
            if (cw == 0) WS_TR(c, 1);
            float G[5];                             // G(c-k, c), k = 1..5
            int lab0;
            {                                       // {G(c-4), G(c-3), G(c-2), G(c-1)}, {label, G(c-5)}
                const float4 r0 = *reinterpret_cast<const float4*>(xring + (c % S) * DP + GOFF);
                const float2 r1 = *reinterpret_cast<const float2*>(xring + (c % S) * DP + GOFF + 4);
                G[0] = r0.w; G[1] = r0.z; G[2] = r0.y; G[3] = r0.x; G[4] = r1.y;
                lab0 = __float_as_int(r1.x);
            }
            float z = sm.asum[c % AR][u];
            if (c & 1) z = fmaf(-g5, G[4], z);
            z = fmaf(-g4, G[3], z);
            z = fmaf(-g3, G[2], z);
            z = fmaf(-g2, G[1], z);
            z = fmaf(-g1, G[0], z);
            z += b1;
            const float h = lc ? act_fwd_t<A1>(z) : 0.f;
            // ---- this warp's partial logits Σ_u W2[o][u] h_u ----
            {
                float pv[16];
#pragma unroll
                for (int o = 0; o < 16; ++o) pv[o] = (o < O) ? w2[o < O ? o : 0] * h : 0.f;
                float p0 = treduce16(pv, lane);
                p0 += __shfl_xor_sync(0xffffffffu, p0, 1);
                if ((lane & 1) == 0 && (lane >> 1) < O) sm.zp[c & 1][cw][lane >> 1] = p0;
            }
            named_bar_sync(1, 32 * NCW);            // the four warps' partials of sample c
            if (cw == 0) WS_TR(c, 2);
            // ---- δ2(c): lane o < 10 of every chain warp forms z2_o and its share of the softmax /
            //      φ2, then every lane takes the ten δ2 by shuffles ----
            float dl[O];
            const int ol = lane < O ? lane : 0;
            const float b2o = sm.b2s[c & 1][ol];    // b2(c)_o
            {
                const float z2 = ((sm.zp[c & 1][0][ol] + sm.zp[c & 1][1][ol]) +
                                  (sm.zp[c & 1][2][ol] + sm.zp[c & 1][3][ol])) + b2o;   // z2 = W2 h + b2 (Eq.2)
                float dmine;
                if constexpr (A2 == PNN_SOFTMAX) {
                    float m = lane < O ? z2 : -INFINITY;
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                    const float ez = lane < O ? __expf(z2 - m) : 0.f;
                    float sum = ez;
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    float inv;
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(sum));
                    dmine = ez * inv - ((lane == lab0) ? 1.f : 0.f);
                } else {
                    // element-wise output (sigmoid / tanh, ½-SSE: Eq.9, R11)
                    const float x2 = act_fwd_t<A2>(z2);
                    dmine = (x2 - ((lane == lab0) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
                }
#pragma unroll
                for (int o = 0; o < O; ++o) dl[o] = __shfl_sync(0xffffffffu, dmine, o);
                // b2(c+1) into the other buffer (the other warps may still read b2(c)): warp 0, lanes < 10
                if (cw == 0 && lane < O) sm.b2s[(c + 1) & 1][lane] = fmaf(-lr, dmine, b2o);
            }
            // ---- δ1, g(c) → the sweeps; W2, b1, b2 updates ----
            float s1 = 0.f;                         // (W2ᵀδ2)_u with the pre-update W2 (R6)
#pragma unroll
            for (int o = 0; o < O; ++o) s1 = fmaf(w2[o], dl[o], s1);
            const float gu = lc ? lr * (s1 * act_deriv_t<A1>(h)) : 0.f;
            sm.gbuf[c % GR][u] = gu;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.gready[c % GR]);
            if (cw == 0) WS_TR(c, 3);
            b1 -= gu;
#pragma unroll
            for (int o = 0; o < O; ++o) w2[o] = fmaf(-(lr * dl[o]), h, w2[o]);
            g5 = g4; g4 = g3; g3 = g2; g2 = g1; g1 = gu;
            if (leader) {
                // every sweep warp passed U(c-1-L) (aready(c)) and every chain warp is past its
                // Gram read of x(c-3): the slot of x(c+PF-S) is free
                if (c + PF < T) issue_x(c + PF);
            }
        }
        if (lc) {
#pragma unroll
            for (int o = 0; o < O; ++o) opaque(W2)[(long long)o * H + u] = w2[o];
            opaque(b1g)[u] = b1;
        }
    }
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    if (warp == 0) tmem::dealloc(sm.tbase, 512);
    if (threadIdx.x == 32 * NSW && T >= 0) {
#pragma unroll
        for (int o = 0; o < O; ++o) opaque(b2g)[o] = sm.b2s[T & 1][o];
    }
}

template <int A1, int A2>
cudaError_t launch_one(const NetDesc& d, float* children, const float* x, const int32_t* y, const float4* rec,
                       long long n_local, int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    if (!rec) return cudaErrorInvalidValue;        // the Gram records of launch_gram are required
    auto kern = sgd_ws_kernel<A1, A2>;
    const size_t smem = kSmemHead + sizeof(float) * (size_t)(S + 1) * DP;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<s_count, NT, smem, st>>>(d, children, x, y, rec, n_local, K_local, s_first, lr, g_trace);
    return cudaGetLastError();
}

}  // namespace

const char* ws_plan(const NetDesc& d, int batch) {
    if (batch != 1) return "per-sample SGD only";
    if (d.L != 2) return "2-layer nets (D-H-O) only";
    const int D = d.n[0], H = d.n[1];
    if (D % 4 != 0 || D <= XC || D > XC + 16) return "built for 768 < inputs <= 784, inputs % 4 == 0";
    if (H > UMAX) return "hidden layer wider than 128";
    if (d.n[2] != O) return "built for 10 outputs";
    if (d.P % 2 != 0) return "odd parameter count (W1 rows are moved as 8-byte pairs)";
    const int a1 = d.act[0], a2 = d.act[1];
    const bool built = (a1 == PNN_RELU && a2 == PNN_SOFTMAX) || (a1 == PNN_TANH && a2 == PNN_SOFTMAX) ||
                       (a1 == PNN_SIGMOID && a2 == PNN_SOFTMAX) || (a1 == PNN_SIGMOID && a2 == PNN_SIGMOID) ||
                       (a1 == PNN_TANH && a2 == PNN_TANH) || (a1 == PNN_RELU && a2 == PNN_SIGMOID) ||
                       (a1 == PNN_LEAKY_RELU && a2 == PNN_SOFTMAX);
    if (!built) return "activation pair not instantiated";
    return nullptr;
}

cudaError_t launch_sgd_ws(const NetDesc& d, float* children, const float* x, const int32_t* y, const float4* rec,
                          long long n_local, int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
#define PNN_ACTS(A1_, A2_) \
    if (d.act[0] == A1_ && d.act[1] == A2_) return launch_one<A1_, A2_>(d, children, x, y, rec, n_local, K_local, s_first, s_count, lr, st);
    PNN_ACTS(PNN_RELU, PNN_SOFTMAX)
    PNN_ACTS(PNN_TANH, PNN_SOFTMAX)
    PNN_ACTS(PNN_SIGMOID, PNN_SOFTMAX)
    PNN_ACTS(PNN_SIGMOID, PNN_SIGMOID)
    PNN_ACTS(PNN_TANH, PNN_TANH)
    PNN_ACTS(PNN_RELU, PNN_SIGMOID)
    PNN_ACTS(PNN_LEAKY_RELU, PNN_SOFTMAX)
#undef PNN_ACTS
    return cudaErrorInvalidValue;
}
