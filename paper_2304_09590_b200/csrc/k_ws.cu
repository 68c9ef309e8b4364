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
// Same data layout and L = 4 lookahead as v11 (k_tmem.cu, R27):
//     z1(t) = W¹(t-L) x(t) - Σ_{k=1..L} g(t-k)·G(t-k,t) + b1(t),  G(s,t) = x(s)·x(t),
// with W¹'s 128 rows split between the register file (6 rows per sweep warp) and tensor
// memory (10 rows per sweep warp + the 16-column tail).  What differs is who runs the chain.
// In v11 the chain of sample c runs on a rotating pair of the 8 sweep warps, whose sweeps
// stop for the chain's whole latency: measured, the per-sample period (~4,300 cycles) was the
// sweep time plus most of a chain.  Here 12 warps in three warpgroups:
//   warps 0-7  (setmaxnreg ↑ kSweepRegs): sweeps only — F(s) = W¹(s-L)·x(s) (row sums to
//              shared memory, arrive aready(s)), U(s) = W¹ -= g(s-L)·x(s-L)ᵀ (wait gready(s-L));
//   warps 8-11 (setmaxnreg ↓ kChainRegs): the chain of every sample, one hidden unit per
//              thread (u = 32·(warp-8) + lane) with W2[:, u], b1[u] and g(c-1..c-4)[u] in
//              registers; the four warps' partial logits meet through shared memory and a named
//              barrier; g(c) goes to shared memory (arrive gready(c)).  The chain warps also
//              form the Gram terms G(c+1-k, c+1) (warp k-1) one sample ahead, stage the labels
//              and issue the x bulk copies.
// The sweeps never run chain code and the chain never waits for a sweep except through
// aready(c) (whose F(c) ran L samples ahead of the chain's need), so the period is
// max(sweep, chain) instead of their sum.
#include <cstddef>
#include <cstdio>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"
#include "pnn_tmem.cuh"

namespace {

using namespace ptx;

constexpr int NSW = 8;          // sweep warps (warpgroups 0, 1)
constexpr int NCW = 4;          // chain warps (warpgroup 2)
constexpr int NT = 32 * (NSW + NCW);
constexpr int RR = 5;           // W¹ rows per sweep warp in registers
constexpr int TR = 10;          // W¹ rows per sweep warp in TMEM
constexpr int SR = RR + TR;     // the warp's row in shared memory (its last row)
constexpr int RPW = RR + TR + 1;// rows per sweep warp
constexpr int UMAX = NSW * RPW; // 128 hidden units
constexpr int NQ = 6;           // column quads per lane: columns [0, 768)
constexpr int NP = 2 * NQ;      // f32x2 pairs per lane per row
constexpr int XC = 768;         // first tail column
constexpr int DP = 800;         // x ring slot stride (floats)
constexpr int LAG = 4;          // lookahead L
constexpr int S = 16;           // x ring slots (+ one zero row at slot S)
constexpr int PF = 8;           // prefetch distance: x(c+PF) issued after chain c
constexpr int O = 10;           // outputs
constexpr int AR = 8;           // row-sum ring slots (> L)
constexpr int GR = 8;           // g ring slots (> L)
constexpr int GT = 4;           // Gram-term ring slots
constexpr int TQCOLS = 4 * TR;  // TMEM columns per quad
constexpr int TTAIL = NQ * TQCOLS;
// Register budgets per thread.  The launch gives every thread 168 (384 threads, one CTA per
// SM); setmaxnreg moves them between warpgroups: 2·kSweepRegs + kChainRegs <= 3·168.
constexpr int kSweepRegs = 224;
constexpr int kChainRegs = 56;
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
    float gterm[GT][4];         // [s % GT][k-1] G(s-k, s)
    float b2s[2][12];           // b2 before sample c at [c & 1]
    float4 wsm[NSW][NQ][32];    // [warp][quad][lane] columns 4·lane + 128·quad .. +3 of row SR
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
__device__ __forceinline__ int pcol(int l, int j) { return 4 * l + 128 * (j >> 1) + 2 * (j & 1); }
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

template <int A1, int A2>
__global__ void __launch_bounds__(NT, 1)
sgd_ws_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X, const int32_t* __restrict__ Y,
              long long n_local, int K_local, int s_first, float lr) {
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
    const int32_t* Yc = Y + row0;
    const uint32_t xbytes = (uint32_t)D * 4u;

    if (warp == 0) tmem::alloc(&sm.tbase, 512);
    if (threadIdx.x == 32) {
        for (int i = 0; i < S; ++i) mbar_init(&sm.xfull[i], 1);
        for (int i = 0; i < AR; ++i) mbar_init(&sm.aready[i], NSW);
        for (int i = 0; i < GR; ++i) mbar_init(&sm.gready[i], NCW);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < (S + 1) * DP; i += blockDim.x) xring[i] = 0.f;   // + the zero row
    for (int i = threadIdx.x; i < GT * 4; i += blockDim.x) (&sm.gterm[0][0])[i] = 0.f;   // G(·, 0) = 0
    for (int i = threadIdx.x; i < 24; i += blockDim.x) (&sm.b2s[0][0])[i] = (i < O) ? b2g[i] : 0.f;
    fence_proxy_async_smem();
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();

    if (warp < NSW) {
        // ============================== sweep warps ==============================
        setmaxnreg_inc<kSweepRegs>();
        const uint32_t tq = sm.tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2);
        const int kr0 = warp * RPW;
        uint64_t w[RR][NP];
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            const bool live = kr0 + r < H;
            const float* src = W1 + (long long)(kr0 + r) * D;
#pragma unroll
            for (int m = 0; m < NP; ++m) w[r][m] = live ? *reinterpret_cast<const uint64_t*>(src + pcol(lane, m)) : 0ull;
        }
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            uint32_t tv[TQCOLS];
#pragma unroll
            for (int t = 0; t < TR; ++t) {
                const bool live = kr0 + RR + t < H;
                const float* src = W1 + (long long)(kr0 + RR + t) * D + 4 * lane + 128 * q;
                // (slabs are 8-byte aligned only: P is even, not a multiple of 4)
                const float2 a = live ? *reinterpret_cast<const float2*>(src) : make_float2(0.f, 0.f);
                const float2 b = live ? *reinterpret_cast<const float2*>(src + 2) : make_float2(0.f, 0.f);
                tv[4 * t] = __float_as_uint(a.x); tv[4 * t + 1] = __float_as_uint(a.y);
                tv[4 * t + 2] = __float_as_uint(b.x); tv[4 * t + 3] = __float_as_uint(b.y);
            }
            tmem::st32(tq + q * TQCOLS, tv);
            tmem::st8(tq + q * TQCOLS + 32, tv + 32);
        }
        {
            const bool live = kr0 + SR < H;
            const float* src = W1 + (long long)(kr0 + SR) * D + 4 * lane;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float2 a = live ? *reinterpret_cast<const float2*>(src + 128 * q) : make_float2(0.f, 0.f);
                const float2 b = live ? *reinterpret_cast<const float2*>(src + 128 * q + 2) : make_float2(0.f, 0.f);
                sm.wsm[warp][q][lane] = make_float4(a.x, a.y, b.x, b.y);
            }
        }
        const int trow = lane >> 1, th8 = lane & 1;     // tail: row kr0 + trow, columns 768 + 8·th8 .. +7
        {
            uint32_t tt[8];
            const bool live = kr0 + trow < H;
            const float* src = W1 + (long long)(kr0 + trow) * D + XC + 8 * th8;
#pragma unroll
            for (int j = 0; j < 8; ++j) tt[j] = __float_as_uint((live && XC + 8 * th8 + j < D) ? src[j] : 0.f);
            tmem::st8(tq + TTAIL, tt);
        }
        tmem::wait_st();

        for (int s = 0; s < T + LAG; ++s) {
            if (s < T) {
                // ---------------- F(s): acc = W¹(s-L)·x(s) ----------------
                const int sl = s % S;
                mbar_wait(&sm.xfull[sl], (uint32_t)((s / S) & 1));
                const float* xn = xring + sl * DP + 4 * lane;
                uint64_t acc[RPW];
#pragma unroll
                for (int r = 0; r < RPW; ++r) acc[r] = 0ull;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    uint32_t tv[TQCOLS];
                    tmem::ld32(tq + q * TQCOLS, tv);
                    tmem::ld8(tq + q * TQCOLS + 32, tv + 32);
                    uint64_t xa, xb;
                    lds4(xn + 128 * q, xa, xb);
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        acc[r] = ffma2(w[r][2 * q], xa, acc[r]);
                        acc[r] = ffma2(w[r][2 * q + 1], xb, acc[r]);
                    }
                    {
                        const ulonglong2 ws = *reinterpret_cast<const ulonglong2*>(&sm.wsm[warp][q][lane]);
                        acc[SR] = ffma2(ws.x, xa, acc[SR]);
                        acc[SR] = ffma2(ws.y, xb, acc[SR]);
                    }
                    tmem::wait_ld_regs<TQCOLS>(tv);
#pragma unroll
                    for (int t = 0; t < TR; ++t) {
                        acc[RR + t] = ffma2(pk(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1])), xa, acc[RR + t]);
                        acc[RR + t] = ffma2(pk(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3])), xb,
                                            acc[RR + t]);
                    }
                }
                float px;
                {
                    uint32_t tt[8];
                    tmem::ld8(tq + TTAIL, tt);
                    const float* xt = xring + sl * DP + XC + 8 * th8;
                    const float4 x0 = *reinterpret_cast<const float4*>(xt), x1 = *reinterpret_cast<const float4*>(xt + 4);
                    tmem::wait_ld_regs<8>(tt);
                    px = __uint_as_float(tt[0]) * x0.x;
                    px = fmaf(__uint_as_float(tt[1]), x0.y, px); px = fmaf(__uint_as_float(tt[2]), x0.z, px);
                    px = fmaf(__uint_as_float(tt[3]), x0.w, px); px = fmaf(__uint_as_float(tt[4]), x1.x, px);
                    px = fmaf(__uint_as_float(tt[5]), x1.y, px); px = fmaf(__uint_as_float(tt[6]), x1.z, px);
                    px = fmaf(__uint_as_float(tt[7]), x1.w, px);
                }
                float v[RPW];
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
                    float lo, hi;
                    upk(acc[r], lo, hi);
                    v[r] = lo + hi;
                }
                float zsum = treduce16(v, lane) + px;
                zsum += __shfl_xor_sync(0xffffffffu, zsum, 1);
                if (th8 == 0) sm.asum[s % AR][kr0 + trow] = zsum;
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.aready[s % AR]);
            }
            // ---------------- U(s-L): W¹ -= g(s-L)·x(s-L)ᵀ ----------------
            const int uu = s - LAG;
            if (uu >= 0 && uu < T) {
                mbar_wait(&sm.gready[uu % GR], (uint32_t)((uu / GR) & 1));
                const float* xo = xring + (uu % S) * DP + 4 * lane;
                uint64_t gp[RPW];                   // (-g, -g) of each row
                {
                    const float4* gv = reinterpret_cast<const float4*>(&sm.gbuf[uu % GR][kr0]);
#pragma unroll
                    for (int i = 0; i < RPW / 4; ++i) {
                        const float4 a = gv[i];
                        gp[4 * i] = pk(-a.x, -a.x); gp[4 * i + 1] = pk(-a.y, -a.y);
                        gp[4 * i + 2] = pk(-a.z, -a.z); gp[4 * i + 3] = pk(-a.w, -a.w);
                    }
                }
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    uint32_t tv[TQCOLS];
                    tmem::ld32(tq + q * TQCOLS, tv);
                    tmem::ld8(tq + q * TQCOLS + 32, tv + 32);
                    uint64_t xa, xb;
                    lds4(xo + 128 * q, xa, xb);
#pragma unroll
                    for (int r = 0; r < RR; ++r) {
                        w[r][2 * q] = ffma2(gp[r], xa, w[r][2 * q]);
                        w[r][2 * q + 1] = ffma2(gp[r], xb, w[r][2 * q + 1]);
                    }
                    {
                        ulonglong2* wp = reinterpret_cast<ulonglong2*>(&sm.wsm[warp][q][lane]);
                        ulonglong2 ws = *wp;
                        ws.x = ffma2(gp[SR], xa, ws.x);
                        ws.y = ffma2(gp[SR], xb, ws.y);
                        *wp = ws;
                    }
                    tmem::wait_ld_regs<TQCOLS>(tv);
#pragma unroll
                    for (int t = 0; t < TR; ++t) {
                        const uint64_t gg = gp[RR + t];
                        const uint64_t a = ffma2(gg, xa, pk(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1])));
                        const uint64_t b = ffma2(gg, xb, pk(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3])));
                        float a0, a1, b0, b1;
                        upk(a, a0, a1);
                        upk(b, b0, b1);
                        tv[4 * t] = __float_as_uint(a0); tv[4 * t + 1] = __float_as_uint(a1);
                        tv[4 * t + 2] = __float_as_uint(b0); tv[4 * t + 3] = __float_as_uint(b1);
                    }
                    tmem::st32(tq + q * TQCOLS, tv);
                    tmem::st8(tq + q * TQCOLS + 32, tv + 32);
                }
                {
                    uint32_t tt[8];
                    tmem::ld8(tq + TTAIL, tt);
                    const float* xt = xring + (uu % S) * DP + XC + 8 * th8;
                    const float4 x0 = *reinterpret_cast<const float4*>(xt), x1 = *reinterpret_cast<const float4*>(xt + 4);
                    const float gt = -sm.gbuf[uu % GR][kr0 + trow];
                    tmem::wait_ld_regs<8>(tt);
                    const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                    for (int j = 0; j < 8; ++j) tt[j] = __float_as_uint(fmaf(gt, xv[j], __uint_as_float(tt[j])));
                    tmem::st8(tq + TTAIL, tt);
                }
                tmem::wait_st();
            }
        }

        // ---- write back this warp's W¹ rows (registers, TMEM, tail) ----
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            if (kr0 + r < H) {
                float* dst = opaque(W1) + (long long)(kr0 + r) * D;
#pragma unroll
                for (int m = 0; m < NP; ++m) *reinterpret_cast<uint64_t*>(dst + pcol(lane, m)) = w[r][m];
            }
        }
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            uint32_t tv[TQCOLS];
            tmem::ld32(tq + q * TQCOLS, tv);
            tmem::ld8(tq + q * TQCOLS + 32, tv + 32);
            tmem::wait_ld_regs<TQCOLS>(tv);
#pragma unroll
            for (int t = 0; t < TR; ++t) {
                if (kr0 + RR + t < H) {
                    float* dst = opaque(W1) + (long long)(kr0 + RR + t) * D + 4 * lane + 128 * q;
                    *reinterpret_cast<float2*>(dst) = make_float2(__uint_as_float(tv[4 * t]), __uint_as_float(tv[4 * t + 1]));
                    *reinterpret_cast<float2*>(dst + 2) =
                        make_float2(__uint_as_float(tv[4 * t + 2]), __uint_as_float(tv[4 * t + 3]));
                }
            }
        }
        if (kr0 + SR < H) {
            float* dst = opaque(W1) + (long long)(kr0 + SR) * D + 4 * lane;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float4 v4 = sm.wsm[warp][q][lane];
                *reinterpret_cast<float2*>(dst + 128 * q) = make_float2(v4.x, v4.y);
                *reinterpret_cast<float2*>(dst + 128 * q + 2) = make_float2(v4.z, v4.w);
            }
        }
        {
            uint32_t tt[8];
            tmem::ld8(tq + TTAIL, tt);
            tmem::wait_ld_regs<8>(tt);
            if (kr0 + trow < H) {
                float* dst = opaque(W1) + (long long)(kr0 + trow) * D + XC + 8 * th8;
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
        float g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f;   // g(c-1) .. g(c-4) of this unit
        auto issue_x = [&](int s) {
            uint64_t* bar = &sm.xfull[s % S];
            mbar_arrive_expect_tx(bar, xbytes);
            bulk_g2s(xring + (s % S) * DP, Xc + (long long)s * D, xbytes, bar);
        };
        if (leader)
            for (int s = 0; s < PF && s < T; ++s) issue_x(s);
        int lab0 = (T > 0) ? __ldg(Yc) : 0;          // labels of samples c, c+1
        int lab1 = (T > 1) ? __ldg(Yc + 1) : 0;
        const int gk = cw + 1;                      // this warp's Gram term: G(s-gk, s)
        for (int c = 0; c < T; ++c) {
            const int lab2 = (c + 2 < T) ? __ldg(Yc + c + 2) : 0;
            // ---- G(c+1-k, c+1), k = cw + 1, one sample ahead (R27) ----
            if (c + 1 < T) {
                const int s1 = c + 1;
                mbar_wait(&sm.xfull[s1 % S], (uint32_t)((s1 / S) & 1));
                const float* xa = xring + (s1 % S) * DP + 4 * lane;
                const float* xb = xring + ((s1 - gk >= 0) ? (s1 - gk) % S : S) * DP + 4 * lane;
                uint64_t ga = 0ull;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    uint64_t a0, a1, b0, b1v;
                    lds4(xa + 128 * q, a0, a1);
                    lds4(xb + 128 * q, b0, b1v);
                    ga = ffma2(a0, b0, ga);
                    ga = ffma2(a1, b1v, ga);
                }
                float glo, ghi;
                upk(ga, glo, ghi);
                float g = glo + ghi;
                if (lane < 4) {                         // columns 768 + 4·lane .. +3 (zero past D)
                    const float4 a = *reinterpret_cast<const float4*>(xa - 4 * lane + XC + 4 * lane);
                    const float4 b = *reinterpret_cast<const float4*>(xb - 4 * lane + XC + 4 * lane);
                    g = fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, fmaf(a.x, b.x, g))));
                }
                g = warp_sum(g);
                if (lane == 0) sm.gterm[s1 % GT][cw] = g;
            }
            // ---- z1(c) = acc - Σ_k g(c-k) G(c-k,c) + b1(c), h(c) ----
            mbar_wait(&sm.aready[c % AR], (uint32_t)((c / AR) & 1));
            const float4 G = *reinterpret_cast<const float4*>(&sm.gterm[c % GT][0]);   // k = 1..4
            float z = sm.asum[c % AR][u];
            z = fmaf(-g4, G.w, z);
            z = fmaf(-g3, G.z, z);
            z = fmaf(-g2, G.y, z);
            z = fmaf(-g1, G.x, z);
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
            // ---- δ2(c) in every thread ----
            float dl[O];
            {
                float z2[O];
                const float4* a = reinterpret_cast<const float4*>(&sm.zp[c & 1][0][0]);
                const float4* b = reinterpret_cast<const float4*>(&sm.zp[c & 1][1][0]);
                const float4* e = reinterpret_cast<const float4*>(&sm.zp[c & 1][2][0]);
                const float4* f = reinterpret_cast<const float4*>(&sm.zp[c & 1][3][0]);
                const float4* bb = reinterpret_cast<const float4*>(&sm.b2s[c & 1][0]);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const float4 x = a[q], y = b[q], v = e[q], t = f[q], bq = bb[q];
                    const float t4[4] = {((x.x + y.x) + (v.x + t.x)) + bq.x, ((x.y + y.y) + (v.y + t.y)) + bq.y,
                                         ((x.z + y.z) + (v.z + t.z)) + bq.z, ((x.w + y.w) + (v.w + t.w)) + bq.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (4 * q + i < O) z2[4 * q + i] = t4[i];   // z2 = W2 h + b2 (Eq.2)
                }
                if constexpr (A2 == PNN_SOFTMAX) {
                    const float m = fmaxf(fmaxf(fmaxf(z2[0], z2[1]), fmaxf(z2[2], z2[3])),
                                          fmaxf(fmaxf(fmaxf(z2[4], z2[5]), fmaxf(z2[6], z2[7])), fmaxf(z2[8], z2[9])));
#pragma unroll
                    for (int o = 0; o < O; ++o) dl[o] = __expf(z2[o] - m);
                    const float sum = ((dl[0] + dl[1]) + (dl[2] + dl[3])) +
                                      (((dl[4] + dl[5]) + (dl[6] + dl[7])) + (dl[8] + dl[9]));
                    float inv;
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(sum));
#pragma unroll
                    for (int o = 0; o < O; ++o) dl[o] = dl[o] * inv - ((o == lab0) ? 1.f : 0.f);
                } else {
                    // element-wise output (sigmoid / tanh, ½-SSE: Eq.9, R11): lane o forms output
                    // o's activation and δ2 once, then every lane takes the ten by shuffles
                    float zsel = z2[0];
#pragma unroll
                    for (int o = 1; o < O; ++o) zsel = (lane == o) ? z2[o] : zsel;
                    const float x2 = act_fwd_t<A2>(zsel);
                    const float dmine = (x2 - ((lane == lab0) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
#pragma unroll
                    for (int o = 0; o < O; ++o) dl[o] = __shfl_sync(0xffffffffu, dmine, o);
                }
            }
            // ---- δ1, g(c) → the sweeps; W2, b1, b2 updates ----
            float s1 = 0.f;                         // (W2ᵀδ2)_u with the pre-update W2 (R6)
#pragma unroll
            for (int o = 0; o < O; ++o) s1 = fmaf(w2[o], dl[o], s1);
            const float gu = lc ? lr * (s1 * act_deriv_t<A1>(h)) : 0.f;
            sm.gbuf[c % GR][u] = gu;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.gready[c % GR]);
            b1 -= gu;
#pragma unroll
            for (int o = 0; o < O; ++o) w2[o] = fmaf(-(lr * dl[o]), h, w2[o]);
            g4 = g3; g3 = g2; g2 = g1; g1 = gu;
            if (leader) {
                // b2(c+1) into the other buffer (the other threads may still read b2(c))
                const float4* bo = reinterpret_cast<const float4*>(&sm.b2s[c & 1][0]);
                float4* bq = reinterpret_cast<float4*>(&sm.b2s[(c + 1) & 1][0]);
                const float4 a = bo[0], b = bo[1], e = bo[2];
                bq[0] = make_float4(fmaf(-lr, dl[0], a.x), fmaf(-lr, dl[1], a.y), fmaf(-lr, dl[2], a.z),
                                    fmaf(-lr, dl[3], a.w));
                bq[1] = make_float4(fmaf(-lr, dl[4], b.x), fmaf(-lr, dl[5], b.y), fmaf(-lr, dl[6], b.z),
                                    fmaf(-lr, dl[7], b.w));
                bq[2] = make_float4(fmaf(-lr, dl[8], e.x), fmaf(-lr, dl[9], e.y), 0.f, 0.f);
                // every sweep warp passed U(c-1-L) (aready(c)) and every chain warp is past its
                // Gram read of x(c-3): the slot of x(c+PF-S) is free
                if (c + PF < T) issue_x(c + PF);
            }
            lab0 = lab1;
            lab1 = lab2;
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
cudaError_t launch_one(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                       int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    auto kern = sgd_ws_kernel<A1, A2>;
    const size_t smem = kSmemHead + sizeof(float) * (size_t)(S + 1) * DP;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<s_count, NT, smem, st>>>(d, children, x, y, n_local, K_local, s_first, lr);
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

cudaError_t launch_sgd_ws(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                          int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
#define PNN_ACTS(A1_, A2_) \
    if (d.act[0] == A1_ && d.act[1] == A2_) return launch_one<A1_, A2_>(d, children, x, y, n_local, K_local, s_first, s_count, lr, st);
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
