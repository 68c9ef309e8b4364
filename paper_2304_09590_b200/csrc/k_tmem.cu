// k_tmem.cu — persistent per-sample SGD, one SM per child network, W¹ resident in
// registers AND tensor memory (variant v11).
//
// A CTA trains one child network (CN) over its whole slice ("Each
// child-network learns only a slice").  Scope: 2-layer nets D-H-O, 768 < D <= 784,
// H <= 128, O = 10, per-sample SGD.  The 128 W¹ rows of the C4 shape
// (784-128-10) are 401 KB: more than the 256 KB register file of an SM, so v8
// (k_resident.cu) splits a CN over a 2-SM cluster and pays a cross-SM exchange in
// every sample's serial chain.  Here the rows are split between the register file
// (6 rows per warp, 144 registers per lane) and the SM's 256 KB tensor memory (TMEM,
// 10 rows per warp), so a CN fits ONE SM and the chain never leaves it.  TMEM rows
// are streamed through registers every pass with tcgen05.ld / tcgen05.st (measured,
// tools/ubench/tmem.cu: a pass over 6 register + 10 TMEM rows per warp runs at the
// same FMA rate as an all-register pass, ~91 FMA/clk/SM).
//
// Per sample, in the paper's sequential order (§3, Eqs.2-13):
//   z1 = W1 x + b1, h = φ1(z1); z2 = W2 h + b2, x2 = φ2(z2)         (Eqs.2-5)
//   δ2 = x2 - e (softmax+CE, Eq.10) or (x2 - e)⊙φ2'(x2) (R11)       (Eqs.9-10)
//   δ1 = (W2ᵀ δ2) ⊙ φ1'(h), with the pre-update W2 (R6)              (Eq.11)
//   W -= η δ xᵀ, b -= η δ                                             (Eqs.12-13)
//
// L-step lookahead (L = 4, R27): with W¹(t) the weights before sample t's
// update and g(s) = η δ1(s),
//     z1(t) = W¹(t-L) x(t) - Σ_{k=1..L} g(t-k)·G(t-k,t) + b1(t),  G(s,t) = x(s)·x(t),
// equal to the paper's pre-activation in real arithmetic.  The Gram terms are formed
// INSIDE this launch from the shared-memory ring (no pre-pass re-reading X).
//
// Warp roles (8 warps; warp w owns hidden units 16w .. 16w+15):
//   F(s)  acc = W¹(s-L)·x(s) for the warp's 16 rows (lane l: columns 4l+128q .. +3,
//         q < 6, and a 16-column tail 768.. held as row l>>1, 8 columns per lane),
//         a 16-value transpose-reduce, row sums → shared memory, arrive aready(s);
//   U(s)  wait gready(s-L), W¹ -= g(s-L)·x(s-L)ᵀ.
// The serial chain of sample c runs on warp pair c mod 4 (warps 2p, 2p+1: different SM
// sub-partitions) after its F(c+1): z1 by the correction, h, the pair's partial logits
// (2 units per lane, a transpose-reduce, the two warps' halves exchanged through
// shared memory + a named barrier), softmax / φ2, δ2, δ1, g(c), the W²/b updates,
// arrive gready(c).  The same pair then issues the bulk copy of x(c+8).  Each warp's F(s)
// also forms one partial Gram term (k = 1 + warp mod 4, one column half), so the chain
// reads G(s-k, s) as two shared-memory sums; warp 0 stages the label.
#include <cstddef>
#include <cstdio>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"
#include "pnn_tmem.cuh"

extern long long* g_trace;   // debug: clock64 timeline (k_resident.cu; tools/trace_tmem.py)

namespace {

using namespace ptx;
constexpr int kTraceT = 64, kTraceP = 16;   // debug timeline: [cta < 2][warp][step][point]

constexpr int NW = 8;          // warps per CTA
constexpr int RR = 6;          // W¹ rows per warp in registers
constexpr int TR = 10;         // W¹ rows per warp in TMEM
constexpr int RPW = RR + TR;   // rows per warp
constexpr int UMAX = NW * RPW; // 128 hidden units
constexpr int NQ = 6;          // column quads per lane: columns [0, 768)
constexpr int NP = 2 * NQ;     // f32x2 pairs per lane per row
constexpr int XC = 768;        // first tail column
constexpr int DP = 800;        // x ring slot stride (floats)
constexpr int LAG = 4;         // lookahead L
constexpr int S = 16;          // x ring slots (+ one zero row at slot S)
constexpr int PF = 8;          // prefetch distance: x(c+PF) issued after chain c
constexpr int O = 10;          // outputs
constexpr int AR = 8;          // row-sum ring slots (> LAG)
constexpr int GR = 8;          // g ring slots (> LAG)
constexpr int GRR = 8;         // Gram-record ring slots
constexpr int TQCOLS = 4 * TR; // TMEM columns per quad (rows t at 4t)
constexpr int TTAIL = NQ * TQCOLS;   // first TMEM column of the tail (240)
static_assert(TTAIL + 8 <= 256, "TMEM half of a lane quadrant");
static_assert(S >= PF + LAG + 4, "x ring: a refilled slot is no longer read");

struct __align__(16) Smem {
    uint64_t xfull[S];             // x(u) landed (bulk copy complete_tx)
    uint64_t aready[AR];           // F(s) of all 8 warps + the end of chain s-1 (count NW + 2)
    uint64_t gready[GR];           // chain c done: g(c) in gbuf (count 2)
    uint32_t tbase;                // TMEM base address
    uint32_t pad[3];
    float asum[AR][UMAX];          // [s % AR][unit] row sums W¹(s-L)·x(s)
    float gbuf[GR][UMAX];          // [c % GR][unit] g(c) = η δ1(c)
    float w2s[UMAX][12];           // W2[o][u] (o < 10), + 2 pad
    float b1s[UMAX];
    float b2s[2][12];              // b2 before sample c at [c & 1]
    float zbuf[4][2][16];          // [pair][half][o] the pair's partial logits
    float gpart[GRR][NW];          // [s % GRR][warp] partial Gram term G(s-k, s), k = 1 + (warp & 3),
                                   // over column half warp >> 2 (formed in F(s))
    int label[GRR];                // [s % GRR] label of sample s (staged in F(s) by warp 0)
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

// 16 values per lane → lane l holds the sum over the warp of value (l >> 1), halves in
// lanes l and l^1 still to be combined (the caller adds its own term first).
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

template <int A1, int A2, bool TRACE>
__global__ void __launch_bounds__(NW * 32, 1)
sgd_tmem_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                const int32_t* __restrict__ Y, long long n_local, int K_local, int s_first, float lr,
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
    const int32_t* Yc = Y + row0;
    const uint32_t xbytes = (uint32_t)D * 4u;

    if (warp == 0) tmem::alloc(&sm.tbase, 512);
    if (threadIdx.x == 32) {
        for (int i = 0; i < S; ++i) mbar_init(&sm.xfull[i], 1);
        for (int i = 0; i < AR; ++i) mbar_init(&sm.aready[i], NW + 2);
        for (int i = 0; i < GR; ++i) mbar_init(&sm.gready[i], 2);
        fence_mbar_init();
        mbar_arrive(&sm.aready[0]);                 // sample 0 has no previous chain
        mbar_arrive(&sm.aready[0]);
    }
    for (int i = threadIdx.x; i < (S + 1) * DP; i += blockDim.x) xring[i] = 0.f;   // + the zero row
    for (int i = threadIdx.x; i < GR * UMAX; i += blockDim.x) (&sm.gbuf[0][0])[i] = 0.f;
    for (int i = threadIdx.x; i < UMAX * 12; i += blockDim.x) {
        const int u = i / 12, o = i % 12;
        sm.w2s[u][o] = (u < H && o < O) ? W2[(long long)o * H + u] : 0.f;
    }
    for (int i = threadIdx.x; i < UMAX; i += blockDim.x) sm.b1s[i] = (i < H) ? b1g[i] : 0.f;
    for (int i = threadIdx.x; i < 24; i += blockDim.x) (&sm.b2s[0][0])[i] = (i < O) ? b2g[i] : 0.f;
    fence_proxy_async_smem();
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tq = sm.tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (uint32_t)(warp >> 2);
    auto issue_x = [&](int u) {
        uint64_t* bar = &sm.xfull[u % S];
        mbar_arrive_expect_tx(bar, xbytes);
        bulk_g2s(xring + (u % S) * DP, Xc + (long long)u * D, xbytes, bar);
    };
    if (threadIdx.x == 0)
        for (int u = 0; u < PF && u < T; ++u) issue_x(u);

    // ---- this warp's W¹ rows: RR in registers, TR in TMEM, the tail in TMEM ----
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
    const int trow = lane >> 1, th8 = lane & 1;     // tail: row kr0 + trow, columns 768 + 8·th8 .. +7
    {
        uint32_t tt[8];
        const bool live = kr0 + trow < H;
        const float* src = W1 + (long long)(kr0 + trow) * D + XC + 8 * th8;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            tt[j] = __float_as_uint((live && XC + 8 * th8 + j < D) ? src[j] : 0.f);
        tmem::st8(tq + TTAIL, tt);
    }
    tmem::wait_st();

    // chain side: warp 2p+h of pair p owns units 64h + lane and 64h + 32 + lane
    const int pair = warp >> 1, half = warp & 1;
    const int u0 = 64 * half + lane, u1 = u0 + 32;
    const bool l0 = u0 < H, l1 = u1 < H;

#define TR(pt)                                                                                   \
    do {                                                                                         \
        if constexpr (TRACE) {                                                                   \
            if (blockIdx.x < 2 && s < kTraceT && lane == 0)                                      \
                trace[(((int)blockIdx.x * NW + warp) * kTraceT + s) * kTraceP + (pt)] = ptx::clock64(); \
        }                                                                                        \
    } while (0)
    for (int s = 0; s < T + LAG; ++s) {
        TR(0);
        if (s < T) {
            // ---------------- F(s): acc = W¹(s-L)·x(s) ----------------
            const int sl = s % S;
            mbar_wait(&sm.xfull[sl], (uint32_t)((s / S) & 1));
            TR(1);
            const float* xn = xring + sl * DP + 4 * lane;
            // this warp's share of the Gram terms (R27): G(s-k, s), k = 1 + (warp & 3), over the
            // column quads of half warp >> 2 (+ the tail for half 1); x(<0) is the zero row
            const int gk = 1 + (warp & 3), gh = warp >> 2;
            const float* xg = xring + ((s - gk >= 0) ? (s - gk) % S : S) * DP + 4 * lane;
            int lab = 0;
            if (warp == 0 && lane == 0) lab = __ldg(Yc + s);
            uint64_t gacc = 0ull;
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
                if (q / 3 == gh) {
                    uint64_t ga, gb;
                    lds4(xg + 128 * q, ga, gb);
                    gacc = ffma2(xa, ga, gacc);
                    gacc = ffma2(xb, gb, gacc);
                }
#pragma unroll
                for (int r = 0; r < RR; ++r) {
                    acc[r] = ffma2(w[r][2 * q], xa, acc[r]);
                    acc[r] = ffma2(w[r][2 * q + 1], xb, acc[r]);
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
            {
                float glo, ghi;
                upk(gacc, glo, ghi);
                float g = glo + ghi;
                if (gh == 1 && lane < 4) {             // the tail columns 768 + 4·lane .. +3
                    const float4 a = *reinterpret_cast<const float4*>(xring + sl * DP + XC + 4 * lane);
                    const float4 b = *reinterpret_cast<const float4*>(xg + XC);
                    g = fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, fmaf(a.x, b.x, g))));
                }
                g = warp_sum(g);
                if (lane == 0) sm.gpart[s % GRR][warp] = g;
                if (warp == 0 && lane == 0) sm.label[s % GRR] = lab;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.aready[s % AR]);
            TR(2);
        }
        // ================= the chain of sample c = s - 1 on warp pair c mod 4 =================
        const int c = s - 1;
        if (c >= 0 && c < T && (c & 3) == pair) {
            mbar_wait(&sm.aready[c % AR], (uint32_t)((c / AR) & 1));
            TR(3);
            float4 G;                                  // G(c-k, c), k = 1..4: the two column halves
            {
                const float4 g0 = *reinterpret_cast<const float4*>(&sm.gpart[c % GRR][0]);
                const float4 g1 = *reinterpret_cast<const float4*>(&sm.gpart[c % GRR][4]);
                G = make_float4(g0.x + g1.x, g0.y + g1.y, g0.z + g1.z, g0.w + g1.w);
            }
            const int label = sm.label[c % GRR];
            const float* gb4 = sm.gbuf[(c + GR - 4) % GR];
            const float* gb3 = sm.gbuf[(c + GR - 3) % GR];
            const float* gb2 = sm.gbuf[(c + GR - 2) % GR];
            const float* gb1 = sm.gbuf[(c + GR - 1) % GR];
            float z0 = sm.asum[c % AR][u0], z1 = sm.asum[c % AR][u1];
            z0 = fmaf(-gb4[u0], G.w, z0); z1 = fmaf(-gb4[u1], G.w, z1);
            z0 = fmaf(-gb3[u0], G.z, z0); z1 = fmaf(-gb3[u1], G.z, z1);
            z0 = fmaf(-gb2[u0], G.y, z0); z1 = fmaf(-gb2[u1], G.y, z1);
            z0 = fmaf(-gb1[u0], G.x, z0); z1 = fmaf(-gb1[u1], G.x, z1);
            z0 += sm.b1s[u0];
            z1 += sm.b1s[u1];
            const float h0 = l0 ? act_fwd_t<A1>(z0) : 0.f;
            const float h1 = l1 ? act_fwd_t<A1>(z1) : 0.f;
            TR(4);
            float wv0[12], wv1[12];                    // W2[:, u] pre-update (R6), kept for δ1
            {
                const float4* q0 = reinterpret_cast<const float4*>(&sm.w2s[u0][0]);
                const float4* q1 = reinterpret_cast<const float4*>(&sm.w2s[u1][0]);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const float4 f = q0[q], g = q1[q];
                    wv0[4 * q] = f.x; wv0[4 * q + 1] = f.y; wv0[4 * q + 2] = f.z; wv0[4 * q + 3] = f.w;
                    wv1[4 * q] = g.x; wv1[4 * q + 1] = g.y; wv1[4 * q + 2] = g.z; wv1[4 * q + 3] = g.w;
                }
            }
            {
                float pv[16];
#pragma unroll
                for (int o = 0; o < 16; ++o) pv[o] = (o < O) ? fmaf(wv1[o < O ? o : 0], h1, wv0[o < O ? o : 0] * h0) : 0.f;
                float p0 = treduce16(pv, lane);
                p0 += __shfl_xor_sync(0xffffffffu, p0, 1);
                const int oi = lane >> 1;
                if ((lane & 1) == 0) sm.zbuf[pair][half][oi] = p0;
            }
            named_bar_sync(1 + pair, 64);
            TR(5);
            float dl[O];
            {
                float z2[O];
                {
                    const float4* a = reinterpret_cast<const float4*>(&sm.zbuf[pair][0][0]);
                    const float4* b = reinterpret_cast<const float4*>(&sm.zbuf[pair][1][0]);
                    const float4* bb = reinterpret_cast<const float4*>(&sm.b2s[c & 1][0]);
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const float4 x = a[q], y = b[q], z = bb[q];
                        const float t4[4] = {(x.x + y.x) + z.x, (x.y + y.y) + z.y, (x.z + y.z) + z.z, (x.w + y.w) + z.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (4 * q + i < O) z2[4 * q + i] = t4[i];
                    }
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
                    for (int o = 0; o < O; ++o) dl[o] = dl[o] * inv - ((o == label) ? 1.f : 0.f);
                } else {
                    float zsel = z2[0];
#pragma unroll
                    for (int o = 1; o < O; ++o) zsel = (lane == o) ? z2[o] : zsel;
                    const float x2 = act_fwd_t<A2>(zsel);
                    const float dmine = (x2 - ((lane == label) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
#pragma unroll
                    for (int o = 0; o < O; ++o) dl[o] = __shfl_sync(0xffffffffu, dmine, o);
                }
            }
            {
                float s0 = 0.f, s1 = 0.f;              // (W2ᵀδ2)_u with the pre-update W2 (R6)
#pragma unroll
                for (int o = 0; o < O; ++o) { s0 = fmaf(wv0[o], dl[o], s0); s1 = fmaf(wv1[o], dl[o], s1); }
                const float g0 = l0 ? lr * (s0 * act_deriv_t<A1>(h0)) : 0.f;
                const float g1 = l1 ? lr * (s1 * act_deriv_t<A1>(h1)) : 0.f;
                sm.gbuf[c % GR][u0] = g0;
                sm.gbuf[c % GR][u1] = g1;
                sm.b1s[u0] -= g0;
                sm.b1s[u1] -= g1;
#pragma unroll
                for (int o = 0; o < O; ++o) {
                    const float e = -(lr * dl[o]);
                    wv0[o] = fmaf(e, h0, wv0[o]);
                    wv1[o] = fmaf(e, h1, wv1[o]);
                }
                float4* q0 = reinterpret_cast<float4*>(&sm.w2s[u0][0]);
                float4* q1 = reinterpret_cast<float4*>(&sm.w2s[u1][0]);
                q0[0] = make_float4(wv0[0], wv0[1], wv0[2], wv0[3]);
                q0[1] = make_float4(wv0[4], wv0[5], wv0[6], wv0[7]);
                q0[2] = make_float4(wv0[8], wv0[9], 0.f, 0.f);
                q1[0] = make_float4(wv1[0], wv1[1], wv1[2], wv1[3]);
                q1[1] = make_float4(wv1[4], wv1[5], wv1[6], wv1[7]);
                q1[2] = make_float4(wv1[8], wv1[9], 0.f, 0.f);
            }
            if (half == 1 && lane == 0) {              // b2(c+1) into the other buffer (the partner
                const float4* bo = reinterpret_cast<const float4*>(&sm.b2s[c & 1][0]);   // may still
                float4* bq = reinterpret_cast<float4*>(&sm.b2s[(c + 1) & 1][0]);        // read b2(c))
                const float4 a = bo[0], b = bo[1], e = bo[2];
                bq[0] = make_float4(fmaf(-lr, dl[0], a.x), fmaf(-lr, dl[1], a.y), fmaf(-lr, dl[2], a.z),
                                    fmaf(-lr, dl[3], a.w));
                bq[1] = make_float4(fmaf(-lr, dl[4], b.x), fmaf(-lr, dl[5], b.y), fmaf(-lr, dl[6], b.z),
                                    fmaf(-lr, dl[7], b.w));
                bq[2] = make_float4(fmaf(-lr, dl[8], e.x), fmaf(-lr, dl[9], e.y), 0.f, 0.f);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.gready[c % GR]);
                if (c + 1 < T) mbar_arrive(&sm.aready[(c + 1) % AR]);
            }
            TR(6);
            // off the critical path: every warp passed U(c-1) (aready(c)), so the slot of
            // x(c+PF-S) is free; then the Gram record of this pair's next sample
            if (half == 0 && lane == 0 && c + PF < T) issue_x(c + PF);
            TR(7);
        }
        // ---------------- U(s): W¹ -= g(s-L)·x(s-L)ᵀ ----------------
        const int uu = s - LAG;
        if (uu >= 0 && uu < T) {
            mbar_wait(&sm.gready[uu % GR], (uint32_t)((uu / GR) & 1));
            TR(8);
            const float* xo = xring + (uu % S) * DP + 4 * lane;
            float gn[RPW];
            {
                const float4* gv = reinterpret_cast<const float4*>(&sm.gbuf[uu % GR][kr0]);
#pragma unroll
                for (int i = 0; i < RPW / 4; ++i) {
                    const float4 a = gv[i];
                    gn[4 * i] = -a.x; gn[4 * i + 1] = -a.y; gn[4 * i + 2] = -a.z; gn[4 * i + 3] = -a.w;
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
                    w[r][2 * q] = ffma2(pk(gn[r], gn[r]), xa, w[r][2 * q]);
                    w[r][2 * q + 1] = ffma2(pk(gn[r], gn[r]), xb, w[r][2 * q + 1]);
                }
                tmem::wait_ld_regs<TQCOLS>(tv);
#pragma unroll
                for (int t = 0; t < TR; ++t) {
                    const uint64_t gg = pk(gn[RR + t], gn[RR + t]);
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
            TR(9);
        }
    }
#undef TR

    // ---- write back: W¹ rows (registers, TMEM, tail), W², b¹, b² ----
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
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    if (warp == 0) tmem::dealloc(sm.tbase, 512);
    for (int i = threadIdx.x; i < H * O; i += blockDim.x) {
        const int o = i / H, u = i % H;
        opaque(W2)[(long long)o * H + u] = sm.w2s[u][o];
    }
    for (int i = threadIdx.x; i < H; i += blockDim.x) opaque(b1g)[i] = sm.b1s[i];
    if (threadIdx.x < O) opaque(b2g)[threadIdx.x] = sm.b2s[T & 1][threadIdx.x];
}

template <int A1, int A2, bool TRACE>
cudaError_t launch_one(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                       int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    auto kern = sgd_tmem_kernel<A1, A2, TRACE>;
    const size_t smem = kSmemHead + sizeof(float) * (size_t)(S + 1) * DP;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<s_count, NW * 32, smem, st>>>(d, children, x, y, n_local, K_local, s_first, lr, g_trace);
    return cudaGetLastError();
}

}  // namespace

const char* tmem_plan(const NetDesc& d, int batch) {
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

cudaError_t launch_sgd_tmem(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                            int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    if (g_trace && d.act[0] == PNN_RELU && d.act[1] == PNN_SOFTMAX)   // debug timeline build
        return launch_one<PNN_RELU, PNN_SOFTMAX, true>(d, children, x, y, n_local, K_local, s_first, s_count, lr, st);
#define PNN_ACTS(A1_, A2_) \
    if (d.act[0] == A1_ && d.act[1] == A2_) return launch_one<A1_, A2_, false>(d, children, x, y, n_local, K_local, s_first, s_count, lr, st);
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
