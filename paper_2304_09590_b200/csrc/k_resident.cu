// k_resident.cu — persistent per-sample SGD with register-resident weights (v8).
//
// A thread-block cluster of C CTAs trains one child network (CN) over its whole
// slice ("Each child-network learns only a slice").  The hidden
// layer is split across the C SMs (C = 2 for the C4 shape 784-128-10): CTA c
// owns units [c·U, c·U+U), U <= 64, served by 8 warps of 8 W¹ rows each; the
// rows live in REGISTERS for the whole slice (loaded once, written back once).
// Scope: 2-layer nets D-H-O, 768 < D <= 784, O = 10, H <= 64·C, per-sample SGD.
//
// Per sample, in the paper's sequential order (§3, Eqs.2-13):
//   z1 = W1 x + b1, h = φ1(z1); z2 = W2 h + b2, x2 = φ2(z2)         (Eqs.2-5)
//   δ2 = x2 - e (softmax+CE, Eq.10) or (x2 - e)⊙φ2'(x2) (R11)       (Eqs.9-10)
//   δ1 = (W2ᵀ δ2) ⊙ φ1'(h), with the pre-update W2 (R6)              (Eq.11)
//   W -= η δ xᵀ, b -= η δ                                             (Eqs.12-13)
//
// L-step lookahead (L = 4).  With W¹(t) the weights before sample t's update
// and g(s) = η δ1(s), W¹(t) = W¹(t-L) - Σ_{s=t-L}^{t-1} g(s) x(s)ᵀ, so
//     z1(t) = W¹(t-L) x(t) - Σ_{k=1..L} g(t-k)·G(t-k,t) + b1(t),  G(s,t) = x(s)·x(t),
// the paper's pre-activation in real arithmetic (R27; only the
// rounding differs).  The Gram terms depend on the data only: gram_kernel
// computes them (and stages the label) for every row before training, and they
// travel with x(t) through the shared-memory ring.
//
// Warp roles.  Every warp sweeps its rows each step s:
//   F(s)  acc = W¹(s-L)·x(s) (lane l: columns 4l+128q .. +3, q < 6, as f32x2
//         pairs, one LDS.128 feeds 16 fma.rn.f32x2; columns 768..783 in shared
//         memory), row sums → shared memory, arrive aready(s);
//   U(s)  wait gready(s-L), W¹ -= g(s-L)·x(s-L)ᵀ.
// The serial per-sample chain runs on ONE warp per CTA at a time: sample c's
// chain is done by warp c mod 8 (after its own F(c+1)), for all of the CTA's
// units, with W², b1, b2 and the g history in shared memory: z1(c) by the
// correction above, h(c), the CTA's partial logits (published to every CTA of
// the cluster through st.async + mbarrier zfull), then z2, softmax / φ2 and
// δ2(c) in every lane, δ1, g(c), the W²/b1/b2 updates, arrive gready(c).  The
// other warps never wait for the chain except through gready(s-L), L samples
// later, so the sweeps run at their own pace while the chain's latency (the
// cross-SM exchange above all) overlaps them.
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
constexpr int NW = 8;         // warps per CTA
constexpr int UMAX = R * NW;  // units per CTA
constexpr int NQ = 6;         // column quads per lane: columns [0, 768)
constexpr int NP = 2 * NQ;    // f32x2 pairs per lane
constexpr int XC = 768;       // first shared-memory column
constexpr int GOFF = 784;     // gram record of sample u sits at its x ring slot + GOFF
constexpr int DP = 800;       // x ring slot stride (floats)
constexpr int LAG = 4;        // lookahead L
constexpr int S = 16;         // x ring slots
constexpr int PF = 8;         // prefetch distance (<= S - 1 - LAG)
constexpr int O = 10;         // outputs
constexpr int AR = 8;         // row-sum ring slots (> LAG + 1)
constexpr int GR = 8;         // g ring slots (> LAG)
static_assert(AR > LAG + 1 && GR > LAG, "ring sizes");
constexpr int ZS = 4;         // partial-logit ring slots
constexpr int CMAX = 4;       // cluster size
// the chain warp of the pair that does not issue the x prefetch updates b2
constexpr int kB2Half = 1;
constexpr int kTraceT = 64, kTraceP = 16;   // debug timeline: [cta][warp][t][point]

struct __align__(16) Smem {
    uint64_t xfull[S];                 // x(u) and its gram record landed
    uint64_t aready[AR];               // all warps' row sums of sample s + the end of chain s-1 (count NW + 2)
    uint64_t gready[GR];               // chain → sweeps: g(c) of every row (the pair: count 2)
    uint64_t zfull[ZS];                // partial logits of sample c from every CTA (count 2 + tx)
    float asum[AR][UMAX][4];           // [s % AR][row][part] partial row sums of acc(s)
    float gbuf[GR][UMAX];              // [c % GR][row] g(c)
    float zbuf[ZS][2 * CMAX][16];      // [c % ZS][2·cta + half][o] partial logits
    float w2s[UMAX][16];               // W2[o][k0 + u] (o < 10), the CTA's units
    float b1s[UMAX];                   // b1 of the CTA's units
    float b2s[2][16];                  // b2 before sample c at [c & 1] (identical in every CTA)
    float hs[2][UMAX];                 // h(c) of the CTA's units, [c & 1]
    float wx[NW][R][16];               // W1 columns 768..783 of each warp's rows
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

constexpr int GCH = 96;                    // least rows per warp chunk (a multiple of the window ring, 6)
constexpr int GR_SLOTS = 6;                // per-warp shared-memory ring (= the register window ring, so the slot of
                                           // a row is a compile-time constant in the unrolled loop): 5 rows in flight
constexpr int GR_STRIDE = 800;             // floats per ring slot
constexpr int GWARPS = 4;                  // warps per CTA
constexpr size_t kGramSmem = sizeof(float) * GWARPS * GR_SLOTS * GR_STRIDE;
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <int N> __device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
struct GramRun {
    const float* X;
    const int32_t* Y;
    float* rec;                             // the records as floats: 8 per row
    float* ring;                            // this warp's shared-memory ring
    int D, lane;
    int ynext;                              // label of the next row, loaded one row ahead
    long long a1, st, nxt_start, base, rem;
};
// x(row) into ring slot `slot` (= (row - chunk start) % GR_SLOTS, a compile-time constant at
// the call sites of the unrolled row loop: a 64-bit row % 6 costs more than the row's dot
// products): each lane copies exactly the columns it reads back (its own cp.async group), so
// no cross-lane synchronisation is needed.  One group per call (empty past the chunk end)
// keeps the wait_group count uniform.
__device__ __forceinline__ void gram_issue(const GramRun& g, long long row, int slot) {
    if (row < g.a1) {
        const float* xr = g.X + row * (long long)g.D;
        float* dst = g.ring + slot * GR_STRIDE;
#pragma unroll
        for (int q = 0; q < 6; ++q) cp_async16(dst + 4 * g.lane + 128 * q, xr + 4 * g.lane + 128 * q);
        if (4 * g.lane + 768 < g.D) cp_async16(dst + 768 + 4 * g.lane, xr + 768 + 4 * g.lane);
    }
    cp_async_commit();
}
__device__ __forceinline__ void gram_zero(float4 (&v)[7]) {
#pragma unroll
    for (int q = 0; q < 7; ++q) v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ uint64_t gpk(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
// dot(a, b): two f32x2 partial sums over the column pairs, folded
__device__ __forceinline__ float gdot(const float4 (&a)[7], const float4 (&b)[7]) {
    uint64_t acc = 0ull;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        acc = ffma2(gpk(a[q].x, a[q].y), gpk(b[q].x, b[q].y), acc);
        acc = ffma2(gpk(a[q].z, a[q].w), gpk(b[q].z, b[q].w), acc);
    }
    float lo, hi;
    upk(acc, lo, hi);
    return lo + hi;
}
// Row `row` at window phase J: x(row-5+k) is in register buffer (J+k)%6 (k < 5); x(row) is read
// from the ring into (J+5)%6, which held x(row-6).
template <int J>
__device__ __forceinline__ void gram_row(GramRun& g, float4 (&b)[6][7], long long row) {
    if (row == g.nxt_start) {               // a new slice begins at this row (R17)
        g.st = row;
        g.nxt_start += g.base + ((row < g.rem * (g.base + 1)) ? 1 : 0);
    }
    // the label rides one row ahead: loaded where it is stored, the row's record store would wait
    // a whole L2 round trip on it
    const int ylab = g.ynext;
    if (row + 1 < g.a1) g.ynext = g.Y[row + 1];
    cp_async_wait_group<GR_SLOTS - 2>();    // x(row) has landed (this lane's part)
    {
        const float* src = g.ring + J * GR_STRIDE;
        float4 (&c)[7] = b[(J + 5) % 6];
#pragma unroll
        for (int q = 0; q < 6; ++q) c[q] = *reinterpret_cast<const float4*>(src + 4 * g.lane + 128 * q);
        c[6] = (4 * g.lane + 768 < g.D) ? *reinterpret_cast<const float4*>(src + 768 + 4 * g.lane)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    gram_issue(g, row + GR_SLOTS - 1, (J + GR_SLOTS - 1) % GR_SLOTS);   // refills the slot x(row-1) used (consumed last row)
    float v[8];
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] = gdot(b[(J + k) % 6], b[(J + 5) % 6]);
    v[5] = v[6] = v[7] = 0.f;
    // the five dot products reduced together: a transpose-reduce of 8 values over the warp
    // (lane 4·i ends with the sum of value i: 9 shuffles instead of 5 × 5)
    const int lane = g.lane;
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    float u4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) u4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, b4 ? v[i] : v[i + 4], 16);
    float u2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) u2[i] = (b3 ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b3 ? u4[i] : u4[i + 2], 8);
    float t = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    // record floats [G(u-4), G(u-3), G(u-2), G(u-1), label, G(u-5), 0, 0]; a term that reaches
    // back past the start of the row's slice is 0
    if ((lane & 3) == 0) {
        const int idx = lane >> 2;
        float val;
        int pos;
        if (idx < 5) {
            val = (row - 5 + idx >= g.st) ? t : 0.f;
            pos = idx == 0 ? 5 : idx - 1;
        } else {
            val = idx == 5 ? __int_as_float(ylab) : 0.f;
            pos = idx == 5 ? 4 : idx;
        }
        g.rec[8 * row + pos] = val;
    }
}
// Gram record of every row of CNs [s_first, s_first + s_count) (shard-local index u):
// rec[2·row] = {x(u-4)·x(u), x(u-3)·x(u), x(u-2)·x(u), x(u-1)·x(u)} (0 before the slice
// start), rec[2·row + 1] = {label bits, x(u-5)·x(u), 0, 0}.  A warp walks a chunk of consecutive
// rows (rows / warps of them, at least GCH): x streams through a per-warp shared-memory ring (cp.async, 5 rows in flight), the last
// five rows stay in registers (lane l: columns 4l + 128q, q < 6, and 768 + 4l for l < 4) as a
// ring indexed at compile time (the row loop unrolled by 6), each dot product is 14
// fma.rn.f32x2, so X is read from HBM about once.
__global__ void __launch_bounds__(GWARPS * 32)
gram_kernel(const float* __restrict__ X, const int32_t* __restrict__ Y, int D, long long n_local,
            int K_local, int s_first, int s_count, float4* __restrict__ rec) {
    extern __shared__ __align__(16) float gring[];
    long long r0, c0, r1, c1;
    shard_of(n_local, K_local, s_first, &r0, &c0);
    shard_of(n_local, K_local, s_first + s_count - 1, &r1, &c1);
    const long long rows = r1 + c1 - r0;
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    GramRun g;
    g.X = X; g.Y = Y; g.rec = reinterpret_cast<float*>(rec); g.D = D; g.lane = lane;
    g.ring = gring + (threadIdx.x >> 5) * (GR_SLOTS * GR_STRIDE);
    g.base = n_local / K_local;
    g.rem = n_local % K_local;
    // one contiguous chunk per warp when the rows allow it (no last partial round of chunks, the
    // 5 window rows re-read once per warp), never shorter than GCH rows
    long long gch = (rows + nwarps - 1) / nwarps;
    gch = max((gch + 5) / 6 * 6, (long long)GCH);
    const long long nchunks = (rows + gch - 1) / gch;
    for (long long ch = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); ch < nchunks; ch += nwarps) {
        const long long a0 = r0 + ch * gch;
        g.a1 = min(a0 + gch, r0 + rows);
        cp_async_wait_all();                   // the previous chunk's (empty) groups
#pragma unroll
        for (int k = 0; k < GR_SLOTS - 1; ++k) gram_issue(g, a0 + k, k);
        g.ynext = Y[a0];
        // the slice holding a0: its start (window rows before it are not loaded) and the next
        const long long sidx = (a0 < g.rem * (g.base + 1)) ? a0 / (g.base + 1)
                                                           : g.rem + (a0 - g.rem * (g.base + 1)) / g.base;
        long long s1, cnt;
        shard_of(n_local, K_local, (int)sidx, &s1, &cnt);
        g.st = s1;
        g.nxt_start = s1 + cnt;
        float4 b[6][7];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const long long pr = a0 - 5 + k;
            if (pr >= g.st) {
                const float* xr = X + pr * (long long)D;
#pragma unroll
                for (int q = 0; q < 6; ++q) b[k][q] = *reinterpret_cast<const float4*>(xr + 4 * lane + 128 * q);
                b[k][6] = (4 * lane + 768 < D) ? *reinterpret_cast<const float4*>(xr + 768 + 4 * lane)
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                gram_zero(b[k]);
            }
        }
        // (rows are uniform over the warp; the chunk length is a multiple of 6, only the last chunk is short)
        const long long n6 = (g.a1 - a0) / 6;
        long long row = a0;
        for (long long i = 0; i < n6; ++i, row += 6) {
            gram_row<0>(g, b, row);
            gram_row<1>(g, b, row + 1);
            gram_row<2>(g, b, row + 2);
            gram_row<3>(g, b, row + 3);
            gram_row<4>(g, b, row + 4);
            gram_row<5>(g, b, row + 5);
        }
        const int left = (int)(g.a1 - row);
        if (left > 0) gram_row<0>(g, b, row);
        if (left > 1) gram_row<1>(g, b, row + 1);
        if (left > 2) gram_row<2>(g, b, row + 2);
        if (left > 3) gram_row<3>(g, b, row + 3);
        if (left > 4) gram_row<4>(g, b, row + 4);
    }
    cp_async_wait_all();
}

// Launch of the Gram pre-pass (its shared-memory ring needs the opt-in size once).
cudaError_t gram_launch(const float* x, const int32_t* labels, int D, long long n_local, int K_local, int s_first,
                        int s_count, float4* rec, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGramSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    gram_kernel<<<148 * 2, GWARPS * 32, kGramSmem, st>>>(x, labels, D, n_local, K_local, s_first, s_count, rec);
    return cudaGetLastError();
}

template <int C, int A1, int A2, bool TRACE>
__global__ void __launch_bounds__(NW * 32, 1)
sgd_resident_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                    const float4* __restrict__ rec, long long n_local, int K_local, int s_first,
                    float lr, long long* __restrict__ trace) {
    extern __shared__ __align__(128) unsigned char smraw[];
    Smem& sm = *reinterpret_cast<Smem*>(smraw);
    float* xring = reinterpret_cast<float*>(smraw + kSmemHead);
    const int D = d.n[0], H = d.n[1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int crank = (C > 1) ? (int)cluster_rank() : 0;
    const int cn = s_first + (int)(blockIdx.x / C);
    const int U = (H + C - 1) / C;                 // units per CTA
    const int k0 = crank * U;
    const int Uown = max(0, min(U, H - k0));

    long long row0, T64;
    shard_of(n_local, K_local, cn, &row0, &T64);
    const int T = (int)T64;
    float* P = children + (long long)cn * d.P;
    float* W1 = P;
    float* b1g = P + (long long)H * D;
    float* W2 = b1g + H;
    float* b2g = W2 + (long long)O * H;
    const float* Xc = X + row0 * (long long)D;
    const float4* Rc = rec + 2 * row0;
    const uint32_t xbytes = (uint32_t)D * 4u;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&sm.xfull[i], 1);
        // aready(s): every warp's F(s) and the end of chain s-1 (its pair arrives), so the
        // chain of s waits once; sample 0 has no previous chain
        for (int i = 0; i < AR; ++i) mbar_init(&sm.aready[i], NW + 2);
        for (int i = 0; i < GR; ++i) mbar_init(&sm.gready[i], 2);
        for (int i = 0; i < ZS; ++i) mbar_init(&sm.zfull[i], 2);
        fence_mbar_init();
        mbar_arrive(&sm.aready[0]);
        mbar_arrive(&sm.aready[0]);
    }
    for (int i = threadIdx.x; i < (S + 1) * DP; i += blockDim.x) xring[i] = 0.f;   // + zero row
    for (int i = threadIdx.x; i < GR * UMAX; i += blockDim.x) (&sm.gbuf[0][0])[i] = 0.f;

    for (int i = threadIdx.x; i < UMAX * 16; i += blockDim.x) {
        const int u = i >> 4, o = i & 15;
        sm.w2s[u][o] = (u < Uown && o < O) ? W2[(long long)o * H + k0 + u] : 0.f;
    }
    for (int i = threadIdx.x; i < UMAX; i += blockDim.x) sm.b1s[i] = (i < Uown) ? b1g[k0 + i] : 0.f;
    for (int i = threadIdx.x; i < 32; i += blockDim.x) (&sm.b2s[0][0])[i] = (i < O) ? b2g[i] : 0.f;
    fence_proxy_async_smem();
    __syncthreads();
    if constexpr (C > 1) cluster_sync_all();       // peers' barriers exist before any st.async
    auto issue_x = [&](int u, int slot) {
        uint64_t* bar = &sm.xfull[slot];
        mbar_arrive_expect_tx(bar, xbytes + 32u);
        bulk_g2s(xring + slot * DP, Xc + (long long)u * D, xbytes, bar);
        bulk_g2s(xring + slot * DP + GOFF, Rc + 2 * u, 32u, bar);
    };
    if (threadIdx.x == 0)
        for (int u = 0; u < PF && u < T; ++u) issue_x(u, u);   // the chain of sample c issues x(c+PF)

#define TR(pt)                                                                                   \
    do {                                                                                         \
        if constexpr (TRACE) {                                                                   \
            if (blockIdx.x < 2 && s < kTraceT && lane == 0)                                      \
                trace[(((int)blockIdx.x * NW + warp) * kTraceT + s) * kTraceP + (pt)] =          \
                    ptx::clock64();                                                              \
        }                                                                                        \
    } while (0)

    // ---- this warp's W1 rows ----
    const int kr0 = warp * R;                      // first row (CTA-local)
    uint64_t w[R][NP];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const bool live = kr0 + r < Uown;
        const float* src = W1 + (long long)(k0 + kr0 + r) * D;
#pragma unroll
        for (int m = 0; m < NP; ++m)
            w[r][m] = live ? *reinterpret_cast<const uint64_t*>(src + pcol(lane, m)) : 0ull;
    }
    const int tr = lane >> 2, tq = lane & 3;       // columns 768+4tq .. +3 of row tr
    const int nx = D - XC - 4 * tq;
    const bool xlive = kr0 + tr < Uown;
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

    // chain side: the pair of warps (2p, 2p+1) runs the chain of samples c ≡ p (mod 4); warp
    // 2p+h owns units 32h + lane (h = warp & 1), the two warps sit on different SM sub-partitions
    const int half = warp & 1;
    const int uc = 32 * half + lane;               // this lane's unit in the chain
    const bool lc = uc < Uown;
    const int zrow = 2 * crank + half;             // this warp's row of zbuf in every CTA
    uint32_t rz[C > 1 ? C - 1 : 1];                // DSMEM address of zbuf[0][zrow][0] in each peer
    if constexpr (C > 1) {
#pragma unroll
        for (int p = 1; p < C; ++p)
            rz[p - 1] = mapa(smem_u32(&sm.zbuf[0][zrow][0]), (uint32_t)((crank + p) % C));
    }
    constexpr uint32_t kZStride = 2 * CMAX * 16 * 4;
    constexpr uint32_t kZfullOff = (uint32_t)offsetof(Smem, zfull) - (uint32_t)offsetof(Smem, zbuf);

    // ===== paired sweeps: step p runs F for samples 2p, 2p+1 with W¹(2p-L) (one pass over the
    // registers for both: 32 fma.rn.f32x2 per pair of x quads), U for samples 2p-4, 2p-3, and
    // the chains of samples 2p-2, 2p-1 on their warp pairs.  Sample 2p+1's forward misses
    // the updates of 2p-4 .. 2p (5 Gram corrections; even samples 4). =====
    const int npair = (T + 1) >> 1;
    auto u_pair = [&](int p) {
    if (p >= 2 && 2 * (p - 2) < T) {
        // ---------------- U(2p-4), U(2p-3): W¹ -= g(u)·x(u)ᵀ in sample order ----------------
        const int u0 = 2 * (p - 2), u1 = u0 + 1;
        const bool v1 = u1 < T;
        const int ul = v1 ? u1 : u0;           // chain u1 done ⇒ chain u0 done
        mbar_wait(&sm.gready[ul % GR], (uint32_t)((ul / GR) & 1));
        const int sl0 = u0 % S, sl1 = v1 ? u1 % S : S;
        const float* xo0 = xring + sl0 * DP + 4 * lane;
        const float* xo1 = xring + sl1 * DP + 4 * lane;
        float gp0[R], gp1[R];
        {
            const float4* g0v = reinterpret_cast<const float4*>(&sm.gbuf[u0 % GR][kr0]);
            const float4* g1v = reinterpret_cast<const float4*>(&sm.gbuf[u1 % GR][kr0]);
            const float4 a0 = g0v[0], a1 = g0v[1];
            float4 c0 = g1v[0], c1 = g1v[1];
            if (!v1) { c0 = make_float4(0.f, 0.f, 0.f, 0.f); c1 = c0; }
            gp0[0] = -a0.x; gp0[1] = -a0.y; gp0[2] = -a0.z; gp0[3] = -a0.w;
            gp0[4] = -a1.x; gp0[5] = -a1.y; gp0[6] = -a1.z; gp0[7] = -a1.w;
            gp1[0] = -c0.x; gp1[1] = -c0.y; gp1[2] = -c0.z; gp1[3] = -c0.w;
            gp1[4] = -c1.x; gp1[5] = -c1.y; gp1[6] = -c1.z; gp1[7] = -c1.w;
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            uint64_t xa, xb, ya, yb;
            lds4(xo0 + 128 * q, xa, xb);
            lds4(xo1 + 128 * q, ya, yb);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                w[r][2 * q] = ffma2(pk(gp0[r], gp0[r]), xa, w[r][2 * q]);
                w[r][2 * q + 1] = ffma2(pk(gp0[r], gp0[r]), xb, w[r][2 * q + 1]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                w[r][2 * q] = ffma2(pk(gp1[r], gp1[r]), ya, w[r][2 * q]);
                w[r][2 * q + 1] = ffma2(pk(gp1[r], gp1[r]), yb, w[r][2 * q + 1]);
            }
        }
        __syncwarp();                          // F's tail reads of wx are done
        float4 w4 = *reinterpret_cast<const float4*>(wxp);
        const float4 x4 = *reinterpret_cast<const float4*>(xring + sl0 * DP + XC + 4 * tq);
        const float4 y4 = *reinterpret_cast<const float4*>(xring + sl1 * DP + XC + 4 * tq);
        const float g0 = -sm.gbuf[u0 % GR][kr0 + tr], g1 = v1 ? -sm.gbuf[u1 % GR][kr0 + tr] : 0.f;
        w4.x = fmaf(g0, x4.x, w4.x); w4.y = fmaf(g0, x4.y, w4.y);
        w4.z = fmaf(g0, x4.z, w4.z); w4.w = fmaf(g0, x4.w, w4.w);
        w4.x = fmaf(g1, y4.x, w4.x); w4.y = fmaf(g1, y4.y, w4.y);
        w4.z = fmaf(g1, y4.z, w4.z); w4.w = fmaf(g1, y4.w, w4.w);
        *reinterpret_cast<float4*>(wxp) = w4;
    }
    };

    const int trow = lane >> 2, tsmp = (lane >> 1) & 1, th8 = lane & 1;   // F's tail: row, sample, 8 columns
    for (int p = 0; p < npair + 3; ++p) {
        const int s = 2 * p;                       // (TR's index)
        TR(0);
        __syncwarp();
        if (p < npair) {
            // ---------------- F(2p), F(2p+1) ----------------
            const int s0 = 2 * p, s1 = 2 * p + 1;
            const bool v1 = s1 < T;
            const int sl0 = s0 % S, sl1 = v1 ? s1 % S : S;   // slot S: the zero row
            mbar_wait(&sm.xfull[sl0], (uint32_t)((s0 / S) & 1));
            if (v1) mbar_wait(&sm.xfull[sl1], (uint32_t)((s1 / S) & 1));
            const float* xn0 = xring + sl0 * DP + 4 * lane;
            const float* xn1 = xring + sl1 * DP + 4 * lane;
            uint64_t acc0[R], acc1[R];
#pragma unroll
            for (int r = 0; r < R; ++r) { acc0[r] = 0ull; acc1[r] = 0ull; }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {             // 32 FFMA2 per quad pair cover the loads
                uint64_t xa, xb, ya, yb;
                lds4(xn0 + 128 * q, xa, xb);
                lds4(xn1 + 128 * q, ya, yb);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    acc0[r] = ffma2(w[r][2 * q], xa, acc0[r]);
                    acc1[r] = ffma2(w[r][2 * q], ya, acc1[r]);
                    acc0[r] = ffma2(w[r][2 * q + 1], xb, acc0[r]);
                    acc1[r] = ffma2(w[r][2 * q + 1], yb, acc1[r]);
                }
            }
            float px;                              // row trow, sample tsmp, columns 768 + 8·th8 .. +7
            {
                const float* wt = &sm.wx[warp][trow][8 * th8];
                const float* xt = xring + (tsmp ? sl1 : sl0) * DP + XC + 8 * th8;
                const float4 w0 = *reinterpret_cast<const float4*>(wt), w1 = *reinterpret_cast<const float4*>(wt + 4);
                const float4 x0 = *reinterpret_cast<const float4*>(xt), x1 = *reinterpret_cast<const float4*>(xt + 4);
                px = w0.x * x0.x;
                px = fmaf(w0.y, x0.y, px); px = fmaf(w0.z, x0.z, px); px = fmaf(w0.w, x0.w, px);
                px = fmaf(w1.x, x1.x, px); px = fmaf(w1.y, x1.y, px); px = fmaf(w1.z, x1.z, px);
                px = fmaf(w1.w, x1.w, px);
            }
            float v[16];                           // v[2r + sample]
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float lo, hi;
                upk(acc0[r], lo, hi);
                v[2 * r] = lo + hi;
                upk(acc1[r], lo, hi);
                v[2 * r + 1] = lo + hi;
            }
            // transpose-reduce 16 values: lane l ends with v[l >> 1] = (row l >> 2, sample (l >> 1) & 1)
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
            float zsum = (b1 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? u2[0] : u2[1], 2) + px;
            zsum += __shfl_xor_sync(0xffffffffu, zsum, 1);
            if (th8 == 0 && (tsmp == 0 || v1))
                *reinterpret_cast<float4*>(&sm.asum[(tsmp ? s1 : s0) % AR][kr0 + trow][0]) =
                    make_float4(zsum, 0.f, 0.f, 0.f);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.aready[s0 % AR]);
                if (v1) mbar_arrive(&sm.aready[s1 % AR]);
            }
        }
        TR(1);
        // ================= the chains of samples 2p-2, 2p-1 (one warp pair each) =================
#pragma unroll 1
        for (int cc = 0; cc < 2; ++cc) {
        const int c = 2 * p - 2 + cc;
        if (c >= 0 && c < T && (c & 3) == (warp >> 1)) {
            const int cs = c % S;                  // ring slot of x(c)
            // every warp's row sums of c and the end of chain c-1 (W2, b, g history in shared memory)
            mbar_wait(&sm.aready[c % AR], (uint32_t)((c / AR) & 1));
            TR(3);
            // ---- z1(c) = acc - Σ_k g(c-k) G(c-k,c) + b1(c), k = 1..4 (+5 for odd c); h(c) of unit uc ----
            const float4 G = *reinterpret_cast<const float4*>(xring + cs * DP + GOFF);
            const int label = __float_as_int(xring[cs * DP + GOFF + 4]);
            const float4 pa = *reinterpret_cast<const float4*>(&sm.asum[c % AR][uc][0]);
            float z = (pa.x + pa.y) + (pa.z + pa.w);
            // the paired sweeps' F misses 4 updates (5 for odd samples)
            if (c & 1) z = fmaf(-sm.gbuf[(c + GR - 5) % GR][uc], xring[cs * DP + GOFF + 5], z);
            z = fmaf(-sm.gbuf[(c + GR - 4) % GR][uc], G.x, z);
            z = fmaf(-sm.gbuf[(c + GR - 3) % GR][uc], G.y, z);
            z = fmaf(-sm.gbuf[(c + GR - 2) % GR][uc], G.z, z);
            z = fmaf(-sm.gbuf[(c + GR - 1) % GR][uc], G.w, z);
            z += sm.b1s[uc];
            const float h = lc ? act_fwd_t<A1>(z) : 0.f;
            TR(7);
            // W2[o][uc] (pre-update: R6), kept for δ1 below
            float wv[12];
            const int zs = c % ZS;
            {
                const float4* wq = reinterpret_cast<const float4*>(&sm.w2s[uc][0]);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const float4 f = wq[q];
                    wv[4 * q] = f.x; wv[4 * q + 1] = f.y; wv[4 * q + 2] = f.z; wv[4 * q + 3] = f.w;
                }
            }
            // ---- this warp's partial logits Σ_u W2[o][u] h_u: transpose-reduce over lanes ----
            float pv0;
            {
                float pv[16];
#pragma unroll
                for (int o = 0; o < 16; ++o) pv[o] = (o < O) ? wv[o < O ? o : 0] * h : 0.f;
                const bool c4 = lane & 16, c3 = lane & 8, c2 = lane & 4, c1 = lane & 2;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    pv[i] = (c4 ? pv[i + 8] : pv[i]) + __shfl_xor_sync(0xffffffffu, c4 ? pv[i] : pv[i + 8], 16);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    pv[i] = (c3 ? pv[i + 4] : pv[i]) + __shfl_xor_sync(0xffffffffu, c3 ? pv[i] : pv[i + 4], 8);
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    pv[i] = (c2 ? pv[i + 2] : pv[i]) + __shfl_xor_sync(0xffffffffu, c2 ? pv[i] : pv[i + 2], 4);
                pv0 = (c1 ? pv[1] : pv[0]) + __shfl_xor_sync(0xffffffffu, c1 ? pv[0] : pv[1], 2);
                pv0 += __shfl_xor_sync(0xffffffffu, pv0, 1);
            }
            TR(8);
            // lane l now holds output (l >> 1) = 8·c4 + 4·c3 + 2·c2 + c1
            {
                const int oi = lane >> 1;
                const bool pub = (lane & 1) == 0 && oi < O;
                if (pub) sm.zbuf[zs][zrow][oi] = pv0;
                if constexpr (C > 1) {
#pragma unroll
                    for (int p = 0; p < C - 1; ++p)
                        st_async_f32_if(pub, rz[p] + zs * kZStride + oi * 4, pv0,
                                        rz[p] + kZfullOff - (uint32_t)(zrow * 64) + zs * 8);
                }
                __syncwarp();
                if (lane == 0) {
                    if constexpr (C > 1) mbar_arrive_expect_tx(&sm.zfull[zs], (uint32_t)((C - 1) * O * 4));
                    else mbar_arrive(&sm.zfull[zs]);
                }
            }
            TR(9);
            // ---- while the exchange is in flight: certify x(c+2+L) for the sweeps' F(c+2+L),
            //      which comes after their wait on gready(c) (first warp of the pair) ----
            // every warp has passed U(c-1) (aready(c) above): the slot of x(c-1-L) is free for x(c+PF)
            TR(4);
            // ---- δ2(c) in every lane: z2 = Σ partials + b2(c) ----
            mbar_wait(&sm.zfull[zs], (uint32_t)((c / ZS) & 1));
            TR(5);
            float dl[O];
            {
                float z2[12];
                {
                    const float4* bq = reinterpret_cast<const float4*>(&sm.b2s[c & 1][0]);
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const float4 f = bq[q];
                        z2[4 * q] = f.x; z2[4 * q + 1] = f.y; z2[4 * q + 2] = f.z; z2[4 * q + 3] = f.w;
                    }
                }
                float zp[12];
#pragma unroll
                for (int o = 0; o < 12; ++o) zp[o] = 0.f;
#pragma unroll
                for (int i = 0; i < 2 * C; ++i) {
                    const float4* zq = reinterpret_cast<const float4*>(&sm.zbuf[zs][i][0]);
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const float4 f = zq[q];
                        zp[4 * q] += f.x; zp[4 * q + 1] += f.y; zp[4 * q + 2] += f.z; zp[4 * q + 3] += f.w;
                    }
                }
#pragma unroll
                for (int o = 0; o < 12; ++o) z2[o] += zp[o];                // z2 = W2 h + b2 (Eq.2)
                if constexpr (A2 == PNN_SOFTMAX) {
                    // max and sum as trees (O = 10: depth 4 instead of 9)
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
                    TR(10);
                } else {
                    // element-wise output (sigmoid / tanh, ½-SSE: Eq.9, R11): lane o forms output
                    // o's activation and δ2 once, then every lane takes the ten by shuffles
                    float zsel = z2[0];
#pragma unroll
                    for (int o = 1; o < O; ++o) zsel = (lane == o) ? z2[o] : zsel;
                    const float x2 = act_fwd_t<A2>(zsel);
                    const float dmine = (x2 - ((lane == label) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
#pragma unroll
                    for (int o = 0; o < O; ++o) dl[o] = __shfl_sync(0xffffffffu, dmine, o);
                }
            }
            // ---- δ1, g(c) of unit uc; W2(c+1), b1(c+1), b2(c+1) ----
            {
                float s1 = 0.f;                    // (W2ᵀδ2)_u with the pre-update W2 (R6)
#pragma unroll
                for (int o = 0; o < O; ++o) s1 = fmaf(wv[o], dl[o], s1);
                const float gu = lc ? lr * (s1 * act_deriv_t<A1>(h)) : 0.f;   // g(c) = η δ1
                sm.gbuf[c % GR][uc] = gu;
                TR(11);
                sm.b1s[uc] -= gu;
#pragma unroll
                for (int o = 0; o < O; ++o) wv[o] = fmaf(-(lr * dl[o]), h, wv[o]);
                float4* wq = reinterpret_cast<float4*>(&sm.w2s[uc][0]);
                wq[0] = make_float4(wv[0], wv[1], wv[2], wv[3]);
                wq[1] = make_float4(wv[4], wv[5], wv[6], wv[7]);
                wq[2] = make_float4(wv[8], wv[9], 0.f, 0.f);
            }
            if (half == kB2Half && lane == 0) {        // b2(c+1) into the other buffer: the pair's
                const float4* bo = reinterpret_cast<const float4*>(&sm.b2s[c & 1][0]);   // partner may
                float4* bq = reinterpret_cast<float4*>(&sm.b2s[(c + 1) & 1][0]);        // still read b2(c)
                const float4 b0 = bo[0], b1v = bo[1], b2v = bo[2];
                bq[0] = make_float4(fmaf(-lr, dl[0], b0.x), fmaf(-lr, dl[1], b0.y), fmaf(-lr, dl[2], b0.z),
                                    fmaf(-lr, dl[3], b0.w));
                bq[1] = make_float4(fmaf(-lr, dl[4], b1v.x), fmaf(-lr, dl[5], b1v.y), fmaf(-lr, dl[6], b1v.z),
                                    fmaf(-lr, dl[7], b1v.w));
                bq[2] = make_float4(fmaf(-lr, dl[8], b2v.x), fmaf(-lr, dl[9], b2v.y), 0.f, 0.f);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.gready[c % GR]);
                if (c + 1 < T) mbar_arrive(&sm.aready[(c + 1) % AR]);   // chain c+1 may start
            }
            // off the critical path: every warp has passed U(c-1) (aready(c) above), so the
            // slot of x(c-1-L) is free for x(c+PF); the sweeps wait for it themselves
            if (half == 0 && lane == 0 && c + PF < T) issue_x(c + PF, (cs + PF) % S);
            TR(6);
        }
        }
        // U after the chains: a chain then starts right after its warps' F
        TR(12);
        u_pair(p);
        TR(2);
    }
#undef TR

    // ---- write back ----
    float* W1o = opaque(W1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (kr0 + r < Uown) {
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
    __syncthreads();                               // the last chain's W2 / b1 / b2 are in shared memory
    float* W2o = opaque(W2);
    for (int i = threadIdx.x; i < Uown * O; i += blockDim.x) {
        const int u = i / O, o = i % O;
        W2o[(long long)o * H + k0 + u] = sm.w2s[u][o];
    }
    for (int i = threadIdx.x; i < Uown; i += blockDim.x) opaque(b1g)[k0 + i] = sm.b1s[i];
    if (crank == 0 && threadIdx.x < O) opaque(b2g)[threadIdx.x] = sm.b2s[T & 1][threadIdx.x];
    if constexpr (C > 1) cluster_sync_all();       // no CTA leaves while a peer may still st.async into it
}

// =====================================================================================
// v10: the per-sample chain on a dedicated CTA.  A cluster of NSW + 1 CTAs trains one
// CN: CTAs 0..NSW-1 hold U = ⌈H/NSW⌉ W¹ rows each in registers and only sweep (F, U as in
// v8, same lookahead R27); CTA NSW runs the chain for all H units (4 warps, one unit per
// lane: W², b1, b2 and the last L g's in registers).  Per sample the sweep CTAs send their
// row-sum parts to the chain CTA (st.async → its aready mbarrier) and the chain sends
// g(c) of each unit back to the owning sweep CTA (st.async → that CTA's gready).  The
// chain never shares an SM sub-partition with a sweep, and the sweeps never run chain
// code, so the period is max(sweep, chain) instead of their contended sum.
// paired sweeps (as v8's): F / U for two samples per pass, one complete row sum per unit
// sent to the chain CTA, 5 Gram corrections for odd samples
constexpr int RS = 16;               // chain CTA: Gram-record ring slots
constexpr int RPF = 8;               // records in flight
constexpr int SPF = S - 2 * LAG - 1; // sweep CTAs: x prefetch distance (slot provably free, see below)
static_assert(SPF >= 4, "x prefetch distance");

struct __align__(16) SplitSmem {
    uint64_t xfull[S];               // sweep: x(u) landed
    uint64_t gready[GR];             // sweep: g(u) of the CTA's rows landed (from the chain CTA)
    uint64_t aready[AR];             // chain: every sweep CTA's row-sum parts of sample c landed
    uint64_t rfull[RS];              // chain: Gram record of sample c landed
    float gbuf[GR][UMAX];            // sweep: g(u) of the CTA's rows
    float asum[AR][2 * UMAX][4];     // chain: [c % AR][unit][part]
    float zp[2][4][16];              // chain: [c & 1][warp][o] partial logits
    float4 rec[RS][2];               // chain: Gram terms of sample c, label
    float wx[NW][R][16];             // sweep: W¹ columns 768..783 of each warp's rows
};
constexpr size_t kSplitHead = ((sizeof(SplitSmem) + 127) / 128) * 128;

template <int NSW, int A1, int A2>
__global__ void __launch_bounds__(NW * 32, 1)
sgd_split_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                 const float4* __restrict__ rec, long long n_local, int K_local, int s_first, float lr) {
    extern __shared__ __align__(128) unsigned char smraw[];
    SplitSmem& sm = *reinterpret_cast<SplitSmem*>(smraw);
    float* xring = reinterpret_cast<float*>(smraw + kSplitHead);
    const int D = d.n[0], H = d.n[1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int crank = (int)cluster_rank();          // 0..NSW-1 sweep CTAs, NSW the chain CTA
    const int cn = s_first + (int)(blockIdx.x / (NSW + 1));
    const int U = (H + NSW - 1) / NSW;               // units per sweep CTA
    long long row0, T64;
    shard_of(n_local, K_local, cn, &row0, &T64);
    const int T = (int)T64;
    float* P = children + (long long)cn * d.P;
    float* W1 = P;
    float* b1g = P + (long long)H * D;
    float* W2 = b1g + H;
    float* b2g = W2 + (long long)O * H;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&sm.xfull[i], 1);
        for (int i = 0; i < GR; ++i) mbar_init(&sm.gready[i], 1);
        for (int i = 0; i < AR; ++i) mbar_init(&sm.aready[i], 1);
        for (int i = 0; i < RS; ++i) mbar_init(&sm.rfull[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();                            // every CTA's barriers exist before any st.async

    if (crank < NSW) {
        // ================= sweep CTA =================
        const int k0 = crank * U;
        const int Uown = max(0, min(U, H - k0));
        const float* Xc = X + row0 * (long long)D;
        const uint32_t xbytes = (uint32_t)D * 4u;
        auto issue_x = [&](int u) {
            const int slot = u % S;
            mbar_arrive_expect_tx(&sm.xfull[slot], xbytes);
            bulk_g2s(xring + slot * DP, Xc + (long long)u * D, xbytes, &sm.xfull[slot]);
        };
        for (int i = threadIdx.x; i < (S + 1) * DP; i += blockDim.x) xring[i] = 0.f;   // + zero row
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0)
            for (int u = 0; u < SPF && u < T; ++u) issue_x(u);
        const int kr0 = warp * R;
        uint64_t w[R][NP];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool live = kr0 + r < Uown;
            const float* src = W1 + (long long)(k0 + kr0 + r) * D;
#pragma unroll
            for (int m = 0; m < NP; ++m)
                w[r][m] = live ? *reinterpret_cast<const uint64_t*>(src + pcol(lane, m)) : 0ull;
        }
        const int tr = lane >> 2, tq = lane & 3;
        const int nx = D - XC - 4 * tq;
        const bool xlive = kr0 + tr < Uown;
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
        // where this lane's row-sum part lands in the chain CTA, and that CTA's aready
        const uint32_t apart = mapa(smem_u32(&sm.asum[0][k0 + kr0 + tr][tq]), (uint32_t)NSW);
        const uint32_t abar = mapa(smem_u32(&sm.aready[0]), (uint32_t)NSW);
        constexpr uint32_t kAStride = 2 * UMAX * 4 * 4;

        const int trow = lane >> 2, tsmp = (lane >> 1) & 1, th8 = lane & 1;
        const bool rlive = kr0 + trow < Uown;
        const uint32_t apart0 = mapa(smem_u32(&sm.asum[0][k0 + kr0 + trow][0]), (uint32_t)NSW);
        auto sweep_f2 = [&](int s0, bool v1) {
            const int s1 = s0 + 1;
            const int sl0 = s0 % S, sl1 = v1 ? s1 % S : S;    // slot S: the zero row
            mbar_wait(&sm.xfull[sl0], (uint32_t)((s0 / S) & 1));
            if (v1) mbar_wait(&sm.xfull[sl1], (uint32_t)((s1 / S) & 1));
            const float* xn0 = xring + sl0 * DP + 4 * lane;
            const float* xn1 = xring + sl1 * DP + 4 * lane;
            uint64_t acc0[R], acc1[R];
#pragma unroll
            for (int r = 0; r < R; ++r) { acc0[r] = 0ull; acc1[r] = 0ull; }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint64_t xa, xb, ya, yb;
                lds4(xn0 + 128 * q, xa, xb);
                lds4(xn1 + 128 * q, ya, yb);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    acc0[r] = ffma2(w[r][2 * q], xa, acc0[r]);
                    acc1[r] = ffma2(w[r][2 * q], ya, acc1[r]);
                    acc0[r] = ffma2(w[r][2 * q + 1], xb, acc0[r]);
                    acc1[r] = ffma2(w[r][2 * q + 1], yb, acc1[r]);
                }
            }
            float px;
            {
                const float* wt = &sm.wx[warp][trow][8 * th8];
                const float* xt = xring + (tsmp ? sl1 : sl0) * DP + XC + 8 * th8;
                const float4 w0 = *reinterpret_cast<const float4*>(wt), w1 = *reinterpret_cast<const float4*>(wt + 4);
                const float4 x0 = *reinterpret_cast<const float4*>(xt), x1 = *reinterpret_cast<const float4*>(xt + 4);
                px = w0.x * x0.x;
                px = fmaf(w0.y, x0.y, px); px = fmaf(w0.z, x0.z, px); px = fmaf(w0.w, x0.w, px);
                px = fmaf(w1.x, x1.x, px); px = fmaf(w1.y, x1.y, px); px = fmaf(w1.z, x1.z, px);
                px = fmaf(w1.w, x1.w, px);
            }
            float v[16];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float lo, hi;
                upk(acc0[r], lo, hi);
                v[2 * r] = lo + hi;
                upk(acc1[r], lo, hi);
                v[2 * r + 1] = lo + hi;
            }
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
            float zsum = (b1 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? u2[0] : u2[1], 2) + px;
            zsum += __shfl_xor_sync(0xffffffffu, zsum, 1);
            const int a = (tsmp ? s1 : s0) % AR;
            st_async_f32_if(rlive && th8 == 0 && (tsmp == 0 || v1), apart0 + (uint32_t)a * kAStride, zsum,
                            abar + (uint32_t)a * 8u);
        };
        auto sweep_u2 = [&](int u0, bool v1) {
            const int u1 = u0 + 1;
            mbar_wait(&sm.gready[u0 % GR], (uint32_t)((u0 / GR) & 1));
            if (v1) mbar_wait(&sm.gready[u1 % GR], (uint32_t)((u1 / GR) & 1));
            const int sl0 = u0 % S, sl1 = v1 ? u1 % S : S;
            const float* xo0 = xring + sl0 * DP + 4 * lane;
            const float* xo1 = xring + sl1 * DP + 4 * lane;
            float gp0[R], gp1[R];
            {
                const float4* g0v = reinterpret_cast<const float4*>(&sm.gbuf[u0 % GR][kr0]);
                const float4* g1v = reinterpret_cast<const float4*>(&sm.gbuf[u1 % GR][kr0]);
                const float4 a0 = g0v[0], a1 = g0v[1];
                float4 c0 = g1v[0], c1 = g1v[1];
                if (!v1) { c0 = make_float4(0.f, 0.f, 0.f, 0.f); c1 = c0; }
                gp0[0] = -a0.x; gp0[1] = -a0.y; gp0[2] = -a0.z; gp0[3] = -a0.w;
                gp0[4] = -a1.x; gp0[5] = -a1.y; gp0[6] = -a1.z; gp0[7] = -a1.w;
                gp1[0] = -c0.x; gp1[1] = -c0.y; gp1[2] = -c0.z; gp1[3] = -c0.w;
                gp1[4] = -c1.x; gp1[5] = -c1.y; gp1[6] = -c1.z; gp1[7] = -c1.w;
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                uint64_t xa, xb, ya, yb;
                lds4(xo0 + 128 * q, xa, xb);
                lds4(xo1 + 128 * q, ya, yb);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    w[r][2 * q] = ffma2(pk(gp0[r], gp0[r]), xa, w[r][2 * q]);
                    w[r][2 * q + 1] = ffma2(pk(gp0[r], gp0[r]), xb, w[r][2 * q + 1]);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    w[r][2 * q] = ffma2(pk(gp1[r], gp1[r]), ya, w[r][2 * q]);
                    w[r][2 * q + 1] = ffma2(pk(gp1[r], gp1[r]), yb, w[r][2 * q + 1]);
                }
            }
            __syncwarp();                          // F's tail reads of wx are done
            float4 w4 = *reinterpret_cast<const float4*>(wxp);
            const float4 x4 = *reinterpret_cast<const float4*>(xring + sl0 * DP + XC + 4 * tq);
            const float4 y4 = *reinterpret_cast<const float4*>(xring + sl1 * DP + XC + 4 * tq);
            const float ga = -sm.gbuf[u0 % GR][kr0 + tr], gb = v1 ? -sm.gbuf[u1 % GR][kr0 + tr] : 0.f;
            w4.x = fmaf(ga, x4.x, w4.x); w4.y = fmaf(ga, x4.y, w4.y);
            w4.z = fmaf(ga, x4.z, w4.z); w4.w = fmaf(ga, x4.w, w4.w);
            w4.x = fmaf(gb, y4.x, w4.x); w4.y = fmaf(gb, y4.y, w4.y);
            w4.z = fmaf(gb, y4.z, w4.z); w4.w = fmaf(gb, y4.w, w4.w);
            *reinterpret_cast<float4*>(wxp) = w4;
            __syncwarp();
        };
        const int npair = (T + 1) >> 1;
        for (int p = 0; p < npair + 2; ++p) {
            const int s0 = 2 * p;
            if (threadIdx.x == 0) {                // g(2p), g(2p+1) of this CTA's rows will arrive
                if (s0 < T) mbar_arrive_expect_tx(&sm.gready[s0 % GR], 4u * (uint32_t)Uown);
                if (s0 + 1 < T) mbar_arrive_expect_tx(&sm.gready[(s0 + 1) % GR], 4u * (uint32_t)Uown);
            }
            if (p < npair) sweep_f2(s0, s0 + 1 < T);
            if (p >= 2 && 2 * (p - 2) < T) sweep_u2(2 * (p - 2), 2 * (p - 2) + 1 < T);
            // x(2p+SPF), x(2p+1+SPF) go to the slots of x(2p-9), x(2p-8): thread 0 waited
            // gready(2p-3) above, so every warp sent its F parts of 2p-3, after its U of ≤ 2p-5
            if (threadIdx.x == 0) {
                if (s0 + SPF < T) issue_x(s0 + SPF);
                if (s0 + 1 + SPF < T) issue_x(s0 + 1 + SPF);
            }
        }
        float* W1o = opaque(W1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (kr0 + r < Uown) {
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
    } else if (warp < 4) {
        // ================= chain CTA: unit u = 32·warp + lane =================
        const int u = 32 * warp + lane;
        const bool lc = u < H;
        const int sr = lc ? u / U : 0;             // owning sweep CTA and its row
        const int r = u - sr * U;
        float w2[O], b2[O];
#pragma unroll
        for (int o = 0; o < O; ++o) {
            w2[o] = lc ? W2[(long long)o * H + u] : 0.f;
            b2[o] = b2g[o];
        }
        float b1 = lc ? b1g[u] : 0.f;
        float g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f, g5 = 0.f;   // g(c-1) .. g(c-5) of this unit
        const uint32_t gdst = mapa(smem_u32(&sm.gbuf[0][r]), (uint32_t)sr);
        const uint32_t gbar = mapa(smem_u32(&sm.gready[0]), (uint32_t)sr);
        const float4* Rc = rec + 2 * row0;
        auto issue_rec = [&](int c) {
            const int slot = c % RS;
            mbar_arrive_expect_tx(&sm.rfull[slot], 32u);
            bulk_g2s(&sm.rec[slot][0], Rc + 2 * c, 32u, &sm.rfull[slot]);
        };
        if (threadIdx.x == 0)
            for (int c = 0; c < RPF && c < T; ++c) issue_rec(c);
        for (int c = 0; c < T; ++c) {
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&sm.aready[c % AR], 4u * (uint32_t)H);   // parts of every unit
                if (c + RPF < T) issue_rec(c + RPF);      // its slot held rec(c+RPF-RS): consumed
            }
            mbar_wait(&sm.rfull[c % RS], (uint32_t)((c / RS) & 1));
            const float4 G = sm.rec[c % RS][0];
            const int label = __float_as_int(sm.rec[c % RS][1].x);
            mbar_wait(&sm.aready[c % AR], (uint32_t)((c / AR) & 1));
            // ---- z1(c) = acc - Σ_k g(c-k) G(c-k,c) + b1(c) (R27), h(c) ----
            const float4 pa = *reinterpret_cast<const float4*>(&sm.asum[c % AR][u][0]);
            float z = pa.x;
            if (c & 1) z = fmaf(-g5, sm.rec[c % RS][1].y, z);
            z = fmaf(-g4, G.x, z);
            z = fmaf(-g3, G.y, z);
            z = fmaf(-g2, G.z, z);
            z = fmaf(-g1, G.w, z);
            z += b1;
            const float h = lc ? act_fwd_t<A1>(z) : 0.f;
            // ---- this warp's partial logits: transpose-reduce over lanes ----
            float pv0;
            {
                float pv[16];
#pragma unroll
                for (int o = 0; o < 16; ++o) pv[o] = (o < O) ? w2[o < O ? o : 0] * h : 0.f;
                const bool c4 = lane & 16, c3 = lane & 8, c2 = lane & 4, c1 = lane & 2;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    pv[i] = (c4 ? pv[i + 8] : pv[i]) + __shfl_xor_sync(0xffffffffu, c4 ? pv[i] : pv[i + 8], 16);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    pv[i] = (c3 ? pv[i + 4] : pv[i]) + __shfl_xor_sync(0xffffffffu, c3 ? pv[i] : pv[i + 4], 8);
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    pv[i] = (c2 ? pv[i + 2] : pv[i]) + __shfl_xor_sync(0xffffffffu, c2 ? pv[i] : pv[i + 2], 4);
                pv0 = (c1 ? pv[1] : pv[0]) + __shfl_xor_sync(0xffffffffu, c1 ? pv[0] : pv[1], 2);
                pv0 += __shfl_xor_sync(0xffffffffu, pv0, 1);
            }
            if ((lane & 1) == 0 && (lane >> 1) < O) sm.zp[c & 1][warp][lane >> 1] = pv0;
            named_bar_sync(1, 128);                // the 4 warps' partials of sample c
            // ---- δ2(c) in every lane ----
            float dl[O];
            {
                float z2[O];
#pragma unroll
                for (int o = 0; o < O; ++o) z2[o] = 0.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (i < (H + 31) / 32) {
#pragma unroll
                        for (int o = 0; o < O; ++o) z2[o] += sm.zp[c & 1][i][o];
                    }
                }
#pragma unroll
                for (int o = 0; o < O; ++o) z2[o] = b2[o] + z2[o];        // z2 = W2 h + b2 (Eq.2)
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
                    // element-wise output (sigmoid / tanh, ½-SSE: Eq.9, R11): lane o forms output
                    // o's activation and δ2 once, then every lane takes the ten by shuffles
                    float zsel = z2[0];
#pragma unroll
                    for (int o = 1; o < O; ++o) zsel = (lane == o) ? z2[o] : zsel;
                    const float x2 = act_fwd_t<A2>(zsel);
                    const float dmine = (x2 - ((lane == label) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
#pragma unroll
                    for (int o = 0; o < O; ++o) dl[o] = __shfl_sync(0xffffffffu, dmine, o);
                }
            }
            // ---- δ1, g(c) → the owning sweep CTA; W2, b1, b2 updates (registers) ----
            float s1 = 0.f;                        // (W2ᵀδ2)_u with the pre-update W2 (R6)
#pragma unroll
            for (int o = 0; o < O; ++o) s1 = fmaf(w2[o], dl[o], s1);
            const float gu = lc ? lr * (s1 * act_deriv_t<A1>(h)) : 0.f;
            if (lc) st_async_f32(gdst + (uint32_t)(c % GR) * (uint32_t)(UMAX * 4), gu, gbar + (uint32_t)(c % GR) * 8u);
            b1 -= gu;
#pragma unroll
            for (int o = 0; o < O; ++o) {
                w2[o] = fmaf(-(lr * dl[o]), h, w2[o]);
                b2[o] = fmaf(-lr, dl[o], b2[o]);
            }
            g5 = g4; g4 = g3; g3 = g2; g2 = g1; g1 = gu;
        }
        if (lc) {
#pragma unroll
            for (int o = 0; o < O; ++o) opaque(W2)[(long long)o * H + u] = w2[o];
            opaque(b1g)[u] = b1;
        }
        if (u == 0) {
#pragma unroll
            for (int o = 0; o < O; ++o) opaque(b2g)[o] = b2[o];
        }
    }
    cluster_sync_all();                            // no CTA leaves while a peer may still st.async into it
}

template <int NSW, int A1, int A2>
cudaError_t launch_split_one(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                             const float4* rec, long long n_local, int K_local, int s_first, int s_count,
                             float lr, cudaStream_t st) {
    auto kern = sgd_split_kernel<NSW, A1, A2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(s_count * (NSW + 1)));
    cfg.blockDim = dim3((unsigned)p.threads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = NSW + 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, d, children, x, rec, n_local, K_local, s_first, lr);
}

template <int NSW>
cudaError_t launch_split(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                         const float4* rec, long long n_local, int K_local, int s_first, int s_count,
                         float lr, cudaStream_t st) {
#define PNN_SPLIT_ACTS(A1_, A2_)                                                                   \
    if (d.act[0] == A1_ && d.act[1] == A2_)                                                      \
        return launch_split_one<NSW, A1_, A2_>(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
    PNN_SPLIT_ACTS(PNN_RELU, PNN_SOFTMAX)
    PNN_SPLIT_ACTS(PNN_TANH, PNN_SOFTMAX)
    PNN_SPLIT_ACTS(PNN_SIGMOID, PNN_SOFTMAX)
    PNN_SPLIT_ACTS(PNN_SIGMOID, PNN_SIGMOID)
    PNN_SPLIT_ACTS(PNN_TANH, PNN_TANH)
    PNN_SPLIT_ACTS(PNN_RELU, PNN_SIGMOID)
    PNN_SPLIT_ACTS(PNN_LEAKY_RELU, PNN_SOFTMAX)
#undef PNN_SPLIT_ACTS
    return cudaErrorInvalidValue;
}

template <int C, int A1, int A2, bool TRACE>
cudaError_t launch_one(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                       const float4* rec, long long n_local, int K_local, int s_first, int s_count,
                       float lr, cudaStream_t st) {
    auto kern = sgd_resident_kernel<C, A1, A2, TRACE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(s_count * C));
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
    return cudaLaunchKernelEx(&cfg, kern, d, children, x, rec, n_local, K_local, s_first, lr, g_trace);
}

template <int C>
cudaError_t launch_c(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                     const float4* rec, long long n_local, int K_local, int s_first, int s_count,
                     float lr, cudaStream_t st) {
#define PNN_ACTS(A1_, A2_)                                                                        \
    if (d.act[0] == A1_ && d.act[1] == A2_)                                                     \
        return g_trace ? launch_one<C, A1_, A2_, true>(p, d, children, x, rec, n_local, K_local, s_first, \
                                                       s_count, lr, st)                           \
                       : launch_one<C, A1_, A2_, false>(p, d, children, x, rec, n_local, K_local, s_first, \
                                                        s_count, lr, st);
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

}  // namespace

// The Gram-record pre-pass, for other kernels that use the same lookahead (k_deep.cu).
cudaError_t launch_gram(const float* x, const int32_t* labels, int D, long long n_local, int K_local, int s_first,
                        int s_count, float4* rec, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    return gram_launch(x, labels, D, n_local, K_local, s_first, s_count, rec, st);
}

ResidentPlan plan_resident(const NetDesc& d, int batch, int concurrent, int variant) {
    ResidentPlan p{};
    auto no = [&](const char* why) {
        p.ok = false;
        snprintf(p.why, sizeof p.why, "%s", why);
        return p;
    };
    if (variant != PNN_VARIANT_AUTO && variant != PNN_VARIANT_RESIDENT_V8 && variant != PNN_VARIANT_RESIDENT_V10 &&
        variant != PNN_VARIANT_RESIDENT_TMEM && variant != PNN_VARIANT_RESIDENT_WS)
        return no("not a resident-kernel variant");
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
                       (a1 == PNN_TANH && a2 == PNN_TANH) || (a1 == PNN_RELU && a2 == PNN_SIGMOID) ||
                       (a1 == PNN_LEAKY_RELU && a2 == PNN_SOFTMAX);
    if (!built) return no("activation pair not instantiated in the resident kernel");
    int c = 1;
    while (c <= CMAX && (H + c - 1) / c > UMAX) c *= 2;
    if (c > CMAX) return no("hidden layer wider than 256");
    // v11 (k_tmem.cu): one SM per CN, W1 in registers + tensor memory, no cross-SM exchange
    // and no Gram pre-pass; H <= 128.
    const bool tm_ok = tmem_plan(d, batch) == nullptr;
    // v10 (the chain on its own CTA) for H <= 128: 1 or 2 sweep CTAs + 1 chain CTA.  It costs one
    // SM more per CN but shortens the per-sample period: measured faster when every CN runs at
    // once (C2 +11 %, C1 +5 %), slower when the SMs are the limit.  AUTO takes it
    // when `concurrent` CNs × its cluster fit (≤ 120 SMs: 3-CTA clusters do not all fit 148 SMs
    // at once; K = 48 measured slower than v8).
    const int c10 = (H + UMAX - 1) / UMAX + 1;
    const bool v10_ok = H <= 2 * UMAX;
    int v = variant;
    if (v == PNN_VARIANT_AUTO) {
        if (v10_ok && concurrent > 0 && (long long)concurrent * c10 <= 120) v = PNN_VARIANT_RESIDENT_V10;
        else if (ws_plan(d, batch) == nullptr) v = PNN_VARIANT_RESIDENT_WS;   // v12: C4 83 M vs v11 67 M samples/s
        else if (tm_ok) v = PNN_VARIANT_RESIDENT_TMEM;
        else v = PNN_VARIANT_RESIDENT_V8;
    }
    if (v == PNN_VARIANT_RESIDENT_TMEM && !tm_ok) return no("TMEM variant: hidden layer wider than 128");
    if (v == PNN_VARIANT_RESIDENT_WS && ws_plan(d, batch) != nullptr) return no("WS variant: hidden layer wider than 128");
    if (v == PNN_VARIANT_RESIDENT_V10 && !v10_ok) return no("v10 variant: hidden layer wider than 128");
    p.groups = 1;
    p.threads = NW * 32;                           // 8 warps; rows >= U are idle
    if (v == PNN_VARIANT_RESIDENT_V8) {
        p.variant = 8;
        p.cluster = c;
        p.smem = kSmemHead + sizeof(float) * (size_t)(S + 1) * DP;
    } else if (v == PNN_VARIANT_RESIDENT_V10) {
        p.variant = 10;
        p.cluster = c10;
        p.smem = kSplitHead + sizeof(float) * (size_t)(S + 1) * DP;   // + the zero row (paired sweeps)
    } else if (v == PNN_VARIANT_RESIDENT_WS) {
        p.variant = 12;
        p.cluster = 1;
        p.threads = 384;
        p.smem = 0;                                // sized by launch_sgd_ws
    } else {
        p.variant = 11;
        p.cluster = 1;
        p.smem = 0;                                // sized by launch_sgd_tmem
    }
    p.ok = true;
    return p;
}

static cudaError_t launch_sgd_resident_only(const ResidentPlan& p, const NetDesc& d, float* children,
                                            const float* x, const float4* rec, long long n_local, int K_local,
                                            int s_first, int s_count, float lr, cudaStream_t st);

cudaError_t launch_sgd_resident(const ResidentPlan& p, const NetDesc& d, float* children,
                                const float* x, const int32_t* labels, float4* rec, long long n_local,
                                int K_local, int s_first, int s_count, float lr, cudaStream_t st,
                                cudaEvent_t ev0, cudaEvent_t ev1) {
    if (s_count <= 0) return cudaSuccess;
    cudaError_t e;
    if (p.variant == 11) {                         // v11 forms its Gram terms in the launch
        if (ev0 && (e = cudaEventRecord(ev0, st)) != cudaSuccess) return e;
        e = launch_sgd_tmem(d, children, x, labels, n_local, K_local, s_first, s_count, lr, st);
        if (e != cudaSuccess || !ev1) return e;
        return cudaEventRecord(ev1, st);
    }
    e = gram_launch(x, labels, d.n[0], n_local, K_local, s_first, s_count, rec, st);
    if (e != cudaSuccess) return e;
    if (ev0) {                                     // timing hook: bracket the SGD launch only
        if ((e = cudaEventRecord(ev0, st)) != cudaSuccess) return e;
        e = launch_sgd_resident_only(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
        if (e != cudaSuccess) return e;
        return cudaEventRecord(ev1, st);
    }
    return launch_sgd_resident_only(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
}

static cudaError_t launch_sgd_resident_only(const ResidentPlan& p, const NetDesc& d, float* children,
                                            const float* x, const float4* rec, long long n_local, int K_local,
                                            int s_first, int s_count, float lr, cudaStream_t st) {
    if (p.variant == 12) return launch_sgd_ws(d, children, x, nullptr, rec, n_local, K_local, s_first, s_count, lr, st);
    if (p.variant == 10) {
        if (p.cluster == 2) return launch_split<1>(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
        if (p.cluster == 3) return launch_split<2>(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
        return cudaErrorInvalidValue;
    }
    switch (p.cluster) {
    case 1: return launch_c<1>(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
    case 2: return launch_c<2>(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
    case 4: return launch_c<4>(p, d, children, x, rec, n_local, K_local, s_first, s_count, lr, st);
    default: return cudaErrorInvalidValue;
    }
}
