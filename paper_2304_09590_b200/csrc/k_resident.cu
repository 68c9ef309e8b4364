// k_resident.cu — persistent per-sample SGD with register-resident weights.
//
// One thread-block cluster of C CTAs trains one child network (CN) over its
// whole slice ("Each child-network learns only a slice").  The
// hidden layer is split across the C SMs: CTA r owns hidden units
// [r·U, r·U+U), U = ceil(H/C) <= 32, and keeps those W^1 rows in REGISTERS
// for the whole launch (loaded once, written back once).  Scope: 2-layer nets
// D-H-O with 768 < D <= 800 and O = 10, per-instance SGD.
//
// Per sample, in the paper's sequential order (§3, Eqs.2-13):
//   z1 = W1 x + b1, h = φ1(z1); z2 = W2 h + b2, x2 = φ2(z2)         (Eqs.2-5)
//   δ2 = x2 - e (softmax+CE, Eq.10) or (x2 - e)⊙φ2'(x2) (R11)       (Eqs.9-10)
//   δ1 = (W2ᵀ δ2) ⊙ φ1'(h), with the pre-update W2 (R6)              (Eq.11)
//   W -= η δ xᵀ, b -= η δ                                             (Eqs.12-13)
//
// Warp roles in a CTA (NPW pass warps, 1 tail warp, 1 helper warp):
//   * pass warps hold W1: R = 8 rows per warp, lane j owns columns j, j+32,
//     ... (conflict-free LDS.32 of x, rows reduced by warp shuffles).  Pass
//     P_t does, per weight, the update of sample t-2 and the forward of
//     sample t in one register sweep
//         w -= g(t-2)·x(t-2)_j ;  acc += w·x(t)_j          ⇒ acc(t) = W1(t-1)·x(t)
//   * the tail warp (lane k = hidden unit k) finishes sample t while the
//     pass warps already sweep sample t+1.  Because W1(t) = W1(t-1) -
//     g(t-1)·x(t-1)ᵀ, the exact pre-activation is recovered as
//         z1(t) = acc(t) - g(t-1)·G(t-1,t) + b1(t),   G(t-1,t) = x(t-1)·x(t)
//     (the lookahead-corrected forward of SURVEY.md §7 hard part 2(ii): the
//     same number in real arithmetic; only the rounding differs from the
//     oracle's direct W1(t)·x(t)).  The tail then computes h, the partial
//     logits of its U units (warp reduce-scatter), exchanges them with every
//     peer CTA (st.async into the peer's shared memory, completing the
//     peer's mbarrier), and every lane redundantly evaluates the output
//     layer (softmax / sigmoid, δ2, b2 update) so no broadcast is needed;
//     then δ1, the W2-column update and g1 = η·δ1 for the pass warps.
//   * the helper warp streams x rows HBM→SMEM with 1-D bulk copies
//     (cp.async.bulk + mbarrier complete_tx) PF samples ahead into an S-slot
//     ring, computes G(t-1,t) for the tail and stages the labels.
// All hand-offs are mbarriers; nothing in the loop uses __syncthreads.  Each
// critical-path wait costs ~100 cycles even when already satisfied, so the
// helper's "x(t+2) landed, G(t+1,t+2) written" signal rides on the tail's
// accfull(t) barrier (NPW + 1 arrivals); g(t) published by the tail thus
// also certifies x(t+2) for pass P_{t+2}, which needs no x wait of its own.
#include <cstdio>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"

long long* g_trace = nullptr;   // debug: clock64 timeline (tools/trace_resident.py)
extern "C" void pnn_debug_set_trace(long long* dev_buf) { g_trace = dev_buf; }

// Critical-path waits: suspending try_wait (default) or polling test_wait.
#ifndef PNN_SPIN_PASS
#define PNN_SPIN_PASS 0
#endif
#ifndef PNN_SPIN_TAIL
#define PNN_SPIN_TAIL 0
#endif
#define PNN_PASS_WAIT(b, p) (PNN_SPIN_PASS ? ptx::mbar_wait_spin(b, p) : ptx::mbar_wait(b, p))
#define PNN_TAIL_WAIT(b, p) (PNN_SPIN_TAIL ? ptx::mbar_wait_spin(b, p) : ptx::mbar_wait(b, p))

namespace {

using namespace ptx;

constexpr int R = 8;          // W1 rows per pass warp
constexpr int MAXPW = 4;      // pass warps per CTA (U <= 32)
constexpr int S = 12;         // x ring slots
constexpr int PF = 6;         // prefetch distance
constexpr int OP = 16;        // outputs padded to 16 in the reduce-scatter
constexpr int CMAX = 8;       // cluster size (portable)
constexpr int kTraceT = 64, kTraceP = 16;

struct __align__(16) Smem {
    uint64_t xfull[S];        // helper → pass/helper: x(t) landed        (tx bytes)
    uint64_t xempty[S];       // pass → helper: slot free again            (NPW arrivals)
    uint64_t accfull[S];      // pass + helper → tail: acc(t) ready, and x(t+2)/G(t+1,t+2)
                              // staged by the helper                      (NPW + 1 arrivals)
    uint64_t gfull[2];        // tail → pass: g(t) ready                   (1 arrival)
    uint64_t lgfull[2];       // peers → tail: partial logits of sample t  (tx bytes)
    float acc[2][32];
    float g[2][32];
    float gram[S];
    int32_t ylab[2][32];
    __align__(16) float logits[2][CMAX][OP];
};

template <int M, int O, int C, int A1, int A2, bool TRACE>
__global__ void __launch_bounds__((MAXPW + 2) * 32, 1)
sgd_resident_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                    const int32_t* __restrict__ Y, long long n_local, int K_local, int s_first,
                    float lr, int npw, long long* __restrict__ trace) {
    constexpr int DP = 32 * M;
    extern __shared__ __align__(128) unsigned char smraw[];
    Smem& sm = *reinterpret_cast<Smem*>(smraw);
    float* xring = reinterpret_cast<float*>(smraw + ((sizeof(Smem) + 127) / 128) * 128);

    const int D = d.n[0], H = d.n[1];
    const int crank = (int)cluster_rank();
    const int cn = s_first + (int)(blockIdx.x / C);
    const int U = (H + C - 1) / C;                 // units per CTA
    const int k0 = crank * U;                      // first hidden unit of this CTA
    const int Uown = max(0, min(U, H - k0));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    long long row0, T;
    shard_of(n_local, K_local, cn, &row0, &T);
    const int Ti = (int)T;
    float* P = children + (long long)cn * d.P;
    float* W1 = P;
    float* b1g = P + (long long)H * D;
    float* W2 = b1g + H;
    float* b2g = W2 + (long long)O * H;

#define TR(pt)                                                                                \
    do {                                                                                      \
        if constexpr (TRACE) {                                                                \
            if (blockIdx.x < 4 && t < kTraceT && lane == 0)                                   \
                trace[((int)blockIdx.x * kTraceT + t) * kTraceP + (pt)] = ptx::clock64();     \
        }                                                                                     \
    } while (0)

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&sm.xfull[i], 1);
            mbar_init(&sm.xempty[i], npw);
            mbar_init(&sm.accfull[i], npw + 1);
            sm.gram[i] = 0.f;
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.gfull[i], 1);
            mbar_init(&sm.lgfull[i], 1);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < S * DP; i += blockDim.x) xring[i] = 0.f;   // pad columns stay 0
    fence_proxy_async_smem();
    __syncthreads();
    if constexpr (C > 1) cluster_sync_all();   // peers' barriers exist before any st.async

    if (warp < npw) {
        // ================================ pass warps ================================
        float w[R][M];
        const int kr0 = warp * R;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int kl = kr0 + r;
            const bool live = kl < Uown;
            const float* src = W1 + (long long)(k0 + kl) * D;
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const int j = lane + 32 * m;
                w[r][m] = (live && j < D) ? src[j] : 0.f;
            }
        }
        int sn = 0, so = S - 2;                    // ring slots of x(t), x(t-2)
        uint32_t xpar = 0;
        for (int t = 0; t < Ti + 2; ++t) {
            if (warp == 0) TR(8);
            float g[R];
#pragma unroll
            for (int r = 0; r < R; ++r) g[r] = 0.f;
            if (t >= 2) {
                PNN_PASS_WAIT(&sm.gfull[t & 1], (uint32_t)(((t - 2) >> 1) & 1));   // g(t-2)
                const float4* gv = reinterpret_cast<const float4*>(&sm.g[t & 1][kr0]);
                const float4 ga = gv[0], gb = gv[1];
                g[0] = ga.x; g[1] = ga.y; g[2] = ga.z; g[3] = ga.w;
                g[4] = gb.x; g[5] = gb.y; g[6] = gb.z; g[7] = gb.w;
            }
            if (warp == 0) TR(9);
            const float* xo = xring + so * DP + lane;                 // x(t-2)
            if (t < Ti) {
                if (t < 2) mbar_wait(&sm.xfull[sn], xpar);   // later: certified by g(t-2)
                if (warp == 0) TR(10);
                const float* xn = xring + sn * DP + lane;             // x(t)
                float acc[R];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = 0.f;
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    const float xnm = xn[32 * m];
                    const float xom = (t >= 2) ? xo[32 * m] : 0.f;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        w[r][m] = fmaf(-g[r], xom, w[r][m]);
                        acc[r] = fmaf(w[r][m], xnm, acc[r]);
                    }
                }
                if (warp == 0) TR(11);
                // transpose-reduce 8 row sums over 32 lanes (4+2+1+1+1 shuffles);
                // afterwards lane l (l % 4 == 0) holds row (l >> 2)
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                float u4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    u4[i] = (b4 ? acc[i + 4] : acc[i]) +
                            __shfl_xor_sync(0xffffffffu, b4 ? acc[i] : acc[i + 4], 16);
                float u2[2];
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    u2[i] = (b3 ? u4[i + 2] : u4[i]) +
                            __shfl_xor_sync(0xffffffffu, b3 ? u4[i] : u4[i + 2], 8);
                float v = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                if ((lane & 3) == 0) sm.acc[t & 1][kr0 + (lane >> 2)] = v;
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.accfull[sn]);
                if (warp == 0) TR(12);
            } else if (t >= 2) {
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    const float xom = xo[32 * m];
#pragma unroll
                    for (int r = 0; r < R; ++r) w[r][m] = fmaf(-g[r], xom, w[r][m]);
                }
            }
            if (t >= 2) {                          // last use of x(t-2) by this warp
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.xempty[so]);
            }
            so = (so + 1 == S) ? 0 : so + 1;
            if (++sn == S) { sn = 0; xpar ^= 1u; }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int kl = kr0 + r;
            if (kl < Uown) {
                float* dst = W1 + (long long)(k0 + kl) * D;
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    const int j = lane + 32 * m;
                    if (j < D) dst[j] = w[r][m];
                }
            }
        }
    } else if (warp == npw) {
        // ================================= tail warp =================================
        const int k = lane;
        const bool unit = k < Uown;
        float w2[O];
#pragma unroll
        for (int o = 0; o < O; ++o) w2[o] = unit ? W2[(long long)o * H + k0 + k] : 0.f;
        float b1 = unit ? b1g[k0 + k] : 0.f;
        float b2[O];                               // every lane (and every CTA) keeps all of b2
#pragma unroll
        for (int o = 0; o < O; ++o) b2[o] = b2g[o];
        float gprev = 0.f;
        // DSMEM addresses of logits[ts][crank][0] and lgfull[ts] in every peer
        // (the peer's window is linear: slot ts adds ts·kLgStride / ts·8 bytes)
        constexpr uint32_t kLgStride = CMAX * OP * 4;
        uint32_t rlg[C > 1 ? C - 1 : 1], rbar[C > 1 ? C - 1 : 1];
        if constexpr (C > 1) {
#pragma unroll
            for (int r = 1; r < C; ++r) {
                const uint32_t peer = (uint32_t)((crank + r) % C);
                rlg[r - 1] = mapa(smem_u32(&sm.logits[0][crank][0]), peer);
                rbar[r - 1] = mapa(smem_u32(&sm.lgfull[0]), peer);
            }
        }
        int as = 0;
        uint32_t apar = 0;
        for (int t = 0; t < Ti; ++t) {
            const int ts = t & 1;
            const uint32_t par = (uint32_t)((t >> 1) & 1);
            TR(0);
            if constexpr (C > 1)
                if (lane == 0) mbar_arrive_expect_tx(&sm.lgfull[ts], (uint32_t)((C - 1) * O * 4));
            PNN_TAIL_WAIT(&sm.accfull[as], apar);
            TR(1);
            const float a = sm.acc[ts][k];
            const float G = sm.gram[as];
            const int label = sm.ylab[(t >> 5) & 1][t & 31];
            if (++as == S) { as = 0; apar ^= 1u; }
            // z1(t) = W1(t-1)x(t) - g(t-1)·G(t-1,t) + b1(t),  b1(t) = b1(t-1) - g(t-1)
            b1 -= gprev;
            const float z1 = fmaf(-gprev, G, a) + b1;
            const float h = unit ? act_fwd_t<A1>(z1) : 0.f;
            // partial logits of this CTA's units: reduce-scatter 16 (O used) values over 32 lanes
            float v[OP];
#pragma unroll
            for (int o = 0; o < OP; ++o) v[o] = (o < O) ? w2[o < O ? o : 0] * h : 0.f;
            const bool b4 = lane & 16, b3 = lane & 8, b2b = lane & 4, b1b = lane & 2;
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
                u2[i] = (b2b ? u4[i + 2] : u4[i]) + __shfl_xor_sync(0xffffffffu, b2b ? u4[i] : u4[i + 2], 4);
            float u1 = (b1b ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b1b ? u2[0] : u2[1], 2);
            u1 += __shfl_xor_sync(0xffffffffu, u1, 1);
            const int idx = (lane >> 1) & 15;      // output index this lane now holds
            TR(2);
            if ((lane & 1) == 0 && idx < O) {
                sm.logits[ts][crank][idx] = u1;
                if constexpr (C > 1) {
#pragma unroll
                    for (int r = 0; r < C - 1; ++r)
                        st_async_f32(rlg[r] + ts * kLgStride + idx * 4, u1, rbar[r] + ts * 8);
                }
            }
            __syncwarp();
            TR(3);
            if constexpr (C > 1) PNN_TAIL_WAIT(&sm.lgfull[ts], par);
            TR(4);
            // output layer, evaluated redundantly (identically) by every lane
            float z2[O];
#pragma unroll
            for (int o = 0; o < O; ++o) z2[o] = 0.f;
#pragma unroll
            for (int r = 0; r < C; ++r) {
                const float4* lr4 = reinterpret_cast<const float4*>(&sm.logits[ts][r][0]);
                float lv[12];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const float4 f = lr4[q];
                    lv[4 * q] = f.x; lv[4 * q + 1] = f.y; lv[4 * q + 2] = f.z; lv[4 * q + 3] = f.w;
                }
#pragma unroll
                for (int o = 0; o < O; ++o) z2[o] += lv[o];
            }
#pragma unroll
            for (int o = 0; o < O; ++o) z2[o] += b2[o];          // z2 = W2 h + b2 (Eq.2 order)
            float d2[O];
            if constexpr (A2 == PNN_SOFTMAX) {
                float m = z2[0];
#pragma unroll
                for (int o = 1; o < O; ++o) m = (z2[o] > m) ? z2[o] : m;
                float e[O], s = 0.f;
#pragma unroll
                for (int o = 0; o < O; ++o) { e[o] = __expf(z2[o] - m); s += e[o]; }
                const float inv = __frcp_rn(s);
#pragma unroll
                for (int o = 0; o < O; ++o) d2[o] = e[o] * inv - ((o == label) ? 1.f : 0.f);
            } else {
#pragma unroll
                for (int o = 0; o < O; ++o) {
                    const float x2 = act_fwd_t<A2>(z2[o]);
                    d2[o] = (x2 - ((o == label) ? 1.f : 0.f)) * act_deriv_t<A2>(x2);
                }
            }
            TR(5);
            float s1 = 0.f;                        // (W2ᵀδ2)_k ascending o, pre-update W2 (R6)
#pragma unroll
            for (int o = 0; o < O; ++o) {
                b2[o] -= lr * d2[o];
                s1 = fmaf(w2[o], d2[o], s1);
                w2[o] = fmaf(-(lr * d2[o]), h, w2[o]);
            }
            const float g1 = unit ? lr * (s1 * act_deriv_t<A1>(h)) : 0.f;
            sm.g[ts][k] = g1;
            gprev = g1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.gfull[ts]);
            TR(6);
        }
        b1 -= gprev;                               // b1(T) = b1(T-1) - g(T-1)
        if (unit) {
#pragma unroll
            for (int o = 0; o < O; ++o) W2[(long long)o * H + k0 + k] = w2[o];
            b1g[k0 + k] = b1;
        }
        if (crank == 0 && lane == 0)
#pragma unroll
            for (int o = 0; o < O; ++o) b2g[o] = b2[o];
    } else {
        // ================================ helper warp ================================
        const uint32_t xbytes = (uint32_t)D * 4u;
        auto issue_x = [&](int u) {
            const int slot = u % S;
            mbar_arrive_expect_tx(&sm.xfull[slot], xbytes);
            bulk_g2s(xring + slot * DP, X + (row0 + u) * (long long)D, xbytes, &sm.xfull[slot]);
        };
        if (lane == 0)
            for (int u = 0; u < PF && u < Ti; ++u) issue_x(u);
        int32_t ycur = (lane < Ti) ? Y[row0 + lane] : 0;
        int32_t ynext = (32 + lane < Ti) ? Y[row0 + 32 + lane] : 0;
        int sn = 0, sp = S - 1;
        uint32_t xpar = 0;
        for (int t = 0; t < Ti + 2; ++t) {
            if (t < Ti) {
                if ((t & 31) == 0) {               // stage the labels of samples [t, t+32)
                    sm.ylab[(t >> 5) & 1][lane] = ycur;
                    ycur = ynext;
                    const int tt = t + 64 + lane;
                    ynext = (tt < Ti) ? Y[row0 + tt] : 0;
                }
                const int u = t + PF;
                if (u < Ti) {
                    if (u >= S) mbar_wait(&sm.xempty[u % S], (uint32_t)(((u / S) - 1) & 1));
                    if (lane == 0) issue_x(u);
                }
                mbar_wait(&sm.xfull[sn], xpar);
                float gsum = 0.f;
                if (t >= 1) {
                    const float* xn = xring + sn * DP + lane;
                    const float* xp = xring + sp * DP + lane;
#pragma unroll
                    for (int m = 0; m < M; ++m) gsum = fmaf(xp[32 * m], xn[32 * m], gsum);
                }
                gsum = warp_sum(gsum);
                if (lane == 0) sm.gram[sn] = gsum;
            }
            // x(t) landed and G(t-1,t) written: certify them on the tail's accfull(t-2)
            __syncwarp();
            if (t >= 2 && lane == 0) mbar_arrive(&sm.accfull[(t - 2) % S]);
            sp = sn;
            if (++sn == S) { sn = 0; xpar ^= 1u; }
        }
    }
    __syncthreads();
    if constexpr (C > 1) cluster_sync_all();   // no CTA leaves while a peer may still st.async into it
#undef TR
}

template <int M, int O, int C, int A1, int A2, bool TRACE>
cudaError_t launch_one(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                       const int32_t* labels, long long n_local, int K_local, int s_first,
                       int s_count, float lr, cudaStream_t st) {
    auto kern = sgd_resident_kernel<M, O, C, A1, A2, TRACE>;
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
    const int npw = p.threads / 32 - 2;
    return cudaLaunchKernelEx(&cfg, kern, d, children, x, labels, n_local, K_local, s_first, lr, npw, g_trace);
}

template <int C, int A1, int A2>
cudaError_t launch_ca(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                      const int32_t* labels, long long n_local, int K_local, int s_first, int s_count,
                      float lr, cudaStream_t st) {
    if constexpr ((C == 1 || C == 4) && ((A1 == PNN_RELU && A2 == PNN_SOFTMAX) ||
                                         (A1 == PNN_SIGMOID && A2 == PNN_SIGMOID)))
        if (g_trace)
            return launch_one<25, 10, C, A1, A2, true>(p, d, children, x, labels, n_local, K_local,
                                                       s_first, s_count, lr, st);
    return launch_one<25, 10, C, A1, A2, false>(p, d, children, x, labels, n_local, K_local, s_first,
                                                s_count, lr, st);
}

template <int C>
cudaError_t launch_c(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                     const int32_t* labels, long long n_local, int K_local, int s_first, int s_count,
                     float lr, cudaStream_t st) {
#define PNN_ACTS(A1_, A2_)                                                                      \
    if (d.act[0] == A1_ && d.act[1] == A2_)                                                   \
        return launch_ca<C, A1_, A2_>(p, d, children, x, labels, n_local, K_local, s_first, s_count, lr, st);
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
    const int D = d.n[0], H = d.n[1], O = d.n[2];
    if (D % 4 != 0) return no("input width must be a multiple of 4 (16-byte bulk copies)");
    if (D > 32 * 25 || D <= 32 * 24) return no("built for 768 < inputs <= 800 (25 columns per lane)");
    if (O != 10) return no("built for 10 outputs");
    const int a1 = d.act[0], a2 = d.act[1];
    const bool built = (a1 == PNN_RELU && a2 == PNN_SOFTMAX) || (a1 == PNN_TANH && a2 == PNN_SOFTMAX) ||
                       (a1 == PNN_SIGMOID && a2 == PNN_SOFTMAX) || (a1 == PNN_SIGMOID && a2 == PNN_SIGMOID) ||
                       (a1 == PNN_TANH && a2 == PNN_TANH) || (a1 == PNN_RELU && a2 == PNN_SIGMOID);
    if (!built) return no("activation pair not instantiated in the resident kernel");
    int c = 1;
    while (c <= CMAX && (H + c - 1) / c > 32) c *= 2;
    if (c > CMAX) return no("hidden layer wider than 256");
    const int U = (H + c - 1) / c;
    p.cluster = c;
    const int npw = (U + R - 1) / R;
    p.threads = (npw + 2) * 32;
    p.smem = ((sizeof(Smem) + 127) / 128) * 128 + sizeof(float) * S * 32 * 25;
    p.variant = 25;
    p.ok = true;
    return p;
}

cudaError_t launch_sgd_resident(const ResidentPlan& p, const NetDesc& d, float* children,
                                const float* x, const int32_t* labels, long long n_local,
                                int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    switch (p.cluster) {
    case 1: return launch_c<1>(p, d, children, x, labels, n_local, K_local, s_first, s_count, lr, st);
    case 2: return launch_c<2>(p, d, children, x, labels, n_local, K_local, s_first, s_count, lr, st);
    case 4: return launch_c<4>(p, d, children, x, labels, n_local, K_local, s_first, s_count, lr, st);
    case 8: return launch_c<8>(p, d, children, x, labels, n_local, K_local, s_first, s_count, lr, st);
    default: return cudaErrorInvalidValue;
    }
}
