// k_resident.cu — persistent per-sample SGD with register-resident weights.
//
// One thread-block cluster of c CTAs trains one child network (CN) over its
// whole slice; the CN's hidden layer is split across the c SMs (CTA r owns
// hidden units [r·U, r·U+U)), and its W^1 rows live in REGISTERS for the
// whole launch (loaded once, written back once).  Scope: 2-layer nets
// (D-H-O, e.g. 784-128-10), per-instance SGD, H <= 32·c, O <= 16.
//
// Per sample (§3, Eqs.2-13), with the paper's sequential order:
//   z1 = W1 x + b1, h = φ1(z1); z2 = W2 h + b2, x2 = φ2(z2)        (Eqs.2-5)
//   δ2 = x2 - e (softmax+CE, Eq.10) or (x2 - e)⊙φ2'(x2) (R11)      (Eqs.9-10)
//   δ1 = (W2ᵀ δ2) ⊙ φ1'(h), pre-update W2 (R6)                      (Eq.11)
//   W -= η δ xᵀ, b -= η δ                                            (Eqs.12-13)
//
// Warp roles inside a CTA:
//   * NPW "pass" warps hold W1 (R=4 rows per warp, lane j owns columns
//     j, j+32, ..., so rows reduce with warp shuffles).  Pass P_t does, per
//     weight, the update of sample t-2 and the forward of sample t in one
//     register sweep:   w -= g(t-2)·x(t-2)_j ;  acc += w·x(t)_j
//     so acc(t) = W1(t-1)·x(t).  It also emits G(t-1,t) = x(t-1)·x(t).
//   * one "tail" warp (lane k = hidden unit k) finishes sample t while the
//     pass warps already sweep sample t+1 ("lookahead-corrected forward",
//     SURVEY.md §7 hard part 2(ii)): since W1(t) = W1(t-1) - g(t-1)x(t-1)ᵀ,
//         z1(t) = acc(t) - g(t-1)·G(t-1,t) + b1(t)
//     exactly in real arithmetic; only the rounding differs from the
//     oracle's direct W1(t)·x(t).  The tail then does the activation, the
//     partial logits of its U units, the cluster exchange (st.async into
//     every peer CTA's shared memory, completing a local mbarrier), softmax,
//     δ2, the W2/b2 update (W2 columns of its units in registers; b2
//     replicated and updated identically by every CTA), δ1 and g1 = η·δ1.
//   * x rows are streamed HBM→SMEM by 1-D bulk copies (cp.async.bulk, mbarrier
//     complete_tx) into an S-slot ring, PF samples ahead.
// Synchronisation is by mbarriers only (no __syncthreads in the loop), so a
// slow tail never stalls the pass of the next sample.
#include <cstdio>
#include "pnn_internal.h"
#include "pnn_device.cuh"

namespace {

constexpr int R = 4;          // W1 rows per pass warp
constexpr int MAXPW = 8;      // pass warps per CTA  (U <= 32)
constexpr int S = 12;         // x ring slots
constexpr int PF = 6;         // prefetch distance (S >= PF + 5, see the slot-reuse note in the pass)
constexpr int OMAX = 16;      // outputs (padded to 16 lanes in the tail reductions)
constexpr int CMAX = 16;      // cluster size

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t tx) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(b)),
                 "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(remote_addr),
                 "r"(__float_as_uint(v)), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

struct __align__(16) Smem {
    uint64_t xfull[S];
    uint64_t accfull[2];
    uint64_t gfull[2];
    uint64_t lgfull[2];
    float acc[2][32];
    float g[2][32];
    float gram[2][MAXPW];
    float logits[2][CMAX][OMAX];
    // x ring follows (dynamic): S × DP floats
};

// --------------------------------------------------------------- the kernel
template <int M>   // columns per lane: D <= 32·M
__global__ void __launch_bounds__((MAXPW + 1) * 32, 1)
sgd_resident_kernel(NetDesc d, float* __restrict__ children, const float* __restrict__ X,
                    const int32_t* __restrict__ Y, long long n_local, int K_local, int s_first,
                    float lr, int npw) {
    constexpr int DP = 32 * M;
    extern __shared__ __align__(128) unsigned char smraw[];
    Smem& sm = *reinterpret_cast<Smem*>(smraw);
    float* xring = reinterpret_cast<float*>(smraw + ((sizeof(Smem) + 127) / 128) * 128);

    const int D = d.n[0], H = d.n[1], O = d.n[2];
    uint32_t csize;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    const int crank = (int)cluster_rank();
    const int cn = s_first + (int)(blockIdx.x / csize);
    const int U = (H + (int)csize - 1) / (int)csize;     // units per CTA
    const int k0 = crank * U;                            // first hidden unit of this CTA
    const int Uown = max(0, min(U, H - k0));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int act1 = d.act[0], act2 = d.act[1];

    long long row0, T;
    shard_of(n_local, K_local, cn, &row0, &T);
    float* P = children + (long long)cn * d.P;
    float* W1 = P;
    float* b1g = P + (long long)H * D;
    float* W2 = b1g + H;
    float* b2g = W2 + (long long)O * H;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&sm.xfull[i], 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sm.accfull[i], npw);
            mbar_init(&sm.gfull[i], 1);
            mbar_init(&sm.lgfull[i], 1);
        }
        fence_mbar_init();
    }
    // zero the ring (the DP - D pad columns stay 0 forever)
    for (int i = threadIdx.x; i < S * DP; i += blockDim.x) xring[i] = 0.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes → async-proxy copies
    __syncthreads();
    cluster_sync_all();   // peers' barriers are initialised before any st.async

    const uint32_t xbytes = (uint32_t)D * 4u;
    auto issue_x = [&](long long t) {   // one thread: bulk-load x(t) into its slot
        const int slot = (int)(t % S);
        mbar_arrive_expect_tx(&sm.xfull[slot], xbytes);
        bulk_g2s(xring + slot * DP, X + (row0 + t) * (long long)D, xbytes, &sm.xfull[slot]);
    };

    if (warp < npw) {
        // =========================== pass warps ===========================
        float w[R][M];
        const int kr0 = warp * R;                // first local row of this warp
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
        if (warp == 0 && lane == 0)
            for (long long t = 0; t < PF && t < T; ++t) issue_x(t);

        // P_t: w -= g(t-2)·x(t-2);  acc += w·x(t);  gram partial x(t-1)·x(t).
        // x(t-2), x(t-1), x(t) are all read from the ring (slot reuse: the
        // copy of x(t+PF) issued at the start of P_t overwrites x(t+PF-S);
        // every warp has finished P_{t-3} (it arrived on accfull(t-3), whose
        // tail produced the g(t-3) warp 0 waited for in P_{t-1}), so any
        // sample <= t-5 is dead: S >= PF + 5.)
        for (long long t = 0; t < T + 2; ++t) {
            const bool fwd = t < T;
            if (warp == 0 && lane == 0 && t + PF < T) issue_x(t + PF);
            float g[R];
#pragma unroll
            for (int r = 0; r < R; ++r) g[r] = 0.f;
            if (t >= 2) {
                const int gs = (int)((t - 2) & 1);
                mbar_wait(&sm.gfull[gs], (uint32_t)(((t - 2) >> 1) & 1));
#pragma unroll
                for (int r = 0; r < R; ++r) g[r] = sm.g[gs][kr0 + r];
            }
            const float* xo = xring + (int)(((t + 2 * S) - 2) % S) * DP + lane;   // x(t-2)
            if (fwd) {
                const int slot = (int)(t % S);
                mbar_wait(&sm.xfull[slot], (uint32_t)((t / S) & 1));
                const float* xn = xring + slot * DP + lane;                         // x(t)
                const float* xp = xring + (int)(((t + S) - 1) % S) * DP + lane;     // x(t-1)
                float acc[R];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = 0.f;
                float gp = 0.f;
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    const float xnm = xn[32 * m];
                    const float xom = (t >= 2) ? xo[32 * m] : 0.f;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        w[r][m] = fmaf(-g[r], xom, w[r][m]);
                        acc[r] = fmaf(w[r][m], xnm, acc[r]);
                    }
                    if (m % npw == warp && t >= 1) gp = fmaf(xp[32 * m], xnm, gp);
                }
                // transpose-reduce the R=4 row sums across 32 lanes (6 shuffles)
                const bool b4 = lane & 16, b3 = lane & 8;
                float u0 = (b4 ? acc[2] : acc[0]) + __shfl_xor_sync(0xffffffffu, b4 ? acc[0] : acc[2], 16);
                float u1 = (b4 ? acc[3] : acc[1]) + __shfl_xor_sync(0xffffffffu, b4 ? acc[1] : acc[3], 16);
                float v = (b3 ? u1 : u0) + __shfl_xor_sync(0xffffffffu, b3 ? u0 : u1, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                gp = warp_sum(gp);
                const int ts = (int)(t & 1);
                // lane holds row (b4 ? 2 : 0) + (b3 ? 1 : 0)
                if ((lane & 7) == 0) sm.acc[ts][kr0 + (b4 ? 2 : 0) + (b3 ? 1 : 0)] = v;
                if (lane == 0) sm.gram[ts][warp] = gp;
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.accfull[ts]);
            } else if (t >= 2) {
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    const float xom = xo[32 * m];
#pragma unroll
                    for (int r = 0; r < R; ++r) w[r][m] = fmaf(-g[r], xom, w[r][m]);
                }
            }
        }
        // write W1 rows back
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
        // ============================ tail warp ============================
        const int k = lane;                     // local hidden unit
        const bool unit = k < Uown;
        float w2[OMAX];
#pragma unroll
        for (int o = 0; o < OMAX; ++o) w2[o] = (unit && o < O) ? W2[(long long)o * H + k0 + k] : 0.f;
        float b1 = unit ? b1g[k0 + k] : 0.f;
        float b2 = (lane < O) ? b2g[lane] : 0.f;       // replicated on every CTA
        float gprev = 0.f;
        // remote addresses of logits[.][crank][.] and lgfull[.] in every peer
        const uint32_t my_lg = smem_u32(&sm.logits[0][crank][0]);
        const uint32_t my_bar = smem_u32(&sm.lgfull[0]);
        const uint32_t lg_bytes = (uint32_t)((csize - 1) * O * 4);
        // labels, one per lane, a block of 32 samples prefetched one block ahead
        int32_t ylab = (lane < T) ? Y[row0 + lane] : 0;
        int32_t ynext = (32 + lane < T) ? Y[row0 + 32 + lane] : 0;
        for (long long t = 0; t < T; ++t) {
            const int ts = (int)(t & 1);
            const uint32_t par = (uint32_t)((t >> 1) & 1);
            if ((t & 31) == 0 && t > 0) {
                ylab = ynext;
                const long long tt = t + 32 + lane;
                ynext = (tt < T) ? Y[row0 + tt] : 0;
            }
            const int label = __shfl_sync(0xffffffffu, ylab, (int)(t & 31));
            if (lane == 0 && csize > 1) mbar_arrive_expect_tx(&sm.lgfull[ts], lg_bytes);
            mbar_wait(&sm.accfull[ts], par);
            float a = unit ? sm.acc[ts][k] : 0.f;
            float G = 0.f;
            for (int w_ = 0; w_ < npw; ++w_) G += sm.gram[ts][w_];
            // z1(t) = W1(t-1)x(t) - g(t-1)·G(t-1,t) + b1(t)
            b1 -= gprev;
            const float z1 = fmaf(-gprev, G, a) + b1;
            const float h = unit ? act_fwd(act1, z1) : 0.f;
            // partial logits of this CTA's units: reduce-scatter 16 values over 32 lanes
            float v[OMAX];
#pragma unroll
            for (int o = 0; o < OMAX; ++o) v[o] = w2[o] * h;
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
            const int idx = (lane >> 1) & 15;   // output index this lane now holds
            if ((lane & 1) == 0 && idx < O) {
                sm.logits[ts][crank][idx] = u1;
                for (uint32_t r = 0; r < csize; ++r) {
                    if ((int)r == crank) continue;
                    const uint32_t off = (uint32_t)((ts * CMAX * OMAX + idx) * 4);
                    st_async_f32(mapa(my_lg + off, r), u1, mapa(my_bar + ts * 8, r));
                }
            }
            __syncwarp();
            if (csize > 1) mbar_wait_cluster(&sm.lgfull[ts], par);
            // output layer: lane o < O owns output o
            float z2 = b2;
            for (uint32_t r = 0; r < csize; ++r) z2 += (lane < O) ? sm.logits[ts][r][lane] : 0.f;
            float x2;
            if (act2 == PNN_SOFTMAX) {
                float m = (lane < O) ? z2 : -INFINITY;
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
                float e = (lane < O) ? expf(z2 - m) : 0.f;
                float ssum = e;
                ssum += __shfl_xor_sync(0xffffffffu, ssum, 8);
                ssum += __shfl_xor_sync(0xffffffffu, ssum, 4);
                ssum += __shfl_xor_sync(0xffffffffu, ssum, 2);
                ssum += __shfl_xor_sync(0xffffffffu, ssum, 1);
                x2 = e / ssum;
            } else {
                x2 = act_fwd(act2, z2);
            }
            const float ev = (lane == label) ? 1.f : 0.f;
            float d2 = (act2 == PNN_SOFTMAX) ? x2 - ev : (x2 - ev) * act_deriv_from_x(act2, x2);
            if (lane >= O) d2 = 0.f;
            if (lane < O) b2 -= lr * d2;
            // hidden delta (pre-update W2) and W2 update for this lane's unit
            float s1 = 0.f;
#pragma unroll
            for (int o = 0; o < OMAX; ++o) {
                if (o < O) {
                    const float dl = __shfl_sync(0xffffffffu, d2, o);
                    s1 = fmaf(w2[o], dl, s1);
                    w2[o] = fmaf(-(lr * dl), h, w2[o]);
                }
            }
            const float g1 = unit ? lr * (s1 * act_deriv_from_x(act1, h)) : 0.f;
            sm.g[ts][k] = g1;
            gprev = g1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.gfull[ts]);
        }
        b1 -= gprev;                            // b1(T) = b1(T-1) - g(T-1)
        if (unit) {
#pragma unroll
            for (int o = 0; o < OMAX; ++o)
                if (o < O) W2[(long long)o * H + k0 + k] = w2[o];
            b1g[k0 + k] = b1;
        }
        if (crank == 0 && lane < O) b2g[lane] = b2;
    }
    __syncthreads();
    cluster_sync_all();   // no CTA leaves while a peer may still st.async into it
}

template <int M>
cudaError_t launch_m(const ResidentPlan& p, const NetDesc& d, float* children, const float* x,
                     const int32_t* labels, long long n_local, int K_local, int s_first, int s_count,
                     float lr, cudaStream_t st) {
    auto kern = sgd_resident_kernel<M>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e != cudaSuccess) return e;
    if (p.cluster > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(s_count * p.cluster));
    cfg.blockDim = dim3((unsigned)p.threads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int npw = p.threads / 32 - 1;
    return cudaLaunchKernelEx(&cfg, kern, d, children, x, labels, n_local, K_local, s_first, lr, npw);
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
    if (D > 32 * 25 || D <= 32 * 24) return no("built for 768 < inputs <= 800 (M = 25 columns per lane)");
    if (O > OMAX) return no("more than 16 outputs");
    if (d.act[0] == PNN_SOFTMAX) return no("softmax hidden layer");
    int c = (H + 31) / 32;
    if (c > CMAX) return no("hidden layer wider than 512");
    // smallest cluster with U = ceil(H/c) <= 32
    const int U = (H + c - 1) / c;
    p.cluster = c;
    const int npw = (U + R - 1) / R;
    p.threads = (npw + 1) * 32;
    p.smem = ((sizeof(Smem) + 127) / 128) * 128 + sizeof(float) * S * 32 * 25;
    p.variant = 25;
    p.ok = true;
    return p;
}

cudaError_t launch_sgd_resident(const ResidentPlan& p, const NetDesc& d, float* children,
                                const float* x, const int32_t* labels, long long n_local,
                                int K_local, int s_first, int s_count, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    switch (p.variant) {
    case 25: return launch_m<25>(p, d, children, x, labels, n_local, K_local, s_first, s_count, lr, st);
    default: return cudaErrorInvalidValue;
    }
}
