// k_cluster.cu — per-sample SGD with the weights resident in the shared memory of a
// thread-block cluster, for networks of any depth whose parameters exceed one SM
// (north_star: "one CTA (or thread-block cluster using distributed shared memory when a
// sub-network's weights exceed one SM's shared memory) per sub-network"; C3's
// 784-300-100-10, 1.04 MB of fp32 parameters, on an 8-CTA cluster).
//
// Layout: CTA r of the C-CTA cluster owns rows R_r(l) = [r·⌈n_l/C⌉, …) of every layer's
// W^l and b^l, in shared memory for the whole slice.  Per sample, in the paper's order
// (§3, Eqs.2-13):
//   forward  l = 1..L: x^l[k] = φ_l(W^l[k]·x^{l-1} + b^l[k]) for own k, stored into every
//            CTA's copy of x^l (st.shared::cluster), cluster barrier — every CTA then
//            holds the full x^l (softmax, max-subtracted (R4), computed redundantly);
//   δ^L      own rows: x^L − e (Eq.10) or (x^L − e)⊙φ'(x^L) (Eq.9, R11);
//   δ^l      l = L-1..1 (Eq.11, pre-update W^{l+1}, R6): CTA r forms the partial
//            Σ_{k∈R_r(l+1)} W^{l+1}[k][j]·δ^{l+1}[k] for every j and sends each j to the
//            CTA owning row j of layer l (a reduce-scatter through DSMEM), cluster
//            barrier, the owner sums the C partials in rank order, × φ'(x^l_j);
//   update   own rows: W^l[k] −= η·δ^l[k]·x^{l-1}, b^l[k] −= η·δ^l[k]  (Eqs.12-13).
// Exchanges are st.async stores completing an mbarrier of the receiver (per layer and sample
// parity; the receiver posts the expected bytes); activations and partials are
// double-buffered by sample parity: a CTA reaching sample t+2 has received every peer's
// data of sample t+1, which each peer sent after finishing sample t.
// x rows stream HBM→SMEM by cp.async.bulk into a 4-slot ring, 2 ahead.
#include <cstdio>
#include "pnn_internal.h"
#include "pnn_device.cuh"
#include "pnn_ptx.cuh"

namespace {

using namespace ptx;

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kRing = 4;          // x ring slots
constexpr int kAhead = 2;         // rows in flight

struct ClusterPlanDev {
    int C;                                   // cluster size
    int rows[PNN_MAX_LAYERS + 1];            // ⌈n_l / C⌉ rows per CTA per layer (n_l if replicated)
    int rep[PNN_MAX_LAYERS + 1];             // layer held in full by every CTA (the small output layer)
    int w_off[PNN_MAX_LAYERS + 1];           // own W^l rows in shared memory (floats)
    int b_off[PNN_MAX_LAYERS + 1];           // own b^l
    int x_off[PNN_MAX_LAYERS + 1];           // full x^l, parity 0 (parity 1 at + x_par)
    int d_off[PNN_MAX_LAYERS + 1];           // own δ^l
    int x_par;                               // floats between the two x buffers
    int recv_off, recv_par, recv_stride;     // [parity][layer][src][rows_max] partial δ
    int recv_layer;                          // floats per layer block (C · recv_stride)
    int ring_off, ring_stride;               // x ring (floats), slot = D + 4 (label in slot[D])
    int total;                               // floats of shared memory
};

__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Σ_j w[j]·x[j] over this lane's share of a row (both 16-byte aligned when n % 4 == 0):
// float4 steps with 2 independent accumulators, scalar tail otherwise.
__device__ __forceinline__ float dot_lanes(const float* w, const float* x, int n, int lane) {
    float a0 = 0.f, a1 = 0.f;
    if ((n & 3) == 0) {
        const float4* w4 = reinterpret_cast<const float4*>(w);
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const int n4 = n >> 2;
        for (int q = lane; q < n4; q += 32) {
            const float4 a = w4[q], b = x4[q];
            a0 = fmaf(a.x, b.x, a0);
            a1 = fmaf(a.y, b.y, a1);
            a0 = fmaf(a.z, b.z, a0);
            a1 = fmaf(a.w, b.w, a1);
        }
    } else {
        for (int j = lane; j < n; j += 32) a0 = fmaf(w[j], x[j], a0);
    }
    return a0 + a1;
}
// w[j] += g·x[j] over this lane's share of a row
__device__ __forceinline__ void axpy_lanes(float* w, const float* x, float g, int n, int lane) {
    if ((n & 3) == 0) {
        float4* w4 = reinterpret_cast<float4*>(w);
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const int n4 = n >> 2;
        for (int q = lane; q < n4; q += 32) {
            float4 a = w4[q];
            const float4 b = x4[q];
            a.x = fmaf(g, b.x, a.x);
            a.y = fmaf(g, b.y, a.y);
            a.z = fmaf(g, b.z, a.z);
            a.w = fmaf(g, b.w, a.w);
            w4[q] = a;
        }
    } else {
        for (int j = lane; j < n; j += 32) w[j] = fmaf(g, x[j], w[j]);
    }
}

// A layer input held in registers, lane l: float4 chunks l, l+32, ... (n % 4 == 0, n <= 1024),
// so that each row of W costs one shared-memory stream instead of two.
struct XRegs {
    static constexpr int Q = 8;
    float4 v[Q];
    bool ok;
    __device__ __forceinline__ void load(const float* x, int n, int lane) {
        ok = (n & 3) == 0 && n <= 128 * Q;
        const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = lane + 32 * q;
            v[q] = (ok && 4 * c < n) ? x4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __device__ __forceinline__ float dot(const float* w, int n, int lane) const {
        const float4* w4 = reinterpret_cast<const float4*>(w);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = lane + 32 * q;
            if (4 * c < n) {
                const float4 a = w4[c];
                a0 = fmaf(a.x, v[q].x, a0);
                a1 = fmaf(a.y, v[q].y, a1);
                a0 = fmaf(a.z, v[q].z, a0);
                a1 = fmaf(a.w, v[q].w, a1);
            }
        }
        return a0 + a1;
    }
    __device__ __forceinline__ void axpy(float* w, float g, int n, int lane) const {
        float4* w4 = reinterpret_cast<float4*>(w);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = lane + 32 * q;
            if (4 * c < n) {
                float4 a = w4[c];
                a.x = fmaf(g, v[q].x, a.x);
                a.y = fmaf(g, v[q].y, a.y);
                a.z = fmaf(g, v[q].z, a.z);
                a.w = fmaf(g, v[q].w, a.w);
                w4[c] = a;
            }
        }
    }
};

__global__ void __launch_bounds__(kThreads, 1)
sgd_cluster_kernel(NetDesc d, ClusterPlanDev pl, float* __restrict__ children, const float* __restrict__ X,
                   const int32_t* __restrict__ Y, long long n_local, int K_local, int s_first, float lr) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) uint64_t xfull[kRing];
    // peers' activations (fwd) / partial δ (bwd) of layer l for samples of parity p landed
    __shared__ __align__(8) uint64_t fbar[PNN_MAX_LAYERS + 1][2], bbar[PNN_MAX_LAYERS + 1][2];
    const int C = pl.C;
    const int r = (int)cluster_rank();
    const int cn = s_first + (int)(blockIdx.x / C);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = d.L, D = d.n[0];
    long long row0, T;
    shard_of(n_local, K_local, cn, &row0, &T);
    float* P = children + (long long)cn * d.P;

    // ---- own rows of every layer into shared memory ----
    for (int l = 1; l <= L; ++l) {
        const int nin = d.n[l - 1], nout = d.n[l], R = pl.rows[l], k0 = pl.rep[l] ? 0 : r * R;
        const float* Wg = P + d.woff[l];
        const float* bg = Wg + (long long)nout * nin;
        for (int i = tid; i < R * nin; i += kThreads) {
            const int k = k0 + i / nin;
            smf[pl.w_off[l] + i] = (k < nout) ? Wg[(long long)k * nin + i % nin] : 0.f;
        }
        for (int i = tid; i < R; i += kThreads) smf[pl.b_off[l] + i] = (k0 + i < nout) ? bg[k0 + i] : 0.f;
    }
    if (tid == 0) {
        for (int i = 0; i < kRing; ++i) mbar_init(&xfull[i], 1);
        for (int l = 0; l <= PNN_MAX_LAYERS; ++l)
            for (int p = 0; p < 2; ++p) {
                mbar_init(&fbar[l][p], 1);
                mbar_init(&bbar[l][p], 1);
            }
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t xbytes = (uint32_t)D * 4u;
    auto issue = [&](long long t) {
        const int slot = (int)(t % kRing);
        float* dst = smf + pl.ring_off + slot * pl.ring_stride;
        mbar_arrive_expect_tx(&xfull[slot], xbytes);
        bulk_g2s(dst, X + (row0 + t) * D, xbytes, &xfull[slot]);
    };
    if (tid == 0)
        for (long long t = 0; t < kAhead && t < T; ++t) issue(t);
    cluster_sync_all();                            // peers' barriers are live before any remote store

    // per-layer tables in shared memory: indexing kernel parameters by a runtime layer
    // number compiles to slow indexed constant loads on the per-sample path
    __shared__ struct {
        int n[PNN_MAX_LAYERS + 1], act[PNN_MAX_LAYERS + 1], rows[PNN_MAX_LAYERS + 1], rep[PNN_MAX_LAYERS + 1];
        int w_off[PNN_MAX_LAYERS + 1], b_off[PNN_MAX_LAYERS + 1], x_off[PNN_MAX_LAYERS + 1],
            d_off[PNN_MAX_LAYERS + 1];
    } sp;
    if (tid <= PNN_MAX_LAYERS) {
        sp.n[tid] = d.n[tid];
        sp.act[tid] = tid < PNN_MAX_LAYERS ? d.act[tid] : 0;
        sp.rows[tid] = pl.rows[tid];
        sp.rep[tid] = pl.rep[tid];
        sp.w_off[tid] = pl.w_off[tid];
        sp.b_off[tid] = pl.b_off[tid];
        sp.x_off[tid] = pl.x_off[tid];
        sp.d_off[tid] = pl.d_off[tid];
    }
    __syncthreads();
    const uint32_t sbase = smem_u32(smf);
    int label_next = (T > 0) ? Y[row0] : 0;        // labels are loaded one sample ahead
#ifdef PNN_CLUSTER_PROFILE
    long long prof[12] = {0};
    long long tp = ptx::clock64();
#define PROF(i) do { if (tid == 0) { const long long tn = ptx::clock64(); prof[i] += tn - tp; tp = tn; } } while (0)
#else
#define PROF(i) do { } while (0)
#endif
    for (long long t = 0; t < T; ++t) {
        const int par = (int)(t & 1);
        const int slot = (int)(t % kRing);
        const int label = label_next;
        if (t + 1 < T) label_next = Y[row0 + t + 1];
        PROF(0);
        mbar_wait(&xfull[slot], (uint32_t)((t / kRing) & 1));
        PROF(1);
        const float* x0 = smf + pl.ring_off + slot * pl.ring_stride;
        // ---------------- forward ----------------
        for (int l = 1; l <= L; ++l) {
            const bool rep = sp.rep[l] != 0;
            const int nin = sp.n[l - 1], nout = sp.n[l], R = sp.rows[l], k0 = rep ? 0 : r * R;
            const float* xin = (l == 1) ? x0 : smf + sp.x_off[l - 1] + par * pl.x_par;
            const int xo = sp.x_off[l] + par * pl.x_par;
            const int a = sp.act[l - 1];
            const int own = max(0, min(R, nout - k0));
            if (tid == 0 && !rep) mbar_arrive_expect_tx(&fbar[l][par], 4u * (uint32_t)(nout - own));
            const uint32_t fb = smem_u32(&fbar[l][par]);
            XRegs xr;
            xr.load(xin, nin, lane);
            for (int i = warp; i < R; i += kWarps) {
                const int k = k0 + i;
                if (k >= nout) break;
                const float* w = smf + sp.w_off[l] + i * nin;
                const float acc = warp_sum(xr.ok ? xr.dot(w, nin, lane) : dot_lanes(w, xin, nin, lane));
                const float z = acc + smf[sp.b_off[l] + i];
                const float v = (a == PNN_SOFTMAX) ? z : act_fwd(a, z);
                if (rep) {                         // replicated layer: every CTA computes every row
                    if (lane == 0) smf[xo + k] = v;
                } else if (lane == r) smf[xo + k] = v;
                else if (lane < C)                 // into peer `lane`'s x^l, completing its fbar
                    st_async_f32(mapa(sbase + 4u * (uint32_t)(xo + k), (uint32_t)lane), v, mapa(fb, (uint32_t)lane));
            }
            PROF(2);
            __syncthreads();                       // own rows of x^l written
            PROF(3);
            if (!rep) mbar_wait(&fbar[l][par], (uint32_t)((t >> 1) & 1));   // peers' rows landed
            PROF(4);
            if (a == PNN_SOFTMAX) {                // the output layer's softmax, redundantly per CTA
                if (warp == 0) softmax_warp(smf + xo, nout, lane);
                __syncthreads();
            }
        }
        // ---------------- δ^L, own rows ----------------
        {
            const int nL = sp.n[L], R = sp.rows[L], k0 = sp.rep[L] ? 0 : r * R, aL = sp.act[L - 1];
            const float* xL = smf + sp.x_off[L] + par * pl.x_par;
            for (int i = tid; i < R; i += kThreads) {
                const int k = k0 + i;
                float dl = 0.f;
                if (k < nL) {
                    const float e = (k == label) ? 1.f : 0.f;
                    dl = (aL == PNN_SOFTMAX) ? xL[k] - e : (xL[k] - e) * act_deriv_from_x(aL, xL[k]);
                }
                smf[sp.d_off[L] + i] = dl;
            }
            __syncthreads();
        }
        // ---------------- δ^l, l = L-1..1: reduce-scatter of the partials ----------------
        for (int l = L - 1; l >= 1; --l) {
            const int nl = sp.n[l], Rn = sp.rows[l + 1], Rl = sp.rows[l];
            if (sp.rep[l + 1]) {
                // W^{l+1} and δ^{l+1} are complete in every CTA: δ^l of the own units directly
                const float* Wn = smf + sp.w_off[l + 1];      // pre-update (R6)
                const float* dn = smf + sp.d_off[l + 1];
                const float* xl = smf + sp.x_off[l] + par * pl.x_par;
                const int k0 = r * Rl;
                for (int i = tid; i < Rl; i += kThreads) {
                    const int k = k0 + i;
                    float acc = 0.f;
                    if (k < nl)
                        for (int q = 0; q < Rn; ++q) acc = fmaf(Wn[q * nl + k], dn[q], acc);
                    smf[sp.d_off[l] + i] = (k < nl) ? acc * act_deriv_from_x(sp.act[l - 1], xl[k]) : 0.f;
                }
                __syncthreads();
                continue;
            }
            const float* Wn = smf + sp.w_off[l + 1];          // own rows of W^{l+1}, pre-update (R6)
            const float* dn = smf + sp.d_off[l + 1];
            const int rv = pl.recv_off + par * pl.recv_par + l * pl.recv_layer;   // per layer: no reuse
                                                                                // within a sample
            const int ownl = max(0, min(Rl, nl - r * Rl));
            if (tid == 0) mbar_arrive_expect_tx(&bbar[l][par], 4u * (uint32_t)((C - 1) * ownl));
            const uint32_t bb = smem_u32(&bbar[l][par]);
            for (int j = tid; j < nl; j += kThreads) {
                float acc = 0.f;
                for (int i = 0; i < Rn; ++i) acc = fmaf(Wn[i * nl + j], dn[i], acc);   // padded rows: δ = 0
                const int q = j / Rl, jj = j - q * Rl;            // owner CTA of unit j, its local index
                const int dst = rv + r * pl.recv_stride + jj;
                if (q == r) smf[dst] = acc;
                else st_async_f32(mapa(sbase + 4u * (uint32_t)dst, (uint32_t)q), acc, mapa(bb, (uint32_t)q));
            }
            PROF(5);
            __syncthreads();
            PROF(6);
            mbar_wait(&bbar[l][par], (uint32_t)((t >> 1) & 1));
            PROF(7);
            const float* xl = smf + sp.x_off[l] + par * pl.x_par;
            const int k0 = r * Rl;
            for (int i = tid; i < Rl; i += kThreads) {
                float s = 0.f;
                for (int src = 0; src < C; ++src) s += smf[rv + src * pl.recv_stride + i];
                const int k = k0 + i;
                smf[sp.d_off[l] + i] = (k < nl) ? s * act_deriv_from_x(sp.act[l - 1], xl[k]) : 0.f;
            }
            __syncthreads();
        }
        // ---------------- update (Eqs.12-13), own rows ----------------
        for (int l = 1; l <= L; ++l) {
            const int nin = sp.n[l - 1], nout = sp.n[l], R = sp.rows[l], k0 = sp.rep[l] ? 0 : r * R;
            const float* xin = (l == 1) ? x0 : smf + sp.x_off[l - 1] + par * pl.x_par;
            XRegs xr;
            xr.load(xin, nin, lane);
            for (int i = warp; i < R; i += kWarps) {
                if (k0 + i >= nout) break;
                const float g = lr * smf[sp.d_off[l] + i];
                if (xr.ok) xr.axpy(smf + sp.w_off[l] + i * nin, -g, nin, lane);
                else axpy_lanes(smf + sp.w_off[l] + i * nin, xin, -g, nin, lane);
                if (lane == 0) smf[sp.b_off[l] + i] -= g;
            }
        }
        PROF(8);
        __syncthreads();                           // x(t)'s ring slot and δ are free
        PROF(9);
        if (tid == 0 && t + kAhead < T) issue(t + kAhead);
    }
#ifdef PNN_CLUSTER_PROFILE
    if (tid == 0 && blockIdx.x < 2)
        printf("cta %d T %lld per-sample cycles: top %lld xwait %lld fwd-compute %lld fwd-sync %lld fwd-wait %lld "
               "bwd-compute %lld bwd-sync %lld bwd-wait %lld update %lld end-sync %lld\n", blockIdx.x, T,
               prof[0] / T, prof[1] / T, prof[2] / T, prof[3] / T, prof[4] / T, prof[5] / T, prof[6] / T,
               prof[7] / T, prof[8] / T, prof[9] / T);
#endif
#undef PROF
    // ---- write back own rows ----
    for (int l = 1; l <= L; ++l) {
        if (pl.rep[l] && r != 0) continue;          // replicated layer: identical copies, CTA 0 writes
        const int nin = d.n[l - 1], nout = d.n[l], R = pl.rows[l], k0 = pl.rep[l] ? 0 : r * R;
        float* Wg = P + d.woff[l];
        float* bg = Wg + (long long)nout * nin;
        for (int i = tid; i < R * nin; i += kThreads) {
            const int k = k0 + i / nin;
            if (k < nout) Wg[(long long)k * nin + i % nin] = smf[pl.w_off[l] + i];
        }
        for (int i = tid; i < R; i += kThreads)
            if (k0 + i < nout) bg[k0 + i] = smf[pl.b_off[l] + i];
    }
    cluster_sync_all();                            // no CTA exits while a peer may still store into it
}

bool make_plan(const NetDesc& d, int C, ClusterPlanDev* pl) {
    ClusterPlanDev p{};
    p.C = C;
    int off = 0;
    int rmax = 1;
    for (int l = 1; l <= d.L; ++l) {
        // the output layer, when small, is replicated in every CTA and updated redundantly: its
        // forward needs no all-gather and the next δ no reduce-scatter (two exchanges fewer)
        p.rep[l] = (C > 1 && l == d.L && (long long)d.n[l] * d.n[l - 1] <= 4096) ? 1 : 0;
        p.rows[l] = p.rep[l] ? d.n[l] : (d.n[l] + C - 1) / C;
        rmax = p.rows[l] > rmax ? p.rows[l] : rmax;
        p.w_off[l] = off;
        off += p.rows[l] * d.n[l - 1];
        off = (off + 3) & ~3;
        p.b_off[l] = off;
        off += (p.rows[l] + 3) & ~3;
    }
    int xs = 0;
    for (int l = 1; l <= d.L; ++l) xs += (d.n[l] + 3) & ~3;
    int xo = off;
    for (int l = 1; l <= d.L; ++l) { p.x_off[l] = xo; xo += (d.n[l] + 3) & ~3; }
    p.x_par = xs;
    off += 2 * xs;
    for (int l = 1; l <= d.L; ++l) { p.d_off[l] = off; off += (p.rows[l] + 3) & ~3; }
    p.recv_stride = (rmax + 3) & ~3;
    p.recv_layer = C * p.recv_stride;
    p.recv_par = (d.L + 1) * p.recv_layer;
    p.recv_off = off;
    off += 2 * p.recv_par;
    p.ring_stride = ((d.n[0] + 4) + 3) & ~3;
    p.ring_off = off;
    off += kRing * p.ring_stride;
    p.total = off;
    *pl = p;
    return (size_t)off * 4 <= 200 * 1024;
}

}  // namespace

ClusterPlan plan_cluster(const NetDesc& d, int batch) {
    ClusterPlan p{};
    auto no = [&](const char* why) {
        p.ok = false;
        snprintf(p.why, sizeof p.why, "%s", why);
        return p;
    };
    if (batch != 1) return no("the cluster kernel is per-sample SGD");
    if (d.n[0] % 4 != 0) return no("input width must be a multiple of 4 (16-byte bulk copies)");
    for (int C : {1, 2, 4, 8}) {
        ClusterPlanDev pd;
        if (make_plan(d, C, &pd)) {
            p.ok = true;
            p.cluster = C;
            p.smem = (size_t)pd.total * 4;
            return p;
        }
    }
    return no("parameters exceed 8 CTAs' shared memory");
}

cudaError_t launch_sgd_cluster(const ClusterPlan& p, const NetDesc& d, float* children, const float* x,
                               const int32_t* labels, long long n_local, int K_local, int s_first,
                               int s_count, float lr, cudaStream_t st) {
    if (s_count <= 0) return cudaSuccess;
    ClusterPlanDev pd;
    make_plan(d, p.cluster, &pd);
    cudaError_t e = cudaFuncSetAttribute(sgd_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p.smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(s_count * p.cluster));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sgd_cluster_kernel, d, pd, children, x, labels, n_local, K_local, s_first, lr);
}
