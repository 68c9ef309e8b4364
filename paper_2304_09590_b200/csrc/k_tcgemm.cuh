// k_tcgemm.cuh — a batched bf16 GEMM on the 5th-generation tensor cores (tcgen05)
// for the mini-batch variant (a10, north_star "mini-batch SGD
// batch 64 on tcgen05 GEMMs"):
//
//     C[z][m][n] = Σ_k A[z][m][k] · B[z][n][k]      (bf16 operands, fp32 accumulate)
//
// Both operands are K-major 3-D tensors [Z][rows][K] read by TMA
// (cp.async.bulk.tensor, 128-byte swizzle, out-of-bounds boxes zero-filled) into a
// STAGES-deep shared-memory ring; one elected thread issues tcgen05.mma
// (cta_group::1, M = 128, N = BN, K = 16 per instruction) accumulating in TMEM;
// tcgen05.commit → mbarrier hands the accumulator to 4 epilogue warps, which read
// it with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31 = tile rows) and apply a
// fused epilogue (EPI_*).  One CTA per 128 × BN output tile and per z.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>
#include "pnn_ptx.cuh"

namespace tc {

using namespace ptx;

constexpr int BM = 128;       // tile rows (UMMA M)
constexpr int BK = 64;        // K per stage: 64 bf16 = one 128-byte swizzle row
// pipeline depth: 8 stages for the narrow tiles (long K: more TMA loads in flight), 2 for BN = 256 (the update GEMMs
// have K = 64, a single stage) so that two CTAs fit per SM
// threads per CTA: the wide update tiles (BN = 256, memory-bound epilogues) use 8 warps, two
// per TMEM lane quadrant, each taking half of the columns
__host__ __device__ constexpr int threads_for(int bn) { return bn >= 64 ? 256 : 128; }
__host__ __device__ constexpr int stages_for(int bn) { return bn >= 256 ? 2 : (bn >= 128 ? 4 : 8); }

enum { EPI_STORE_F32 = 0, EPI_FWD = 1, EPI_BWD = 2, EPI_UPD = 3 };

// Epilogue operands (per z strides in elements).  Only the fields of the chosen mode
// are used.
struct Epi {
    int M, N, nvalid;         // logical rows, columns; columns >= nvalid are not written
    // EPI_STORE_F32: out_f32[z][m][n]
    float* out_f32;
    long long zs_out;
    // EPI_FWD: y = relu(acc + bias[m]); out_bm[z][n][m] (bf16), out_mb[z][m][n] (bf16, nullable)
    const float* bias;
    long long zs_bias;
    __nv_bfloat16* out_bm;
    __nv_bfloat16* out_mb;
    long long zs_act;         // M·N elements per z for both activation layouts
    //          optional (w3 != nullptr): the next layer's partial pre-activations of this
    //          row tile, z3part[z][blockIdx.x][n][o] = Σ_{m in tile} w3[z][o][m]·y[m][n], o < 16
    //          (the 10-wide output layer fused into the producing GEMM, a10)
    const __nv_bfloat16* w3;
    float* z3part;
    // EPI_BWD: d = acc ⊙ [mask[z][m][n] > 0]; out_mb[z][m][n] = bf16(d);
    //          bias[m] -= scale · Σ_{n < nvalid} d  (the layer's bias update)
    const __nv_bfloat16* mask;
    float* bias_upd;
    // EPI_UPD: master[z][m][n] -= scale · acc; wb[z][m][n] = bf16(master); wbt[z][n][m] (nullable)
    float* master;
    long long zs_master;
    __nv_bfloat16* wb;
    __nv_bfloat16* wbt;
    long long zs_w;
    float scale;
    // z of blockIdx.z = 0 is zoff; when lr > 0 the update scale of tensor z is lr / bsz(z),
    // bsz(z) = the rows of CN (zoff + z)'s slice in mini-batch `step` (short last batch, R14)
    int zoff;
    float lr;
    long long n_local;
    int K_local, step, batch;
    // A (the weight operand) was complete before the previous kernel of the stream started
    // (it comes from an earlier kernel or another stream's joined kernel): its first stages'
    // loads may be issued before griddep_wait, under the previous kernel's tail (PDL)
    bool a_early;
    // debug timeline (nullable; tools/trace_tc.py): per CTA 24 entries — [0] %globaltimer at
    // entry, then clock64 at: [1] entry, [2] after the prologue, [3] after griddep_wait,
    // [4 + kt] (kt < 16) each stage's full-barrier wait done (MMA thread), [20] epilogue
    // start (accumulator complete), [23] first chunk read from TMEM, [22] chunk loop done, [21] end
    long long* trace;
};

__device__ __forceinline__ float update_scale(const Epi& ep, int z) {
    if (ep.lr <= 0.f) return ep.scale;
    long long st, cnt;
    const long long base = ep.n_local / ep.K_local, rem = ep.n_local % ep.K_local;
    cnt = base + ((z < rem) ? 1 : 0);
    (void)st;
    long long b = cnt - (long long)ep.step * ep.batch;
    b = b < 0 ? 0 : (b > ep.batch ? ep.batch : b);
    return b > 0 ? ep.lr / (float)b : 0.f;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// 32 lanes × 16 consecutive 32-bit TMEM columns: thread t gets lane (base lane + t), cols c..c+15
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes × 32 consecutive 32-bit TMEM columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor of a K-major tile written by TMA with the 128-byte swizzle:
// rows of 128 bytes, 8-row core groups 1024 bytes apart (SBO), LBO unused, version 1
// (sm_100), layout type 2 = SWIZZLE_128B.  Advancing along K inside the swizzle atom adds
// the byte offset to the start address.
__device__ __forceinline__ uint64_t sdesc_kmajor_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);            // start address   [0,14)
    d |= (uint64_t)(1) << 16;                          // LBO (ignored)   [16,30)
    d |= (uint64_t)(1024 >> 4) << 32;                  // SBO             [32,46)
    d |= (uint64_t)1 << 46;                            // version         [46,48)
    d |= (uint64_t)2 << 61;                            // SWIZZLE_128B    [61,64)
    return d;
}
// Instruction descriptor, kind::f16: D f32, A/B bf16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
    return (1u << 4)                 // D format F32
           | (1u << 7)               // A format BF16
           | (1u << 10)              // B format BF16
           | ((uint32_t)(n >> 3) << 17)
           | ((uint32_t)(BM >> 4) << 24);
}

template <int BN>
struct __align__(1024) GemmSmem {
    static constexpr int STAGES = stages_for(BN);
    __nv_bfloat16 a[STAGES][BM * BK];     // 16 KB per stage
    __nv_bfloat16 b[STAGES][BN * BK];
    uint64_t full[STAGES], empty[STAGES], accf;
    uint32_t tmem;
};

// the wide update tiles run two CTAs per SM (smem 2 × ~97 KB, TMEM 2 × 256 columns): the
// register budget must allow it (≤ 128 per thread at 2 × 256 threads)
__host__ __device__ constexpr int min_ctas_for(int bn) { return bn >= 256 ? 2 : 1; }

template <int BN, int EPI>
__global__ void __launch_bounds__(threads_for(BN), min_ctas_for(BN))
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K, Epi ep) {
    extern __shared__ __align__(1024) unsigned char raw[];
    GemmSmem<BN>& s = *reinterpret_cast<GemmSmem<BN>*>(
        raw + ((1024 - (smem_u32(raw) & 1023)) & 1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, z = blockIdx.z + ep.zoff;
    const int nk = (K + BK - 1) / BK;
    constexpr int STAGES = GemmSmem<BN>::STAGES;
    long long* trc = ep.trace ? ep.trace + 24LL * (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z))
                              : nullptr;
    auto tstamp = [&](int i) {
        if (trc) {
            long long t;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
            trc[i] = t;
        }
    };
    if (trc && threadIdx.x == 0) {
        long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        trc[0] = g;
        tstamp(1);
    }
    constexpr int NWE = threads_for(BN) / 32;     // epilogue warps: 4, or 8 (two per lane quadrant)
    constexpr int CSPAN = BN / (NWE / 4);          // columns per epilogue warp
    static_assert(sizeof(GemmSmem<BN>::a) + sizeof(GemmSmem<BN>::b) >=
                      NWE * 32 * 33 * sizeof(float) + (EPI == EPI_FWD ? 4 * BN * 16 * sizeof(float) : 0),
                  "epilogue tiles");

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&s.full[i], 1);
            mbar_init(&s.empty[i], 1);
        }
        mbar_init(&s.accf, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&s.tmem, BN < 32 ? 32 : BN);
    if (threadIdx.x == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = s.tmem;
    // everything above overlaps the previous kernel's tail (PDL); every global read and
    // write below comes after it has completed
    if (threadIdx.x == 0) tstamp(2);
    constexpr uint32_t kStageBytes = (BM + BN) * BK * 2;
    const int npre = ep.a_early ? (nk < STAGES ? nk : STAGES) : 0;
    if (warp == 0 && lane == 0) {
        for (int kt = 0; kt < npre; ++kt) {        // stage kt: expect A and B, issue A now
            mbar_arrive_expect_tx(&s.full[kt], kStageBytes);
            tma_load_3d(s.a[kt], &tmA, kt * BK, m0, z, &s.full[kt]);
        }
    }
    griddep_wait();
    griddep_launch();
    if (threadIdx.x == 0) tstamp(3);
    // the next layer's weights of this row tile (EPI_FWD with w3): staged by warps 2-3 while
    // the producer and MMA threads run (read after the accumulator barrier)
    __shared__ __align__(16) float w3s[EPI == EPI_FWD ? 16 * BM : 1];
    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        for (int kt = 0; kt < nk; ++kt) {
            const int st = kt % STAGES;
            if (kt >= STAGES) mbar_wait(&s.empty[st], (uint32_t)(((kt / STAGES) - 1) & 1));
            if (kt >= npre) {
                mbar_arrive_expect_tx(&s.full[st], kStageBytes);
                tma_load_3d(s.a[st], &tmA, kt * BK, m0, z, &s.full[st]);
            }
            tma_load_3d(s.b[st], &tmB, kt * BK, n0, z, &s.full[st]);
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_bf16(BN);
        for (int kt = 0; kt < nk; ++kt) {
            const int st = kt % STAGES;
            mbar_wait(&s.full[st], (uint32_t)((kt / STAGES) & 1));
            if (kt < 16) tstamp(4 + kt);
            fence_after();
            const uint32_t sa = smem_u32(s.a[st]), sb = smem_u32(s.b[st]);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
                mma_bf16(tmem, sdesc_kmajor_sw128(sa + kk * 32), sdesc_kmajor_sw128(sb + kk * 32), idesc,
                         (kt | kk) != 0);
            mma_commit(&s.empty[st]);                  // frees the stage once these MMAs read it
        }
        mma_commit(&s.accf);                           // accumulator complete
    }
    if constexpr (EPI == EPI_FWD) {
        if (ep.w3 && warp >= 2 && warp < 4) {      // 64 threads × 2 rows × 16 outputs; all loads
            const int rr = (threadIdx.x - 64) * 2; // issued first (a generic pointer may alias
                                                   // shared memory: stores would serialise them)
            uint32_t v[16];
            const __nv_bfloat16* w3 = ep.w3 + (long long)z * 16 * ep.M + m0 + rr;
            const bool ok = m0 + rr + 1 < ep.M && ((ep.M & 1) == 0);
#pragma unroll
            for (int o = 0; o < 16; ++o)
                v[o] = ok ? __ldg(reinterpret_cast<const unsigned int*>(w3 + (long long)o * ep.M)) : 0u;
#pragma unroll
            for (int o = 0; o < 16; ++o) {
                float2 f = ok ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[o])) : make_float2(0.f, 0.f);
                if (!ok) {
                    if (m0 + rr < ep.M) f.x = __bfloat162float(ep.w3[((long long)z * 16 + o) * ep.M + m0 + rr]);
                    if (m0 + rr + 1 < ep.M) f.y = __bfloat162float(ep.w3[((long long)z * 16 + o) * ep.M + m0 + rr + 1]);
                }
                w3s[rr * 16 + o] = f.x;            // [row][o]: a row's 16 weights are one
                w3s[(rr + 1) * 16 + o] = f.y;      // broadcast 4 × 16-byte read
            }
        }
    }
    // ---------------- epilogue: all 4 warps ----------------
    // Per 32-column chunk: (1) lane = tile row (the TMEM lane layout): per-row work and the
    // [n][m] outputs, which are coalesced in this mapping; (2) through a padded shared tile,
    // lane = column: the [m][n] outputs, coalesced 128-byte rows.  The operand stages are
    // free once the accumulator is complete, so the transpose tile reuses them.
    const int quad = warp & 3, chalf = warp >> 2;  // TMEM lanes 32·quad.., column half
    const int mrow0 = m0 + 32 * quad;
    // EPI_UPD: the fp32 master values of the next chunk are loaded one chunk ahead (the first
    // chunk's while the MMAs run): the epilogue is a chain of memory round trips otherwise.
    // (Lane = column, 32 rows: each load instruction is one coalesced 128-byte row segment; a
    // lane-per-row layout with vector accesses touches 32 lines per instruction and ran 1.7x
    // slower.)
    float old[EPI == EPI_UPD ? 32 : 1];
    auto load_old = [&](int c) {
        if constexpr (EPI == EPI_UPD) {
            const int n = n0 + c + lane;
            const float* ms = ep.master + (long long)z * ep.zs_master + (mrow0 * ep.N + n);
            const bool full = n < ep.nvalid && mrow0 + 32 <= ep.M;
#pragma unroll
            for (int r = 0; r < 32; ++r)
                old[r] = (full || (n < ep.nvalid && mrow0 + r < ep.M)) ? ms[r * ep.N] : 0.f;
        }
    };
    load_old(chalf * CSPAN);
    const int m = mrow0 + lane;                        // phase-1 row of this thread
    const bool mok = m < ep.M;
    // EPI_FWD / EPI_BWD operands that do not depend on the accumulator, loaded before it is
    // complete: the bias of this row; the ReLU mask of the first chunk (the next chunk's at
    // the end of each chunk) and the bias being updated
    float bias_pre = 0.f;
    if constexpr (EPI == EPI_FWD) bias_pre = mok ? ep.bias[(long long)z * ep.zs_bias + m] : 0.f;
    if constexpr (EPI == EPI_BWD) bias_pre = (mok && chalf == 0) ? ep.bias_upd[(long long)z * ep.zs_bias + m] : 0.f;
    __nv_bfloat16 mv[EPI == EPI_BWD ? 32 : 1];
    auto load_mask = [&](int c) {
        if constexpr (EPI == EPI_BWD) {
            const int n = n0 + c + lane;
            const __nv_bfloat16* mk = ep.mask + (long long)z * ep.zs_act + (mrow0 * ep.N + n);
            const int rows = (ep.M - mrow0) < 32 ? (ep.M - mrow0) : 32;
            const bool full = rows == 32 && n < ep.nvalid;
#pragma unroll
            for (int r = 0; r < 32; ++r)
                mv[r] = (full || (r < rows && n < ep.nvalid)) ? mk[r * ep.N] : __float2bfloat16_rn(0.f);
        }
    };
    load_mask(chalf * CSPAN);
    __syncwarp();
    mbar_wait(&s.accf, 0u);
    if (threadIdx.x == 0) tstamp(20);
    __syncwarp();
    fence_after();
    if constexpr (EPI == EPI_FWD) {
        if (ep.w3) __syncthreads();                // w3s staged
    }
    float (*tile)[33] = reinterpret_cast<float (*)[33]>(&s.a[0][0]) + 32 * warp;   // a then b: free now
    float rowsum = 0.f;
    float scale = 0.f;
    if constexpr (EPI == EPI_UPD || EPI == EPI_BWD) scale = update_scale(ep, z);
    // the epilogue is latency-bound (few warps): per-CN base pointers once, 32-bit offsets,
    // and a predicate-free path for full 32-row × 32-column chunks
    const int Mv = ep.M, Nv = ep.N, NVv = ep.nvalid;
    const int rows = Mv - mrow0 < 0 ? 0 : (Mv - mrow0 > 32 ? 32 : Mv - mrow0);
#pragma unroll 1
    for (int c = chalf * CSPAN; c < (chalf + 1) * CSPAN; c += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)c, v);
        if (threadIdx.x == 0 && c == 0) tstamp(23);
        const int nb = n0 + c;
        // ---- phase 1: lane = row
        if constexpr (EPI == EPI_FWD) {
            const float b = bias_pre;
            __nv_bfloat16* obm = ep.out_bm + (long long)z * ep.zs_act + m;   // [n][m]
            const bool fullc = mok && nb + 32 <= NVv;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const __nv_bfloat16 yb = __float2bfloat16_rn(fmaxf(v[i] + b, 0.f));   // ReLU (Eq.4), bias once (R1)
                if (fullc || (mok && nb + i < NVv)) obm[(nb + i) * Mv] = yb;
                v[i] = __bfloat162float(yb);
            }
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) tile[lane][i] = v[i];
        __syncwarp();
        // ---- phase 2: lane = column n = nb + lane
        const int n = nb + lane;
        const bool nok = n < NVv;
        const bool full = nok && rows == 32;
        const int off0 = mrow0 * Nv + n;               // [m][n] offset of (mrow0, n) in one CN's matrix
        if constexpr (EPI == EPI_STORE_F32) {
            float* o = ep.out_f32 + (long long)z * ep.zs_out + off0;
            if (full) {
#pragma unroll
                for (int r = 0; r < 32; ++r) o[r * Nv] = tile[r][lane];
            } else if (nok) {
#pragma unroll
                for (int r = 0; r < 32; ++r)
                    if (r < rows) o[r * Nv] = tile[r][lane];
            }
        } else if constexpr (EPI == EPI_FWD) {
            if (ep.out_mb) {
                __nv_bfloat16* omb = ep.out_mb + (long long)z * ep.zs_act + off0;
                if (full) {
#pragma unroll
                    for (int r = 0; r < 32; ++r) omb[r * Nv] = __float2bfloat16_rn(tile[r][lane]);
                } else if (nok) {
#pragma unroll
                    for (int r = 0; r < 32; ++r)
                        if (r < rows) omb[r * Nv] = __float2bfloat16_rn(tile[r][lane]);
                }
            }
            if (ep.w3) {                           // this warp's 32 rows' share of z3[n][o]
                float zp[16];
#pragma unroll
                for (int o = 0; o < 16; ++o) zp[o] = 0.f;
#pragma unroll 4
                for (int r = 0; r < 32; ++r) {
                    const float y = tile[r][lane];
                    const float4* wr = reinterpret_cast<const float4*>(w3s + (32 * quad + r) * 16);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float4 w4 = wr[u];
                        zp[4 * u] = fmaf(w4.x, y, zp[4 * u]);
                        zp[4 * u + 1] = fmaf(w4.y, y, zp[4 * u + 1]);
                        zp[4 * u + 2] = fmaf(w4.z, y, zp[4 * u + 2]);
                        zp[4 * u + 3] = fmaf(w4.w, y, zp[4 * u + 3]);
                    }
                }
                float* zr = reinterpret_cast<float*>(&s.a[0][0]) + NWE * 32 * 33;   // [4][BN][16]
#pragma unroll
                for (int o = 0; o < 16; ++o) zr[(quad * BN + (c + lane)) * 16 + o] = zp[o];
            }
        } else if constexpr (EPI == EPI_BWD) {
            // d = acc ⊙ [mask > 0] (ReLU'(z) from the stored activation, R9), mask [m][n]
            __nv_bfloat16* omb = ep.out_mb + (long long)z * ep.zs_act + off0;
            const bool nin = n < Nv;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                const float d = (__bfloat162float(mv[r]) > 0.f) ? tile[r][lane] : 0.f;
                tile[r][lane] = d;
                if ((rows == 32 && nin) || (r < rows && nin)) omb[r * Nv] = __float2bfloat16_rn(d);
            }
            if (c + 32 < (chalf + 1) * CSPAN) load_mask(c + 32);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 32; ++i) rowsum += tile[lane][i];     // phase 3: lane = row
        } else {  // EPI_UPD: W -= η·(Σ/B), bf16 copy
            float* ms = ep.master + (long long)z * ep.zs_master + off0;
            __nv_bfloat16* wb = ep.wb + (long long)z * ep.zs_w + off0;
            auto upd = [&](int r) {
                const float w = fmaf(-scale, tile[r][lane], old[r]);
                ms[r * Nv] = w;
                const __nv_bfloat16 w16 = __float2bfloat16_rn(w);
                wb[r * Nv] = w16;
                tile[r][lane] = __bfloat162float(w16);
            };
            if (full) {
#pragma unroll
                for (int r = 0; r < 32; ++r) upd(r);
            } else if (nok) {
#pragma unroll
                for (int r = 0; r < 32; ++r)
                    if (r < rows) upd(r);
            }
            if (c + 32 < (chalf + 1) * CSPAN) load_old(c + 32);
            if (ep.wbt) {                              // ---- phase 3: lane = row again, [n][m] copy
                __syncwarp();
                __nv_bfloat16* wt = ep.wbt + (long long)z * ep.zs_w + m;
                if (mok && nb + 32 <= NVv) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) wt[(nb + i) * Mv] = __float2bfloat16_rn(tile[lane][i]);
                } else if (mok) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (nb + i < NVv) wt[(nb + i) * Mv] = __float2bfloat16_rn(tile[lane][i]);
                }
            }
        }
        __syncwarp();
    }
    if (threadIdx.x == 0) tstamp(22);
    if constexpr (EPI == EPI_FWD) {
        if (ep.w3) {                               // sum the 4 row groups, in order
            __syncthreads();
            const float* zr = reinterpret_cast<const float*>(&s.a[0][0]) + NWE * 32 * 33;
            for (int i = threadIdx.x; i < BN * 16; i += blockDim.x) {
                const float t = ((zr[i] + zr[BN * 16 + i]) + zr[2 * BN * 16 + i]) + zr[3 * BN * 16 + i];
                if (n0 + i / 16 < ep.nvalid)
                    ep.z3part[(((long long)z * gridDim.x + blockIdx.x) * ep.N + n0 + i / 16) * 16 + (i % 16)] = t;
            }
        }
    }
    if constexpr (EPI == EPI_BWD) {
        if constexpr (NWE == 8) {                  // the two column halves of a row, in order
            float* rs = reinterpret_cast<float*>(&s.b[0][0]);
            if (chalf == 1) rs[32 * quad + lane] = rowsum;
            __syncthreads();
            if (chalf == 0) rowsum += rs[32 * quad + lane];
        }
        if (mok && chalf == 0) ep.bias_upd[(long long)z * ep.zs_bias + m] = bias_pre - scale * rowsum;   // b -= η·(Σδ/B)
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, BN < 32 ? 32 : BN);
    if (threadIdx.x == 0) tstamp(21);
}

template <int BN>
constexpr size_t smem_bytes() { return sizeof(GemmSmem<BN>) + 1024; }

}  // namespace tc
