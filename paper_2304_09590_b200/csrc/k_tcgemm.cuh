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
constexpr int STAGES = 4;

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
    // EPI_BWD: d = acc ⊙ [mask[z][n][m] > 0]; out_mb[z][m][n] = bf16(d);
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
    __nv_bfloat16 a[STAGES][BM * BK];     // 16 KB per stage
    __nv_bfloat16 b[STAGES][BN * BK];
    uint64_t full[STAGES], empty[STAGES], accf;
    uint32_t tmem;
};

template <int BN, int EPI>
__global__ void __launch_bounds__(128, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K, Epi ep) {
    extern __shared__ __align__(1024) unsigned char raw[];
    GemmSmem<BN>& s = *reinterpret_cast<GemmSmem<BN>*>(
        raw + ((1024 - (smem_u32(raw) & 1023)) & 1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, z = blockIdx.z + ep.zoff;
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&s.full[i], 1);
            mbar_init(&s.empty[i], 1);
        }
        mbar_init(&s.accf, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&s.tmem, BN < 32 ? 32 : BN);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = s.tmem;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        constexpr uint32_t bytes = (BM + BN) * BK * 2;
        for (int kt = 0; kt < nk; ++kt) {
            const int st = kt % STAGES;
            if (kt >= STAGES) mbar_wait(&s.empty[st], (uint32_t)(((kt / STAGES) - 1) & 1));
            mbar_arrive_expect_tx(&s.full[st], bytes);
            tma_load_3d(s.a[st], &tmA, kt * BK, m0, z, &s.full[st]);
            tma_load_3d(s.b[st], &tmB, kt * BK, n0, z, &s.full[st]);
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_bf16(BN);
        for (int kt = 0; kt < nk; ++kt) {
            const int st = kt % STAGES;
            mbar_wait(&s.full[st], (uint32_t)((kt / STAGES) & 1));
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
    // ---------------- epilogue: all 4 warps ----------------
    __syncwarp();
    mbar_wait(&s.accf, 0u);
    __syncwarp();
    fence_after();
    const int m = m0 + 32 * warp + lane;               // this thread's tile row
    const bool mok = m < ep.M;
    float rowsum = 0.f;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c, v);
        const int nb = n0 + c;
        if (!mok) continue;
        if constexpr (EPI == EPI_STORE_F32) {
            float* o = ep.out_f32 + (long long)z * ep.zs_out + (long long)m * ep.N + nb;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (nb + i < ep.nvalid) o[i] = v[i];
        } else if constexpr (EPI == EPI_FWD) {
            const float b = ep.bias[(long long)z * ep.zs_bias + m];
            __nv_bfloat16* obm = ep.out_bm + (long long)z * ep.zs_act;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float y = fmaxf(v[i] + b, 0.f);    // φ = ReLU (Eq.4), bias once (R1)
                const __nv_bfloat16 yb = __float2bfloat16_rn(y);
                if (nb + i < ep.nvalid) {
                    obm[(long long)(nb + i) * ep.M + m] = yb;
                    if (ep.out_mb) ep.out_mb[(long long)z * ep.zs_act + (long long)m * ep.N + nb + i] = yb;
                }
            }
        } else if constexpr (EPI == EPI_BWD) {
            const __nv_bfloat16* mk = ep.mask + (long long)z * ep.zs_act;
            __nv_bfloat16* omb = ep.out_mb + (long long)z * ep.zs_act + (long long)m * ep.N;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (nb + i < ep.nvalid) {
                    const float d = (__bfloat162float(mk[(long long)(nb + i) * ep.M + m]) > 0.f) ? v[i] : 0.f;
                    omb[nb + i] = __float2bfloat16_rn(d);
                    rowsum += d;
                } else if (nb + i < ep.N) {
                    omb[nb + i] = __float2bfloat16_rn(0.f);
                }
            }
        } else {  // EPI_UPD
            const float scale = update_scale(ep, z);
            float* ms = ep.master + (long long)z * ep.zs_master + (long long)m * ep.N + nb;
            __nv_bfloat16* wb = ep.wb + (long long)z * ep.zs_w + (long long)m * ep.N + nb;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (nb + i < ep.nvalid) {
                    const float w = fmaf(-scale, v[i], ms[i]);   // W -= η·(Σ/B)
                    ms[i] = w;
                    const __nv_bfloat16 w16 = __float2bfloat16_rn(w);
                    wb[i] = w16;
                    if (ep.wbt) ep.wbt[(long long)z * ep.zs_w + (long long)(nb + i) * ep.M + m] = w16;
                }
            }
        }
    }
    if constexpr (EPI == EPI_BWD) {
        if (mok) ep.bias_upd[(long long)z * ep.zs_bias + m] -= update_scale(ep, z) * rowsum;   // b -= η·(Σδ/B)
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, BN < 32 ? 32 : BN);
}

template <int BN>
constexpr size_t smem_bytes() { return sizeof(GemmSmem<BN>) + 1024; }

}  // namespace tc
