// k_minibatch.cu — the bf16 mini-batch variant (a10) on tcgen05 GEMMs, and a test hook
// for the GEMM alone.  See k_tcgemm.cuh for the GEMM kernel.
#include <cstdio>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "pnn_internal.h"
#include "k_tcgemm.cuh"

namespace {

using PFN_encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encode encode_fn() {
    static PFN_encode fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encode>(p);
    }
    return fn;
}

}  // namespace

// A K-major bf16 tensor [Z][rows][K] as a TMA map with a 64 × box_rows box, 128-byte
// swizzle, zero fill out of bounds.  Returns false on failure.
bool make_tmap_kmajor(CUtensorMap* tm, const void* base, int K, int rows, int Z, int box_rows) {
    PFN_encode fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)Z};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)K * rows * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int EPI>
static cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int Z, int M, int N, int K,
                               const tc::Epi& ep, cudaStream_t st) {
    auto kern = tc::gemm_kernel<BN, EPI>;
    const size_t smem = tc::smem_bytes<BN>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((M + tc::BM - 1) / tc::BM), (unsigned)((N + BN - 1) / BN), (unsigned)Z);
    kern<<<grid, 128, smem, st>>>(ta, tb, K, ep);
    return cudaGetLastError();
}

// Test hook (tests/test_gpu_tcgemm.py): C[z][m][n] = Σ_k A[z][m][k]·B[z][n][k], fp32 out.
extern "C" int pnn_debug_tc_gemm(const void* A, const void* B, float* C, int Z, int M, int N, int K, int bn) {
    CUtensorMap ta, tb;
    if (!make_tmap_kmajor(&ta, A, K, M, Z, tc::BM)) return 1;
    if (!make_tmap_kmajor(&tb, B, K, N, Z, bn)) return 2;
    tc::Epi ep{};
    ep.M = M;
    ep.N = N;
    ep.nvalid = N;
    ep.out_f32 = C;
    ep.zs_out = (long long)M * N;
    cudaError_t e;
    switch (bn) {
    case 64: e = launch_gemm<64, tc::EPI_STORE_F32>(ta, tb, Z, M, N, K, ep, 0); break;
    case 128: e = launch_gemm<128, tc::EPI_STORE_F32>(ta, tb, Z, M, N, K, ep, 0); break;
    case 256: e = launch_gemm<256, tc::EPI_STORE_F32>(ta, tb, Z, M, N, K, ep, 0); break;
    default: return 3;
    }
    if (e != cudaSuccess) return 10 + (int)e;
    e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 1000 + (int)e;
}
