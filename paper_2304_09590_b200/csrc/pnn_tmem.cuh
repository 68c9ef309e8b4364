// pnn_tmem.cuh — tensor-memory (TMEM) access for the CUDA-core kernels that keep data in
// TMEM outside a tcgen05.mma (k_tmem.cu: W¹ rows; k_mbres.cu: the mini-batch W¹ gradient).
// 32x32b shapes: thread t of the warp ↔ TMEM lane (32·(warp % 4) + t); N consecutive 32-bit
// columns per instruction.  Measured (tools/ubench/tmem.cu): ~1.7-4 KB/clk/SM load,
// ~0.95 KB/clk/SM store, 38-cycle load latency.
#pragma once
#include <cstdint>
#include "pnn_ptx.cuh"

namespace tmem {

__device__ __forceinline__ void alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// wait::ld, then tie the loaded registers to it: an empty volatile asm that "rewrites" each
// register keeps the compiler from hoisting their uses above the wait.
template <int N> __device__ __forceinline__ void wait_ld_regs(uint32_t* a) {
    wait_ld();
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("" : "+r"(a[i]));
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#define PNN_TM_R4(a, i) "=r"(a[i]), "=r"(a[i + 1]), "=r"(a[i + 2]), "=r"(a[i + 3])
#define PNN_TM_W4(a, i) "r"(a[i]), "r"(a[i + 1]), "r"(a[i + 2]), "r"(a[i + 3])
__device__ __forceinline__ void ld4(uint32_t t, uint32_t* a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : PNN_TM_R4(a, 0) : "r"(t));
}
__device__ __forceinline__ void ld8(uint32_t t, uint32_t* a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : PNN_TM_R4(a, 0), PNN_TM_R4(a, 4)
                 : "r"(t));
}
__device__ __forceinline__ void ld16(uint32_t t, uint32_t* a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : PNN_TM_R4(a, 0), PNN_TM_R4(a, 4), PNN_TM_R4(a, 8), PNN_TM_R4(a, 12)
                 : "r"(t));
}
__device__ __forceinline__ void ld32(uint32_t t, uint32_t* a) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : PNN_TM_R4(a, 0), PNN_TM_R4(a, 4), PNN_TM_R4(a, 8), PNN_TM_R4(a, 12), PNN_TM_R4(a, 16), PNN_TM_R4(a, 20),
          PNN_TM_R4(a, 24), PNN_TM_R4(a, 28)
        : "r"(t));
}
__device__ __forceinline__ void st4(uint32_t t, const uint32_t* a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(t), PNN_TM_W4(a, 0) : "memory");
}
__device__ __forceinline__ void st8(uint32_t t, const uint32_t* a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t), PNN_TM_W4(a, 0),
                 PNN_TM_W4(a, 4)
                 : "memory");
}
__device__ __forceinline__ void st16(uint32_t t, const uint32_t* a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(t), PNN_TM_W4(a, 0), PNN_TM_W4(a, 4), PNN_TM_W4(a, 8), PNN_TM_W4(a, 12)
                 : "memory");
}
__device__ __forceinline__ void st32(uint32_t t, const uint32_t* a) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t),
        PNN_TM_W4(a, 0), PNN_TM_W4(a, 4), PNN_TM_W4(a, 8), PNN_TM_W4(a, 12), PNN_TM_W4(a, 16), PNN_TM_W4(a, 20),
        PNN_TM_W4(a, 24), PNN_TM_W4(a, 28)
        : "memory");
}
#undef PNN_TM_R4
#undef PNN_TM_W4

}  // namespace tmem
