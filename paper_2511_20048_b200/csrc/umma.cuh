// tcgen05 (5th-generation tensor core) helpers for sm_100a: shared-memory matrix
// descriptors, instruction descriptors, MMA issue/commit, tensor-memory alloc/ld/st.
// Layout conventions are the canonical UMMA layouts (CUTLASS cute/atom/mma_traits_sm100.hpp,
// read for the bit positions only):
//   K-major SWIZZLE_128B  ((8,m),(T,2)):((8T,SBO),(1,T)) in 16-B units -- rows of 128 B,
//       8-row atoms SBO bytes apart; a K step of 16 bf16 advances the start address 32 B
//       inside the 128-B row (the hardware applies the swizzle to the address bits, so the
//       atom base must be 1024-B aligned).
//   MN-major SWIZZLE_128B ((8,n),(8,k)):((1,LBO),(8,SBO)) -- 64 bf16 of MN contiguous per
//       128-B row, the next 64 MN elements LBO bytes on, 8 K-rows per atom, the next 8 K-rows
//       SBO bytes on.
// TMA with CU_TENSOR_MAP_SWIZZLE_128B writes exactly the 128-B swizzle these layouts expect
// (16-B chunk c of row r lands at chunk c ^ (r % 8) of its 1024-B atom).
#pragma once
#include <cstdint>

namespace spa {
namespace umma {

// ---------------------------------------------------------------- shared-memory descriptors
__device__ __forceinline__ uint64_t desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= uint64_t((smem_addr >> 4) & 0x3FFF);            // start address        [0,14)
    d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;      // leading byte offset  [16,30)
    d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;      // stride byte offset   [32,46)
    d |= uint64_t(1) << 46;                              // version = 1 (sm_100) [46,48)
    //    base offset [49,52) = 0, LBO mode [52] = 0 (legacy)
    d |= uint64_t(2) << 61;                              // layout: SWIZZLE_128B [61,64)
    return d;
}
// K-major SW128 (A or B operand with K contiguous): LBO unused (1), SBO = 8-row atom stride
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t smem_addr, uint32_t sbo_bytes) {
    return desc_sw128(smem_addr, 16, sbo_bytes);
}
// MN-major SW128 (B operand with N contiguous): LBO = stride between 64-element MN atoms,
// SBO = stride between 8-row K groups
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return desc_sw128(smem_addr, lbo_bytes, sbo_bytes);
}

// ---------------------------------------------------------------- instruction descriptor
// kind::f16: bf16 x bf16 -> fp32, dense.  a_mn / b_mn: operand is MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, bool a_mn, bool b_mn) {
    return (1u << 4)                          // c_format F32        [4,6)
           | (1u << 7)                        // a_format BF16       [7,10)
           | (1u << 10)                       // b_format BF16       [10,13)
           | (uint32_t(a_mn) << 15)           // a_major             [15]
           | (uint32_t(b_mn) << 16)           // b_major             [16]
           | (uint32_t(N >> 3) << 17)         // N >> 3              [17,23)
           | (uint32_t(M >> 4) << 24);        // M >> 4              [24,29)
}

// ---------------------------------------------------------------- MMA issue (one thread)
// D[tmem] (+)= A[smem desc] x B[smem desc]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       bool accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(uint32_t(accumulate))
        : "memory");
}
// D[tmem] (+)= A[tmem] x B[smem desc]   (A: M lanes x K, two bf16 per 32-bit column)
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       bool accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(uint32_t(accumulate))
        : "memory");
}
// arrive (once) on an mbarrier when every MMA issued so far by this thread has completed
__device__ __forceinline__ void commit(uint32_t mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
                 : "memory");
}

// elect one lane of the (converged) warp: the MMA issuer of a warp-uniform loop
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, %1;\n@px mov.s32 %0, 1;\n}\n"
        : "+r"(pred)
        : "r"(0xffffffffu));
    return pred != 0;
}

// ---------------------------------------------------------------- tensor memory
__device__ __forceinline__ void tmem_alloc(uint32_t smem_dst, uint32_t ncols) {   // one warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_dst), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {   // the same warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 consecutive fp32 columns of this thread's lane (warp w reads lanes 32 (w % 4) + 0..31)
__device__ __forceinline__ void ld32(uint32_t taddr, float* v) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
// 16 consecutive 32-bit columns of this thread's lane
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
// 32 consecutive 32-bit columns of this thread's lane
__device__ __forceinline__ void st32(uint32_t taddr, const float* v) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// byte offset of 16-B chunk `c` (0..7) of row `r` inside a 128-B-swizzled tile of 128-B rows
__host__ __device__ constexpr uint32_t sw128_offset(uint32_t r, uint32_t c) {
    return (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
}

}  // namespace umma
}  // namespace spa
