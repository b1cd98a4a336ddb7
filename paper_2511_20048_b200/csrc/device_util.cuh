// Device helpers shared by the sm_100a kernels (PTX wrappers: mbarrier, TMA, ldmatrix,
// mma.sync, scoped atomics) and the PDL launch helper.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

namespace spa {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// D(16x8, f32) += A(16x16, bf16, row) * B(16x8, bf16, col)
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* addr, int v) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(addr), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void red_add_release_gpu(int* addr, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release_gpu(int* addr, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_gpu(const int* addr) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(addr) : "memory");
    return v;
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

// Launch with programmatic stream serialization (PDL): the kernel may start while the
// previous kernel on the stream drains; every kernel here begins with griddepcontrol.wait
// before touching memory the previous one wrote.  SPA_NO_PDL=1 disables it (A/B runs).
template <typename... KArgs, typename... Args>
static int launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, void* stream, Args&&... args) {
    static const bool no_pdl = std::getenv("SPA_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = no_pdl ? 0 : 1;
    return int(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// ============================================================================ a6 core: one warp merges one head
// Split-KV partial-LSE merge of records [s0, s1) of one (request, head) (oracle:
// merge_partials; include/spa.h spa_merge_splits):
//     LSE = m + ln sum_{s live} exp(LSE_s - m),  O = sum_s exp(LSE_s - LSE) O_s,
//     all partials -inf -> O = 0, LSE = -inf.
// Lanes own records for the LSE reduction (shuffle max / sum) and float4 columns for O;
// partials are read with ld.global.cg (L2): they were written by other SMs.
template <int DT>   // DT = head_dim if known at compile time, 0 = runtime `dim`
__device__ __forceinline__ void warp_merge_head(const float* part_o, const float* part_lse, int H, int s0, int s1,
                                                int head, __nv_bfloat16* orow, long long o_sh, float* lrow,
                                                long long l_sh, int lane, int dim = DT) {
    const int D = DT ? DT : dim;
    orow += (long long)head * o_sh;
    if (s1 - s0 <= 16 && D <= 128) {
        // few records (<= 2 x the automatic split cap): issue the LSE loads and every partial
        // O load back to back -- one L2 round trip -- then reduce in registers
        const int S = s1 - s0;
        const int c = lane * 4;
        const float ls = lane < S ? __ldcg(part_lse + (long long)(s0 + lane) * H + head) : -INFINITY;
        float4 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            v[j] = (j < S && c < D)
                       ? __ldcg(reinterpret_cast<const float4*>(part_o + ((long long)(s0 + j) * H + head) * D + c))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        float m = ls;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float e = (ls != -INFINITY) ? expf(ls - m) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        const float lse = (m == -INFINITY) ? -INFINITY : m + logf(e);
        const float w = (ls != -INFINITY) ? expf(ls - lse) : 0.f;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float wj = __shfl_sync(0xffffffffu, w, j);
            if (j < S && wj != 0.f) {
                a.x += wj * v[j].x;
                a.y += wj * v[j].y;
                a.z += wj * v[j].z;
                a.w += wj * v[j].w;
            }
        }
        if (c < D) {
            *reinterpret_cast<__nv_bfloat162*>(orow + c) = __floats2bfloat162_rn(a.x, a.y);
            *reinterpret_cast<__nv_bfloat162*>(orow + c + 2) = __floats2bfloat162_rn(a.z, a.w);
        }
        if (lane == 0 && lrow) lrow[(long long)head * l_sh] = lse;
        return;
    }
    if (s1 - s0 <= 32) {
        // common case: one record per lane, the LSEs are read once (one L2 round trip for
        // the LSEs, one for the partial O rows, issued back to back)
        const int S = s1 - s0;
        const float ls = lane < S ? __ldcg(part_lse + (long long)(s0 + lane) * H + head) : -INFINITY;
        float m = ls;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float e = (ls != -INFINITY) ? expf(ls - m) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        const float lse = (m == -INFINITY) ? -INFINITY : m + logf(e);
        const float w = (ls != -INFINITY) ? expf(ls - lse) : 0.f;
        for (int c = lane * 4; c - lane * 4 < D; c += 128) {
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
            for (int j = 0; j < S; ++j) {
                const float wj = __shfl_sync(0xffffffffu, w, j);
                if (c < D && wj != 0.f) {
                    const float4 v =
                        __ldcg(reinterpret_cast<const float4*>(part_o + ((long long)(s0 + j) * H + head) * D + c));
                    a.x += wj * v.x;
                    a.y += wj * v.y;
                    a.z += wj * v.z;
                    a.w += wj * v.w;
                }
            }
            if (c < D) {
                *reinterpret_cast<__nv_bfloat162*>(orow + c) = __floats2bfloat162_rn(a.x, a.y);
                *reinterpret_cast<__nv_bfloat162*>(orow + c + 2) = __floats2bfloat162_rn(a.z, a.w);
            }
        }
        if (lane == 0 && lrow) lrow[(long long)head * l_sh] = lse;
        return;
    }
    float m = -INFINITY;
    for (int sb = s0; sb < s1; sb += 32) {
        const int s = sb + lane;
        if (s < s1) m = fmaxf(m, __ldcg(part_lse + (long long)s * H + head));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float sum = 0.f;
    if (m != -INFINITY) {
        for (int sb = s0; sb < s1; sb += 32) {
            const int s = sb + lane;
            if (s < s1) {
                const float ls = __ldcg(part_lse + (long long)s * H + head);
                if (ls != -INFINITY) sum += expf(ls - m);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float lse = (m == -INFINITY) ? -INFINITY : m + logf(sum);
    for (int c = lane * 4; c - lane * 4 < D; c += 128) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m != -INFINITY) {
            for (int sb = s0; sb < s1; sb += 32) {
                const int s = sb + lane;
                float w = 0.f;
                if (s < s1) {
                    const float ls = __ldcg(part_lse + (long long)s * H + head);
                    if (ls != -INFINITY) w = expf(ls - lse);
                }
                const int n = min(32, s1 - sb);
#pragma unroll 8
                for (int j = 0; j < n; ++j) {
                    const float wj = __shfl_sync(0xffffffffu, w, j);
                    if (c < D) {
                        const float4 v = __ldcg(reinterpret_cast<const float4*>(part_o + ((long long)(sb + j) * H + head) * D + c));
                        a.x += wj * v.x;
                        a.y += wj * v.y;
                        a.z += wj * v.z;
                        a.w += wj * v.w;
                    }
                }
            }
        }
        if (c < D) {
            *reinterpret_cast<__nv_bfloat162*>(orow + c) = __floats2bfloat162_rn(a.x, a.y);
            *reinterpret_cast<__nv_bfloat162*>(orow + c + 2) = __floats2bfloat162_rn(a.z, a.w);
        }
    }
    if (lane == 0 && lrow) lrow[(long long)head * l_sh] = lse;
}

}  // namespace spa
