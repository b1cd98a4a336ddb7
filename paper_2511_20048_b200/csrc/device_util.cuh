// Device helpers shared by the sm_100a kernels (PTX wrappers: mbarrier, TMA, ldmatrix,
// mma.sync, scoped atomics) and the PDL launch helper.
#pragma once

#include <atomic>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
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

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// non-blocking: has the phase of parity `parity` completed?
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
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

// F4 (fp8 KV): f16 MMA (fp32 accumulate), e4m3x2 -> f16x2 conversion, 4-B shared loads
__device__ __forceinline__ void mma16816_f16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

#ifndef SPA_F8_INTCVT
#define SPA_F8_INTCVT 0
#endif
// Two e4m3 codes (bits 7:0 -> low half, 15:8 -> high half) as f16x2.  SPA_F8_INTCVT = 0: the
// hardware conversion (value exact).  SPA_F8_INTCVT = 1: integer bit moves -- each code's
// byte at the top of its half, shifted right once, the sign carried back up -- which yield
// value * 2^-8 exactly (normals and subnormals; kF8Unit) for the caller to fold into its scales.
constexpr float kF8Unit = SPA_F8_INTCVT ? 256.f : 1.f;
__device__ __forceinline__ uint32_t e4m3x2_to_f16x2(uint32_t two_codes) {   // low byte -> low half
    uint32_t r;
#if defined(SPA_F8_EXP) && SPA_F8_EXP == 2   // timing experiment only: no conversion
    return two_codes;
#endif
#if SPA_F8_INTCVT
    uint32_t x;
    asm("prmt.b32 %0, %1, 0, 0x1404;" : "=r"(x) : "r"(two_codes));   // halves (b0 << 8, b1 << 8)
    const uint32_t y = x >> 1;                                       // sign lands on bit 14
    r = y + (y & 0x40004000u);                                       // ... and carries into bit 15
#else
    asm("{ .reg .b16 t; cvt.u16.u32 t, %1; cvt.rn.f16x2.e4m3x2 %0, t; }" : "=r"(r) : "r"(two_codes));
#endif
    return r;
}

// Four e4m3 codes (one 4-B fragment load) -> two f16x2 registers: bytes 0,1 -> lo, 2,3 -> hi.
// The 32-bit word is split into its b16 halves in PTX so ptxas can read the upper half in
// place instead of shifting it down first.
__device__ __forceinline__ void e4m3x4_to_f16x2x2(uint32_t w, uint32_t& lo, uint32_t& hi) {
#if SPA_F8_INTCVT || (defined(SPA_F8_EXP) && SPA_F8_EXP == 2)
    lo = e4m3x2_to_f16x2(w);
    hi = e4m3x2_to_f16x2(w >> 16);
#else
    asm("{ .reg .b16 l, h; mov.b32 {l, h}, %2; cvt.rn.f16x2.e4m3x2 %0, l; cvt.rn.f16x2.e4m3x2 %1, h; }"
        : "=r"(lo), "=r"(hi)
        : "r"(w));
#endif
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t w) {
    return pack_f16(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
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

// F1: output fan-out for the fused decode + all-gather.  Every
// output element is stored at its local address and at the same offset of each peer
// rank's gathered buffer: delta[k] is the byte distance from this rank's buffer to rank
// k's as mapped in this process (NVLink peer memory via CUDA IPC; delta[rank] = 0).
// fan == nullptr or n <= 1: the plain local store.
constexpr int kMaxPeers = 8;
struct OutFan {
    int n;
    int pad;
    long long delta[kMaxPeers];
};

__device__ __forceinline__ void st_out2(const OutFan* fan, __nv_bfloat16* p, float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    if (!fan || fan->n <= 1) {
        *reinterpret_cast<__nv_bfloat162*>(p) = v;
        return;
    }
    for (int k = 0; k < fan->n; ++k)
        *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<char*>(p) + fan->delta[k]) = v;
}

__device__ __forceinline__ void st_out1(const OutFan* fan, float* p, float v) {
    if (!fan || fan->n <= 1) {
        *p = v;
        return;
    }
    for (int k = 0; k < fan->n; ++k) *reinterpret_cast<float*>(reinterpret_cast<char*>(p) + fan->delta[k]) = v;
}

__device__ __forceinline__ void st_release_sys(unsigned* addr, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* addr) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(addr) : "memory");
    return v;
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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device context: remember it per
// device (bit d of *done), so a process driving several devices raises the limit on each.
template <typename... KArgs>
static int set_smem_attr_once(void (*kernel)(KArgs...), int smem, std::atomic<unsigned long long>* done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return int(e);
    const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
    if (bit && (done->load(std::memory_order_acquire) & bit)) return 0;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e) return int(e);
    done->fetch_or(bit, std::memory_order_acq_rel);
    return 0;
}

// Merge the split partials of G <= 8 consecutive heads [head0, head0 + G) of one request
// row, G x S <= 32 (S = s1 - s0 <= 16 records), D <= 128, in one warp pass: the LSEs of all
// G heads and the float4 columns [4 lane, 4 lane + 4) of all G x S partial rows are loaded
// back to back (one L2 round trip).  Per head the arithmetic (butterfly max and sum over
// lanes j < S, FMAs in record order) is that of warp_merge_head's S <= 16 path, so a head
// merged alone or within its group gets the same bits.
template <int DT>
__device__ __forceinline__ void warp_merge_group_small(const float* part_o, const float* part_lse, int H, int s0, int s1,
                                                       int head0, int G, __nv_bfloat16* orow, long long o_sh,
                                                       float* lrow, long long l_sh, int lane, int dim = DT,
                                                       const OutFan* fan = nullptr) {
    const int D = DT ? DT : dim;
    const int S = s1 - s0, GS = G * S;
    const int c = lane * 4;
    // every LSE (lane j < S holds record j of head hh in ls[hh]) and every partial row
    // (head-major, record-minor: v[hh * S + j]) in flight together
    float ls[8];
#pragma unroll
    for (int hh = 0; hh < 8; ++hh)
        ls[hh] = (hh < G && lane < S) ? __ldcg(part_lse + (long long)(s0 + lane) * H + head0 + hh) : -INFINITY;
    const long long rs = (long long)H * D;
    const float* pj = part_o + ((long long)s0 * H + head0) * D + c;
    float4 v[32];
    int jr = 0;
#pragma unroll
    for (int idx = 0; idx < 32; ++idx) {
        v[idx] = (idx < GS && c < D) ? __ldcg(reinterpret_cast<const float4*>(pj)) : make_float4(0.f, 0.f, 0.f, 0.f);
        pj += rs;
        if (++jr == S) {
            jr = 0;
            pj += D - S * rs;
        }
    }
    // per head: warp_merge_head's reduction; the weight of (hh, j) moves to lane hh * S + j
    float wflat = 0.f;
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
        if (hh < G) {
            float m = ls[hh];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float e = (ls[hh] != -INFINITY) ? expf(ls[hh] - m) : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
            const float lse = (m == -INFINITY) ? -INFINITY : m + logf(e);
            const float w = (ls[hh] != -INFINITY) ? expf(ls[hh] - lse) : 0.f;
            const int src = lane - hh * S;
            const float wm = __shfl_sync(0xffffffffu, w, src & 31);
            if (src >= 0 && src < S) wflat = wm;
            if (lane == 0 && lrow) st_out1(fan, lrow + (long long)(head0 + hh) * l_sh, lse);
        }
    }
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    int jj = 0, hc = 0;
#pragma unroll
    for (int idx = 0; idx < 32; ++idx) {
        if (idx < GS) {
            const float wj = __shfl_sync(0xffffffffu, wflat, idx);
            if (wj != 0.f) {
                a.x += wj * v[idx].x;
                a.y += wj * v[idx].y;
                a.z += wj * v[idx].z;
                a.w += wj * v[idx].w;
            }
            if (++jj == S) {
                if (c < D) {
                    __nv_bfloat16* op = orow + (long long)(head0 + hc) * o_sh + c;
                    st_out2(fan, op, a.x, a.y);
                    st_out2(fan, op + 2, a.z, a.w);
                }
                a = make_float4(0.f, 0.f, 0.f, 0.f);
                jj = 0;
                ++hc;
            }
        }
    }
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
                                                long long l_sh, int lane, int dim = DT,
                                                const OutFan* fan = nullptr) {
    const int D = DT ? DT : dim;
    orow += (long long)head * o_sh;
    if (s1 - s0 <= 16 && D <= 128) {
        // few records: issue the LSE loads and every partial O load back to back (one L2
        // round trip), then reduce in registers (warp_merge_group_small repeats this
        // arithmetic per head, so both give the same bits)
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
            if (j < S) {
                const float wj = __shfl_sync(0xffffffffu, w, j);
                if (wj != 0.f) {
                    a.x += wj * v[j].x;
                    a.y += wj * v[j].y;
                    a.z += wj * v[j].z;
                    a.w += wj * v[j].w;
                }
            }
        }
        if (c < D) {
            st_out2(fan, orow + c, a.x, a.y);
            st_out2(fan, orow + c + 2, a.z, a.w);
        }
        if (lane == 0 && lrow) st_out1(fan, lrow + (long long)head * l_sh, lse);
        return;
    }
    if (s1 - s0 <= 128 && D <= 128) {
        // up to 128 records: every LSE in one round trip (4 per lane), then the partial O rows
        // in chunks of 16 records, each chunk's loads issued back to back (one round trip each)
        const int S = s1 - s0;
        const int c = lane * 4;
        float ls[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            ls[k] = lane + 32 * k < S ? __ldcg(part_lse + (long long)(s0 + lane + 32 * k) * H + head) : -INFINITY;
        float m = fmaxf(fmaxf(ls[0], ls[1]), fmaxf(ls[2], ls[3]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float e = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) e += (ls[k] != -INFINITY) ? expf(ls[k] - m) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        const float lse = (m == -INFINITY) ? -INFINITY : m + logf(e);
        float w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = (ls[k] != -INFINITY) ? expf(ls[k] - lse) : 0.f;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int cb = 0; cb < S; cb += 16) {
            float4 v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
                v[j] = (cb + j < S && c < D)
                           ? __ldcg(reinterpret_cast<const float4*>(part_o + ((long long)(s0 + cb + j) * H + head) * D + c))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            const int k = cb >> 5;
            const float wk = k == 0 ? w[0] : k == 1 ? w[1] : k == 2 ? w[2] : w[3];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float wj = __shfl_sync(0xffffffffu, wk, (cb & 31) + j);
                if (cb + j < S && wj != 0.f) {
                    a.x += wj * v[j].x;
                    a.y += wj * v[j].y;
                    a.z += wj * v[j].z;
                    a.w += wj * v[j].w;
                }
            }
        }
        if (c < D) {
            st_out2(fan, orow + c, a.x, a.y);
            st_out2(fan, orow + c + 2, a.z, a.w);
        }
        if (lane == 0 && lrow) st_out1(fan, lrow + (long long)head * l_sh, lse);
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
            st_out2(fan, orow + c, a.x, a.y);
            st_out2(fan, orow + c + 2, a.z, a.w);
        }
    }
    if (lane == 0 && lrow) st_out1(fan, lrow + (long long)head * l_sh, lse);
}

// A whole (row, KV head) task with exactly S = 2 records (a shared range + a tail: the common
// case of prefix sharing), G <= 8 heads: every lane loads both LSEs and its float4 column of
// both partial rows of every head up front (one L2 round trip, no shuffles), then reduces in
// registers.  Per head the arithmetic is warp_merge_head's S <= 16 path (max; butterfly sum
// of exp(LSE_j - m), which for two live lanes is e_0 + e_1; weights exp(LSE_j - LSE); FMAs in
// record order), so the result has the same bits.
template <int DT>
__device__ __forceinline__ void warp_merge_task_s2(const float* part_o, const float* part_lse, int H, int s0,
                                                   int head0, int G, __nv_bfloat16* orow, long long o_sh,
                                                   float* lrow, long long l_sh, int lane) {
    constexpr int D = DT;
    const int c = lane * 4;
    float l0[8], l1[8];
    float4 v0[8], v1[8];
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
        if (hh < G) {
            l0[hh] = __ldcg(part_lse + (long long)s0 * H + head0 + hh);
            l1[hh] = __ldcg(part_lse + (long long)(s0 + 1) * H + head0 + hh);
            if (c < D) {
                v0[hh] = __ldcg(reinterpret_cast<const float4*>(part_o + ((long long)s0 * H + head0 + hh) * D + c));
                v1[hh] = __ldcg(reinterpret_cast<const float4*>(part_o + ((long long)(s0 + 1) * H + head0 + hh) * D + c));
            }
        }
    }
#pragma unroll
    for (int hh = 0; hh < 8; ++hh) {
        if (hh < G) {
            const float m = fmaxf(l0[hh], l1[hh]);
            const float e0 = (l0[hh] != -INFINITY) ? expf(l0[hh] - m) : 0.f;
            const float e1 = (l1[hh] != -INFINITY) ? expf(l1[hh] - m) : 0.f;
            const float e = e0 + e1;
            const float lse = (m == -INFINITY) ? -INFINITY : m + logf(e);
            const float w0 = (l0[hh] != -INFINITY) ? expf(l0[hh] - lse) : 0.f;
            const float w1 = (l1[hh] != -INFINITY) ? expf(l1[hh] - lse) : 0.f;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
            if (w0 != 0.f) {
                a.x += w0 * v0[hh].x;
                a.y += w0 * v0[hh].y;
                a.z += w0 * v0[hh].z;
                a.w += w0 * v0[hh].w;
            }
            if (w1 != 0.f) {
                a.x += w1 * v1[hh].x;
                a.y += w1 * v1[hh].y;
                a.z += w1 * v1[hh].z;
                a.w += w1 * v1[hh].w;
            }
            if (c < D) {
                __nv_bfloat16* op = orow + (long long)(head0 + hh) * o_sh + c;
                st_out2(nullptr, op, a.x, a.y);
                st_out2(nullptr, op + 2, a.z, a.w);
            }
            if (lane == 0 && lrow) st_out1(nullptr, lrow + (long long)(head0 + hh) * l_sh, lse);
        }
    }
}

// Merge heads [head0, head0 + G) of one request row: all G in one warp pass when
// G x S <= 32, else head by head (warp_merge_head).  Bit-identical to merging each head
// alone with warp_merge_head, so every merge mode and path of the library agrees bitwise.
template <int DT>
__device__ __forceinline__ void warp_merge_group(const float* part_o, const float* part_lse, int H, int s0, int s1,
                                                 int head0, int G, __nv_bfloat16* orow, long long o_sh, float* lrow,
                                                 long long l_sh, int lane, int dim = DT,
                                                 const OutFan* fan = nullptr) {
    const int D = DT ? DT : dim;
    if (G <= 8 && G * (s1 - s0) <= 32 && s1 - s0 <= 16 && D <= 128) {
        warp_merge_group_small<DT>(part_o, part_lse, H, s0, s1, head0, G, orow, o_sh, lrow, l_sh, lane, dim, fan);
        return;
    }
    for (int hh = 0; hh < G; ++hh)
        warp_merge_head<DT>(part_o, part_lse, H, s0, s1, head0 + hh, orow, o_sh, lrow, l_sh, lane, dim, fan);
}

}  // namespace spa
