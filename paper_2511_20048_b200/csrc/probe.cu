// Bandwidth probes (measurement infrastructure, include/spa_debug.h): the read ceilings the
// decode kernel's achieved HBM bandwidth is compared against in the same bench run.
//   ldg_read_kernel      streaming 16-B loads (ld.global.nc.L1::no_allocate), 8 in flight
//                        per thread, persistent grid
//   tma_pool_read_kernel the decode kernel's memory pipeline with the math removed:
//                        per-warp rings of NS stages, 2 (page, head) K+V pairs per stage,
//                        static round-robin assignment of stages to warps.  Copy modes:
//                          0  the pool's 3-D tensor maps, one 64 x 16 x d/64 box per
//                             page-head (exactly the decode kernel's copies)
//                          1  3-D map ordered (64, d/64, rows): same bytes, [row][block] layout
//                          2  1-D bulk copies (cp.async.bulk), 4 KB per page-head, no swizzle
#include <dlfcn.h>

#include "device_util.cuh"
#include "spa_internal.h"
#include "umma.cuh"
#include "../../include/spa_debug.h"

namespace spa {

__global__ void __launch_bounds__(256) ldg_read_kernel(const uint4* __restrict__ p, size_t n, unsigned* sink) {
    unsigned acc = 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                         : "l"(p + i + k * stride));
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    for (; i < n; i += stride) acc ^= p[i].x;
    if (acc == 0x9e3779b9u) sink[0] = acc;   // practically never: defeats dead-code elimination
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}

// unit u: layer = u / (pairs * Hkv), then (page pair, head); 2 pages x (K, V) per stage
template <int D, int MODE>
__global__ void __launch_bounds__(kWarps * 32, 1)
    tma_pool_read_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                         const uint16_t* kp, const uint16_t* vp, int units, int pairs_per_layer, int Hkv,
                         int num_pages) {
    constexpr int PAGE_BYTES = kPageSize * D * 2;
    constexpr int STAGE_BYTES = 2 * 2 * PAGE_BYTES;
    constexpr int NS = (kSmemBudget - 1024) / (kWarps * STAGE_BYTES);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t ring = smem_u32(smem) + warp * NS * STAGE_BYTES;
    const uint32_t bars = smem_u32(smem) + kWarps * NS * STAGE_BYTES + warp * NS * 8;
    if (lane == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(bars + s * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
    const int my_units = gw < units ? (units - gw + nw - 1) / nw : 0;
    int next = 0;   // next of my units to issue
    auto issue = [&](int slot) {
        const int u = gw + next * nw;
        ++next;
        const int layer = u / (pairs_per_layer * Hkv);
        const int rem = u - layer * pairs_per_layer * Hkv;
        const int pair = rem / Hkv, h = rem - pair * Hkv;
        const uint32_t bar = bars + slot * 8;
        mbar_expect_tx(bar, STAGE_BYTES);
        for (int j = 0; j < 2; ++j) {
            const int page = pair * 2 + j;
            const int row = ((layer * num_pages + page) * Hkv + h) * kPageSize;
            const uint32_t dk = ring + slot * STAGE_BYTES + j * 2 * PAGE_BYTES;
            if (MODE == 0) {
                tma_load_3d(dk, &tmk, 0, row, 0, bar, policy);
                tma_load_3d(dk + PAGE_BYTES, &tmv, 0, row, 0, bar, policy);
            } else if (MODE == 1) {
                tma_load_3d(dk, &tmk, 0, 0, row, bar, policy);
                tma_load_3d(dk + PAGE_BYTES, &tmv, 0, 0, row, bar, policy);
            } else {
                bulk_load(dk, kp + size_t(row) * D, PAGE_BYTES, bar, policy);
                bulk_load(dk + PAGE_BYTES, vp + size_t(row) * D, PAGE_BYTES, bar, policy);
            }
        }
    };
    if (lane == 0)
        for (int s = 0; s < NS && s < my_units; ++s) issue(s);
    uint32_t phase = 0;
    int slot = 0;
    for (int k = 0; k < my_units; ++k) {
        mbar_wait(bars + slot * 8, phase);
        __syncwarp();
        if (lane == 0 && next < my_units) issue(slot);
        if (++slot == NS) {
            slot = 0;
            phase ^= 1u;
        }
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_3d_maps(const spa_pool* p, CUtensorMap* mk, CUtensorMap* mv) {
    static EncodeTiledFn enc = nullptr;
    if (!enc) {
        void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (h) enc = reinterpret_cast<EncodeTiledFn>(dlsym(h, "cuTensorMapEncodeTiled"));
    }
    if (!enc) return false;
    const auto& c = p->cfg;
    const cuuint64_t rows = cuuint64_t(c.num_layers) * c.num_pages * c.num_kv_heads * c.page_size;
    cuuint64_t dims[3] = {64, cuuint64_t(c.head_dim / 64), rows};
    cuuint64_t strides[2] = {128, cuuint64_t(c.head_dim) * 2};
    cuuint32_t box[3] = {64, cuuint32_t(c.head_dim / 64), 16};
    cuuint32_t estr[3] = {1, 1, 1};
    void* ptrs[2] = {p->k_pool, p->v_pool};
    CUtensorMap* maps[2] = {mk, mv};
    for (int i = 0; i < 2; ++i)
        if (enc(maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, ptrs[i], dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    return true;
}

template <int D, int MODE>
static cudaError_t launch_probe(const spa_pool* pool, const CUtensorMap& mk, const CUtensorMap& mv, int units,
                                int pairs, cudaStream_t s) {
    const int smem = kSmemBudget + 1024;
    cudaFuncSetAttribute(tma_pool_read_kernel<D, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma_pool_read_kernel<D, MODE><<<pool->sm_count, kWarps * 32, smem, s>>>(
        mk, mv, static_cast<const uint16_t*>(pool->k_pool), static_cast<const uint16_t*>(pool->v_pool), units, pairs,
        pool->cfg.num_kv_heads, pool->cfg.num_pages);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- tcgen05 self-test
// One CTA: S = Q K^T (M=128, N=16 per page, K=128 in 8 steps) from 128-B-swizzled shared
// memory into tensor memory, P = bf16(S) stored back to tensor memory, O = P V (A from
// tensor memory, V as an MN-major operand, one K=16 MMA per page).  Checks the descriptor
// and tensor-memory conventions the extend kernel relies on against a host reference.
__global__ void __launch_bounds__(192, 1)
    umma_selftest_kernel(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v, float* out_s,
                         float* out_o) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t QB = sbase, KB = sbase + 32768, VB = KB + 8192, BAR = VB + 8192, TSLOT = BAR + 64;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // stage operands: Q [128][128] -> two 16-KB column chunks; K, V [32][128] -> 2 pages of
    // [chunk][16 rows][128 B], exactly as the TMA boxes of the pool land
    for (int i = tid; i < 128 * 16; i += blockDim.x) {
        const int r = i >> 4, u = i & 15;   // 16-B unit u of row r (8 bf16)
        const uint4 val = reinterpret_cast<const uint4*>(q + r * 128)[u];
        *reinterpret_cast<uint4*>(smem + (u >> 3) * 16384 + umma::sw128_offset(r, u & 7)) = val;
    }
    for (int i = tid; i < 32 * 16; i += blockDim.x) {
        const int r = i >> 4, u = i & 15, pg = r >> 4, rr = r & 15;
        const uint32_t off = pg * 4096 + (u >> 3) * 2048 + umma::sw128_offset(rr, u & 7);
        *reinterpret_cast<uint4*>(smem + 32768 + off) = reinterpret_cast<const uint4*>(k + r * 128)[u];
        *reinterpret_cast<uint4*>(smem + 32768 + 8192 + off) = reinterpret_cast<const uint4*>(v + r * 128)[u];
    }
    if (tid == 0) {
        for (int b = 0; b < 3; ++b) mbar_init(BAR + b * 8, b == 1 ? 128 : 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_proxy_async_smem();
    __syncthreads();
    if (warp == 0) umma::tmem_alloc(TSLOT, 256);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (TSLOT - sbase));
    const uint32_t S_COL = 0, P_COL = 32, O_COL = 128;
    if (tid == 32) {
        const uint32_t id_s = umma::idesc_bf16_f32(128, 16, false, false);
        for (int pg = 0; pg < 2; ++pg)
            for (int ks = 0; ks < 8; ++ks) {
                const uint64_t a = umma::desc_k_sw128(QB + (ks >> 2) * 16384 + (ks & 3) * 32, 1024);
                const uint64_t b = umma::desc_k_sw128(KB + pg * 4096 + (ks >> 2) * 2048 + (ks & 3) * 32, 1024);
                umma::mma_ss(tmem + S_COL + pg * 16, a, b, id_s, ks > 0);
            }
        umma::commit(BAR);
    }
    const bool wg = warp >= 2;
    const int row = 32 * (warp & 3) + lane;
    const uint32_t lane_off = uint32_t(32 * (warp & 3)) << 16;
    if (wg) {
        mbar_wait(BAR, 0);
        umma::fence_after();
        float s[32];
        umma::ld32(tmem + lane_off + S_COL, s);
        umma::wait_ld();
        uint32_t pk[16];
        for (int i = 0; i < 32; ++i) out_s[row * 32 + i] = s[i];
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(s[2 * i], s[2 * i + 1]);
        umma::st16(tmem + lane_off + P_COL, pk);
        umma::wait_st();
        umma::fence_before();
        mbar_arrive(BAR + 8);
    }
    if (tid == 32) {
        mbar_wait(BAR + 8, 0);
        umma::fence_after();
        const uint32_t id_o = umma::idesc_bf16_f32(128, 128, false, true);
        for (int pg = 0; pg < 2; ++pg)
            umma::mma_ts(tmem + O_COL, tmem + P_COL + pg * 8, umma::desc_mn_sw128(VB + pg * 4096, 2048, 1024), id_o,
                         pg > 0);
        umma::commit(BAR + 16);
    }
    if (wg) {
        mbar_wait(BAR + 16, 0);
        umma::fence_after();
        for (int c = 0; c < 4; ++c) {
            float o[32];
            umma::ld32(tmem + lane_off + O_COL + c * 32, o);
            umma::wait_ld();
            for (int i = 0; i < 32; ++i) out_o[row * 128 + c * 32 + i] = o[i];
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem, 256);
}

}  // namespace spa

using namespace spa;

extern "C" {

spa_status spa_debug_read_bw_ldg(const void* buf, size_t bytes, void* sink4, void* stream) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ldg_read_kernel<<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint4*>(buf),
                                                                            bytes / 16, static_cast<unsigned*>(sink4));
    cudaError_t e = cudaGetLastError();
    return e ? fail(SPA_ERR_CUDA, cudaGetErrorString(e)) : SPA_OK;
}

spa_status spa_debug_pool_read_tma(const spa_pool* pool, int32_t layers, int32_t mode, void* stream) {
    if (!pool || pool->metadata_only) return fail(SPA_ERR_INVALID_ARG, "device pool needed");
    if (pool->kv_fp8) return fail(SPA_ERR_UNSUPPORTED, "the TMA read probe is written for bf16 pools");
    const auto& c = pool->cfg;
    if (layers <= 0 || layers > c.num_layers) return fail(SPA_ERR_INVALID_ARG, "layers out of range");
    if (mode < 0 || mode > 2) return fail(SPA_ERR_INVALID_ARG, "mode must be 0, 1 or 2");
    const int pairs = c.num_pages / 2;
    const int units = layers * pairs * c.num_kv_heads;
    CUtensorMap mk = *reinterpret_cast<const CUtensorMap*>(pool->tmap_k.bytes);
    CUtensorMap mv = *reinterpret_cast<const CUtensorMap*>(pool->tmap_v.bytes);
    if (mode == 1 && !make_3d_maps(pool, &mk, &mv)) return fail(SPA_ERR_CUDA, "3-D tensor map encode failed");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (c.head_dim == 128)
        e = mode == 0   ? launch_probe<128, 0>(pool, mk, mv, units, pairs, s)
            : mode == 1 ? launch_probe<128, 1>(pool, mk, mv, units, pairs, s)
                        : launch_probe<128, 2>(pool, mk, mv, units, pairs, s);
    else
        e = mode == 0   ? launch_probe<64, 0>(pool, mk, mv, units, pairs, s)
            : mode == 1 ? launch_probe<64, 1>(pool, mk, mv, units, pairs, s)
                        : launch_probe<64, 2>(pool, mk, mv, units, pairs, s);
    return e ? fail(SPA_ERR_CUDA, cudaGetErrorString(e)) : SPA_OK;
}

spa_status spa_debug_umma_selftest(const void* q, const void* k, const void* v, float* out_s, float* out_o,
                                   void* stream) {
    const int smem = 1024 + 32768 + 16384 + 128;
    cudaError_t e = cudaFuncSetAttribute(spa::umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) {
        spa::umma_selftest_kernel<<<1, 192, smem, static_cast<cudaStream_t>(stream)>>>(
            static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
            static_cast<const __nv_bfloat16*>(v), out_s, out_o);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return spa::fail(SPA_ERR_CUDA, std::string("umma selftest: ") + cudaGetErrorString(e));
    return SPA_OK;
}

}  // extern "C"
