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

}  // extern "C"
