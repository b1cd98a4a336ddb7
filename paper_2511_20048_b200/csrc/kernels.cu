// sm_100a kernels of the shared-prefix paged GQA decode-attention step, and their launchers.
//
//   append_kernel  a2: scatter new K/V rows of all layers into their (page, slot)
//   cow_kernel     a3: copy-on-write of a fork's partial last page, all layers
//   decode_kernel  a5: persistent, one 1-warp (or 2-warp) team per work-item stream:
//                  TMA (cp.async.bulk.tensor, 128-B swizzle) page staging into an
//                  mbarrier ring, ldmatrix + mma.sync bf16 QK^T and PV tiles over all
//                  R = members x G query rows of a group (so a shared page is read once
//                  per KV head and group), warp-shuffle online softmax in fp32 (exp2).
//   merge_kernel   a6: split-KV partial-LSE merge.
// Shapes and readings: include/spa.h, DESIGN.md Sec. 3-5.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "spa_internal.h"

namespace spa {

// ============================================================================ host utilities
int device_sm_count(int* dev_out) {
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return -int(e);
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return -int(e);
    *dev_out = dev;
    return sms;
}

const char* cuda_error_string(int err) { return cudaGetErrorString(cudaError_t(err)); }

static size_t pool_bytes(const spa_pool* p) {
    const auto& c = p->cfg;
    return size_t(c.num_layers) * c.num_pages * c.num_kv_heads * c.page_size * c.head_dim * 2;
}

int memset_pool(spa_pool* p) {
    cudaError_t e = cudaMemset(p->k_pool, 0, pool_bytes(p));
    if (e == cudaSuccess) e = cudaMemset(p->v_pool, 0, pool_bytes(p));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return int(e);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) fn = reinterpret_cast<EncodeTiledFn>(dlsym(h, "cuTensorMapEncodeTiled"));
    }
    return fn;
}

// 2-D view of a pool: rows = L * num_pages * Hkv * 16 (one row = one token of one head),
// cols = d; box = 16 rows x 64 cols (128 B, 128-B swizzle): one page-half per TMA op.
bool make_tensor_maps(spa_pool* p, std::string* err) {
    static_assert(sizeof(CUtensorMap) == sizeof(spa_tmap), "CUtensorMap size");
    EncodeTiledFn enc = encode_fn();
    if (!enc) {
        *err = "libcuda.so.1 / cuTensorMapEncodeTiled not available";
        return false;
    }
    const auto& c = p->cfg;
    const cuuint64_t rows = cuuint64_t(c.num_layers) * c.num_pages * c.num_kv_heads * c.page_size;
    cuuint64_t dims[2] = {cuuint64_t(c.head_dim), rows};
    cuuint64_t strides[1] = {cuuint64_t(c.head_dim) * 2};
    cuuint32_t box[2] = {64, 16};
    cuuint32_t estr[2] = {1, 1};
    void* ptrs[2] = {p->k_pool, p->v_pool};
    spa_tmap* maps[2] = {&p->tmap_k, &p->tmap_v};
    for (int i = 0; i < 2; ++i) {
        CUresult r = enc(reinterpret_cast<CUtensorMap*>(maps[i]->bytes), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptrs[i],
                         dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            *err = "CUresult " + std::to_string(int(r));
            return false;
        }
    }
    return true;
}

// ============================================================================ device helpers
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

// ============================================================================ a2: append
constexpr int kAppendMax = 896;

struct AppendParams {
    const uint4* k_src;
    const uint4* v_src;
    uint4* k_dst;
    uint4* v_dst;
    long long layer_stride;  // in uint4 units: num_pages * Hkv * ps * d / 8
    int T_total, t0, n, Hkv, dvec, ps;
    int slots[kAppendMax];   // page * ps + slot, per token of this launch
};

__global__ void append_kernel(const __grid_constant__ AppendParams p) {
    const int i = blockIdx.x, layer = blockIdx.y;
    const int slot = p.slots[i];
    const int page = slot / p.ps, s = slot - page * p.ps;
    for (int tid = threadIdx.x; tid < p.Hkv * p.dvec; tid += blockDim.x) {
        const int h = tid / p.dvec, c = tid - h * p.dvec;
        const long long src = ((long long)(layer)*p.T_total + p.t0 + i) * p.Hkv * p.dvec + (long long)h * p.dvec + c;
        const long long dst = layer * p.layer_stride + (((long long)page * p.Hkv + h) * p.ps + s) * p.dvec + c;
        p.k_dst[dst] = p.k_src[src];
        p.v_dst[dst] = p.v_src[src];
    }
}

int launch_append(const spa_pool* pool, const void* k_new, const void* v_new, int32_t T_total,
                  const std::vector<int32_t>& slots, void* stream) {
    const auto& c = pool->cfg;
    AppendParams p{};
    p.k_src = static_cast<const uint4*>(k_new);
    p.v_src = static_cast<const uint4*>(v_new);
    p.k_dst = static_cast<uint4*>(pool->k_pool);
    p.v_dst = static_cast<uint4*>(pool->v_pool);
    p.dvec = c.head_dim / 8;
    p.layer_stride = (long long)c.num_pages * c.num_kv_heads * c.page_size * p.dvec;
    p.T_total = T_total;
    p.Hkv = c.num_kv_heads;
    p.ps = c.page_size;
    const int threads = std::min(256, ((p.Hkv * p.dvec + 31) / 32) * 32);
    for (int t0 = 0; t0 < T_total; t0 += kAppendMax) {
        p.t0 = t0;
        p.n = std::min(kAppendMax, T_total - t0);
        std::memcpy(p.slots, slots.data() + t0, sizeof(int) * p.n);
        append_kernel<<<dim3(p.n, c.num_layers), threads, 0, static_cast<cudaStream_t>(stream)>>>(p);
    }
    return int(cudaGetLastError());
}

// ============================================================================ a3: copy-on-write
__global__ void cow_kernel(const uint4* __restrict__ k, const uint4* __restrict__ v, uint4* kd, uint4* vd,
                           long long layer_stride, int src_page, int dst_page, int rows, int Hkv, int dvec, int ps) {
    const int layer = blockIdx.x, h = blockIdx.y;
    const long long sb = layer * layer_stride + ((long long)src_page * Hkv + h) * ps * dvec;
    const long long db = layer * layer_stride + ((long long)dst_page * Hkv + h) * ps * dvec;
    for (int t = threadIdx.x; t < rows * dvec; t += blockDim.x) {
        kd[db + t] = k[sb + t];
        vd[db + t] = v[sb + t];
    }
}

int launch_cow(const spa_pool* pool, int32_t src_page, int32_t dst_page, int32_t rows, void* stream) {
    const auto& c = pool->cfg;
    const int dvec = c.head_dim / 8;
    const long long ls = (long long)c.num_pages * c.num_kv_heads * c.page_size * dvec;
    cow_kernel<<<dim3(c.num_layers, c.num_kv_heads), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(pool->k_pool), static_cast<const uint4*>(pool->v_pool),
        static_cast<uint4*>(pool->k_pool), static_cast<uint4*>(pool->v_pool), ls, src_page, dst_page, rows,
        c.num_kv_heads, dvec, c.page_size);
    return int(cudaGetLastError());
}

// ============================================================================ a5: decode
struct DecodeParams {
    const int32_t* meta;
    const __nv_bfloat16* q;
    long long q_sr, q_sh;
    __nv_bfloat16* o;
    long long o_sr, o_sh;
    float* lse;
    long long l_sr, l_sh;
    float* part_o;
    float* part_lse;
    float scale_log2;
    int layer_row_base;  // layer * num_pages * Hkv * 16
    int num_q_heads, group_size, num_kv_heads;
    int fused_merge;     // 1: the last item of a (request, KV head) merges its partials in-kernel
};

template <int D, int MT>
struct DecodeCfg {
    static constexpr int TEAMS = kWarps / MT;
    static constexpr int PAGE_BYTES = kPageSize * D * 2;  // K (or V) of one page, one head
    static constexpr int STAGE_BYTES = kPagesPerStage * 2 * PAGE_BYTES;
    static constexpr int NS = (kSmemBudget - 1024) / (TEAMS * STAGE_BYTES);
    static constexpr int RING_BYTES = TEAMS * NS * STAGE_BYTES;
    static constexpr int QN = NS + 2;   // popped-item queue entries per team
    static constexpr int SMEM = 1024 + RING_BYTES + TEAMS * NS * 2 * 8 + TEAMS * 4 + TEAMS * QN * 4;
    static_assert(NS >= 2, "pipeline needs >= 2 stages");
};

int stages_per_team(int head_dim, int mt) {
    if (head_dim == 64) return mt == 1 ? DecodeCfg<64, 1>::NS : DecodeCfg<64, 2>::NS;
    return mt == 1 ? DecodeCfg<128, 1>::NS : DecodeCfg<128, 2>::NS;
}

size_t decode_smem_bytes(int head_dim, int mt) {
    if (head_dim == 64) return mt == 1 ? DecodeCfg<64, 1>::SMEM : DecodeCfg<64, 2>::SMEM;
    return mt == 1 ? DecodeCfg<128, 1>::SMEM : DecodeCfg<128, 2>::SMEM;
}

template <int D, int MT>
__global__ void __launch_bounds__(kWarps * 32, 1)
    decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const DecodeParams p) {
    using C = DecodeCfg<D, MT>;
    constexpr int PPS = kPagesPerStage;
    constexpr int KS = D / 16;   // k16 steps over the head dimension
    constexpr int NT = D / 8;    // n8 tiles of the output
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int team = warp / MT, wt = warp - team * MT;
    const uint32_t ring = smem_u32(smem) + team * C::NS * C::STAGE_BYTES;
    const uint32_t bars = smem_u32(smem) + C::RING_BYTES;
    auto full_bar = [&](int s) { return bars + (team * C::NS + s) * 8; };
    auto empty_bar = [&](int s) { return bars + (C::TEAMS * C::NS + team * C::NS + s) * 8; };
    uint32_t* team_slot = reinterpret_cast<uint32_t*>(smem + C::RING_BYTES + C::TEAMS * C::NS * 2 * 8) + team;
    int32_t* team_q = reinterpret_cast<int32_t*>(smem + C::RING_BYTES + C::TEAMS * C::NS * 2 * 8 + C::TEAMS * 4);
    auto team_sync = [&]() {
        if constexpr (MT == 1) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(MT * 32) : "memory");
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::TEAMS * C::NS; ++i) {
            mbar_init(bars + i * 8, 1);
            mbar_init(bars + (C::TEAMS * C::NS + i) * 8, MT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // programmatic dependent launch: everything above overlapped the previous kernel's
    // tail; from here on we read what it (and earlier stream work) wrote.  Let the next
    // kernel (the split merge / the next layer) start its own prologue early.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");

    const int32_t* meta = p.meta;
    const Desc* descs = reinterpret_cast<const Desc*>(meta + meta[H_OFF_DESC]);
    const Member* mems = reinterpret_cast<const Member*>(meta + meta[H_OFF_MEMBER]);
    const Item* items = reinterpret_cast<const Item*>(meta + meta[H_OFF_ITEM]);
    const int32_t* queue = meta + meta[H_OFF_QUEUE];
    const int32_t* pages = meta + meta[H_OFF_PAGES];
    const int32_t* rec_ptr = meta + meta[H_OFF_REC_PTR];
    int32_t* counters = const_cast<int32_t*>(meta) + meta[H_OFF_COUNTERS];
    int32_t* sched = const_cast<int32_t*>(meta) + meta[H_OFF_SCHED];
    const int n_items = meta[H_N_ITEMS];
    int32_t* tq = team_q + team * C::QN;   // items this team popped, in order (producer -> consumers)

    const int G = p.group_size, Hq = p.num_q_heads, Hkv = p.num_kv_heads;
    const bool leader = (wt == 0) && (lane == 0);
    uint64_t policy = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

    // ---- producer (one elected thread per team): pops items from the dynamic LPT queue
    //      and streams their (stage) page pairs into the ring, NS stages ahead.  When the
    //      queue is empty it publishes -1 and completes the slot's barrier without data.
    int p_item = -1, p_st = 0, p_n = 0;
    bool p_done = false;
    Item p_itm{0, 0};
    Desc p_dsc{};
    auto issue_next = [&](int slot) {
        if (p_done) return;
        if (p_item < 0) {
            const int qi = atomicAdd(sched, 1);
            const int it = qi < n_items ? queue[qi] : -1;
            tq[p_n % C::QN] = it;
            ++p_n;
            if (it < 0) {
                p_done = true;
                mbar_arrive(full_bar(slot));
                return;
            }
            p_item = it;
            p_st = 0;
            p_itm = items[it];
            p_dsc = descs[p_itm.desc];
        }
        const int p0 = p_st * PPS;
        const int npg = min(PPS, p_dsc.n_pages - p0);
        const uint32_t fb = full_bar(slot);
        mbar_expect_tx(fb, npg * 2 * C::PAGE_BYTES);
        const uint32_t sb = ring + slot * C::STAGE_BYTES;
        for (int j = 0; j < npg; ++j) {
            const int page = pages[p_dsc.page_off + p0 + j];
            const int row = p.layer_row_base + (page * Hkv + p_itm.kv_head) * kPageSize;
#pragma unroll
            for (int hf = 0; hf < D / 64; ++hf) {
                tma_load_2d(sb + j * 2 * C::PAGE_BYTES + hf * 2048, &tmk, hf * 64, row, fb, policy);
                tma_load_2d(sb + j * 2 * C::PAGE_BYTES + C::PAGE_BYTES + hf * 2048, &tmv, hf * 64, row, fb, policy);
            }
        }
        if (++p_st * PPS >= p_dsc.n_pages) p_item = -1;
    };
    if (leader) {
        for (int s = 0; s < C::NS; ++s) issue_next(s);
    }

    int slot = 0, c_n = 0;
    uint32_t phase = 0;
    while (true) {
        // the first stage of the next item (or the end-of-queue marker) has landed
        mbar_wait(full_bar(slot), phase);
        const int it = tq[c_n % C::QN];
        ++c_n;
        if (it < 0) break;
        const Item itm = items[it];
        const Desc dsc = descs[itm.desc];
        const int R = dsc.n_members * G;
        const bool active = wt * 16 < R;
        const int row0 = wt * 16 + (lane >> 2), row1 = row0 + 8;

        // ---- per-row setup: member, window bound, query fragments
        int lo0 = 0x7fffffff, lo1 = 0x7fffffff;
        uint32_t qa[KS][4];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) qa[ks][0] = qa[ks][1] = qa[ks][2] = qa[ks][3] = 0u;
        if (active) {
            const __nv_bfloat16* q0 = nullptr;
            const __nv_bfloat16* q1 = nullptr;
            if (row0 < R) {
                const int mb = row0 / G;
                const Member m = mems[dsc.member_off + mb];
                lo0 = m.lo;
                q0 = p.q + m.row * p.q_sr + (itm.kv_head * G + row0 - mb * G) * p.q_sh;
            }
            if (row1 < R) {
                const int mb = row1 / G;
                const Member m = mems[dsc.member_off + mb];
                lo1 = m.lo;
                q1 = p.q + m.row * p.q_sr + (itm.kv_head * G + row1 - mb * G) * p.q_sh;
            }
            const int cq = 2 * (lane & 3);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                if (q0) {
                    qa[ks][0] = *reinterpret_cast<const uint32_t*>(q0 + ks * 16 + cq);
                    qa[ks][2] = *reinterpret_cast<const uint32_t*>(q0 + ks * 16 + cq + 8);
                }
                if (q1) {
                    qa[ks][1] = *reinterpret_cast<const uint32_t*>(q1 + ks * 16 + cq);
                    qa[ks][3] = *reinterpret_cast<const uint32_t*>(q1 + ks * 16 + cq + 8);
                }
            }
        }
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        float acc[NT][4];
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;

        const int nst = (dsc.n_pages + PPS - 1) / PPS;
        for (int st = 0; st < nst; ++st) {
            if (st > 0) mbar_wait(full_bar(slot), phase);
            if (active) {
                const uint32_t sb = ring + slot * C::STAGE_BYTES;
                const int npg = min(PPS, dsc.n_pages - st * PPS);
                const int tok0 = dsc.tok_start + st * PPS * kPageSize;
                float s[PPS][2][4];
#pragma unroll
                for (int j = 0; j < PPS; ++j) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) s[j][0][e] = s[j][1][e] = 0.f;
                    if (j < npg) {
                        const uint32_t kb = sb + j * 2 * C::PAGE_BYTES;
                        const int key = ((lane >> 4) << 3) + (lane & 7);
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) {
                            const int dcol = ks * 16 + ((lane >> 3) & 1) * 8;
                            const uint32_t addr =
                                kb + (dcol >> 6) * 2048 + key * 128 + ((((dcol & 63) >> 3) ^ (key & 7)) << 4);
                            uint32_t b0, b1, b2, b3;
                            ldsm_x4(b0, b1, b2, b3, addr);
                            mma16816(s[j][0], qa[ks], b0, b1);
                            mma16816(s[j][1], qa[ks], b2, b3);
                        }
                    }
                }
                // mask + scale (log2 domain), row max
                float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
                for (int j = 0; j < PPS; ++j) {
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int tok = tok0 + j * kPageSize + nt * 8 + 2 * (lane & 3) + (e & 1);
                            const int lo = (e < 2) ? lo0 : lo1;
                            const bool ok = (j < npg) && (tok < dsc.tok_end) && (tok >= lo);
                            const float v = ok ? s[j][nt][e] * p.scale_log2 : -INFINITY;
                            s[j][nt][e] = v;
                            if (e < 2) mx0 = fmaxf(mx0, v);
                            else mx1 = fmaxf(mx1, v);
                        }
                    }
                }
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
                const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
                const float mu0 = (mn0 == -INFINITY) ? 0.f : mn0;
                const float mu1 = (mn1 == -INFINITY) ? 0.f : mn1;
                const float al0 = fast_exp2(m0 - mu0), al1 = fast_exp2(m1 - mu1);
                m0 = mn0;
                m1 = mn1;
                l0 *= al0;
                l1 *= al1;
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    acc[n][0] *= al0;
                    acc[n][1] *= al0;
                    acc[n][2] *= al1;
                    acc[n][3] *= al1;
                }
                // P = exp2(s - m): l accumulates the fp32 P (so the LSE carries no bf16
                // rounding); the PV MMA takes P rounded to bf16 (A fragments).
#pragma unroll
                for (int j = 0; j < PPS; ++j) {
                    if (j < npg) {
                        float e[2][4];
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt) {
                            e[nt][0] = fast_exp2(s[j][nt][0] - mu0);
                            e[nt][1] = fast_exp2(s[j][nt][1] - mu0);
                            e[nt][2] = fast_exp2(s[j][nt][2] - mu1);
                            e[nt][3] = fast_exp2(s[j][nt][3] - mu1);
                            l0 += e[nt][0] + e[nt][1];
                            l1 += e[nt][2] + e[nt][3];
                        }
                        uint32_t pa[4];
                        pa[0] = pack_bf16(e[0][0], e[0][1]);
                        pa[1] = pack_bf16(e[0][2], e[0][3]);
                        pa[2] = pack_bf16(e[1][0], e[1][1]);
                        pa[3] = pack_bf16(e[1][2], e[1][3]);
                        const uint32_t vb = sb + j * 2 * C::PAGE_BYTES + C::PAGE_BYTES;
                        const int key = (((lane >> 3) & 1) << 3) + (lane & 7);
#pragma unroll
                        for (int dn = 0; dn < KS; ++dn) {
                            const int dchunk = 2 * dn + (lane >> 4);
                            const uint32_t addr = vb + (dchunk >> 3) * 2048 + key * 128 + (((dchunk & 7) ^ (key & 7)) << 4);
                            uint32_t b0, b1, b2, b3;
                            ldsm_x4_t(b0, b1, b2, b3, addr);
                            mma16816(acc[2 * dn], pa, b0, b1);
                            mma16816(acc[2 * dn + 1], pa, b2, b3);
                        }
                    }
                }
            }
            // ---- release the stage and refill it NS stages ahead
            __syncwarp();
            if constexpr (MT == 1) {
                if (leader) issue_next(slot);
            } else {
                if (lane == 0) mbar_arrive(empty_bar(slot));
                if (leader) {
                    mbar_wait(empty_bar(slot), phase);
                    issue_next(slot);
                }
            }
            if (++slot == C::NS) {
                slot = 0;
                phase ^= 1u;
            }
        }

        // ---- epilogue: normalise, write final O/LSE or an fp32 partial record
        if (active) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
            l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
            l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
            l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int row = rr ? row1 : row0;
                if (row < R) {
                    const int mb = row / G;
                    const Member m = mems[dsc.member_off + mb];
                    const int head = itm.kv_head * G + (row - mb * G);
                    const float l = rr ? l1 : l0;
                    const float mm = rr ? m1 : m0;
                    const float inv = l > 0.f ? 1.f / l : 0.f;
                    const float lse = l > 0.f ? (mm + log2f(l)) * 0.69314718055994531f : -INFINITY;
                    const int c0 = 2 * (lane & 3);
                    if (m.rec < 0) {
                        __nv_bfloat16* orow = p.o + m.row * p.o_sr + head * p.o_sh;
#pragma unroll
                        for (int n = 0; n < NT; ++n)
                            *reinterpret_cast<__nv_bfloat162*>(orow + n * 8 + c0) =
                                __floats2bfloat162_rn(acc[n][2 * rr] * inv, acc[n][2 * rr + 1] * inv);
                        if ((lane & 3) == 0 && p.lse) p.lse[m.row * p.l_sr + head * p.l_sh] = lse;
                    } else {
                        float* prow = p.part_o + ((long long)m.rec * Hq + head) * D;
#pragma unroll
                        for (int n = 0; n < NT; ++n)
                            *reinterpret_cast<float2*>(prow + n * 8 + c0) =
                                make_float2(acc[n][2 * rr] * inv, acc[n][2 * rr + 1] * inv);
                        if ((lane & 3) == 0) p.part_lse[(long long)m.rec * Hq + head] = lse;
                    }
                }
            }
        }

        // ---- fused split merge (a6): the last item to finish a (request, KV head) merges
        //      that request's partial records for the G query heads of this KV head.
        bool any_partial = false;
        for (int mb = 0; mb < dsc.n_members; ++mb) any_partial |= mems[dsc.member_off + mb].rec >= 0;
        if (any_partial && p.fused_merge) {
            // the team barrier orders every lane's partial stores before the leader's
            // acq_rel arrival (release is cumulative); the last arriver acquires all of them
            team_sync();
            uint32_t mask = 0;
            if (leader) {
                for (int mb = 0; mb < dsc.n_members; ++mb) {
                    const Member mm = mems[dsc.member_off + mb];
                    if (mm.rec < 0) continue;
                    const int nrec = rec_ptr[mm.row + 1] - rec_ptr[mm.row];
                    int* c = counters + mm.row * Hkv + itm.kv_head;
                    if (atom_add_acq_rel_gpu(c, 1) == nrec - 1) {
                        mask |= 1u << mb;
                        *c = 0;    // every arrival of this launch is in: ready for the next layer
                    }
                }
            }
            if constexpr (MT == 1) {
                mask = __shfl_sync(0xffffffffu, mask, 0);
            } else {
                if (leader) *team_slot = mask;
                team_sync();
                mask = *team_slot;
            }
            while (mask) {
                const int mb = __ffs(mask) - 1;
                mask &= mask - 1;
                const Member mm = mems[dsc.member_off + mb];
                for (int hh = wt; hh < G; hh += MT)
                    warp_merge_head<D>(p.part_o, p.part_lse, Hq, rec_ptr[mm.row], rec_ptr[mm.row + 1],
                                       itm.kv_head * G + hh, p.o + mm.row * p.o_sr, p.o_sh,
                                       p.lse ? p.lse + mm.row * p.l_sr : nullptr, p.l_sh, lane);
            }
        }
    }
    // the last team to drain the queue rewinds it for the next launch (stream-ordered)
    if (leader) {
        if (atomicAdd(sched + 1, 1) == int(gridDim.x) * C::TEAMS - 1) {
            sched[0] = 0;
            sched[1] = 0;
        }
    }
}

// ============================================================================ a6: merge
struct MergeParams {
    const int32_t* rec_ptr;
    const float* part_o;
    const float* part_lse;
    __nv_bfloat16* o;
    long long o_sr, o_sh;
    float* lse;
    long long l_sr, l_sh;
    int n_req, H, D;
};

// One warp per (request, head); lanes stride over float4 columns.
__global__ void __launch_bounds__(256) merge_kernel(const MergeParams p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // partials come from the decode kernel
    asm volatile("griddepcontrol.launch_dependents;");
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int pair = gw; pair < p.n_req * p.H; pair += warps) {
        const int r = pair / p.H, h = pair - r * p.H;
        const int s0 = p.rec_ptr[r], s1 = p.rec_ptr[r + 1];
        if (s0 == s1) continue;
        warp_merge_head<0>(p.part_o, p.part_lse, p.H, s0, s1, h, p.o + r * p.o_sr, p.o_sh,
                           p.lse ? p.lse + r * p.l_sr : nullptr, p.l_sh, lane, p.D);
    }
}

int launch_merge(int32_t n_req, int32_t num_heads, int32_t head_dim, const int32_t* rec_ptr, const float* part_o,
                 const float* part_lse, void* o, int64_t o_sr, int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh,
                 int grid_hint, void* stream) {
    MergeParams p{rec_ptr, part_o, part_lse, static_cast<__nv_bfloat16*>(o), o_sr, o_sh, lse, l_sr, l_sh,
                  n_req, num_heads, head_dim};
    const int pairs = n_req * num_heads;
    int blocks = (pairs + 7) / 8;
    if (grid_hint > 0) blocks = std::min(blocks, grid_hint * 8);
    blocks = std::max(blocks, 1);
    return launch_pdl(merge_kernel, dim3(blocks), dim3(256), 0, stream, p);
}

// ============================================================================ plan device buffers
int plan_upload(spa_plan* P, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    if (!P->upload_event) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e) return int(e);
        P->upload_event = ev;
    }
    if (P->upload_pending) {   // the pinned staging buffer may still be read by the last upload
        e = cudaEventSynchronize(static_cast<cudaEvent_t>(P->upload_event));
        if (e) return int(e);
        P->upload_pending = false;
    }
    const size_t words = P->host.size();
    if (words > P->pinned_words) {
        if (P->pinned) cudaFreeHost(P->pinned);
        P->pinned = nullptr;
        const size_t nw = words + words / 2 + 1024;
        e = cudaMallocHost(reinterpret_cast<void**>(&P->pinned), nw * 4);
        if (e) return int(e);
        P->pinned_words = nw;
    }
    std::memcpy(P->pinned, P->host.data(), words * 4);
    if (words > P->d_meta_words) {
        if (P->d_meta) cudaFree(P->d_meta);
        P->d_meta = nullptr;
        const size_t nw = words + words / 2 + 1024;
        e = cudaMalloc(reinterpret_cast<void**>(&P->d_meta), nw * 4);
        if (e) return int(e);
        P->d_meta_words = nw;
        P->generation++;
    }
    const size_t records = size_t(P->host[H_N_RECORDS]);
    if (records > P->part_records) {
        const auto& c = P->pool->cfg;
        if (P->d_part_o) cudaFree(P->d_part_o);
        if (P->d_part_lse) cudaFree(P->d_part_lse);
        P->d_part_o = nullptr;
        P->d_part_lse = nullptr;
        const size_t nr = records + records / 4 + 64;
        e = cudaMalloc(reinterpret_cast<void**>(&P->d_part_o), nr * c.num_q_heads * c.head_dim * 4);
        if (!e) e = cudaMalloc(reinterpret_cast<void**>(&P->d_part_lse), nr * c.num_q_heads * 4);
        if (e) return int(e);
        P->part_records = nr;
        P->generation++;
    }
    e = cudaMemcpyAsync(P->d_meta, P->pinned, words * 4, cudaMemcpyHostToDevice, s);
    if (e) return int(e);
    e = cudaEventRecord(static_cast<cudaEvent_t>(P->upload_event), s);
    if (e) return int(e);
    P->upload_pending = true;
    return 0;
}

void plan_release(spa_plan* P) {
    if (P->upload_event) {
        cudaEventSynchronize(static_cast<cudaEvent_t>(P->upload_event));
        cudaEventDestroy(static_cast<cudaEvent_t>(P->upload_event));
    }
    if (P->pinned) cudaFreeHost(P->pinned);
    if (P->d_meta) cudaFree(P->d_meta);
    if (P->d_part_o) cudaFree(P->d_part_o);
    if (P->d_part_lse) cudaFree(P->d_part_lse);
    P->upload_event = nullptr;
    P->pinned = nullptr;
    P->d_meta = nullptr;
    P->d_part_o = nullptr;
    P->d_part_lse = nullptr;
}

// ============================================================================ decode launcher
template <int D, int MT>
static int launch_decode_t(const spa_plan* P, const DecodeParams& dp, void* stream) {
    using C = DecodeCfg<D, MT>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(decode_kernel<D, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e) return int(e);
        attr_set = true;
    }
    const CUtensorMap* tk = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_k.bytes);
    const CUtensorMap* tv = reinterpret_cast<const CUtensorMap*>(P->pool->tmap_v.bytes);
    return launch_pdl(decode_kernel<D, MT>, dim3(P->num_ctas), dim3(kWarps * 32), C::SMEM, stream, *tk, *tv, dp);
}

int launch_decode(const spa_plan* P, int32_t layer, const void* q, int64_t q_sr, int64_t q_sh, void* o, int64_t o_sr,
                  int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh, float scale, void* stream) {
    const auto& c = P->pool->cfg;
    const int32_t* H = P->host.data();
    if (H[H_N_ITEMS] == 0) return 0;
    DecodeParams dp{};
    dp.meta = P->d_meta;
    dp.q = static_cast<const __nv_bfloat16*>(q);
    dp.q_sr = q_sr;
    dp.q_sh = q_sh;
    dp.o = static_cast<__nv_bfloat16*>(o);
    dp.o_sr = o_sr;
    dp.o_sh = o_sh;
    dp.lse = lse;
    dp.l_sr = l_sr;
    dp.l_sh = l_sh;
    dp.part_o = P->d_part_o;
    dp.part_lse = P->d_part_lse;
    dp.scale_log2 = float(double(scale) * 1.4426950408889634);
    dp.layer_row_base = layer * c.num_pages * c.num_kv_heads * kPageSize;
    dp.num_q_heads = c.num_q_heads;
    dp.num_kv_heads = c.num_kv_heads;
    dp.group_size = c.num_q_heads / c.num_kv_heads;
    dp.fused_merge = P->cfg.fused_merge ? 1 : 0;
    int err = 0;
    if (c.head_dim == 64)
        err = P->mt == 1 ? launch_decode_t<64, 1>(P, dp, stream) : launch_decode_t<64, 2>(P, dp, stream);
    else
        err = P->mt == 1 ? launch_decode_t<128, 1>(P, dp, stream) : launch_decode_t<128, 2>(P, dp, stream);
    if (err) return err;
    if (H[H_N_RECORDS] > 0 && !dp.fused_merge)
        err = launch_merge(H[H_N_REQ], c.num_q_heads, c.head_dim, P->d_meta + H[H_OFF_REC_PTR], P->d_part_o,
                           P->d_part_lse, o, o_sr, o_sh, lse, l_sr, l_sh, P->num_ctas, stream);
    return err;
}

}  // namespace spa
