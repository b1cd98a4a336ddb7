// sm_100a kernels of the shared-prefix paged GQA decode-attention step, and their launchers.
//
//   append_kernel  a2: scatter new K/V rows of all layers into their (page, slot)
//   append_f8_kernel  a2 for FP8 pools (S8(f) F4): quantise to e4m3 on the way in
//   cow_kernel     a3: copy-on-write of a fork's partial last page, all layers
//   decode_kernel  a5 (decode.cu): persistent, teams of warps per work-item stream:
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

#include "device_util.cuh"
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

int current_device() {
    int dev = -1;
    return cudaGetDevice(&dev) == cudaSuccess ? dev : -1;
}

const char* cuda_error_string(int err) { return cudaGetErrorString(cudaError_t(err)); }

static size_t pool_bytes(const spa_pool* p) {
    const auto& c = p->cfg;
    return size_t(c.num_layers) * c.num_pages * c.num_kv_heads * c.page_size * c.head_dim * 2;
}

int memset_pool(spa_pool* p) {
    // fp8: ONE interleaved buffer of the same byte size (K and V^T blocks alternate per page-head)
    cudaError_t e = cudaMemset(p->k_pool, 0, pool_bytes(p));
    if (e == cudaSuccess && !p->kv_fp8) e = cudaMemset(p->v_pool, 0, pool_bytes(p));
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

// 3-D view of a pool: (64 channels, row, d/64 channel blocks) with row = one token of one
// head (L * num_pages * Hkv * 16 rows, stride d*2 B) and channel blocks 128 B apart.  A box
// of 64 x 16 x d/64 is one whole (page, head) block in ONE TMA op, landing in shared memory
// as [channel block][16 rows][128 B] with 128-B swizzle (the layout ldmatrix reads
// conflict-free).
bool make_tensor_maps(spa_pool* p, std::string* err) {
    static_assert(sizeof(CUtensorMap) == sizeof(spa_tmap), "CUtensorMap size");
    EncodeTiledFn enc = encode_fn();
    if (!enc) {
        *err = "libcuda.so.1 / cuTensorMapEncodeTiled not available";
        return false;
    }
    const auto& c = p->cfg;
    const cuuint64_t rows = cuuint64_t(c.num_layers) * c.num_pages * c.num_kv_heads * c.page_size;
    if (p->kv_fp8) {
        // F4, d = 128: the interleaved buffer as rows of 128 bytes -- 16 K rows (one token
        // each) then 16 V^T rows (8 channels x 16 slots each) per page-head -- so a whole
        // page-head, K and V, is ONE 128 x 32 box (4 KB, as a bf16 page-head's K box), landing
        // 128-B swizzled (the kernel's 4-B fragment loads are conflict-free through the XOR).
        // A unit third dimension keeps the 3-D TMA call of the bf16 maps.
        cuuint64_t kd[3] = {128, rows * 2, 1};
        cuuint64_t ks[2] = {128, rows * 2 * 128};
        cuuint32_t kb[3] = {128, 32, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(reinterpret_cast<CUtensorMap*>(p->tmap_k.bytes), CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, p->k_pool,
                         kd, ks, kb, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        std::memcpy(p->tmap_v.bytes, p->tmap_k.bytes, sizeof(p->tmap_v.bytes));
        if (r != CUDA_SUCCESS) {
            *err = "CUresult " + std::to_string(int(r));
            return false;
        }
        return true;
    }
    cuuint64_t dims[3] = {64, rows, cuuint64_t(c.head_dim / 64)};
    cuuint64_t strides[2] = {cuuint64_t(c.head_dim) * 2, 128};
    cuuint32_t box[3] = {64, 16, cuuint32_t(c.head_dim / 64)};
    cuuint32_t estr[3] = {1, 1, 1};
    void* ptrs[2] = {p->k_pool, p->v_pool};
    spa_tmap* maps[2] = {&p->tmap_k, &p->tmap_v};
    for (int i = 0; i < 3; ++i) {
        cuuint32_t bx[3] = {box[0], box[1], i < 2 ? box[2] : 1u};
        CUresult r = enc(reinterpret_cast<CUtensorMap*>(i < 2 ? maps[i]->bytes : p->tmap_k1.bytes),
                         CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, i < 2 ? ptrs[i] : p->k_pool, dims, strides, bx, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            *err = "CUresult " + std::to_string(int(r));
            return false;
        }
    }
    return true;
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

// F4: quantise to e4m3 on the way in (oracle/fp8.py: code = RNE_SATFINITE(fp32(x) /
// scale), the division IEEE fp32).  One thread per (token, head, 8 channels): K's 8 codes
// are one 8-B store into the token's row; V's go to 8 channel rows of the page's V^T block
// at the slot's permuted column kF8VCol(slot).
struct AppendF8Params {
    const uint4* k_src;
    const uint4* v_src;
    uint8_t* k_dst;          // the interleaved buffer
    const float* scale;      // [L][Hkv][2]
    long long layer_stride;  // bytes: num_pages * Hkv * 4096 (interleaved K / V^T blocks)
    int T_total, t0, n, Hkv;
    int slots[kAppendMax];
};

__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d) {
    uint16_t lo, hi;   // cvt packs its first source operand into the upper byte
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
    return uint32_t(lo) | (uint32_t(hi) << 16);
}

__global__ void append_f8_kernel(const __grid_constant__ AppendF8Params p) {
    const int i = blockIdx.x, layer = blockIdx.y;
    const int slot = p.slots[i];
    const int page = slot >> 4, s = slot & 15;
    const int vcol = kF8VCol(s);
    for (int tid = threadIdx.x; tid < p.Hkv * 16; tid += blockDim.x) {
        const int h = tid >> 4, c8 = tid & 15;
        const long long src = ((long long)(layer)*p.T_total + p.t0 + i) * p.Hkv * 16 + (long long)h * 16 + c8;
        const float ks = p.scale[(layer * p.Hkv + h) * 2], vs = p.scale[(layer * p.Hkv + h) * 2 + 1];
        const uint4 kr = p.k_src[src], vr = p.v_src[src];
        float kf[8], vf[8];
        const uint32_t kw[4] = {kr.x, kr.y, kr.z, kr.w}, vw[4] = {vr.x, vr.y, vr.z, vr.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            kf[2 * e] = __fdiv_rn(__uint_as_float(kw[e] << 16), ks);
            kf[2 * e + 1] = __fdiv_rn(__uint_as_float(kw[e] & 0xffff0000u), ks);
            vf[2 * e] = __fdiv_rn(__uint_as_float(vw[e] << 16), vs);
            vf[2 * e + 1] = __fdiv_rn(__uint_as_float(vw[e] & 0xffff0000u), vs);
        }
        const long long pb = layer * p.layer_stride + ((long long)page * p.Hkv + h) * 4096;
        uint2 kc;
        kc.x = e4m3x4(kf[0], kf[1], kf[2], kf[3]);
        kc.y = e4m3x4(kf[4], kf[5], kf[6], kf[7]);
        *reinterpret_cast<uint2*>(p.k_dst + pb + s * 128 + c8 * 8) = kc;
        const uint32_t v0 = e4m3x4(vf[0], vf[1], vf[2], vf[3]), v1 = e4m3x4(vf[4], vf[5], vf[6], vf[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e)
            p.k_dst[pb + 2048 + (c8 * 8 + e) * 16 + vcol] = uint8_t(((e < 4 ? v0 : v1) >> (8 * (e & 3))) & 0xff);
    }
}

int launch_append(const spa_pool* pool, const void* k_new, const void* v_new, int32_t T_total,
                  const std::vector<int32_t>& slots, void* stream) {
    const auto& c = pool->cfg;
    if (pool->kv_fp8) {
        AppendF8Params p{};
        p.k_src = static_cast<const uint4*>(k_new);
        p.v_src = static_cast<const uint4*>(v_new);
        p.k_dst = static_cast<uint8_t*>(pool->k_pool);
        p.scale = pool->kv_scale;
        p.layer_stride = (long long)c.num_pages * c.num_kv_heads * 4096;
        p.T_total = T_total;
        p.Hkv = c.num_kv_heads;
        const int threads = std::min(256, ((p.Hkv * 16 + 31) / 32) * 32);
        for (int t0 = 0; t0 < T_total; t0 += kAppendMax) {
            p.t0 = t0;
            p.n = std::min(kAppendMax, T_total - t0);
            std::memcpy(p.slots, slots.data() + t0, sizeof(int) * p.n);
            append_f8_kernel<<<dim3(p.n, c.num_layers), threads, 0, static_cast<cudaStream_t>(stream)>>>(p);
        }
        return int(cudaGetLastError());
    }
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
    int dvec = c.head_dim / 8;
    if (pool->kv_fp8) {
        // interleaved 4-KB page-head blocks (K rows + the permuted V^T block): copy them whole
        // as 32 "rows" of 128 B of the one buffer (slots past the fork point are overwritten
        // by the child's appends before they are read)
        const long long ls = (long long)c.num_pages * c.num_kv_heads * 256;   // uint4 per layer
        cow_kernel<<<dim3(c.num_layers, c.num_kv_heads), 128, 0, static_cast<cudaStream_t>(stream)>>>(
            static_cast<const uint4*>(pool->k_pool), static_cast<const uint4*>(pool->k_pool),
            static_cast<uint4*>(pool->k_pool), static_cast<uint4*>(pool->k_pool), ls, src_page, dst_page, 32,
            c.num_kv_heads, 8, 32);
        return int(cudaGetLastError());
    }
    const long long ls = (long long)c.num_pages * c.num_kv_heads * c.page_size * dvec;
    cow_kernel<<<dim3(c.num_layers, c.num_kv_heads), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(pool->k_pool), static_cast<const uint4*>(pool->v_pool),
        static_cast<uint4*>(pool->k_pool), static_cast<uint4*>(pool->v_pool), ls, src_page, dst_page, rows,
        c.num_kv_heads, dvec, c.page_size);
    return int(cudaGetLastError());
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
__global__ void __launch_bounds__(256, 1) merge_kernel(const MergeParams p) {
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

// A plan's split merge as its own launch (the tcgen05 extend path): one warp per merge
// subtask of the plan's list (a whole (row, KV head) task -- all G heads x S records loaded in
// one L2 round trip -- or one head of it), the whole list in one wave.  The plan metadata is
// read before the programmatic-dependency wait (it was uploaded earlier in stream order),
// the partials after it.
template <int D, bool S2>   // S2: every subtask is a whole task of exactly 2 records (lean registers)
__global__ void __launch_bounds__(128) merge_tasks_kernel(const int32_t* meta, const MergeParams p, int G, int Hkv) {
    const int lane = threadIdx.x & 31;
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int n_sub = meta[H_N_MTASK];
    int code = 0, s0 = 0, s1 = 0;
    if (t < n_sub) {
        code = meta[meta[H_OFF_MTASK] + t];
        const int row = (code >> 8) / Hkv;
        s0 = p.rec_ptr[row];
        s1 = p.rec_ptr[row + 1];
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");   // partials come from the attention kernel
    asm volatile("griddepcontrol.launch_dependents;");
    if (t >= n_sub) return;
    const int task = code >> 8, sub = code & 255;
    const int row = task / Hkv, kvh = task - row * Hkv;
    __nv_bfloat16* orow = p.o + row * p.o_sr;
    float* lrow = p.lse ? p.lse + row * p.l_sr : nullptr;
    if (S2)
        warp_merge_task_s2<D>(p.part_o, p.part_lse, p.H, s0, kvh * G, G, orow, p.o_sh, lrow, p.l_sh, lane);
    else if (sub == 0)
        warp_merge_group<D>(p.part_o, p.part_lse, p.H, s0, s1, kvh * G, G, orow, p.o_sh, lrow, p.l_sh, lane);
    else
        warp_merge_head<D>(p.part_o, p.part_lse, p.H, s0, s1, kvh * G + sub - 1, orow, p.o_sh, lrow, p.l_sh, lane);
}

int launch_merge_tasks(const spa_plan* P, void* o, int64_t o_sr, int64_t o_sh, float* lse, int64_t l_sr, int64_t l_sh,
                       void* stream) {
    const auto& c = P->pool->cfg;
    const int32_t* H = P->host.data();
    const int n_sub = H[H_N_MTASK];
    if (n_sub == 0) return 0;
    MergeParams mp{P->d_meta + H[H_OFF_REC_PTR], P->d_part_o, P->d_part_lse, static_cast<__nv_bfloat16*>(o), o_sr, o_sh,
                   lse, l_sr, l_sh, H[H_N_REQ], c.num_q_heads, c.head_dim};
    const int G = c.num_q_heads / c.num_kv_heads;
    const dim3 grid((n_sub + 3) / 4);
    const int32_t* m = P->d_meta;
    if (P->merge_all_s2 && G <= 8)
        return c.head_dim == 128
                   ? launch_pdl(merge_tasks_kernel<128, true>, grid, dim3(128), 0, stream, m, mp, G, c.num_kv_heads)
                   : launch_pdl(merge_tasks_kernel<64, true>, grid, dim3(128), 0, stream, m, mp, G, c.num_kv_heads);
    return c.head_dim == 128
               ? launch_pdl(merge_tasks_kernel<128, false>, grid, dim3(128), 0, stream, m, mp, G, c.num_kv_heads)
               : launch_pdl(merge_tasks_kernel<64, false>, grid, dim3(128), 0, stream, m, mp, G, c.num_kv_heads);
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
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t plan_workspace_need(const spa_plan* P) {
    const auto& c = P->pool->cfg;
    const size_t records = size_t(P->host[H_N_RECORDS]);
    return align256(P->host.size() * 4) + align256(records * c.num_q_heads * c.head_dim * 4) +
           records * c.num_q_heads * 4;
}

// Upload the host plan into the caller's workspace (S8(b): all device memory is caller-owned).
// Returns kUploadNoWorkspace when the workspace is missing or too small (nothing enqueued),
// else a cudaError_t.  Under stream capture the upload becomes a memcpy node that re-reads
// the pinned staging buffer at every replay (which also re-zeroes the queue and merge
// counters, so a captured plan + its decode launches replay consistently); no event is
// waited on or recorded then, and the staging buffer must already be large enough.
int plan_upload(spa_plan* P, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    P->ws_need = plan_workspace_need(P);
    if (!P->ws || P->ws_need > P->ws_bytes) return kUploadNoWorkspace;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    e = cudaStreamIsCapturing(s, &cap);
    if (e) return int(e);
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    if (!capturing && !P->upload_event) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e) return int(e);
        P->upload_event = ev;
    }
    if (!capturing && P->upload_pending) {   // the pinned staging buffer may still be read by the last upload
        e = cudaEventSynchronize(static_cast<cudaEvent_t>(P->upload_event));
        if (e) return int(e);
        P->upload_pending = false;
    }
    const size_t words = P->host.size();
    if (words > P->pinned_words) {   // host staging memory (library-owned host metadata)
        if (capturing) return int(cudaErrorStreamCaptureUnsupported);
        if (P->pinned) cudaFreeHost(P->pinned);
        P->pinned = nullptr;
        P->pinned_words = 0;
        const size_t nw = words + words / 2 + 1024;
        e = cudaMallocHost(reinterpret_cast<void**>(&P->pinned), nw * 4);
        if (e) return int(e);
        P->pinned_words = nw;
    }
    std::memcpy(P->pinned, P->host.data(), words * 4);
    const auto& c = P->pool->cfg;
    const size_t records = size_t(P->host[H_N_RECORDS]);
    char* base = static_cast<char*>(P->ws);
    P->d_meta = reinterpret_cast<int32_t*>(base);
    P->d_part_o = reinterpret_cast<float*>(base + align256(words * 4));
    P->d_part_lse = reinterpret_cast<float*>(base + align256(words * 4) +
                                             align256(records * c.num_q_heads * c.head_dim * 4));
    e = cudaMemcpyAsync(P->d_meta, P->pinned, words * 4, cudaMemcpyHostToDevice, s);
    if (e) return int(e);
    if (!capturing) {
        e = cudaEventRecord(static_cast<cudaEvent_t>(P->upload_event), s);
        if (e) return int(e);
        P->upload_pending = true;
    }
    return 0;
}

void plan_release(spa_plan* P) {
    if (P->upload_event) {
        cudaEventSynchronize(static_cast<cudaEvent_t>(P->upload_event));
        cudaEventDestroy(static_cast<cudaEvent_t>(P->upload_event));
    }
    if (P->pinned) cudaFreeHost(P->pinned);
    P->upload_event = nullptr;
    P->pinned = nullptr;
    P->d_meta = nullptr;
    P->d_part_o = nullptr;
    P->d_part_lse = nullptr;
}

}  // namespace spa
