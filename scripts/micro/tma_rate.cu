// TMA issue-rate microbenchmark (sm_100a): how fast can P producer warps per SM stream
// paged K boxes into a shared-memory ring, as a function of the box size (2 KB = one
// 64-channel chunk of a 16-row page, 4 KB = both chunks) and of the number of issuing
// warps?  Answers whether the extend kernel's single producer thread (12 boxes per 32-KB
// stage) is bounded by per-thread TMA issue cost or by the SM's TMA unit.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu -lcuda
//   ./tma_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
            bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar,
                                     uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
        : "memory");
}

constexpr int SMEM = 200 * 1024;
constexpr int STAGE = 16384;   // bytes per ring stage (per issuing warp ring)

// each of P producer warps owns SMEM / P / STAGE stages; a stage = 16 KB = 16KB/box boxes.
// box_chunks 1: 2-KB boxes (64 ch x 16 rows x 1 chunk, 8 per stage); 2: 4-KB boxes (4 per stage)
__global__ void __launch_bounds__(512, 1) stream_kernel(const __grid_constant__ CUtensorMap m1,
                                                        const __grid_constant__ CUtensorMap m2, int box_chunks,
                                                        int producers, int stages_per_warp, long long pages,
                                                        unsigned long long* issue_cycles, int lanes, int seq) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= producers) return;
    const int ns = (SMEM / producers) / STAGE;
    const uint32_t ring = uint32_t(__cvta_generic_to_shared(smem)) + warp * ns * STAGE;
    __shared__ uint64_t bars[64];
    const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(&bars[warp * 8]));
    if (lane == 0)
        for (int s = 0; s < ns; ++s) mbar_init(bar0 + s * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    if (lane >= lanes) return;
    const unsigned lmask = lanes == 32 ? 0xffffffffu : ((1u << lanes) - 1u);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const long long gw = blockIdx.x * producers + warp, nw = (long long)gridDim.x * producers;
    unsigned long long icyc = 0;
    long long pg = gw * 4;   // 4 pages per 16-KB stage
    const CUtensorMap* m = box_chunks == 1 ? &m1 : &m2;
    auto issue = [&](int s) {
        const uint32_t b = bar0 + s * 8, d = ring + s * STAGE;
        const long long t0 = clock64();
        if (lane == 0) mbar_expect_tx(b, STAGE);
        __syncwarp(lmask);
        const int nbox = box_chunks == 1 ? 8 : 4;
        for (int x = lane; x < nbox; x += lanes) {
            const int j = box_chunks == 1 ? (x >> 1) : x;
            // pseudo-random page (paged KV: pages are scattered) or consecutive pages
            const long long p = seq ? (pg + j) % pages : ((pg + j) * 2654435761ll) % pages;
            const int row = int(p * 16);
            if (box_chunks == 1)
                tma3(d + (x & 1) * 8192 + j * 2048, m, 0, row, x & 1, b, pol);
            else
                tma3(d + j * 4096, m, 0, row, 0, b, pol);
        }
        __syncwarp(lmask);
        icyc += clock64() - t0;
        pg += 4 * nw;
    };
    for (int s = 0; s < ns; ++s) issue(s);
    uint32_t ph = 0;
    int s = 0;
    for (int k = 0; k < stages_per_warp; ++k) {
        mbar_wait(bar0 + s * 8, ph);
        __syncwarp(lmask);
        if (k + ns < stages_per_warp) issue(s);
        if (++s == ns) {
            s = 0;
            ph ^= 1u;
        }
    }
    if (lane == 0) atomicAdd(issue_cycles, icyc);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const long long pages = (6ll << 30) / 4096;   // 6 GB of 4-KB page-heads (>> L2)
    void* buf;
    cudaMalloc(&buf, pages * 4096);
    cudaMemset(buf, 1, pages * 4096);
    CUtensorMap m1, m2;
    cuuint64_t dims[3] = {64, cuuint64_t(pages * 16), 2};   // (channel, row, chunk): chunk stride 128 B
    cuuint64_t str[2] = {256, 128};
    cuuint32_t box1[3] = {64, 16, 1}, box2[3] = {64, 16, 2}, es[3] = {1, 1, 1};
    // dims order (64 ch, rows, 2 chunks) with strides row 256 B, chunk 128 B
    CUresult r1 = cuTensorMapEncodeTiled(&m1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box1, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = cuTensorMapEncodeTiled(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box2, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 || r2) {
        printf("encode failed %d %d\n", int(r1), int(r2));
        return 1;
    }
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM + 1024);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* ic;
    cudaMalloc(&ic, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("seq lanes box_KB producers stages/warp  GB/s   ns_per_box_per_SM  issue_cycles_per_box\n");
    for (int seq : {0, 1})
    for (int lanes : {1, 4, 8})
    for (int bc : {1, 2})
        for (int P : {1, 2, 4}) {
            if (lanes == 8 && bc == 2) continue;
            const long long total_stages = 2ll * 1024 * 1024 * 1024 / STAGE;   // 2 GB per run
            const int spw = int(total_stages / (sms * P));
            float best = 1e30f;
            unsigned long long cyc = 0;
            for (int rep = 0; rep < 4; ++rep) {
                cudaMemset(ic, 0, 8);
                cudaEventRecord(e0);
                stream_kernel<<<sms, 32 * P, SMEM + 1024>>>(m1, m2, bc, P, spw, pages, ic, lanes, seq);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) {
                    best = ms;
                    cudaMemcpy(&cyc, ic, 8, cudaMemcpyDeviceToHost);
                }
            }
            cudaError_t err = cudaGetLastError();
            if (err) {
                printf("error %s\n", cudaGetErrorString(err));
                return 1;
            }
            const double bytes = double(spw) * sms * P * STAGE;
            const double boxes = bytes / (2048.0 * bc);
            printf("%3d %5d %6d %9d %11d %7.0f %12.1f %16.1f\n", seq, lanes, 2 * bc, P, spw, bytes / (best * 1e-3) / 1e9,
                   best * 1e6 / (boxes / sms), double(cyc) / boxes);
        }
    return 0;
}
