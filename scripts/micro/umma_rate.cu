// tcgen05.mma issue / completion cost of SMALL MMAs on sm_100a (one CTA, one issuing thread):
// the shapes an fp8 decode step would use (M64 / M128, N 16-128, kind::f8f6f4 K32) next to the
// bf16 kind::f16 K16 shapes of the extend kernel.  Operands are zero tiles in shared memory
// (K-major, 128-B swizzle); D goes to tensor memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2511_20048_b200/csrc -o /tmp/umma_rate umma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "device_util.cuh"
#include "umma.cuh"

using namespace spa;

__device__ __forceinline__ void mma_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(uint32_t(acc))
        : "memory");
}

__host__ __device__ constexpr uint32_t idesc_f8(int M, int N) {   // e4m3 x e4m3 -> f32, K-major both
    return (1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// KIND 0: f8f6f4 (K = 32 per MMA), 1: f16/bf16 (K = 16 per MMA).  MODE 0: thread 0 issues
// (descriptors built per MMA); MODE 1: warp 0 runs the loop warp-uniformly, elect.sync issues,
// descriptors advanced by adding to the 64-bit descriptor (what a tuned issuer does).
template <int KIND, int MODE>
__global__ void k(int M, int N, int n_mma, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* s = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x < 32) umma::tmem_alloc(smem_u32(&tbase), 512);
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_proxy_async_smem();
    __syncthreads();
    umma::fence_after();
    const uint32_t t = tbase;
    const uint32_t a = smem_u32(s), b = smem_u32(s + 32 * 1024);
    const uint32_t idesc = KIND == 0 ? idesc_f8(M, N) : umma::idesc_bf16_f32(M, N, false, false);
    if (MODE == 0 && threadIdx.x == 0) {
        long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i) {
            const uint64_t ad = umma::desc_k_sw128(a + (i & 3) * 32, 1024), bd = umma::desc_k_sw128(b + (i & 3) * 32, 1024);
            if (KIND == 0) mma_f8(t + (i & 1) * 256, ad, bd, idesc, i > 1);
            else umma::mma_ss(t + (i & 1) * 256, ad, bd, idesc, i > 1);
        }
        long long t1 = clock64();
        umma::commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        long long t2 = clock64();
        out[blockIdx.x * 2 + 0] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
    if (MODE == 1 && threadIdx.x < 32) {
        const uint64_t ad0 = umma::desc_k_sw128(a, 1024), bd0 = umma::desc_k_sw128(b, 1024);
        long long t0 = clock64();
        for (int i = 0; i < n_mma; i += 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (umma::elect_one()) {
                    if (KIND == 0) mma_f8(t + (j & 1) * 256, ad0 + 2 * j, bd0 + 2 * j, idesc, i + j > 1);
                    else umma::mma_ss(t + (j & 1) * 256, ad0 + 2 * j, bd0 + 2 * j, idesc, i + j > 1);
                }
                __syncwarp();
            }
        }
        long long t1 = clock64();
        if (umma::elect_one()) umma::commit(smem_u32(&bar));
        __syncwarp();
        mbar_wait(smem_u32(&bar), 0);
        long long t2 = clock64();
        if (threadIdx.x == 0) {
            out[blockIdx.x * 2 + 0] = t1 - t0;
            out[blockIdx.x * 2 + 1] = t2 - t0;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_dealloc(t, 512);
}

template <int KIND, int MODE>
void run(int M, int N, long long* d) {
    cudaFuncSetAttribute(k<KIND, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    for (int n : {8, 64, 512}) {
        k<KIND, MODE><<<1, 128, 70 * 1024>>>(M, N, n, d);
        k<KIND, MODE><<<1, 128, 70 * 1024>>>(M, N, n, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const double flop = 2.0 * M * N * (KIND == 0 ? 32 : 16);
        printf("%-5s mode %d M%-3d N%-3d  n=%3d  issue %6.1f cyc/mma  done %7.1f cyc/mma  (%.0f flop/cyc)\n",
               KIND == 0 ? "f8" : "bf16", MODE, M, N, n, double(h[0]) / n, double(h[1]) / n, flop * n / double(h[1]));
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 4096);
    const int shapes[][2] = {{64, 16}, {64, 64}, {64, 128}, {128, 16}, {128, 64}, {128, 128}, {128, 256}};
    for (auto sh : shapes) { run<0, 0>(sh[0], sh[1], d); run<0, 1>(sh[0], sh[1], d); }
    for (auto sh : shapes) run<1, 1>(sh[0], sh[1], d);
    return 0;
}
