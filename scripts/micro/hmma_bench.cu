// mma.sync m16n8k16 bf16 latency / throughput on sm_100a (one SM).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(float* c, const unsigned* a, unsigned b0, unsigned b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int CH>
__global__ void k(float* out, long long* cyc, int iters) {
    unsigned a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u};
    float c[CH][4] = {};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) mma(c[ch], a, 0x3f803f80u + i, 0x3f80u);
    long long t1 = clock64();
    float s = 0;
    for (int ch = 0; ch < CH; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
void run(int warps) {
    float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64);
    const int iters = 4096;
    k<CH><<<1, warps * 32>>>(out, cyc, 16);
    k<CH><<<1, warps * 32>>>(out, cyc, iters);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("chains=%2d warps=%2d  cycles/iter=%7.1f  cycles per HMMA per warp=%6.2f  SM HMMA/clk=%.3f\n", CH, warps,
           double(h) / iters, double(h) / iters / CH, double(CH) * warps * iters / double(h));
    cudaFree(out); cudaFree(cyc);
}
int main() {
    run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<16>(1);
    run<1>(4); run<8>(4); run<16>(4); run<8>(8); run<16>(8); run<8>(16);
    return 0;
}
