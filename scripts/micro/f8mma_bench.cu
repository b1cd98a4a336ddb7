// fp8 mma.sync m16n8k32 (e4m3 x e4m3, e5m2 x e4m3) vs bf16 m16n8k16 latency / throughput on
// sm_100a (one SM), plus the XU-pipe conversions the fp8 decode path uses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/f8mma f8mma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__device__ __forceinline__ void mma(float* c, const unsigned* a, unsigned b0, unsigned b1) {
    if constexpr (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    else if constexpr (KIND == 1)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    else
        asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e5m2.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int KIND, int CH>
__global__ void k(float* out, long long* cyc, int iters) {
    unsigned a[4] = {threadIdx.x & 0x3f3f3f3fu, (threadIdx.x * 3u) & 0x3f3f3f3fu, 0x30303030u, 0x28282828u};
    float c[CH][4] = {};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) mma<KIND>(c[ch], a, 0x38383838u + (i & 7), 0x30303030u);
    long long t1 = clock64();
    float s = 0;
    for (int ch = 0; ch < CH; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// conversion throughput: OP 0 cvt.rn.f16x2.e4m3x2, 1 cvt.rn.satfinite.e4m3x2.f32, 2 ex2.approx,
// 3 cvt.rn.satfinite.e5m2x2.f32
template <int OP>
__global__ void kc(unsigned* out, long long* cyc, int iters) {
    unsigned v[8];
    float f[8];
    for (int j = 0; j < 8; ++j) { v[j] = threadIdx.x * 977u + j; f[j] = 0.001f * (threadIdx.x + j); }
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (OP == 0) {
                unsigned r;
                asm volatile("{ .reg .b16 l; mov.b32 {l, _}, %1; cvt.rn.f16x2.e4m3x2 %0, l; }" : "=r"(r) : "r"(v[j]));
                v[j] ^= r;
            } else if constexpr (OP == 1) {
                unsigned short r;
                asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(f[j]), "f"(f[(j + 1) & 7]));
                f[j] += float(r);
            } else if constexpr (OP == 2) {
                float r;
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[j]));
                f[j] = r * 0.5f;
            } else {
                unsigned short r;
                asm volatile("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(f[j]), "f"(f[(j + 1) & 7]));
                f[j] += float(r);
            }
        }
    }
    long long t1 = clock64();
    unsigned s = 0;
    for (int j = 0; j < 8; ++j) s += v[j] + __float_as_uint(f[j]);
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int KIND, int CH>
void run(int warps) {
    float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64);
    const int iters = 4096;
    k<KIND, CH><<<1, warps * 32>>>(out, cyc, 16);
    k<KIND, CH><<<1, warps * 32>>>(out, cyc, iters);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const char* name = KIND == 0 ? "bf16 m16n8k16" : KIND == 1 ? "e4m3 m16n8k32" : "e5m2xe4m3 k32";
    printf("%s chains=%2d warps=%2d  cycles per MMA per warp=%6.2f  SM MMA/clk=%.3f\n", name, CH, warps,
           double(h) / iters / CH, double(CH) * warps * iters / double(h));
    cudaFree(out); cudaFree(cyc);
}

template <int OP>
void runc(int warps) {
    unsigned* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64);
    const int iters = 2048;
    kc<OP><<<1, warps * 32>>>(out, cyc, 16);
    kc<OP><<<1, warps * 32>>>(out, cyc, iters);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const char* name = OP == 0 ? "cvt f16x2<-e4m3x2" : OP == 1 ? "cvt e4m3x2<-f32x2" : OP == 2 ? "ex2.approx" : "cvt e5m2x2<-f32x2";
    printf("%s warps=%2d  SM warp-instr/clk=%.3f\n", name, warps, 8.0 * warps * iters / double(h));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    run<0, 1>(1); run<0, 8>(1); run<0, 8>(4); run<0, 8>(8); run<0, 8>(16);
    run<1, 1>(1); run<1, 8>(1); run<1, 8>(4); run<1, 8>(8); run<1, 8>(16);
    run<2, 1>(1); run<2, 8>(1); run<2, 8>(8);
    runc<0>(4); runc<0>(16); runc<1>(4); runc<1>(16); runc<2>(4); runc<2>(16); runc<3>(16);
    return 0;
}
