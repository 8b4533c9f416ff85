// mma.sync (tf32, bf16) vs FFMA2 issue throughput on this GPU: the measurement
// behind keeping the tile products on FFMA2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_vs_ffma2 scripts/mma_vs_ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void k_mma(float *out, int iters) {
    float d[8][4] = {};
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u}, b0 = threadIdx.x ^ 5u, b1 = 11u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_mma_bf16(float *out, int iters) {
    float d[8][4] = {};
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u}, b0 = threadIdx.x ^ 5u, b1 = 11u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_ffma2(float *out, int iters) {
    unsigned long long acc[16];
    for (int j = 0; j < 16; ++j) acc[j] = threadIdx.x + j;
    unsigned long long w = 0x3f8000003f800000ull, f = 0x3f0000003f000000ull;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j]) : "l"(w), "l"(f));
    }
    unsigned long long s = 0;
    for (int j = 0; j < 16; ++j) s ^= acc[j];
    if (s == 12345) out[0] = 1;
}
int main() {
    float *o; cudaMalloc(&o, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a); k_mma<<<blocks, threads>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 16 * 8 * 8 * 8 * double(iters) * blocks * threads / 32;
        printf("mma tf32 m16n8k8: %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
        cudaEventRecord(a); k_mma_bf16<<<blocks, threads>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl = 2.0 * 16 * 8 * 16 * 8 * double(iters) * blocks * threads / 32;
        printf("mma bf16 m16n8k16: %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
        cudaEventRecord(a); k_ffma2<<<blocks, threads>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl = 2.0 * 2 * 16 * double(iters) * blocks * threads;
        printf("ffma2: %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    }
    return 0;
}
