// stage_bench.cu -- cost of staging a camera column's feature rows and depth
// weights (the tiled reduction's phase-1 loads) by access pattern, config S:
// features (6, 80, 32, 88) f32 + dist (6, 118, 32, 88) f32 = 13.4 MB.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/stage_bench scripts/stage_bench.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

constexpr int N = 6, C = 80, H = 32, W = 88, D = 118, HW = H * W;

// (a) one CTA per column (n, w): lane = row, 32 lines per load
__global__ void col_tile(const float *f, const float *dw, float *sink) {
    const int n = blockIdx.x / W, w = blockIdx.x % W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float acc = 0.f;
    for (int c = warp; c < C; c += 8) acc += __ldg(f + ((n * C + c) * H + lane) * W + w);
    for (int d = warp; d < D; d += 8) acc += __ldg(dw + ((n * D + d) * H + lane) * W + w);
    if (acc == 12345.f) sink[0] = acc;
}
// (a2) same, 4 channels per iteration unrolled (more loads in flight)
__global__ void col_tile_u(const float *f, const float *dw, float *sink) {
    const int n = blockIdx.x / W, w = blockIdx.x % W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float acc = 0.f;
#pragma unroll 10
    for (int c = warp; c < C; c += 8) acc += __ldg(f + ((n * C + c) * H + lane) * W + w);
#pragma unroll 15
    for (int d = warp; d < D; d += 8) acc += __ldg(dw + ((n * D + d) * H + lane) * W + w);
    if (acc == 12345.f) sink[0] = acc;
}
// (b) cluster of 8 columns: CTA rank r loads channels r, r+8, ... for 8 columns x 32 rows
__global__ void __cluster_dims__(8, 1, 1) cluster8(const float *f, const float *dw, float *sink) {
    namespace cg = cooperative_groups;
    const int rank = cg::this_cluster().block_rank();
    const int n = blockIdx.x / W, w0 = (blockIdx.x % W) - rank;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = lane & 7, r0 = lane >> 3;
    float acc = 0.f;
    for (int c = rank + 8 * warp; c < C; c += 64)
#pragma unroll
        for (int m = 0; m < 8; ++m) acc += __ldg(f + ((n * C + c) * H + r0 + 4 * m) * W + w0 + j);
    for (int d = rank + 8 * warp; d < D; d += 64)
#pragma unroll
        for (int m = 0; m < 8; ++m) acc += __ldg(dw + ((n * D + d) * H + r0 + 4 * m) * W + w0 + j);
    if (acc == 12345.f) sink[0] = acc;
}
// (c) same bytes, coalesced: CTA reads a contiguous 25 KB block
__global__ void coalesced(const float4 *f, const float4 *dw, float *sink) {
    const long per_f = (long)N * C * HW / 4 / (N * W), per_d = (long)N * D * HW / 4 / (N * W);
    float acc = 0.f;
    for (long i = threadIdx.x; i < per_f; i += 256) { float4 v = __ldg(f + blockIdx.x * per_f + i); acc += v.x; }
    for (long i = threadIdx.x; i < per_d; i += 256) { float4 v = __ldg(dw + blockIdx.x * per_d + i); acc += v.x; }
    if (acc == 12345.f) sink[0] = acc;
}

template <typename F>
float timeit(F f, char *flush) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ts;
    for (int r = 0; r < 23; ++r) {
        cudaMemsetAsync(flush, r, 512u << 20);
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) ts.push_back(ms * 1e3f);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

int main() {
    float *f, *dw, *sink;
    char *flush;
    cudaMalloc(&f, sizeof(float) * N * C * HW);
    cudaMalloc(&dw, sizeof(float) * N * D * HW);
    cudaMalloc(&sink, 64);
    cudaMalloc(&flush, 512u << 20);
    cudaMemset(f, 0, sizeof(float) * N * C * HW);
    cudaMemset(dw, 0, sizeof(float) * N * D * HW);
    printf("col_tile   %7.1f us\n", timeit([&] { col_tile<<<N * W, 256>>>(f, dw, sink); }, flush));
    printf("col_tile_u %7.1f us\n", timeit([&] { col_tile_u<<<N * W, 256>>>(f, dw, sink); }, flush));
    printf("cluster8   %7.1f us\n", timeit([&] { cluster8<<<N * W, 256>>>(f, dw, sink); }, flush));
    printf("coalesced  %7.1f us\n", timeit([&] { coalesced<<<N * W, 256>>>((const float4 *)f, (const float4 *)dw, sink); }, flush));
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
