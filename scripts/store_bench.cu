// store_bench.cu -- what does writing the (C, n_cells) channel-major map cost
// on this B200, by access pattern?  (Guides the phase-2 design of tile.cu.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/store_bench scripts/store_bench.cu
//
// Each variant writes 80 x 129600 floats (41.5 MB); times are CUDA-event
// medians of 20, with and without a 512 MiB L2-flushing write before each rep.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int C = 80;
constexpr long NC = 129600;

// A: 32 cells per CTA (256 threads), warp w writes channels w, w+8, ... (128 B each)
__global__ void store32(float *out) {
    const long c0 = blockIdx.x * 32L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int ch = warp; ch < C; ch += 8) out[ch * NC + c0 + lane] = 1.f;
}
// A2: same with incompressible values
__global__ void store32_rand(float *out) {
    const long c0 = blockIdx.x * 32L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int ch = warp; ch < C; ch += 8) {
        unsigned x = unsigned(ch * NC + c0 + lane) * 2654435761u;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        out[ch * NC + c0 + lane] = __uint_as_float((x & 0x007FFFFFu) | 0x3F000000u);
    }
}
__global__ void fill_rand(float *p, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        unsigned x = unsigned(i) * 2654435761u + 12345u;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        p[i] = __uint_as_float((x & 0x007FFFFFu) | 0x3F000000u);
    }
}
// B: 128 cells per CTA: a warp writes 512 B of one channel row (float4 per lane)
__global__ void store128v4(float *out) {
    const long c0 = blockIdx.x * 128L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int ch = warp; ch < C; ch += 8)
        reinterpret_cast<float4 *>(out + ch * NC + c0)[lane] = make_float4(1.f, 1.f, 1.f, 1.f);
}
// C: grid-stride linear float4 (memset-like)
__global__ void store_linear(float4 *out, long n4) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
        out[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}
// D: per-CTA channel-major slab, CTA owns a channel range x all cells? (one row per CTA)
__global__ void store_rows(float4 *out) {
    const long row = blockIdx.x;  // channel
    float4 *r = out + row * (NC / 4);
    for (long i = threadIdx.x; i < NC / 4; i += blockDim.x) r[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}
// E: like A, plus a read of a contiguous 320 B row per non-empty cell (36% of cells)
__global__ void store32_read(float *out, const float *rows) {
    __shared__ float tile[32][97];
    const long c0 = blockIdx.x * 32L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int u = 0; u < 4; ++u) {
        const int cl = warp + 8 * u;
        const long c = c0 + cl;
        float a0 = 0, a1 = 0, a2 = 0;
        if ((c * 2654435761u) % 100 < 36) {
            const float *r = rows + ((c * 7) % 56548) * C;
            a0 = r[lane]; a1 = r[lane + 32]; if (lane < 16) a2 = r[lane + 64];
        }
        tile[cl][lane] = a0; tile[cl][lane + 32] = a1; tile[cl][lane + 64] = a2;
    }
    __syncthreads();
    for (int ch = warp; ch < C; ch += 8) out[ch * NC + c0 + lane] = tile[lane][ch];
}

// F: like E but the row index comes from a dependent load (cell -> first
// segment), as in the tiled finalize; rows of consecutive cells are adjacent
__global__ void store32_dep(float *out, const float *rows, const unsigned *first) {
    __shared__ float tile[32][97];
    const long c0 = blockIdx.x * 32L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned f = first[c0 + lane], f1 = first[c0 + 32];
    for (int u = 0; u < 4; ++u) {
        const int cl = warp + 8 * u;
        const unsigned s0 = __shfl_sync(~0u, f, cl), s1 = cl < 31 ? __shfl_sync(~0u, f, cl + 1) : f1;
        float a0 = 0, a1 = 0, a2 = 0;
        if (s1 > s0) {
            const float *r = rows + (long)s0 * C;
            a0 = r[lane]; a1 = r[lane + 32]; if (lane < 16) a2 = r[lane + 64];
        }
        tile[cl][lane] = a0; tile[cl][lane + 32] = a1; tile[cl][lane + 64] = a2;
    }
    __syncthreads();
    for (int ch = warp; ch < C; ch += 8) out[ch * NC + c0 + lane] = tile[lane][ch];
}
// G: only the dependent-load chain (no map stores)
__global__ void dep_only(float *sink, const float *rows, const unsigned *first) {
    const long c0 = blockIdx.x * 32L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned f = first[c0 + lane], f1 = first[c0 + 32];
    float acc = 0;
    for (int u = 0; u < 4; ++u) {
        const int cl = warp + 8 * u;
        const unsigned s0 = __shfl_sync(~0u, f, cl), s1 = cl < 31 ? __shfl_sync(~0u, f, cl + 1) : f1;
        if (s1 > s0) acc += rows[(long)s0 * C + lane];
    }
    if (acc == 1234.f) sink[0] = acc;
}

template <typename F>
float timeit(F f, char *flush, bool do_flush) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ts;
    for (int r = 0; r < 23; ++r) {
        if (do_flush) cudaMemsetAsync(flush, r, 512u << 20);
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
    float *out, *rows;
    char *flush;
    cudaMalloc(&out, sizeof(float) * C * NC);
    cudaMalloc(&rows, sizeof(float) * C * 56548);
    cudaMalloc(&flush, 512u << 20);
    cudaMemset(rows, 0, sizeof(float) * C * 56548);
    const bool rnd = true;
    if (rnd) fill_rand<<<1024, 256>>>(rows, (long)C * 56548);
    unsigned *first;
    cudaMalloc(&first, sizeof(unsigned) * (NC + 1));
    {
        std::vector<unsigned> h(NC + 1);
        unsigned acc = 0;
        for (long c = 0; c <= NC; ++c) { h[c] = acc; if ((c * 2654435761u) % 100 < 36) acc += 1 + (c % 5 == 0); }
        printf("segments %u\n", acc);
        cudaMemcpy(first, h.data(), sizeof(unsigned) * (NC + 1), cudaMemcpyHostToDevice);
    }
    for (int fl = 0; fl < 2; ++fl) {
        printf("flush=%d\n", fl);
        printf("  memset           %7.1f us\n", timeit([&] { cudaMemsetAsync(out, 0, sizeof(float) * C * NC); }, flush, fl));
        printf("  store32          %7.1f us\n", timeit([&] { store32<<<NC / 32, 256>>>(out); }, flush, fl));
        printf("  store32_rand     %7.1f us\n", timeit([&] { store32_rand<<<NC / 32, 256>>>(out); }, flush, fl));
        printf("  store128v4       %7.1f us\n", timeit([&] { store128v4<<<NC / 128, 256>>>(out); }, flush, fl));
        printf("  store_linear     %7.1f us\n", timeit([&] { store_linear<<<148 * 8, 256>>>((float4 *)out, C * NC / 4); }, flush, fl));
        printf("  store_rows       %7.1f us\n", timeit([&] { store_rows<<<C, 1024>>>((float4 *)out); }, flush, fl));
        printf("  store32_read     %7.1f us\n", timeit([&] { store32_read<<<NC / 32, 256>>>(out, rows); }, flush, fl));
        printf("  store32_dep      %7.1f us\n", timeit([&] { store32_dep<<<NC / 32, 256>>>(out, rows, first); }, flush, fl));
        printf("  dep_only         %7.1f us\n", timeit([&] { dep_only<<<NC / 32, 256>>>(out, rows, first); }, flush, fl));
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
