// Microbenchmark: gather 320-byte rows (C=80 fp32) from an L2-resident
// 16,896-row table -- the access pattern of the interval kernel.
//   ldg-strided : warp w takes points [w*U, w*U+U), then strides by all warps
//   ldg-chunk   : warp w walks a contiguous chunk of CH points (like a task)
// for (a) uniformly random rows and (b) the real S-config rank order
// (scratch/pix_S.u32, written by the oracle).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2g scripts/l2_gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int C = 80;

template <int U>
__global__ void __launch_bounds__(256) gather_strided(const float *__restrict__ tab, const uint32_t *__restrict__ idx,
                                                      int64_t n, float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t base = warp * U; base < n; base += nw * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = base + u;
            if (j < n && lane < 20) v[u] = __ldg(reinterpret_cast<const float4 *>(tab + size_t(idx[j]) * C) + lane);
            else v[u] = make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    if (acc.x == 123.f) out[0] = acc.y + acc.z + acc.w;
}

template <int U>
__global__ void __launch_bounds__(256) gather_chunk(const float *__restrict__ tab, const uint32_t *__restrict__ idx,
                                                    int64_t n, int chunk, float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t a = warp * chunk, e = a + chunk < n ? a + chunk : n;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t base = a; base < e; base += U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = base + u;
            if (j < e && lane < 20) v[u] = __ldg(reinterpret_cast<const float4 *>(tab + size_t(idx[j]) * C) + lane);
            else v[u] = make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    if (acc.x == 123.f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
    const int64_t rows = 16896;
    std::vector<uint32_t> real;
    if (FILE *f = fopen("scratch/pix_S.u32", "rb")) {
        fseek(f, 0, SEEK_END);
        real.resize(ftell(f) / 4);
        fseek(f, 0, SEEK_SET);
        if (fread(real.data(), 4, real.size(), f) != real.size()) real.clear();
        fclose(f);
    }
    const int64_t n = real.empty() ? 1742580 : (int64_t)real.size();
    std::vector<uint32_t> rnd(n);
    uint64_t s = 88172645463325252ull;
    for (auto &x : rnd) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = s % rows; }
    float *tab, *out; uint32_t *d_rnd, *d_real; void *flush;
    CK(cudaMalloc(&tab, rows * C * 4)); CK(cudaMalloc(&out, 4));
    CK(cudaMalloc(&d_rnd, n * 4)); CK(cudaMalloc(&d_real, n * 4));
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMemset(tab, 0, rows * C * 4));
    CK(cudaMemcpy(d_rnd, rnd.data(), n * 4, cudaMemcpyHostToDevice));
    if (!real.empty()) CK(cudaMemcpy(d_real, real.data(), n * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        float best = 1e9;
        for (int i = 0; i < 10; ++i) {
            CK(cudaMemsetAsync(flush, 0, 512 << 20));
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        printf("%-44s %8.1f us  %7.2f TB/s (row bytes)\n", name, best * 1e3, n * C * 4.0 / (best * 1e-3) / 1e12);
    };
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("n=%lld real=%d\n", (long long)n, (int)!real.empty());
    for (int which = 0; which < (real.empty() ? 1 : 2); ++which) {
        const uint32_t *idx = which ? d_real : d_rnd;
        const char *tag = which ? "real" : "rand";
        char nm[96];
        for (int occ : {4, 8}) {
            snprintf(nm, 96, "%s strided U=4 blocks/SM=%d", tag, occ);
            timeit(nm, [&] { gather_strided<4><<<sms * occ, 256>>>(tab, idx, n, out); });
        }
        for (int chunk : {32, 128, 384}) {
            const int64_t warps = (n + chunk - 1) / chunk;
            snprintf(nm, 96, "%s chunk=%d U=4", tag, chunk);
            timeit(nm, [&] { gather_chunk<4><<<(warps * 32 + 255) / 256, 256>>>(tab, idx, n, chunk, out); });
            snprintf(nm, 96, "%s chunk=%d U=8", tag, chunk);
            timeit(nm, [&] { gather_chunk<8><<<(warps * 32 + 255) / 256, 256>>>(tab, idx, n, chunk, out); });
        }
    }
    return 0;
}
