// Microbenchmark: how fast can B200 gather 320-byte rows (C = 80 fp32) from an
// L2-resident 16,896-row table, as a function of the bytes each SM keeps in
// flight?  The access pattern of the interval kernel (the real S-config rank
// order when scratch/pix_S.u32 exists, else uniform random rows).
//   reg U        : one point per warp instruction (20 lanes x 16 B), U rows loaded
//                  before they are summed (U rows in flight per warp)
//   grp U        : 8 points per instruction (4 lanes x 5 x 16 B), U steps in flight
//   ring D       : grp layout, rows land in a per-lane shared-memory ring via
//                  cp.async, D steps in flight (no registers held)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gmlp scripts/gather_mlp_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
constexpr int C = 80;

template <int U>
__global__ void reg_kernel(const float *__restrict__ tab, const uint32_t *__restrict__ idx, int64_t n, int chunk, float *out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t a = w * chunk, e = min(a + chunk, n);
    float4 acc = make_float4(0, 0, 0, 0);
    const int l = lane < 20 ? lane : 0;
    for (int64_t j = a; j < e; j += U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t jj = min(j + u, e - 1);
            v[u] = __ldg(reinterpret_cast<const float4 *>(tab + size_t(__ldg(idx + jj)) * C) + l);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    if (acc.x == 123.f) out[0] = acc.y + acc.z + acc.w;
}

// group layout: 8 groups x 4 lanes, lane li loads chunks li, li+4, ... (5 float4)
template <int U>
__global__ void grp_kernel(const float *__restrict__ tab, const uint32_t *__restrict__ idx, int64_t n, int chunk, float *out) {
    const int lane = threadIdx.x & 31, g = lane >> 2, li = lane & 3;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t a = w * chunk, e = min(a + chunk, n);
    float acc[20] = {0};
    for (int64_t j = a; j < e; j += 8 * U) {
        float4 v[U][5];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t jj = min(j + u * 8 + g, e - 1);
            const float4 *r = reinterpret_cast<const float4 *>(tab + size_t(__ldg(idx + jj)) * C) + li;
#pragma unroll
            for (int k = 0; k < 5; ++k) v[u][k] = __ldg(r + 4 * k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 5; ++k) { acc[4*k] += v[u][k].x; acc[4*k+1] += v[u][k].y; acc[4*k+2] += v[u][k].z; acc[4*k+3] += v[u][k].w; }
    }
    float s = 0; for (int k = 0; k < 20; ++k) s += acc[k];
    if (s == 123.f) out[0] = s;
}

__device__ __forceinline__ void cpa16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
template <int D>
__global__ void ring_kernel(const float *__restrict__ tab, const uint32_t *__restrict__ idx, int64_t n, int chunk, float *out) {
    extern __shared__ float4 ring[];  // [warps][D+1][5][32]
    const int lane = threadIdx.x & 31, g = lane >> 2, li = lane & 3, warp = threadIdx.x >> 5;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t a = w * chunk, e = min(a + chunk, n);
    float4 *my = ring + warp * (D + 1) * 5 * 32;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(my));
    float acc[20] = {0};
    const int64_t steps = (e - a + 7) / 8;
    auto issue = [&](int64_t s) {
        const int slot = static_cast<int>(s % (D + 1));
        const int64_t jj = min(a + s * 8 + g, e - 1);
        const float4 *r = reinterpret_cast<const float4 *>(tab + size_t(__ldg(idx + jj)) * C) + li;
#pragma unroll
        for (int k = 0; k < 5; ++k) cpa16(base + ((slot * 5 + k) * 32 + lane) * 16, r + 4 * k);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int s = 0; s < D; ++s) {
        if (s < steps) issue(s);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int64_t s = 0; s < steps; ++s) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        const int slot = static_cast<int>(s % (D + 1));
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const float4 v = my[(slot * 5 + k) * 32 + lane];
            acc[4*k] += v.x; acc[4*k+1] += v.y; acc[4*k+2] += v.z; acc[4*k+3] += v.w;
        }
        if (s + D < steps) issue(s + D);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    float s = 0; for (int k = 0; k < 20; ++k) s += acc[k];
    if (s == 123.f) out[0] = s;
}

int main() {
    const int64_t rows = 16896;
    std::vector<uint32_t> real;
    if (FILE *f = fopen("scratch/pix_S.u32", "rb")) {
        fseek(f, 0, SEEK_END); real.resize(ftell(f) / 4); fseek(f, 0, SEEK_SET);
        if (fread(real.data(), 4, real.size(), f) != real.size()) real.clear();
        fclose(f);
    }
    const int64_t n = real.empty() ? 1742580 : (int64_t)real.size();
    if (real.empty()) { real.resize(n); uint64_t s = 88172645463325252ull; for (auto &x : real) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = s % rows; } }
    float *tab, *out; uint32_t *d_idx; void *flush;
    CK(cudaMalloc(&tab, rows * C * 4)); CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&d_idx, n * 4)); CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMemset(tab, 0, rows * C * 4));
    CK(cudaMemcpy(d_idx, real.data(), n * 4, cudaMemcpyHostToDevice));
    cudaEvent_t ea, eb; cudaEventCreate(&ea); cudaEventCreate(&eb);
    auto timeit = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int i = 0; i < 10; ++i) {
            CK(cudaMemsetAsync(flush, 0, 512 << 20));
            cudaEventRecord(ea); launch(); cudaEventRecord(eb); cudaEventSynchronize(eb);
            float ms; cudaEventElapsedTime(&ms, ea, eb); best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        printf("%-40s %8.1f us  %6.2f TB/s\n", name, best * 1e3, n * C * 4.0 / (best * 1e-3) / 1e12);
    };
    char nm[96];
    for (int chunk : {128, 512}) {
        const int64_t warps = (n + chunk - 1) / chunk;
        const unsigned blocks = (warps * 32 + 255) / 256;
        snprintf(nm, 96, "reg U=4 chunk=%d", chunk); timeit(nm, [&] { reg_kernel<4><<<blocks, 256>>>(tab, d_idx, n, chunk, out); });
        snprintf(nm, 96, "reg U=8 chunk=%d", chunk); timeit(nm, [&] { reg_kernel<8><<<blocks, 256>>>(tab, d_idx, n, chunk, out); });
        snprintf(nm, 96, "reg U=16 chunk=%d", chunk); timeit(nm, [&] { reg_kernel<16><<<blocks, 256>>>(tab, d_idx, n, chunk, out); });
        snprintf(nm, 96, "grp U=1 chunk=%d", chunk); timeit(nm, [&] { grp_kernel<1><<<blocks, 256>>>(tab, d_idx, n, chunk, out); });
        snprintf(nm, 96, "grp U=2 chunk=%d", chunk); timeit(nm, [&] { grp_kernel<2><<<blocks, 256>>>(tab, d_idx, n, chunk, out); });
        snprintf(nm, 96, "grp U=4 chunk=%d", chunk); timeit(nm, [&] { grp_kernel<4><<<blocks, 256>>>(tab, d_idx, n, chunk, out); });
        {
            const size_t sm2 = 8 * 3 * 5 * 32 * 16; cudaFuncSetAttribute(ring_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
            snprintf(nm, 96, "ring D=2 chunk=%d", chunk); timeit(nm, [&] { ring_kernel<2><<<blocks, 256, sm2>>>(tab, d_idx, n, chunk, out); });
            const size_t sm4 = 8 * 5 * 5 * 32 * 16; cudaFuncSetAttribute(ring_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
            snprintf(nm, 96, "ring D=4 chunk=%d", chunk); timeit(nm, [&] { ring_kernel<4><<<blocks, 256, sm4>>>(tab, d_idx, n, chunk, out); });
            const size_t sm8 = 8 * 9 * 5 * 32 * 16; cudaFuncSetAttribute(ring_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8);
            snprintf(nm, 96, "ring D=8 chunk=%d", chunk); timeit(nm, [&] { ring_kernel<8><<<blocks, 256, sm8>>>(tab, d_idx, n, chunk, out); });
        }
    }
    return 0;
}
