// Microbenchmark: gather 320-byte rows (C=80 fp32) from an L2-resident table
// in random order -- the access pattern of the interval kernel -- two ways:
//   (a) LDG.128 from registers, 20 lanes x 16 B per row, U rows in flight/warp
//   (b) cp.async.bulk (TMA 1-D bulk copy) global -> shared, one lane per row,
//       completion on an mbarrier
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2g scripts/l2_gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int C = 80;

template <int U>
__global__ void __launch_bounds__(256) gather_ldg(const float *__restrict__ tab, const uint32_t *__restrict__ idx,
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

__device__ __forceinline__ void mbar_init(uint64_t *m, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t *m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
    asm volatile("{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}" ::"r"((uint32_t)__cvta_generic_to_shared(m)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(m)) : "memory");
}

// each warp: S-stage ring of 32 rows
template <int S>
__global__ void __launch_bounds__(128) gather_tma(const float *__restrict__ tab, const uint32_t *__restrict__ idx,
                                                  int64_t n, float *__restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *buf = reinterpret_cast<float *>(smem) + wid * S * 32 * C;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 4 * 32 * C * S * 4) + wid * S;
    if (lane == 0) for (int s = 0; s < S; ++s) mbar_init(bar + s, 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const int64_t nchunks = (n + 31) / 32;
    float acc = 0.f;
    int64_t issue = warp, consume = warp;
    uint32_t phase[S] = {};
    int t_issue = 0, t_cons = 0;
    for (int s = 0; s < S - 1 && issue < nchunks; ++s, issue += nw, ++t_issue) {
        const int64_t j = issue * 32 + lane;
        const int st = t_issue % S;
        const uint32_t cnt = (uint32_t)(n - issue * 32 < 32 ? n - issue * 32 : 32);
        if (lane == 0) mbar_expect(bar + st, cnt * C * 4);
        if (j < n) bulk_g2s(buf + (st * 32 + lane) * C, tab + size_t(idx[j]) * C, C * 4, bar + st);
    }
    for (; consume < nchunks; consume += nw, ++t_cons) {
        if (issue < nchunks) {
            const int64_t j = issue * 32 + lane;
            const int st = t_issue % S;
            const uint32_t cnt = (uint32_t)(n - issue * 32 < 32 ? n - issue * 32 : 32);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (lane == 0) mbar_expect(bar + st, cnt * C * 4);
            if (j < n) bulk_g2s(buf + (st * 32 + lane) * C, tab + size_t(idx[j]) * C, C * 4, bar + st);
            issue += nw;
            ++t_issue;
        }
        const int st = t_cons % S;
        mbar_wait(bar + st, phase[st]);
        phase[st] ^= 1;
        const float *rb = buf + st * 32 * C;
        for (int k = 0; k < 32; ++k)
            if (lane < 20) { float4 v = reinterpret_cast<const float4 *>(rb + k * C)[lane]; acc += v.x + v.y + v.z + v.w; }
        __syncwarp();
    }
    if (acc == 123.f) out[0] = acc;
}

int main() {
    const int64_t rows = 16896;  // S config pixels: 5.4 MB table
    const int64_t n = 1742580;   // gathers
    std::vector<uint32_t> h(n);
    uint64_t s = 88172645463325252ull;
    for (auto &x : h) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = s % rows; }
    float *tab, *out; uint32_t *idx; void *flush;
    CK(cudaMalloc(&tab, rows * C * 4)); CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&idx, n * 4));
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMemset(tab, 0, rows * C * 4));
    CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        float best = 1e9;
        for (int i = 0; i < 10; ++i) {
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        printf("%-28s %8.1f us  %7.2f TB/s (row bytes)\n", name, best * 1e3, n * C * 4.0 / (best * 1e-3) / 1e12);
    };
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {4, 8, 16})
    {
        char nm[64];
        snprintf(nm, 64, "ldg U=4 blocks/SM=%d", occ);
        timeit(nm, [&] { gather_ldg<4><<<sms * occ, 256>>>(tab, idx, n, out); });
        snprintf(nm, 64, "ldg U=8 blocks/SM=%d", occ);
        timeit(nm, [&] { gather_ldg<8><<<sms * occ, 256>>>(tab, idx, n, out); });
    }
    for (int S : {2, 3, 4}) {
        const size_t smem = 4 * 32 * C * S * 4 + 4 * S * 8;
        for (int cta : {1, 2, 3, 4}) {
            if (smem * cta > 227 * 1024) continue;
            char nm[64];
            snprintf(nm, 64, "tma S=%d ctas/SM=%d", S, cta);
            if (S == 2) { cudaFuncSetAttribute(gather_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); timeit(nm, [&] { gather_tma<2><<<sms * cta, 128, smem>>>(tab, idx, n, out); }); }
            if (S == 3) { cudaFuncSetAttribute(gather_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); timeit(nm, [&] { gather_tma<3><<<sms * cta, 128, smem>>>(tab, idx, n, out); }); }
            if (S == 4) { cudaFuncSetAttribute(gather_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); timeit(nm, [&] { gather_tma<4><<<sms * cta, 128, smem>>>(tab, idx, n, out); }); }
        }
    }
    // sequential streaming read for reference (L2-resident table re-read)
    return 0;
}
