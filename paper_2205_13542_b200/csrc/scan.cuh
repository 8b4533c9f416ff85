// scan.cuh -- device-wide exclusive scan (reduce / scan partials / downsweep).
#pragma once

#include "common.cuh"

namespace bvp {

// ---- device-wide exclusive scan (3 phases) ---------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanChunk = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *warp_sums, T &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    T wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
        const T s = warp_sums[w];
        if (w < warp) wpre += s;
        tot += s;
    }
    __syncthreads();
    total = tot;
    return wpre + x - v;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads)
scan_reduce_kernel(const T *__restrict__ in, int64_t n, T *__restrict__ partials) {
    __shared__ T ws[kScanThreads / 32];
    const int64_t base = blockIdx.x * (int64_t)kScanChunk;
    T s = 0;
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t e = base + k * kScanThreads + threadIdx.x;
        if (e < n) s += in[e];
    }
    T tot;
    block_excl_scan<T>(s, ws, tot);
    if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads)
scan_partials_kernel(T *__restrict__ partials, int64_t nb, T *__restrict__ total_out) {
    __shared__ T ws[kScanThreads / 32];
    T carry = 0;
    for (int64_t b = 0; b < nb; b += kScanThreads) {
        const int64_t e = b + threadIdx.x;
        const T v = e < nb ? partials[e] : T(0);
        T tot;
        const T ex = block_excl_scan<T>(v, ws, tot);
        if (e < nb) partials[e] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads)
scan_down_kernel(const T *__restrict__ in, int64_t n, const T *__restrict__ partials,
                 T *__restrict__ out) {
    __shared__ T ws[kScanThreads / 32];
    const int64_t base = blockIdx.x * (int64_t)kScanChunk;
    T carry = partials[blockIdx.x];
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t e = base + k * kScanThreads + threadIdx.x;
        const T v = e < n ? in[e] : T(0);
        T tot;
        const T ex = block_excl_scan<T>(v, ws, tot);
        if (e < n) out[e] = carry + ex;
        carry += tot;
    }
}

template <typename T>
static int64_t scan_partials_len(int64_t n) { return ceil_div(n, kScanChunk) + 1; }

// Exclusive scan of n elements (in may equal out).  partials must hold
// scan_partials_len(n) elements; *total (device) receives the sum.
template <typename T>
static void device_excl_scan(const T *in, T *out, int64_t n, T *partials, T *total,
                             cudaStream_t s) {
    const int64_t nb = ceil_div(n, kScanChunk);
    if (nb == 0) {
        cudaMemsetAsync(total, 0, sizeof(T), s);
        return;
    }
    scan_reduce_kernel<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partials);
    scan_partials_kernel<T><<<1, kScanThreads, 0, s>>>(partials, nb, total);
    scan_down_kernel<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partials, out);
}

}  // namespace bvp
