// scan.cuh -- device-wide exclusive scan (reduce / scan partials / downsweep).
//
// A block owns a chunk of kScanChunk elements; each of its 8 warps owns a
// contiguous 512-element slice and walks it 32 elements at a time with warp
// shuffles only, so a chunk costs one block barrier instead of one per round.
// T: an integer or floating type, or uint4 (four independent counters scanned
// together).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace bvp {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanChunk = kScanThreads * kScanItems;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kScanSlice = kScanChunk / kScanWarps;  // elements per warp

__device__ __forceinline__ uint4 operator+(uint4 a, uint4 b) {
    return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ uint4 &operator+=(uint4 &a, uint4 b) { return a = a + b; }

template <typename T>
__device__ __forceinline__ T shfl_up_t(T v, int o) { return __shfl_up_sync(0xFFFFFFFFu, v, o); }
template <>
__device__ __forceinline__ uint4 shfl_up_t<uint4>(uint4 v, int o) {
    return make_uint4(__shfl_up_sync(0xFFFFFFFFu, v.x, o), __shfl_up_sync(0xFFFFFFFFu, v.y, o),
                      __shfl_up_sync(0xFFFFFFFFu, v.z, o), __shfl_up_sync(0xFFFFFFFFu, v.w, o));
}
template <typename T>
__device__ __forceinline__ T shfl_t(T v, int src) { return __shfl_sync(0xFFFFFFFFu, v, src); }
template <typename T>
__device__ __forceinline__ T shfl_xor_t(T v, int o) { return __shfl_xor_sync(0xFFFFFFFFu, v, o); }
template <>
__device__ __forceinline__ uint4 shfl_xor_t<uint4>(uint4 v, int o) {
    return make_uint4(__shfl_xor_sync(0xFFFFFFFFu, v.x, o), __shfl_xor_sync(0xFFFFFFFFu, v.y, o),
                      __shfl_xor_sync(0xFFFFFFFFu, v.z, o), __shfl_xor_sync(0xFFFFFFFFu, v.w, o));
}
template <>
__device__ __forceinline__ uint4 shfl_t<uint4>(uint4 v, int src) {
    return make_uint4(__shfl_sync(0xFFFFFFFFu, v.x, src), __shfl_sync(0xFFFFFFFFu, v.y, src),
                      __shfl_sync(0xFFFFFFFFu, v.z, src), __shfl_sync(0xFFFFFFFFu, v.w, src));
}

// Inclusive warp scan.
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = shfl_up_t(x, o);
        if (lane >= o) x += y;
    }
    return x;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads)
scan_reduce_kernel(const T *__restrict__ in, int64_t n, T *__restrict__ partials) {
    __shared__ T ws[kScanWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = blockIdx.x * (int64_t)kScanChunk + warp * kScanSlice;
    T s{};
#pragma unroll 4
    for (int k = 0; k < kScanSlice / 32; ++k) {
        const int64_t e = base + k * 32 + lane;
        if (e < n) s += in[e];
    }
    s = warp_incl_scan(s, lane);
    if (lane == 31) ws[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t{};
#pragma unroll
        for (int w = 0; w < kScanWarps; ++w) t += ws[w];
        partials[blockIdx.x] = t;
    }
}

// Exclusive scan of the block partials (one block; nb is small).
template <typename T>
__global__ void __launch_bounds__(kScanThreads)
scan_partials_kernel(T *__restrict__ partials, int64_t nb, T *__restrict__ total_out) {
    __shared__ T ws[kScanWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T carry{};
    for (int64_t b = 0; b < nb; b += kScanThreads) {
        const int64_t e = b + threadIdx.x;
        const T v = e < nb ? partials[e] : T{};
        const T x = warp_incl_scan(v, lane);
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        T wpre{}, tot{};
#pragma unroll
        for (int w = 0; w < kScanWarps; ++w) {
            const T s = ws[w];
            if (w < warp) wpre += s;
            tot += s;
        }
        __syncthreads();
        // exclusive prefix of this thread: carry + wpre + (x - v), with the
        // warp-exclusive part taken from the neighbouring lane
        T wex = shfl_up_t(x, 1);
        if (lane == 0) wex = T{};
        if (e < nb) partials[e] = carry + wpre + wex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads)
scan_down_kernel(const T *__restrict__ in, int64_t n, const T *__restrict__ partials,
                 T *__restrict__ out) {
    __shared__ T ws[kScanWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = blockIdx.x * (int64_t)kScanChunk + warp * kScanSlice;
    constexpr int R = kScanSlice / 32;
    T ex[R];
    T run{};
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int64_t e = base + k * 32 + lane;
        const T v = e < n ? in[e] : T{};
        const T x = warp_incl_scan(v, lane);
        T wex = shfl_up_t(x, 1);
        if (lane == 0) wex = T{};
        ex[k] = run + wex;
        run += shfl_t(x, 31);
    }
    if (lane == 0) ws[warp] = run;
    __syncthreads();
    T pre = partials[blockIdx.x];
#pragma unroll
    for (int w = 0; w < kScanWarps; ++w)
        if (w < warp) pre += ws[w];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int64_t e = base + k * 32 + lane;
        if (e < n) out[e] = pre + ex[k];
    }
}

// ---- single pass (integer T): decoupled look-back ----------------------------
// Chunks take tickets in the order their CTAs start; chunk t publishes its
// aggregate (flag 1), looks back over chunks t-1, t-2, ... adding aggregates
// until one with its inclusive prefix (flag 2), then publishes its own
// inclusive prefix.  A chunk only waits on chunks that started before it, so
// the scan cannot deadlock.  The look-back's decomposition depends on
// timing, so only exact (integer) sums use it; floating types keep the
// three-pass scan (deterministic rounding).
template <typename T>
struct is_exact_scan : std::integral_constant<bool, std::is_integral<T>::value> {};
template <>
struct is_exact_scan<uint4> : std::true_type {};

template <typename T>
__device__ __forceinline__ T ld_cg(const T *p) { return __ldcg(p); }
template <>
__device__ __forceinline__ uint4 ld_cg<uint4>(const uint4 *p) { return __ldcg(p); }

// part: [agg: nb][incl: nb] T, then [flags: nb][ticket] uint32 (zeroed by the caller)
template <typename T>
struct ScanIdentity {
    __device__ __forceinline__ T operator()(T v) const { return v; }
};

template <typename T, typename In = T, typename Xf = ScanIdentity<T>>
__global__ void __launch_bounds__(kScanThreads)
scan_onepass_kernel(const In *__restrict__ in, int64_t n, T *out, T *part, int64_t nb,
                    T *__restrict__ total, Xf xf = Xf{}) {
    __shared__ T ws[kScanWarps];
    __shared__ T s_excl;
    __shared__ uint32_t s_tile;
    T *agg = part, *incl = part + nb;
    uint32_t *flags = reinterpret_cast<uint32_t *>(part + 2 * nb), *ticket = flags + nb;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // (a programmatic dependent launch waits here for its producer; else a no-op)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanChunk + warp * kScanSlice;
    constexpr int R = kScanSlice / 32;
    T ex[R];
    T run{};
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int64_t e = base + k * 32 + lane;
        const T v = e < n ? xf(in[e]) : T{};
        const T x = warp_incl_scan(v, lane);
        T wex = shfl_up_t(x, 1);
        if (lane == 0) wex = T{};
        ex[k] = run + wex;
        run += shfl_t(x, 31);
    }
    if (lane == 0) ws[warp] = run;
    __syncthreads();
    // warp 0: publish the aggregate, then look back 32 chunks at a time (lane
    // i reads chunk base - i): the nearest chunk with its inclusive prefix
    // bounds the window; the aggregates before it are summed across lanes
    if (warp == 0) {
        T tot{};
#pragma unroll
        for (int w = 0; w < kScanWarps; ++w) tot += ws[w];
        T excl{};
        if (tile == 0) {
            if (lane == 0) {
                incl[0] = tot;
                __threadfence();
                atomicExch(flags, 2u);
            }
        } else {
            if (lane == 0) {
                agg[tile] = tot;
                __threadfence();
                atomicExch(flags + tile, 1u);
            }
            for (int64_t hi = tile - 1;; hi -= 32) {
                const int64_t j = hi - lane;
                uint32_t f = 2u;  // past chunk 0: nothing to add (acts as a stop)
                if (j >= 0) {
                    do {
                        f = atomicAdd(flags + j, 0u);
                    } while (f == 0u);
                }
                __threadfence();
                const unsigned stop = __ballot_sync(0xFFFFFFFFu, f == 2u);
                const int first = stop ? __ffs(stop) - 1 : 32;  // nearest inclusive lane
                T v{};
                if (j >= 0 && lane <= first && lane < 32)
                    v = lane == first ? ld_cg(incl + j) : ld_cg(agg + j);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += shfl_xor_t(v, o);
                excl += v;
                if (stop) break;
            }
            if (lane == 0) {
                incl[tile] = excl + tot;
                __threadfence();
                atomicExch(flags + tile, 2u);
            }
        }
        if (lane == 0) {
            s_excl = excl;
            if (tile == nb - 1 && total) *total = excl + tot;
        }
    }
    __syncthreads();
    T pre = s_excl;
#pragma unroll
    for (int w = 0; w < kScanWarps; ++w)
        if (w < warp) pre += ws[w];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int64_t e = base + k * 32 + lane;
        if (e < n) out[e] = pre + ex[k];
    }
}

template <typename T>
static int64_t scan_partials_len(int64_t n) {
    const int64_t nb = ceil_div(n, kScanChunk);
    // three-pass: nb + 1 partials; single pass: 2 nb values + nb + 1 flags
    return 2 * nb + ceil_div((nb + 1) * int64_t(sizeof(uint32_t)), int64_t(sizeof(T))) + 1;
}

// Exclusive scan of xf(in[i]) (integer T, one pass): out[i] = sum_{j<i} xf(in[j]).
// flags_zeroed: the caller already zeroed scan_flags(partials, n) earlier on
// the stream (e.g. beside other resets), so the scan follows its producer
// directly.
template <typename T>
static void *scan_flags(T *partials, int64_t n, size_t *bytes) {
    const int64_t nb = ceil_div(n, kScanChunk);
    *bytes = size_t(nb + 1) * sizeof(uint32_t);
    return partials + 2 * nb;
}

// pdl: launched as a programmatic dependent of the kernel before it on s
// (the kernel waits for that grid before its first access).
template <typename T, typename In, typename Xf>
static void device_excl_scan_xf(const In *in, T *out, int64_t n, T *partials, T *total, Xf xf,
                                cudaStream_t s, bool flags_zeroed = false, bool pdl = false) {
    static_assert(is_exact_scan<T>::value, "the transformed scan is the one-pass form");
    const int64_t nb = ceil_div(n, kScanChunk);
    if (nb == 0) {
        cudaMemsetAsync(total, 0, sizeof(T), s);
        return;
    }
    if (!flags_zeroed) cudaMemsetAsync(partials + 2 * nb, 0, size_t(nb + 1) * sizeof(uint32_t), s);
    if (pdl && flags_zeroed) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)nb);
        cfg.blockDim = dim3(kScanThreads);
        cfg.stream = s;
        cudaLaunchAttribute at1[1];
        at1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at1[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at1;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, scan_onepass_kernel<T, In, Xf>, in, n, out, partials, nb, total,
                           xf);
        return;
    }
    scan_onepass_kernel<T, In, Xf><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, out, partials, nb,
                                                                        total, xf);
}

// Exclusive scan of n elements (in may equal out).  partials must hold
// scan_partials_len(n) elements; *total (device) receives the sum.  Integer
// types: one pass (a flag reset and one kernel); floating: three passes.
template <typename T>
static void device_excl_scan(const T *in, T *out, int64_t n, T *partials, T *total,
                             cudaStream_t s) {
    const int64_t nb = ceil_div(n, kScanChunk);
    if (nb == 0) {
        cudaMemsetAsync(total, 0, sizeof(T), s);
        return;
    }
    if constexpr (is_exact_scan<T>::value) {
        cudaMemsetAsync(partials + 2 * nb, 0, size_t(nb + 1) * sizeof(uint32_t), s);
        scan_onepass_kernel<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, out, partials, nb,
                                                                    total);
        return;
    }
    scan_reduce_kernel<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partials);
    scan_partials_kernel<T><<<1, kScanThreads, 0, s>>>(partials, nb, total);
    scan_down_kernel<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partials, out);
}

}  // namespace bvp
