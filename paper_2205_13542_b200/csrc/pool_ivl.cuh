// pool_ivl.cuh -- the fast (fp32-accumulating) interval-reduction kernel over
// the chunk schedule (work.cu), sm_100a.
//
// Restates the reference's interval_reduce (_kernels.py:22-63): fast mode
// (fp32 accumulation; tolerance 1e-5 against the fp64 reference) and, with
// EXACT, the bit-exact fp64 mode (whole intervals here, the intervals longer
// than a chunk in order by pool_exact_long_kernel, pool_kernel.cuh).
//
// Design (measured, profiles/ + scripts/gather_mlp_bench.cu): the path is a
// gather of 320-byte feature rows from an L2-resident table; B200 sustains
// ~13.6 TB/s of such gathers when every SM keeps enough rows in flight and
// each warp instruction carries several points.  So:
//   * a warp is G = 32 / L lane groups; group g owns ONE chunk (<= chunk
//     consecutive sorted points of one interval) and walks it sequentially,
//     its L lanes holding CPL VEC-wide slices of the channel row (C = 80
//     fp32: L = 4 lanes x 5 float4, 8 chunks = 8 points per warp step);
//   * chunks come longest first, so the 8 groups of a warp finish together;
//   * no cross-group combine, no shared memory, ~60 registers: 32 warps per
//     SM keep ~256 rows in flight;
//   * chunks of equal length stay in cell order (work.cu), so a warp's
//     groups store to neighbouring cells; a chunk that is a whole interval
//     stores its cell's column; chunks of a longer interval store fp32
//     partials that pool_ivl_combine_kernel adds in chunk order --
//     deterministic, independent of timing and launch shape;
//   * the map is zero-filled first (cudaMemsetAsync) so the scattered column
//     stores hit valid L2 lines.  Measured alternatives, both slower: zeroing
//     only the empty cells in-kernel (+15 us, partial-sector write misses),
//     combining split intervals in the last-finishing chunk (+14 us), and
//     walking intervals longer than a chunk with a whole warp (8 slices,
//     butterfly combine; +9 us).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "pool_kernel.cuh"
#include "pool_ref.cuh"

namespace bvp {

constexpr uint32_t kIvlSplit = 0x80000000u;  // work.cu kSplitDest

// A row chunk as loaded (packed) and its fp32 unpacking.
template <typename Elem, int VEC>
struct RawChunk;
template <>
struct RawChunk<float, 4> {
    using type = float4;
    template <bool STREAM>
    __device__ __forceinline__ static float4 load(const float *p) {
        return STREAM ? ldg_stream_f4(p) : ldg_f4(p);
    }
    __device__ __forceinline__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
    __device__ __forceinline__ static void unpack(const float4 &t, float (&v)[4]) {
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
};
template <>
struct RawChunk<float, 1> {
    using type = float;
    template <bool STREAM>
    __device__ __forceinline__ static float load(const float *p) { return __ldg(p); }
    __device__ __forceinline__ static float zero() { return 0.f; }
    __device__ __forceinline__ static void unpack(float t, float (&v)[1]) { v[0] = t; }
};
template <>
struct RawChunk<__nv_bfloat16, 8> {
    using type = uint4;
    template <bool STREAM>
    __device__ __forceinline__ static uint4 load(const __nv_bfloat16 *p) {
        return __ldg(reinterpret_cast<const uint4 *>(p));
    }
    __device__ __forceinline__ static uint4 zero() { return make_uint4(0u, 0u, 0u, 0u); }
    __device__ __forceinline__ static void unpack(const uint4 &t, float (&v)[8]) {
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
};
template <>
struct RawChunk<__nv_bfloat16, 1> {
    using type = float;
    template <bool STREAM>
    __device__ __forceinline__ static float load(const __nv_bfloat16 *p) { return __bfloat162float(p[0]); }
    __device__ __forceinline__ static float zero() { return 0.f; }
    __device__ __forceinline__ static void unpack(float t, float (&v)[1]) { v[0] = t; }
};
#ifndef BVP_IVL_MIN_BLOCKS
#define BVP_IVL_MIN_BLOCKS 3
#endif

// Accumulation of one point into a lane's channel slices.  EXACT: fp64, the
// fp32 x fp32 product exact, one rounding per add -- the reference's
// arithmetic, so a chunk that is a whole interval reproduces its sum bit for
// bit.
template <bool EXACT, int CPL, int VEC, bool IS_MAX, bool ARG>
__device__ __forceinline__ void ivl_acc(std::conditional_t<EXACT, double, float> (&acc)[CPL][VEC],
                                        uint32_t (&arg)[ARG ? CPL : 1][ARG ? VEC : 1],
                                        uint32_t j, float w, const float (&v)[CPL][VEC]) {
    if constexpr (!EXACT) {
        gacc<CPL, VEC, IS_MAX, ARG>(acc, arg, j, true, w, v);
        return;
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
        for (int x = 0; x < VEC; ++x) {
            const double pv = double(w) * double(v[k][x]);
            if (IS_MAX) {
                if (pv > acc[k][x]) {
                    acc[k][x] = pv;
                    if (ARG) arg[ARG ? k : 0][ARG ? x : 0] = j;
                }
            } else {
                acc[k][x] += pv;
            }
        }
}

template <typename Elem, int VEC, int CPL, bool IS_MAX, int SRC, bool ARG = IS_MAX,
          bool EXACT = false>
__global__ void __launch_bounds__(kPoolThreads, EXACT ? 2
                                                : sizeof(Elem) == 2 ? BVP_IVL_MIN_BLOCKS + 1
                                                                    : BVP_IVL_MIN_BLOCKS)
pool_ivl_kernel(const PoolParams P, int L, int lg) {
    using Acc = std::conditional_t<EXACT, double, float>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.y;
    const int C = P.C;
    const int G = 32 >> lg;
    const int g = lane >> lg, li = lane & (L - 1);
    const int nch = C / VEC;
    uint32_t live = 0;  // bit k: chunk li + k*L exists
#pragma unroll
    for (int k = 0; k < CPL; ++k)
        if (li + k * L < nch) live |= 1u << k;
    const Elem *rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride + li * VEC;
    const float *wdist = static_cast<const float *>(P.wsrc) + (SRC == kSrcDist ? b * P.w_bstride : 0);
    const uint32_t Cu = static_cast<uint32_t>(C);
    const int64_t n_work = P.work_counts[0];
    const int64_t n_part = P.max_splits > 0 ? P.work_counts[2] : 0;
    const int64_t nwarps = int64_t(gridDim.x) * kPoolWarps;

    auto rec_of = [&](uint32_t j) -> uint2 {
        if (SRC == kSrcX) return make_uint2(__ldg(P.ranks + j), 0u);
        return __ldg(P.meta + j);
    };

#pragma unroll 1
    for (int64_t batch = int64_t(blockIdx.x) * kPoolWarps + warp; batch * G < n_work;
         batch += nwarps) {
        const int64_t item = batch * G + g;
        uint4 r = make_uint4(0u, 0u, 0u, 0u);
        if (item < n_work) r = __ldg(P.work + item);
        const uint32_t j0 = r.x;
        // EXACT: chunks of split intervals belong to pool_exact_long_kernel
        const uint32_t len = (EXACT && (r.z & kIvlSplit)) ? 0u : r.y - r.x;
        uint32_t steps = len;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) steps = max(steps, __shfl_xor_sync(0xFFFFFFFFu, steps, o));

        Acc acc[CPL][VEC];
        uint32_t arg[ARG ? CPL : 1][ARG ? VEC : 1];
#pragma unroll
        for (int k = 0; k < CPL; ++k)
#pragma unroll
            for (int x = 0; x < VEC; ++x) {
                acc[k][x] = IS_MAX ? Acc(-INFINITY) : Acc(0);
                if (ARG) arg[ARG ? k : 0][ARG ? x : 0] = 0xFFFFFFFFu;
            }
        // rows of two steps in flight: fetch(s + 1) is issued before the
        // FMAs of step s; each fetch also loads the next step's record
        uint2 m = len > 0 ? rec_of(j0) : make_uint2(0u, 0u);
        // rows stay packed (bf16: 4 registers per 8 values) until the FMAs
        using Raw = typename RawChunk<Elem, VEC>::type;
        auto fetch = [&](uint32_t s, float &w, Raw (&v)[CPL]) {
            const bool ok = s < len;
            w = 1.f;
            if (SRC == kSrcDist) w = ok ? __ldg(wdist + m.y) : 0.f;
            const Elem *rp = rows + m.x * Cu;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                if (k == 0 || ((live >> k) & 1u))
                    v[k] = RawChunk<Elem, VEC>::template load<SRC == kSrcX>(rp + k * L * VEC);
                else v[k] = RawChunk<Elem, VEC>::zero();
            }
            if (s + 1 < len) m = rec_of(j0 + s + 1);
        };
        auto consume = [&](uint32_t j, float w, const Raw (&raw)[CPL]) {
            float v[CPL][VEC];
#pragma unroll
            for (int k = 0; k < CPL; ++k) RawChunk<Elem, VEC>::unpack(raw[k], v[k]);
            ivl_acc<EXACT, CPL, VEC, IS_MAX, ARG>(acc, arg, j, w, v);
        };
        float wa, wb;
        Raw va[CPL], vb[CPL];
        if (steps > 0) fetch(0, wa, va);
#pragma unroll 1
        for (uint32_t s = 0; s < steps; s += 2) {
            if (s + 1 < steps) fetch(s + 1, wb, vb);
            if (s < len) consume(j0 + s, wa, va);
            if (s + 1 >= steps) break;
            if (s + 2 < steps) fetch(s + 2, wa, va);
            if (s + 1 < len) consume(j0 + s + 1, wb, vb);
        }
        if (item >= n_work || (EXACT && (r.z & kIvlSplit))) continue;
        if (!(r.z & kIvlSplit)) {  // the chunk is the whole interval: store its cell
            const Acc inv = P.mean ? Acc(1) / Acc(len) : Acc(1);
            float *out = P.out + int64_t(b) * C * P.n_cells + r.z;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int ch = li + k * L;
                if (ch < nch)
#pragma unroll
                    for (int x = 0; x < VEC; ++x) {
                        const int c = ch * VEC + x;
                        out[int64_t(c) * P.n_cells] = static_cast<float>(
                            P.mean == 2 ? acc[k][x] / Acc(len) : acc[k][x] * inv);
                        if (ARG && P.argmax)
                            P.argmax[(b * P.n_int_max + r.w) * C + c] =
                                __ldg(P.ranks + arg[ARG ? k : 0][ARG ? x : 0]);
                    }
            }
        } else {  // one chunk of a split interval: its partial
            const int64_t slot = int64_t(b) * n_part + (r.z & ~kIvlSplit);
            float *pp = P.partials + slot * C;
            uint32_t *pa = ARG ? P.partial_arg + slot * C : nullptr;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
                const int ch = li + k * L;
                if (ch < nch)
#pragma unroll
                    for (int x = 0; x < VEC; ++x) {
                        pp[ch * VEC + x] = static_cast<float>(acc[k][x]);
                        if (ARG) pa[ch * VEC + x] = arg[ARG ? k : 0][ARG ? x : 0];
                    }
            }
        }
    }
}

// One thread per (split interval, channel): add the interval's chunk
// partials in chunk order (MAX: the first maximum in rank order), scale
// (MEAN), store the cell's value.  Loads of up to 8 chunks are issued before
// the in-order adds, so a thread waits ~2 memory latencies, not one per chunk.
template <bool IS_MAX, bool ARG = IS_MAX>
__global__ void __launch_bounds__(kPoolThreads)
pool_ivl_combine_kernel(const PoolParams P) {
    const int b = blockIdx.y;
    const int C = P.C;
    const int64_t n_split = P.work_counts[1], n_part = P.work_counts[2];
    const int64_t total = n_split * C;
#pragma unroll 1
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = e / C;
        const int c = static_cast<int>(e - s * C);
        const uint4 sp = __ldg(P.splits + s);  // interval, cell, first slot, chunks
        const float *pp = P.partials + (int64_t(b) * n_part + sp.z) * C + c;
        const uint32_t *pa = ARG ? P.partial_arg + (int64_t(b) * n_part + sp.z) * C + c : nullptr;
        float v = 0.f;
        uint32_t a = 0u;
        for (uint32_t k0 = 0; k0 < sp.w; k0 += 8) {
            float x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = k0 + q < sp.w ? pp[int64_t(k0 + q) * C] : 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (k0 + q >= sp.w) break;
                if (IS_MAX) {
                    if (k0 + q == 0 || x[q] > v) {
                        v = x[q];
                        if (ARG) a = pa[int64_t(k0 + q) * C];
                    }
                } else {
                    v = (k0 + q == 0) ? x[q] : v + x[q];
                }
            }
        }
        float inv = 1.f;
        if (P.mean) inv = 1.f / float(__ldg(P.starts + sp.x + 1) - __ldg(P.starts + sp.x));
        P.out[int64_t(b) * C * P.n_cells + int64_t(c) * P.n_cells + sp.y] = v * inv;
        if (ARG && P.argmax) P.argmax[(b * P.n_int_max + sp.x) * C + c] = __ldg(P.ranks + a);
    }
}

// Zero fill of the map's EMPTY cells only (cell_first[c] == cell_first[c+1]),
// on a side stream beside the chunk kernel: no interval writes those cells, so
// the two need no ordering, and the fill's HBM writes overlap the chunk
// kernel's L2-bound gathers instead of preceding them (a full memset of the
// 41.5 MB map is ~8 us in front of the reduction at config S).  128 threads
// at <= 32 registers: one block per SM fits beside the chunk kernel's three
// (3 x 256 threads x 80 registers of 64 K).  Consecutive warps take
// neighbouring 32-cell groups of one 16-channel slab, so the masked stores of
// a slab stream through DRAM pages in order.
constexpr int kZeroThreads = 128;
static __global__ void __launch_bounds__(kZeroThreads, 16)
zero_empty_cells_kernel(const uint32_t *__restrict__ cell_first, int64_t n_cells, int C, int B,
                        float *__restrict__ out) {
    constexpr int kCh = 16;
    const int64_t groups = (n_cells + 31) / 32;
    const int nchg = (C + kCh - 1) / kCh;
    const int64_t items = groups * nchg * B;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t(gridDim.x) * kZeroThreads) >> 5;
#pragma unroll 1
    for (int64_t it = (int64_t(blockIdx.x) * kZeroThreads + threadIdx.x) >> 5; it < items;
         it += nw) {
        const int64_t grp = it % groups, rest = it / groups;
        const int chg = static_cast<int>(rest % nchg), b = static_cast<int>(rest / nchg);
        const int64_t c = grp * 32 + lane;
        const bool empty = c < n_cells && __ldg(cell_first + c) == __ldg(cell_first + c + 1);
        if (!__any_sync(0xFFFFFFFFu, empty)) continue;
        float *o = out + (int64_t(b) * C + chg * kCh) * n_cells + c;
        const int ce = min(kCh, C - chg * kCh);
#pragma unroll 4
        for (int k = 0; k < ce; ++k)
            if (empty) o[int64_t(k) * n_cells] = 0.f;
    }
}

// Bytes of the split partials for B samples of C channels (values, + the
// argmax positions for MAX).
inline size_t ivl_scratch_bytes(int64_t n_partials, int B, int C, bool is_max) {
    return size_t(B) * n_partials * C * (is_max ? 8 : 4);
}

// Zero-fill + chunk kernel + combine.  BVP_ERR_UNSUPPORTED: shape not covered
// (the caller falls back).
// EXACT: fp64 accumulation; chunks that are whole intervals here, the split
// intervals (longer than a chunk) walked in order by pool_exact_long_kernel
// on a forked stream -- every cell bit-identical to the reference.
template <typename Elem, int VEC, int SRC, bool EXACT = false>
int run_pool_ivl(const PoolParams &p0, int B, bool is_max, cudaStream_t s) {
    void *scratch = p0.scratch;
    const size_t scratch_bytes = p0.scratch_bytes;
    int L, lg, cpl;
    if (!p0.work || !choose_group(p0.C / VEC, VEC, L, lg, cpl)) return BVP_ERR_UNSUPPORTED;
    BVP_REQUIRE(SRC == kSrcX || p0.meta, BVP_ERR_INVALID,
                "the cache's point gather table (point_meta) is required");
    const size_t need =
        EXACT ? 0 : ivl_scratch_bytes(p0.max_splits > 0 ? p0.chunk_partials : 0, B, p0.C, is_max);
    BVP_REQUIRE(scratch_bytes >= need, BVP_ERR_INVALID,
                "pool scratch too small: need %zu bytes (bvp_pool_scratch_bytes)", need);
    PoolParams p = p0;
    p.partials = static_cast<float *>(scratch);
    const bool arg = is_max && p0.argmax;  // MAX winners only for autograd
    p.partial_arg = arg && !EXACT ? reinterpret_cast<uint32_t *>(static_cast<float *>(scratch) +
                                                                 size_t(B) * p0.chunk_partials * p0.C)
                                  : nullptr;
    // the scattered column stores need a zero-filled map
    if (!p.out_zeroed) cudaMemsetAsync(p.out, 0, size_t(B) * p.C * p.n_cells * sizeof(float), s);
    const int G = 32 >> lg;
    const int64_t batches = ceil_div(p.max_work, G);
    const dim3 grid(static_cast<unsigned>(std::max<int64_t>(
                        1, std::min<int64_t>(ceil_div(batches, kPoolWarps),
                                             int64_t(kNumSms) * BVP_IVL_MIN_BLOCKS * 4))),
                    static_cast<unsigned>(B));
    SideFork fork(s);
    if (EXACT && p.max_splits > 0) {  // the split intervals, in order, meanwhile
        auto ke = is_max ? pool_exact_long_kernel<VEC, true, true>
                         : pool_exact_long_kernel<VEC, false, true>;
        const int T = std::min(128, kExactTile / p.C);
        const size_t esmem = size_t(T) * (p.C + 1) * sizeof(float);
        if (esmem > 48 * 1024)
            cudaFuncSetAttribute(ke, cudaFuncAttributeMaxDynamicSharedMemorySize, int(esmem));
        ke<<<dim3(static_cast<unsigned>(p.max_splits), static_cast<unsigned>(B)), kPoolThreads,
             esmem, fork.side>>>(p);
    }
#define BVP_IVL_LAUNCH(CPLV)                                                          \
    if (cpl == CPLV) {                                                                \
        auto k = !is_max ? pool_ivl_kernel<Elem, VEC, CPLV, false, SRC, false, EXACT> \
                 : arg   ? pool_ivl_kernel<Elem, VEC, CPLV, true, SRC, true, EXACT>   \
                         : pool_ivl_kernel<Elem, VEC, CPLV, true, SRC, false, EXACT>; \
        k<<<grid, kPoolThreads, 0, s>>>(p, L, lg);                                    \
    }
    BVP_IVL_LAUNCH(1) BVP_IVL_LAUNCH(2) BVP_IVL_LAUNCH(3)
    BVP_IVL_LAUNCH(4) BVP_IVL_LAUNCH(5) BVP_IVL_LAUNCH(6)
#undef BVP_IVL_LAUNCH
    fork.join();
    if (!EXACT && p.max_splits > 0) {
        const dim3 cg(static_cast<unsigned>(std::max<int64_t>(
                          1, std::min<int64_t>(ceil_div(p.max_splits * p.C, kPoolThreads),
                                               kNumSms * 16))),
                      static_cast<unsigned>(B));
        if (arg) pool_ivl_combine_kernel<true, true><<<cg, kPoolThreads, 0, s>>>(p);
        else if (is_max) pool_ivl_combine_kernel<true, false><<<cg, kPoolThreads, 0, s>>>(p);
        else pool_ivl_combine_kernel<false><<<cg, kPoolThreads, 0, s>>>(p);
    }
    return BVP_OK;
}

// Fast-mode dispatch: the chunk kernel when the cache carries a chunk
// schedule and a lane layout fits C, else the reference-order kernel
// (pool_ref.cuh).
template <typename Elem, int VEC, int SRC>
int run_pool_fast(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    const int rc = run_pool_ivl<Elem, VEC, SRC>(p, B, is_max, s);
    if (rc != BVP_ERR_UNSUPPORTED) return rc;
    return run_pool_ref<Elem, SRC>(p, B, is_max, s);  // channel widths the chunk kernel lacks
}

}  // namespace bvp
