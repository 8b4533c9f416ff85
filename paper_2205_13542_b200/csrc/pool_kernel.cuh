// pool_kernel.cuh -- the interval-reduction kernel (forward), sm_100a.
//
// Restates the reference's interval_reduce (_kernels.py:22-63).
//
// Work decomposition (the choice is measured):
//   * The cached schedule cuts the BEV grid into work UNITS: runs of at most
//     kUnitCells consecutive cells of one row holding at most a budget of
//     in-range points (a heavier single cell is a unit of its own).  A unit's
//     intervals occupy one contiguous range [J0, J1) of the rank-ordered
//     point stream.
//   * One WARP owns one unit and walks its point stream in rank order.  The
//     lanes span the channel row (16-byte chunks), so every point's row is
//     one coalesced warp load and interval boundaries are warp-uniform: the
//     accumulation is sequential in rank order per interval, exactly like the
//     reference.  With Acc = double the sums are therefore bit-identical to
//     interval_reduce (fp32 x fp32 products are exact in fp64); Acc = float is
//     the fast mode.
//   * Per point the warp reads a precomputed gather record (feature row,
//     weight index) -- no division in the loop -- and the next U rows are in
//     flight while the current U are accumulated (register double buffer).
//     The kernel is a gather from L2: it needs occupancy, so its footprint is
//     kept small (no per-lane shuffles, one small shared tile per warp).
//   * A finished interval is parked in the warp's shared [C][kUnitCells] tile;
//     the warp then writes its cells' output columns once -- zeros of empty
//     cells included -- so there is no memset and exactly one non-atomic store
//     per (channel, cell).
//
// Sources (SRC):
//   kSrcDist  : rows = NHWC features (f32), weight = dist[n,d,h,w] (f32)
//   kSrcX     : rows = materialised frustum x[p, :] (f32), weight = 1
//   kSrcFused : rows = NHWC context (bf16), weight = exp(logit - lse[pixel])
#pragma once

#include "common.cuh"

namespace bvp {

constexpr int kPoolWarps = 8;
constexpr int kPoolThreads = 32 * kPoolWarps;
constexpr int kUnitPitch = kUnitCells + 1;

enum { kSrcDist = 0, kSrcX = 1, kSrcFused = 2 };

struct PoolParams {
    const void *rows;        // f32 NHWC features | f32 x (P,C) | bf16 NHWC context
    const void *wsrc;        // f32 dist (N,D,H,W) | bf16 logits (N,D,H,W) | unused
    const float *lse;        // fused: per-pixel log-sum-exp (N,H,W)
    const uint32_t *ranks;
    const uint32_t *starts;  // n_int + 1 entries (sentinel = n_in)
    const uint32_t *icells;
    const uint32_t *cell_first;  // n_cells + 1: first interval with cell >= c
    const uint32_t *units;   // work units: (first cell, cell count) pairs
    const int64_t *n_units;  // device count of units
    const uint2 *meta;       // per sorted point: (feature row, weight index)
    float *out;              // (B, C, n_cells)
    uint32_t *argmax;        // MAX only, optional: (B, n_int_max, C)
    int C, D, HW, NHW;
    int mean;
    int nx, ny;
    int64_t n_cells, n_int_max;
    int64_t max_units;       // grid size (>= *n_units)
    int64_t rows_bstride;    // elements of rows per batch sample
    int64_t w_bstride;       // elements of wsrc per batch sample
};

template <typename Elem, int VEC>
struct Loader;

template <>
struct Loader<float, 4> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const float *p, float (&v)[4]) {
        const float4 t = STREAM ? ldg_stream_f4(p) : ldg_f4(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
};
template <>
struct Loader<float, 1> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const float *p, float (&v)[1]) { v[0] = __ldg(p); }
};
template <>
struct Loader<__nv_bfloat16, 8> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const __nv_bfloat16 *p, float (&v)[8]) {
        const uint4 t = __ldg(reinterpret_cast<const uint4 *>(p));
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
};
template <>
struct Loader<__nv_bfloat16, 1> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const __nv_bfloat16 *p, float (&v)[1]) {
        v[0] = __bfloat162float(p[0]);
    }
};

// Gather record of sorted point j: (feature row, weight index).
template <int SRC>
__device__ __forceinline__ uint2 point_record(const PoolParams &P, uint32_t j) {
    if (SRC == kSrcX) return make_uint2(__ldg(P.ranks + j), 0u);
    return __ldg(P.meta + j);
}

template <int SRC>
__device__ __forceinline__ float point_weight(const PoolParams &P, int b, uint2 m) {
    if (SRC == kSrcX) return 1.f;
    if (SRC == kSrcDist) return __ldg(static_cast<const float *>(P.wsrc) + b * P.w_bstride + m.y);
    const float l =
        __bfloat162float(static_cast<const __nv_bfloat16 *>(P.wsrc)[b * P.w_bstride + m.y]);
    return __expf(l - __ldg(P.lse + int64_t(b) * P.NHW + m.x));
}

// CH = 16-byte (VEC-element) chunks of the channel row per lane.
template <typename Acc, typename Elem, int VEC, int CH, bool IS_MAX, int SRC>
__global__ void __launch_bounds__(kPoolThreads)
pool_stream_kernel(const PoolParams P) {
    extern __shared__ float s_all[];  // per warp: [C][kUnitPitch]
    // rows per pipeline step (x2 buffers in registers)
    constexpr int U = CH == 1 ? 4 : (CH == 2 ? 2 : 1);
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int C = P.C;
    const int nchunks = C / VEC;
    const int b = blockIdx.y;
    float *s_tile = s_all + warp * C * kUnitPitch;

    const int64_t k = int64_t(blockIdx.x) * kPoolWarps + warp;
    if (k >= *P.n_units) return;
    const int64_t cell0 = __ldg(P.units + 2 * k);
    const int ncell = static_cast<int>(__ldg(P.units + 2 * k + 1));
    const uint32_t i0 = __ldg(P.cell_first + cell0), i1 = __ldg(P.cell_first + cell0 + ncell);
    const uint32_t J0 = __ldg(P.starts + i0), J1 = __ldg(P.starts + i1);
    // which of the unit's cells own an interval (bit x <-> cell0 + x)
    bool mine = false;
    if (lane < ncell)
        mine = __ldg(P.cell_first + cell0 + lane + 1) > __ldg(P.cell_first + cell0 + lane);
    const unsigned has = __ballot_sync(0xFFFFFFFFu, mine);

    const Elem *rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride;
    Acc acc[CH][VEC];
    uint32_t arg[IS_MAX ? CH : 1][IS_MAX ? VEC : 1];
    auto reset = [&]() {
#pragma unroll
        for (int q = 0; q < CH; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                acc[q][e] = IS_MAX ? Acc(-INFINITY) : Acc(0);
                if (IS_MAX) arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = kNone;
            }
    };
    uint32_t iv = i0, lo = J0, hi = __ldg(P.starts + i0 + 1);
    auto park = [&]() {  // interval iv = [lo, hi) complete
        const int lc = static_cast<int>(int64_t(__ldg(P.icells + iv)) - cell0);
        const Acc inv = P.mean ? Acc(1) / Acc(hi - lo) : Acc(1);
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int ch = lane + 32 * q;
            if (ch < nchunks)
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const int c = ch * VEC + e;
                    const Acc r = P.mean ? acc[q][e] * inv : acc[q][e];
                    s_tile[c * kUnitPitch + lc] = static_cast<float>(r);
                    if (IS_MAX && P.argmax)
                        P.argmax[(b * P.n_int_max + iv) * C + c] =
                            __ldg(P.ranks + arg[IS_MAX ? q : 0][IS_MAX ? e : 0]);
                }
        }
    };
    reset();

    // software pipeline: rows of step t+1 are in flight while step t is summed
    float v[2][U][CH][VEC];
    float w[2][U];
    uint2 mrec[U];
    auto issue = [&](int buf, uint32_t j) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = j + u < J1;
            w[buf][u] = ok ? point_weight<SRC>(P, b, mrec[u]) : 0.f;
            const Elem *rp = rows + size_t(mrec[u].x) * C;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int ch = lane + 32 * q;
                if (ok && ch < nchunks) {
                    Loader<Elem, VEC>::template load<SRC == kSrcX>(rp + ch * VEC, v[buf][u][q]);
                } else {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) v[buf][u][q][e] = 0.f;
                }
            }
        }
    };
    auto fetch_rec = [&](uint32_t j) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            mrec[u] = (j + u < J1) ? point_record<SRC>(P, j + u) : make_uint2(0u, 0u);
    };

    // accumulate step j out of buffer CUR (compile-time, so v stays in registers)
    auto consume = [&](auto cur_c, uint32_t j) {
        constexpr int cur = decltype(cur_c)::value;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t jj = j + u;
            if (jj < J1) {
                if (jj == hi) {  // interval boundary (warp-uniform)
                    park();
                    reset();
                    ++iv;
                    lo = hi;
                    hi = __ldg(P.starts + iv + 1);
                }
#pragma unroll
                for (int q = 0; q < CH; ++q)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        if (IS_MAX) {
                            const Acc pv = Acc(w[cur][u]) * Acc(v[cur][u][q][e]);
                            if (pv > acc[q][e]) {
                                acc[q][e] = pv;
                                arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = jj;
                            }
                        } else {
                            acc[q][e] += Acc(w[cur][u]) * Acc(v[cur][u][q][e]);
                        }
                    }
            }
        }
    };
    using B0 = std::integral_constant<int, 0>;
    using B1 = std::integral_constant<int, 1>;

    if (J1 > J0) {
        fetch_rec(J0);
        issue(0, J0);
        fetch_rec(J0 + U);
#pragma unroll 1
        for (uint32_t j = J0; j < J1; j += 2 * U) {
            if (j + U < J1) {  // warp-uniform
                issue(1, j + U);
                fetch_rec(j + 2 * U);
            }
            consume(B0{}, j);
            if (j + U >= J1) break;
            if (j + 2 * U < J1) {
                issue(0, j + 2 * U);
                fetch_rec(j + 3 * U);
            }
            consume(B1{}, j + U);
        }
        park();
    }
    __syncwarp();
    float *out = P.out + int64_t(b) * C * P.n_cells + cell0;
    for (int idx = lane; idx < C * ncell; idx += 32) {
        const int c = idx / ncell, x = idx - c * ncell;
        out[int64_t(c) * P.n_cells + x] = ((has >> x) & 1u) ? s_tile[c * kUnitPitch + x] : 0.f;
    }
}

// Channel chunks per lane for a row of `nchunks` VEC-element chunks.
inline int choose_ch(int nchunks) {
    for (int ch : {1, 2, 4, 8})
        if (32 * ch >= nchunks) return ch;
    return 0;
}

// pool.cu
PoolParams make_pool_params(const uint32_t *ranks, const uint32_t *starts, const uint32_t *icells,
                            const uint32_t *cell_first, const uint32_t *units,
                            const uint32_t *point_meta, const int64_t *n_units, int64_t max_units,
                            int C, int nx, int ny, float *out, int mode);
template <typename T>
void launch_to_nhwc(const T *src, int64_t NB, int A, int HW, T *dst, cudaStream_t s);

// Launch the instantiated kernel for (Acc, Elem, VEC, SRC) and the shape of
// p.C.  Defined (and explicitly instantiated) in the pool_*.cu / fused.cu
// translation units so the kernel families compile in parallel.
template <typename Acc, typename Elem, int VEC, int SRC>
int run_pool(const PoolParams &p, int B, bool is_max, cudaStream_t s);
#define BVP_DECLARE_RUN_POOL(A, E, V, S) \
    template <>                          \
    int run_pool<A, E, V, S>(const PoolParams &p, int B, bool is_max, cudaStream_t s);
BVP_DECLARE_RUN_POOL(float, float, 4, kSrcDist)          // pool_fast.cu
BVP_DECLARE_RUN_POOL(float, float, 1, kSrcDist)          // pool_fast.cu
BVP_DECLARE_RUN_POOL(double, float, 4, kSrcDist)         // pool_exact.cu
BVP_DECLARE_RUN_POOL(double, float, 1, kSrcDist)         // pool_exact.cu
BVP_DECLARE_RUN_POOL(float, float, 4, kSrcX)             // pool_x.cu
BVP_DECLARE_RUN_POOL(float, float, 1, kSrcX)             // pool_x.cu
BVP_DECLARE_RUN_POOL(float, __nv_bfloat16, 8, kSrcFused) // fused.cu
BVP_DECLARE_RUN_POOL(float, __nv_bfloat16, 1, kSrcFused) // fused.cu
#undef BVP_DECLARE_RUN_POOL

template <typename Acc, typename Elem, int VEC, int SRC>
int run_pool_impl(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    const int ch = choose_ch(p.C / VEC);
    BVP_REQUIRE(ch > 0, BVP_ERR_UNSUPPORTED, "channel count %d not supported (max %d)", p.C,
                256 * VEC);
    const size_t smem = size_t(kPoolWarps) * p.C * kUnitPitch * sizeof(float);
    BVP_REQUIRE(smem <= 227 * 1024, BVP_ERR_UNSUPPORTED, "channel count %d too large", p.C);
    BVP_REQUIRE(SRC == kSrcX || p.meta, BVP_ERR_INVALID,
                "the cache's point gather table (point_meta) is required");
    const dim3 grid(static_cast<unsigned>(ceil_div(p.max_units, kPoolWarps)),
                    static_cast<unsigned>(B));
#define BVP_LAUNCH_CH(CHV)                                                                   \
    if (ch == CHV) {                                                                         \
        auto k = is_max ? pool_stream_kernel<Acc, Elem, VEC, CHV, true, SRC>                 \
                        : pool_stream_kernel<Acc, Elem, VEC, CHV, false, SRC>;               \
        if (smem > 48 * 1024)                                                                \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        k<<<grid, kPoolThreads, smem, s>>>(p);                                               \
        return BVP_OK;                                                                       \
    }
    BVP_LAUNCH_CH(1) BVP_LAUNCH_CH(2) BVP_LAUNCH_CH(4) BVP_LAUNCH_CH(8)
#undef BVP_LAUNCH_CH
    set_error("no kernel instance for %d chunks per lane", ch);
    return BVP_ERR_UNSUPPORTED;
}

}  // namespace bvp
