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
    const uint32_t *units;       // work units: (first cell, cell count | long flag)
    const uint2 *meta;           // per sorted point: (feature row, weight index)
    const uint32_t *long_units;  // indices of the long (split) units
    const int64_t *sched_counts; // device: n_units, n_long
    float *out;              // (B, C, n_cells)
    uint32_t *argmax;        // MAX only, optional: (B, n_int_max, C)
    int C, D, HW, NHW;
    int mean;
    int nx, ny;
    int64_t n_cells, n_int_max;
    int64_t max_units, max_long;  // launch sizes (>= the device counts)
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

// Walk the sorted points [a, e) in rank order, calling f(jj, w, v) for each
// with the point's weight and this lane's CH x VEC slice of its row.  Gather
// records are read 32 at a time, one per lane, two blocks ahead; the block's
// weights one block ahead; rows one step (U points) ahead into a register
// double buffer -- so a step costs issue time, not a memory latency.
template <typename Elem, int VEC, int CH, int SRC, typename F>
__device__ __forceinline__ void warp_walk(const PoolParams &P, int b, const Elem *rows, uint32_t a,
                                          uint32_t e, F &&f) {
    constexpr int U = CH == 1 ? 4 : (CH == 2 ? 2 : 1);
    constexpr int STEPS = 32 / U;
    const int lane = threadIdx.x & 31;
    const int C = P.C;
    const int nchunks = C / VEC;
    auto rec_of = [&](uint32_t j) {
        return j < e ? point_record<SRC>(P, j) : make_uint2(0u, 0u);
    };
    uint32_t jb = a;
    uint2 r0 = rec_of(jb + lane);
    uint2 r1 = rec_of(jb + 32 + lane);
    float w0 = (jb + lane < e) ? point_weight<SRC>(P, b, r0) : 0.f;
    float v[2][U][CH][VEC];
    // rows of step s of the block whose records are `r` (block start jbb)
    auto issue = [&](int buf, int s, uint2 r, uint32_t jbb) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t rx = __shfl_sync(0xFFFFFFFFu, r.x, s * U + u);
            const bool ok = jbb + s * U + u < e;
            const Elem *rp = rows + size_t(rx) * C;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int ch = lane + 32 * q;
                if (ok && ch < nchunks) {
                    Loader<Elem, VEC>::template load<SRC == kSrcX>(rp + ch * VEC, v[buf][u][q]);
                } else {
#pragma unroll
                    for (int k = 0; k < VEC; ++k) v[buf][u][q][k] = 0.f;
                }
            }
        }
    };
    issue(0, 0, r0, jb);
#pragma unroll 1
    for (; jb < e; jb += 32) {
        const uint2 r2 = rec_of(jb + 64 + lane);
        const float w1 = (jb + 32 + lane < e) ? point_weight<SRC>(P, b, r1) : 0.f;
#pragma unroll
        for (int s = 0; s < STEPS; ++s) {
            if (jb + s * U >= e) break;  // warp-uniform
            if (s + 1 < STEPS) {
                if (jb + (s + 1) * U < e) issue((s + 1) & 1, s + 1, r0, jb);
            } else if (jb + 32 < e) {
                issue(0, 0, r1, jb + 32);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t jj = jb + s * U + u;
                const float w = __shfl_sync(0xFFFFFFFFu, w0, s * U + u);
                if (jj < e) f(jj, w, v[s & 1][u]);
            }
        }
        r0 = r1;
        r1 = r2;
        w0 = w1;
    }
}

template <typename Acc, int CH, int VEC, bool IS_MAX>
__device__ __forceinline__ void acc_point(Acc (&acc)[CH][VEC],
                                          uint32_t (&arg)[IS_MAX ? CH : 1][IS_MAX ? VEC : 1],
                                          uint32_t jj, float w, const float (&v)[CH][VEC]) {
#pragma unroll
    for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            if (IS_MAX) {
                const Acc pv = Acc(w) * Acc(v[q][k]);
                if (pv > acc[q][k]) {
                    acc[q][k] = pv;
                    arg[IS_MAX ? q : 0][IS_MAX ? k : 0] = jj;  // sorted position
                }
            } else {
                acc[q][k] += Acc(w) * Acc(v[q][k]);
            }
        }
}

constexpr uint32_t kLongUnit = 0x80000000u;  // unit flag: split by pool_long_kernel

// One warp per work unit.  SPLIT: units flagged long are left to
// pool_long_kernel (fast mode); the exact mode walks them here, in order.
template <typename Acc, typename Elem, int VEC, int CH, bool IS_MAX, int SRC, bool SPLIT>
__global__ void __launch_bounds__(kPoolThreads)
pool_stream_kernel(const PoolParams P) {
    extern __shared__ float s_all[];  // per warp: [C][kUnitPitch]
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int C = P.C;
    const int nchunks = C / VEC;
    const int b = blockIdx.y;
    float *s_tile = s_all + warp * C * kUnitPitch;

    const int64_t k = int64_t(blockIdx.x) * kPoolWarps + warp;
    if (k >= P.sched_counts[0]) return;
    const int64_t cell0 = __ldg(P.units + 2 * k);
    const uint32_t word = __ldg(P.units + 2 * k + 1);
    if (SPLIT && (word & kLongUnit)) return;
    const int ncell = static_cast<int>(word & 0xFFu);
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
    if (J1 > J0) {
        warp_walk<Elem, VEC, CH, SRC>(P, b, rows, J0, J1,
                                      [&](uint32_t jj, float w, const float (&v)[CH][VEC]) {
            if (jj == hi) {  // interval boundary (warp-uniform)
                park();
                reset();
                ++iv;
                lo = hi;
                hi = __ldg(P.starts + iv + 1);
            }
            acc_point<Acc, CH, VEC, IS_MAX>(acc, arg, jj, w, v);
        });
        park();
    }
    __syncwarp();
    float *out = P.out + int64_t(b) * C * P.n_cells + cell0;
    for (int idx = lane; idx < C * ncell; idx += 32) {
        const int c = idx / ncell, x = idx - c * ncell;
        out[int64_t(c) * P.n_cells + x] = ((has >> x) & 1u) ? s_tile[c * kUnitPitch + x] : 0.f;
    }
}

// Fast mode: one CTA per heavy cell (a single interval above the unit point
// budget).  Its 8 warps walk equal slices of the interval; the slices'
// partial results are combined in slice order in shared memory, so the sum
// is deterministic and the heavy cell no longer sets the kernel's critical
// path.
template <typename Elem, int VEC, int CH, bool IS_MAX, int SRC>
__global__ void __launch_bounds__(kPoolThreads)
pool_long_kernel(const PoolParams P) {
    extern __shared__ float s_all[];  // [kPoolWarps][C] values + [kPoolWarps][C] argmax
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int C = P.C;
    const int nchunks = C / VEC;
    const int b = blockIdx.y;
    if (int64_t(blockIdx.x) >= P.sched_counts[1]) return;
    const uint32_t k = __ldg(P.long_units + blockIdx.x);
    const int64_t cell = __ldg(P.units + 2 * size_t(k));
    const uint32_t iv = __ldg(P.cell_first + cell);
    const uint32_t lo = __ldg(P.starts + iv), hi = __ldg(P.starts + iv + 1);
    const uint32_t L = hi - lo;
    const uint32_t a = lo + uint32_t(uint64_t(L) * warp / kPoolWarps);
    const uint32_t e = lo + uint32_t(uint64_t(L) * (warp + 1) / kPoolWarps);
    const Elem *rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride;
    float acc[CH][VEC];
    uint32_t arg[IS_MAX ? CH : 1][IS_MAX ? VEC : 1];
#pragma unroll
    for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int x = 0; x < VEC; ++x) {
            acc[q][x] = IS_MAX ? -INFINITY : 0.f;
            if (IS_MAX) arg[IS_MAX ? q : 0][IS_MAX ? x : 0] = kNone;
        }
    if (e > a)
        warp_walk<Elem, VEC, CH, SRC>(P, b, rows, a, e,
                                      [&](uint32_t jj, float w, const float (&v)[CH][VEC]) {
            acc_point<float, CH, VEC, IS_MAX>(acc, arg, jj, w, v);
        });
    float *s_val = s_all;
    uint32_t *s_arg = reinterpret_cast<uint32_t *>(s_all + kPoolWarps * C);
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int ch = lane + 32 * q;
        if (ch < nchunks)
#pragma unroll
            for (int x = 0; x < VEC; ++x) {
                s_val[warp * C + ch * VEC + x] = acc[q][x];
                if (IS_MAX) s_arg[warp * C + ch * VEC + x] = arg[IS_MAX ? q : 0][IS_MAX ? x : 0];
            }
    }
    __syncthreads();
    float *out = P.out + int64_t(b) * C * P.n_cells + cell;
    const float inv = P.mean ? 1.f / float(L) : 1.f;
    for (int c = threadIdx.x; c < C; c += kPoolThreads) {
        float run = s_val[c];
        uint32_t ra = IS_MAX ? s_arg[c] : 0u;
        for (int wv = 1; wv < kPoolWarps; ++wv) {
            const float x = s_val[wv * C + c];
            if (IS_MAX) {
                const uint32_t xa = s_arg[wv * C + c];
                if (x > run || (x == run && xa < ra)) {
                    run = x;
                    ra = xa;
                }
            } else {
                run += x;
            }
        }
        out[int64_t(c) * P.n_cells] = run * inv;
        if (IS_MAX && P.argmax) P.argmax[(b * P.n_int_max + iv) * C + c] = __ldg(P.ranks + ra);
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
                            const uint32_t *cell_first, const bvp_schedule *sched, int C, int nx,
                            int ny, float *out, int mode);
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
    // fast mode: heavy cells are split over a CTA by pool_long_kernel; the
    // exact mode must walk every interval in order and does not split
    constexpr bool kSplit = sizeof(Acc) == sizeof(float);
    const dim3 grid(static_cast<unsigned>(ceil_div(p.max_units, kPoolWarps)),
                    static_cast<unsigned>(B));
    const size_t lsmem = size_t(kPoolWarps) * p.C * 2 * sizeof(float);
#define BVP_LAUNCH_CH(CHV)                                                                   \
    if (ch == CHV) {                                                                         \
        auto k = is_max ? pool_stream_kernel<Acc, Elem, VEC, CHV, true, SRC, kSplit>         \
                        : pool_stream_kernel<Acc, Elem, VEC, CHV, false, SRC, kSplit>;       \
        if (smem > 48 * 1024)                                                                \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        k<<<grid, kPoolThreads, smem, s>>>(p);                                               \
        if (kSplit && p.max_long > 0) {                                                      \
            auto kl = is_max ? pool_long_kernel<Elem, VEC, CHV, true, SRC>                   \
                             : pool_long_kernel<Elem, VEC, CHV, false, SRC>;                 \
            if (lsmem > 48 * 1024)                                                           \
                cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                     int(lsmem));                                            \
            kl<<<dim3(static_cast<unsigned>(p.max_long), static_cast<unsigned>(B)),          \
                 kPoolThreads, lsmem, s>>>(p);                                               \
        }                                                                                    \
        return BVP_OK;                                                                       \
    }
    BVP_LAUNCH_CH(1) BVP_LAUNCH_CH(2) BVP_LAUNCH_CH(4) BVP_LAUNCH_CH(8)
#undef BVP_LAUNCH_CH
    set_error("no kernel instance for %d chunks per lane", ch);
    return BVP_ERR_UNSUPPORTED;
}

}  // namespace bvp
