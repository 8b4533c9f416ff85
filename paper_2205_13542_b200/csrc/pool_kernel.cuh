// pool_kernel.cuh -- the interval-reduction kernels (forward), sm_100a.
//
// Restates the reference's interval_reduce (_kernels.py:22-63).
//
// Work decomposition (measured; DESIGN.md §4 records the alternatives):
//   * The cached schedule (units.cu) cuts the BEV grid into UNITS -- runs of
//     at most kUnitCells consecutive cells of one row -- and groups
//     consecutive units into TASKS of about a fixed number of in-range
//     points.  Units and tasks are in cell order, so a task's intervals are
//     one contiguous range [J0, J1) of the rank-ordered point stream.
//   * One WARP walks one task's stream in rank order.  The lanes span the
//     channel row (16-byte chunks), so a point's row is one coalesced warp
//     load and interval boundaries are warp-uniform: every interval is
//     accumulated sequentially in rank order, exactly like the reference.
//     With Acc = double the sums are bit-identical to interval_reduce (fp32 x
//     fp32 products are exact in fp64); Acc = float is the fast mode.
//   * Gather records (feature row, weight index; precomputed per sorted point
//     so the loop never divides) are read 32 at a time, one per lane, two
//     blocks ahead; weights one block ahead; rows one 4-point step ahead into
//     a register double buffer.  Interval boundaries are tested once per
//     step; steps inside one interval take a branch-free path, and the next
//     interval's end and cell are prefetched.
//   * Finished intervals are parked in the warp's shared [C][kUnitCells] tile
//     of the current unit; when the stream leaves a unit the warp writes its
//     cells' output columns once -- zeros of empty cells included -- so there
//     is no memset and exactly one non-atomic store per (channel, cell).
//   * Fast mode only: a cell holding more points than the unit budget is a
//     "long" unit (its own task); pool_long_kernel splits it over the 8 warps
//     of a CTA and combines the slices in order in shared memory, so a heavy
//     cell does not set the kernel's critical path.
//
// Sources (SRC):
//   kSrcDist  : rows = NHWC features (f32), weight = dist[n,d,h,w] (f32)
//   kSrcX     : rows = materialised frustum x[p, :] (f32), weight = 1
//   kSrcFused : rows = NHWC context (bf16), weight = exp(logit - lse[pixel])
#pragma once

#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace bvp {

constexpr int kPoolWarps = 8;
constexpr int kPoolThreads = 32 * kPoolWarps;

// The interval kernels' map is zero-filled by a memset beside the feature
// staging (bvp_pool_prepare_f32) before their scattered column stores.
constexpr int kUnitPitch = kUnitCells + 1;
constexpr uint32_t kLongUnit = 0x80000000u;  // unit / task flag: split by pool_long_kernel

enum { kSrcDist = 0, kSrcX = 1, kSrcFused = 2 };

struct PoolParams {
    const void *rows;        // f32 NHWC features | f32 x (P,C) | bf16 NHWC context
    const void *wsrc;        // f32 dist (N,D,H,W) | bf16 logits (N,D,H,W) | unused
    const float *lse;        // fused: per-pixel log-sum-exp (N,H,W)
    const uint32_t *ranks;
    const uint32_t *starts;  // n_int + 1 entries (sentinel = n_in)
    const uint32_t *icells;
    const uint32_t *cell_first;  // n_cells + 1: first interval with cell >= c
    const uint32_t *units;       // (first cell, ncell | has << 8 | long flag)
    const uint2 *meta;           // per sorted point: (feature row, weight index)
    const uint32_t *long_units;  // indices of the long (split) units
    const uint4 *tasks;          // 2 x uint4 per task (units.cu)
    const int64_t *sched_counts; // device: n_units, n_long, n_tasks
    float *out;              // (B, C, n_cells)
    uint32_t *argmax;        // MAX only, optional: (B, n_int_max, C)
    int C, D, HW, NHW;
    int mean;
    int nx, ny;
    int64_t n_cells, n_int_max;
    int64_t max_units, max_long, max_tasks;  // launch sizes (>= the device counts)
    const uint32_t *order;   // optional launch order of the units (2D blocks)
    int64_t order_rep;       // units per warp
    // chunk schedule (work.cu); work == nullptr: not built
    const uint4 *work;
    const uint4 *splits;
    const int64_t *work_counts;
    int64_t max_work, max_splits, chunk_partials;
    int chunk;
    void *scratch;           // caller's scratch for the split partials
    size_t scratch_bytes;
    int long_only;           // group kernel: long cells only
    int debug;               // experiment switches (BVP_IVL_DEBUG), 0 in production
    int out_zeroed;          // the caller already zero-filled out (chunk kernel skips it)
    float *partials;         // split intervals: [B][n_chunks of splits][C] (workspace)
    uint32_t *partial_arg;   // MAX: sorted position of each partial's max
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

// Per-warp gather context: pointers batch-offset once, the lane's chunk
// folded into the row base, 32-bit element offsets in the loop (callers
// guarantee rows * C < 2^32).  Lanes beyond the row read chunk 0 of the same
// row (same sectors: no extra traffic, no predicates in the loop).
template <typename Elem, int VEC, int CH, int SRC>
struct Gather {
    static constexpr int U = CH == 1 ? 4 : (CH == 2 ? 2 : 1);  // rows per step
    static constexpr int STEPS = 32 / U;
    const Elem *rows;   // + this lane's chunk offset
    const float *wdist;
    const __nv_bfloat16 *wlog;
    const float *lse;
    const uint2 *meta;
    const uint32_t *ranks;
    uint32_t C;
    int nchunks;
    int lane;

    __device__ __forceinline__ Gather(const PoolParams &P, int b) {
        lane = threadIdx.x & 31;
        nchunks = P.C / VEC;
        const int ch0 = lane < nchunks ? lane : 0;
        rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride + ch0 * VEC;
        wdist = static_cast<const float *>(P.wsrc) + (SRC == kSrcDist ? b * P.w_bstride : 0);
        wlog = static_cast<const __nv_bfloat16 *>(P.wsrc) + (SRC == kSrcFused ? b * P.w_bstride : 0);
        lse = P.lse + (SRC == kSrcFused ? int64_t(b) * P.NHW : 0);
        meta = P.meta;
        ranks = P.ranks;
        C = static_cast<uint32_t>(P.C);
    }
    __device__ __forceinline__ uint2 rec(uint32_t j, uint32_t e) const {
        if (j >= e) return make_uint2(0u, 0u);
        if (SRC == kSrcX) return make_uint2(__ldg(ranks + j), 0u);
        return __ldg(meta + j);
    }
    __device__ __forceinline__ float weight(uint2 m, bool ok) const {
        if (!ok) return 0.f;
        if (SRC == kSrcX) return 1.f;
        if (SRC == kSrcDist) return __ldg(wdist + m.y);
        return __expf(__bfloat162float(wlog[m.y]) - __ldg(lse + m.x));
    }
    // rows of step s of the block whose records are `r`.  FULL: the whole
    // step lies before e (no per-point test); otherwise points >= e load row
    // 0 (their weight is 0 and MAX skips them).
    template <bool FULL>
    __device__ __forceinline__ void issue(float (&v)[U][CH][VEC], int s, uint2 r, uint32_t jbb,
                                          uint32_t e) const {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t rx = __shfl_sync(0xFFFFFFFFu, r.x, s * U + u);
            if (!FULL && jbb + s * U + u >= e) rx = 0;
            const Elem *rp = rows + rx * C;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                if (q == 0 || lane + 32 * q < nchunks)
                    Loader<Elem, VEC>::template load<SRC == kSrcX>(rp + 32 * q * VEC, v[u][q]);
                else
#pragma unroll
                    for (int k = 0; k < VEC; ++k) v[u][q][k] = 0.f;
            }
        }
    }
};

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

template <typename Acc, int CH, int VEC, bool IS_MAX>
__device__ __forceinline__ void acc_reset(Acc (&acc)[CH][VEC],
                                          uint32_t (&arg)[IS_MAX ? CH : 1][IS_MAX ? VEC : 1]) {
#pragma unroll
    for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            acc[q][k] = IS_MAX ? Acc(-INFINITY) : Acc(0);
            if (IS_MAX) arg[IS_MAX ? q : 0][IS_MAX ? k : 0] = 0xFFFFFFFFu;
        }
}

// The gather pipeline over sorted points [a, e): calls on_step(js, ws, v)
// for every full step inside one block (caller decides fast / slow path).
// Kept as a macro-free template so both kernels share it.
template <typename G, typename Buf, typename StepFn>
__device__ __forceinline__ void gather_stream(const G &g, uint32_t a, uint32_t e, Buf &v,
                                              StepFn &&on_step) {
    constexpr int U = G::U, STEPS = G::STEPS;
    const int lane = g.lane;
    uint32_t jb = a;
    uint2 r0 = g.rec(jb + lane, e), r1 = g.rec(jb + 32 + lane, e);
    float w0 = g.weight(r0, jb + lane < e);
    if (jb + U <= e) g.template issue<true>(v[0], 0, r0, jb, e);
    else g.template issue<false>(v[0], 0, r0, jb, e);
#pragma unroll 1
    for (; jb < e; jb += 32) {
        const uint2 r2 = g.rec(jb + 64 + lane, e);
        const float w1 = g.weight(r1, jb + 32 + lane < e);
#pragma unroll
        for (int s = 0; s < STEPS; ++s) {
            const uint32_t js = jb + s * U;
            if (js >= e) break;  // warp-uniform
            if (s + 1 < STEPS) {
                const uint32_t jn = js + U;
                if (jn + U <= e) g.template issue<true>(v[(s + 1) & 1], s + 1, r0, jb, e);
                else if (jn < e) g.template issue<false>(v[(s + 1) & 1], s + 1, r0, jb, e);
            } else {
                const uint32_t jn = jb + 32;
                if (jn + U <= e) g.template issue<true>(v[0], 0, r1, jn, e);
                else if (jn < e) g.template issue<false>(v[0], 0, r1, jn, e);
            }
            float ws[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ws[u] = __shfl_sync(0xFFFFFFFFu, w0, s * U + u);
            on_step(js, ws, v[s & 1]);
        }
        r0 = r1;
        r1 = r2;
        w0 = w1;
    }
}

// One warp per work unit (<= 8 cells, <= budget points): the simple loop the
// gather microbenchmark (scripts/l2_gather_bench.cu) shows is fastest on
// B200 -- U rows per step, every lane loading the step's gather records and
// weights itself (same address across the warp: one L1 transaction), no
// register double buffer, so the kernel stays near 40 registers and the SM
// holds enough warps to cover the L2 latency.  SPLIT: long units are left to
// pool_long_kernel (fast mode); the exact mode walks them here, in order.
#ifndef BVP_UNIT_MIN_BLOCKS
#define BVP_UNIT_MIN_BLOCKS 6  // 48 warps/SM: caps registers at 40
#endif
template <typename Acc, typename Elem, int VEC, int CH, bool IS_MAX, int SRC, bool SPLIT>
__global__ void __launch_bounds__(kPoolThreads, BVP_UNIT_MIN_BLOCKS)
pool_unit_kernel(const PoolParams P) {
    constexpr int U = CH == 1 ? 4 : (CH == 2 ? 2 : 1);
    extern __shared__ float s_all[];  // per warp: [C][kUnitPitch]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.y;
    const int64_t n_units = P.sched_counts[0];
    const int rep = static_cast<int>(P.order_rep);
#pragma unroll 1
    for (int r = 0; r < rep; ++r) {
    const int64_t kk = (int64_t(blockIdx.x) * rep + r) * kPoolWarps + warp;
    if (kk >= n_units) break;
    const int64_t k = P.order ? int64_t(__ldg(P.order + kk)) : kk;
    const uint4 ur = __ldg(reinterpret_cast<const uint4 *>(P.units) + k);
    if (SPLIT && (ur.y & kLongUnit)) continue;
    const uint4 un = __ldg(reinterpret_cast<const uint4 *>(P.units) + k + 1);
    const int64_t cell0 = ur.x;
    const int ncell = static_cast<int>(ur.y & 0xFFu);
    const uint32_t has = (ur.y >> 8) & 0xFFu;
    const uint32_t J0 = ur.w, J1 = un.w;
    const int C = P.C;
    const int nchunks = C / VEC;
    const uint32_t *starts = P.starts;
    float *s_tile = s_all + warp * C * kUnitPitch;
    const Gather<Elem, VEC, CH, SRC> g(P, b);

    Acc acc[CH][VEC];
    uint32_t arg[IS_MAX ? CH : 1][IS_MAX ? VEC : 1];
    acc_reset<Acc, CH, VEC, IS_MAX>(acc, arg);
    uint32_t iv = ur.z, lo = J0;
    uint32_t hi = J1 > J0 ? __ldg(starts + iv + 1) : 0u;
    auto park = [&]() {  // interval iv = [lo, hi) complete
        const int lc = static_cast<int>(int64_t(__ldg(P.icells + iv)) - cell0);
        const Acc inv = P.mean ? Acc(1) / Acc(hi - lo) : Acc(1);
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int ch = lane + 32 * q;
            if (ch < nchunks)
#pragma unroll
                for (int x = 0; x < VEC; ++x) {
                    const int c = ch * VEC + x;
                    s_tile[c * kUnitPitch + lc] = static_cast<float>(
                        P.mean == 2 ? acc[q][x] / Acc(hi - lo) : acc[q][x] * inv);
                    if (IS_MAX && P.argmax)
                        P.argmax[(b * P.n_int_max + iv) * C + c] =
                            __ldg(P.ranks + arg[IS_MAX ? q : 0][IS_MAX ? x : 0]);
                }
        }
    };
#pragma unroll 1
    for (uint32_t js = J0; js < J1; js += U) {
        float w[U];
        float v[U][CH][VEC];
        const bool full = js + U <= J1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = full || js + u < J1;
            const uint2 m = g.rec(ok ? js + u : J0, J1);
            w[u] = g.weight(m, ok);
            const Elem *rp = g.rows + m.x * g.C;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                if (q == 0 || lane + 32 * q < nchunks)
                    Loader<Elem, VEC>::template load<SRC == kSrcX>(rp + 32 * q * VEC, v[u][q]);
                else
#pragma unroll
                    for (int x = 0; x < VEC; ++x) v[u][q][x] = 0.f;
            }
        }
        if (js + U <= hi) {  // whole step inside the current interval
#pragma unroll
            for (int u = 0; u < U; ++u) acc_point<Acc, CH, VEC, IS_MAX>(acc, arg, js + u, w[u], v[u]);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t jj = js + u;
                if (jj >= J1) break;
                if (jj == hi) {  // interval boundary (warp-uniform)
                    park();
                    acc_reset<Acc, CH, VEC, IS_MAX>(acc, arg);
                    ++iv;
                    lo = hi;
                    hi = __ldg(starts + iv + 1);
                }
                acc_point<Acc, CH, VEC, IS_MAX>(acc, arg, jj, w[u], v[u]);
            }
        }
    }
    if (J1 > J0) park();
    __syncwarp();
    float *out = P.out + int64_t(b) * C * P.n_cells + cell0;
    const int64_t n_cells = P.n_cells;
    for (int idx = lane; idx < C * ncell; idx += 32) {
        const int c = idx / ncell, x = idx - c * ncell;
        out[int64_t(c) * n_cells + x] = ((has >> x) & 1u) ? s_tile[c * kUnitPitch + x] : 0.f;
    }
    __syncwarp();
    }
}

// Fast mode: one CTA per heavy cell (a single interval above the unit point
// budget).  Its 8 warps walk equal slices of the interval; the slices'
// partial results are combined in slice order in shared memory, so the sum
// is deterministic and the heavy cell no longer sets the critical path.
template <typename Elem, int VEC, int CH, bool IS_MAX, int SRC>
__global__ void __launch_bounds__(kPoolThreads)
pool_long_kernel(const PoolParams P) {
    using G = Gather<Elem, VEC, CH, SRC>;
    constexpr int U = G::U;
    extern __shared__ float s_all[];  // [kPoolWarps][C] values + [kPoolWarps][C] argmax
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int C = P.C;
    const int b = blockIdx.y;
    if (int64_t(blockIdx.x) >= P.sched_counts[1]) return;
    const uint32_t k = __ldg(P.long_units + blockIdx.x);
    const int64_t cell = __ldg(P.units + 4 * size_t(k));
    const uint32_t iv = __ldg(P.cell_first + cell);
    const uint32_t lo = __ldg(P.starts + iv), hi = __ldg(P.starts + iv + 1);
    const uint32_t L = hi - lo;
    const uint32_t a = lo + uint32_t(uint64_t(L) * warp / kPoolWarps);
    const uint32_t e = lo + uint32_t(uint64_t(L) * (warp + 1) / kPoolWarps);
    const G g(P, b);
    float acc[CH][VEC];
    uint32_t arg[IS_MAX ? CH : 1][IS_MAX ? VEC : 1];
    acc_reset<float, CH, VEC, IS_MAX>(acc, arg);
    if (e > a) {
        float v[2][U][CH][VEC];
        gather_stream(g, a, e, v, [&](uint32_t js, const float (&ws)[U],
                                      const float (&vb)[U][CH][VEC]) {
#pragma unroll
            for (int k2 = 0; k2 < U; ++k2)
                if (!IS_MAX || js + k2 < e)
                    acc_point<float, CH, VEC, IS_MAX>(acc, arg, js + k2, ws[k2], vb[k2]);
        });
    }
    float *s_val = s_all;
    uint32_t *s_arg = reinterpret_cast<uint32_t *>(s_all + kPoolWarps * C);
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int ch = lane + 32 * q;
        if (ch < g.nchunks)
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

// Exact mode: one CTA per heavy cell (a long unit), summed in rank order
// like every other cell -- but with the gathers batched.  The cell's points
// are walked in tiles of T = kExactTile / C rows: all 256 threads load the
// next tile's rows (and weights) into registers while the channel threads
// run the current tile's sequential fp64 FMAs out of shared memory, so the
// cell costs ~L / T gather latencies instead of ~L / 4.
constexpr int kExactTile = 8192;                  // floats per staged tile
constexpr int kExactRegs = kExactTile / kPoolThreads;  // per thread (32)

// SPLITS: the cells are the chunk schedule's split intervals (work.cu),
// else the long units (units.cu).
template <int VEC, bool IS_MAX, bool SPLITS = false>
__global__ void __launch_bounds__(kPoolThreads)
pool_exact_long_kernel(const PoolParams P) {
    extern __shared__ float s_ex[];  // [T][C] rows, [T] weights
    const int C = P.C, tid = threadIdx.x;
    const int b = blockIdx.y;
    if (int64_t(blockIdx.x) >= (SPLITS ? P.work_counts[1] : P.sched_counts[1])) return;
    const int T = min(128, kExactTile / C);
    float *s_rows = s_ex, *s_w = s_ex + T * C;
    int64_t cell;
    uint32_t iv;
    if (SPLITS) {
        const uint4 sp = __ldg(P.splits + blockIdx.x);  // interval, cell, slot, chunks
        iv = sp.x;
        cell = sp.y;
    } else {
        const uint32_t k = __ldg(P.long_units + blockIdx.x);
        cell = __ldg(P.units + 4 * size_t(k));
        iv = __ldg(P.cell_first + cell);
    }
    const uint32_t lo = __ldg(P.starts + iv), hi = __ldg(P.starts + iv + 1);
    const float *rows = static_cast<const float *>(P.rows) + b * P.rows_bstride;
    const float *wd = static_cast<const float *>(P.wsrc) + b * P.w_bstride;
    const int cv = C / VEC;          // vectors per row
    constexpr int R = kExactRegs / VEC;  // vectors per thread per tile

    float buf[R][VEC];
    float wbuf = 0.f;
    auto load = [&](uint32_t j0) {  // tile starting at sorted point j0 -> registers
        const int n = static_cast<int>(min(uint32_t(T), hi - j0));
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int e = tid + q * kPoolThreads;
            const int t = e / cv;
            if (t < n) {
                const uint2 m = __ldg(P.meta + j0 + t);
                const float *src = rows + size_t(m.x) * C + (e - t * cv) * VEC;
                if (VEC == 4) {
                    const float4 v = ldg_f4(src);
                    buf[q][0] = v.x; buf[q][VEC > 1 ? 1 : 0] = v.y;
                    buf[q][VEC > 2 ? 2 : 0] = v.z; buf[q][VEC > 3 ? 3 : 0] = v.w;
                } else {
                    buf[q][0] = __ldg(src);
                }
            }
        }
        if (tid < n) wbuf = __ldg(wd + __ldg(P.meta + j0 + tid).y);
    };
    auto stash = [&](uint32_t j0) {
        const int n = static_cast<int>(min(uint32_t(T), hi - j0));
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int e = tid + q * kPoolThreads;
            if (e / cv < n)
#pragma unroll
                for (int x = 0; x < VEC; ++x) s_rows[e * VEC + x] = buf[q][x];
        }
        if (tid < n) s_w[tid] = wbuf;
    };

    constexpr int A = 1024 / kPoolThreads;  // channels per thread (C <= 1024)
    double acc[A];
    uint32_t arg[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
        acc[a] = IS_MAX ? -INFINITY : 0.0;
        arg[a] = lo;
    }
    load(lo);
    for (uint32_t j0 = lo; j0 < hi; j0 += T) {
        __syncthreads();  // the previous tile is consumed
        stash(j0);
        __syncthreads();
        if (j0 + T < hi) load(j0 + T);  // in flight during the sums below
        const int n = static_cast<int>(min(uint32_t(T), hi - j0));
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const int c = tid + a * kPoolThreads;
            if (c >= C) break;
            double r = acc[a];
            uint32_t ra = arg[a];
            for (int t = 0; t < n; ++t) {
                const double pv = double(s_w[t]) * double(s_rows[t * C + c]);
                if (IS_MAX) {
                    if (pv > r) {
                        r = pv;
                        ra = j0 + t;
                    }
                } else {
                    r += pv;
                }
            }
            acc[a] = r;
            arg[a] = ra;
        }
    }
    float *out = P.out + int64_t(b) * C * P.n_cells + cell;
    const double inv = P.mean ? 1.0 / double(hi - lo) : 1.0;
#pragma unroll
    for (int a = 0; a < A; ++a) {
        const int c = tid + a * kPoolThreads;
        if (c >= C) break;
        out[int64_t(c) * P.n_cells] =
            static_cast<float>(P.mean == 2 ? acc[a] / double(hi - lo) : acc[a] * inv);
        if (IS_MAX && P.argmax) P.argmax[(b * P.n_int_max + iv) * C + c] = __ldg(P.ranks + arg[a]);
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

// Launch the instantiated kernels for (Acc, Elem, VEC, SRC) and the shape of
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
BVP_DECLARE_RUN_POOL(float, __nv_bfloat16, 8, kSrcDist)  // fused.cu (precomputed softmax)
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
    BVP_REQUIRE(p.units && p.tasks && p.sched_counts, BVP_ERR_INVALID,
                "the schedule's units / tasks are required (built without units?)");
    // heavy cells go to a CTA each: split over its warps in the fast mode
    // (pool_long_kernel), walked in order with batched gathers in the exact
    // mode (pool_exact_long_kernel)
    constexpr bool kSplit = true;
    constexpr bool kExact = sizeof(Acc) == sizeof(double);
    const dim3 grid(static_cast<unsigned>(ceil_div(p.max_units, kPoolWarps * p.order_rep)),
                    static_cast<unsigned>(B));
    const size_t lsmem = size_t(kPoolWarps) * p.C * 2 * sizeof(float);
#define BVP_LAUNCH_CH(CHV)                                                                   \
    if (ch == CHV) {                                                                         \
        auto k = is_max ? pool_unit_kernel<Acc, Elem, VEC, CHV, true, SRC, kSplit>           \
                        : pool_unit_kernel<Acc, Elem, VEC, CHV, false, SRC, kSplit>;         \
        if (smem > 48 * 1024)                                                                \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        if (kExact && p.max_long > 0) {                                                      \
            /* heavy cells on a side stream, overlapping the unit kernel */                  \
            auto ke = is_max ? pool_exact_long_kernel<VEC, true>                             \
                             : pool_exact_long_kernel<VEC, false>;                           \
            const int T = std::min(128, kExactTile / p.C);                                   \
            const size_t esmem = size_t(T) * (p.C + 1) * sizeof(float);                      \
            if (esmem > 48 * 1024)                                                           \
                cudaFuncSetAttribute(ke, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                     int(esmem));                                            \
            SideFork fork(s);                                                                \
            ke<<<dim3(static_cast<unsigned>(p.max_long), static_cast<unsigned>(B)),          \
                 kPoolThreads, esmem, fork.side>>>(p);                                       \
            k<<<grid, kPoolThreads, smem, s>>>(p);                                           \
            fork.join();                                                                     \
            return BVP_OK;                                                                   \
        }                                                                                    \
        k<<<grid, kPoolThreads, smem, s>>>(p);                                               \
        if (kExact) {                                                                        \
        } else if (kSplit && p.max_long > 0) {                                               \
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
