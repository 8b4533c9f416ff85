// pool_kernel.cuh -- the interval-reduction kernel (forward), sm_100a.
//
// Restates the reference's interval_reduce (_kernels.py:22-63).
//
// Work decomposition
//   * A tile is 32 consecutive cells of one BEV row (ix fixed).  One WARP
//     owns one tile: it reduces every interval of the tile and writes the
//     tile's (C x 32) output block -- zeros of empty cells included -- as
//     128-byte row segments.  Exactly one non-atomic store per (channel,
//     cell); no __syncthreads anywhere.
//   * The kWarps warps of a CTA own the tiles of kWarps consecutive BEV rows
//     at the same y-range: a CTA covers a kWarps x 32 block of cells, so the
//     feature rows its intervals gather (a ray crosses neighbouring rows at
//     neighbouring depths) are re-used out of L1.
//   * Inside a warp, groups of LPP lanes each own ONE interval at a time and
//     walk its points sequentially in rank order (CPL 16-byte chunks of the
//     channel row per lane).  Groups that finish pick the next interval of
//     the tile (warp-uniform refill via ballot), so the warp stays busy until
//     the tile's total work is done.  Because each interval is accumulated by
//     one group in rank order, Acc = double reproduces the reference's 64-bit
//     sums bit for bit (products of two fp32 are exact in fp64); Acc = float
//     is the fast mode.
//   * Points are taken U = LPP at a time: each lane of the group fetches one
//     point's rank + depth weight, shuffles broadcast them, and the group
//     issues U x CPL independent 16-byte loads.  The next block's ranks are
//     prefetched while the current block's gathers are in flight.
//
// Sources (SRC):
//   kSrcDist  : rows = NHWC features (f32), weight = dist[n,d,h,w] (f32)
//   kSrcX     : rows = materialised frustum x[p, :] (f32), weight = 1
//   kSrcFused : rows = NHWC context (bf16), weight = exp(logit - lse[pixel])
#pragma once

#include "common.cuh"

namespace bvp {

constexpr int kPoolWarps = 4;
constexpr int kPoolThreads = 32 * kPoolWarps;
constexpr int kTilePitch = kTileCells + 1;

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
    int nx, ny, tiles_y;     // BEV rows, cells per row, 32-cell tiles per row
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

// Park one finished interval (MEAN scaling, argmax) in the warp's tile.
template <typename Acc, int VEC, int LPP, int CPL, bool IS_MAX>
__device__ __forceinline__ void store_interval(const PoolParams &P, float *s_out,
                                               const Acc (&acc)[CPL][VEC],
                                               const uint32_t (&arg)[IS_MAX ? CPL : 1]
                                                                    [IS_MAX ? VEC : 1],
                                               uint32_t iv, uint32_t hi, int64_t cell0, int b,
                                               int sub, int nchunks) {
    const int lc = static_cast<int>(int64_t(__ldg(P.icells + iv)) - cell0);
    const uint32_t len = hi - __ldg(P.starts + iv);
    const Acc inv = P.mean ? Acc(1) / Acc(len) : Acc(1);
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
        const int ch = sub + q * LPP;
        if (ch < nchunks) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const int c = ch * VEC + e;
                const Acc r = P.mean ? acc[q][e] * inv : acc[q][e];
                s_out[c * kTilePitch + lc] = static_cast<float>(r);
                if (IS_MAX && P.argmax)
                    P.argmax[(b * P.n_int_max + iv) * P.C + c] = arg[IS_MAX ? q : 0][IS_MAX ? e : 0];
            }
        }
    }
}

template <typename Acc, typename Elem, int VEC, int LPP, int CPL, bool IS_MAX, int SRC>
__global__ void __launch_bounds__(kPoolThreads)
pool_tile_kernel(const PoolParams P) {
    extern __shared__ float s_all[];  // [kPoolWarps][C][kTilePitch]
    // points per block per group (bounded so the block's rows fit registers)
    constexpr int U = LPP < 4 ? LPP : (CPL > 5 ? 2 : 4);
    constexpr int NG = 32 / LPP;  // interval groups per warp
    // fast mode may split one long interval over all groups (exact may not)
    constexpr bool kCoop = sizeof(Acc) == sizeof(float);
    constexpr uint32_t kCoopMin = 64;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPP, sub = lane % LPP, gbase = g * LPP;
    const int C = P.C;
    const int nchunks = C / VEC;
    const int b = blockIdx.y;
    float *s_out = s_all + warp * C * kTilePitch;

    // work unit of this warp: a run of <= 32 cells of one row tile
    const int64_t k = int64_t(blockIdx.x) * kPoolWarps + warp;
    if (k >= *P.n_units) return;
    const int64_t cell0 = __ldg(P.units + 2 * k);
    const int ncell = static_cast<int>(__ldg(P.units + 2 * k + 1));
    const uint32_t i0 = __ldg(P.cell_first + cell0), i1 = __ldg(P.cell_first + cell0 + ncell);

    const Elem *rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride;
    uint32_t written = 0;  // bit x: cell cell0+x received an interval

    // group state (replicated over the group's lanes)
    uint32_t cur = 0xFFFFFFFFu, j = 0, hi = 0;
    uint32_t next_i = i0;
    uint32_t stride = U;
    Acc acc[CPL][VEC];
    uint32_t arg[IS_MAX ? CPL : 1][IS_MAX ? VEC : 1];
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
            acc[q][e] = IS_MAX ? Acc(-INFINITY) : Acc(0);
            if (IS_MAX) arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = 0xFFFFFFFFu;
        }
    uint32_t pf_rank = 0;
    bool pf_ok = false;

    // fast mode, a unit that is one long interval: every group walks a
    // strided share of it and the shares are combined at the end
    bool coop = false;
    if (kCoop && i1 == i0 + 1) {
        const uint32_t lo = __ldg(P.starts + i0), h = __ldg(P.starts + i0 + 1);
        if (h - lo > kCoopMin) {
            coop = true;
            cur = i0;
            j = lo + g * U;
            hi = h;
            stride = NG * U;
            next_i = i1;
            if (j >= hi) cur = 0xFFFFFFFEu;  // nothing for this group
        }
    }

    while (true) {
        // ---- refill: groups without an interval take the next ones --------
        const bool need = (cur == 0xFFFFFFFFu);
        const unsigned ask = __ballot_sync(0xFFFFFFFFu, need && sub == 0);
        if (ask) {
            if (need) {
                const uint32_t mine = next_i + __popc(ask & ((1u << gbase) - 1u));
                if (mine < i1) {
                    cur = mine;
                    j = __ldg(P.starts + mine);
                    hi = __ldg(P.starts + mine + 1);
                    pf_ok = false;
#pragma unroll
                    for (int q = 0; q < CPL; ++q)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            acc[q][e] = IS_MAX ? Acc(-INFINITY) : Acc(0);
                            if (IS_MAX) arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = 0xFFFFFFFFu;
                        }
                } else {
                    cur = 0xFFFFFFFEu;  // retired
                }
            }
            next_i += __popc(ask);
        }
        const bool active = cur < 0xFFFFFFFEu;
        if (!__any_sync(0xFFFFFFFFu, active)) break;

        // ---- one block of U points per active group --------------------------
        uint32_t p = 0, row = 0;
        float wt = 0.f;
        const bool mine_ok = active && sub < U && (j + sub < hi);
        if (mine_ok) {
            p = pf_ok ? pf_rank : __ldg(P.ranks + j + sub);
            // prefetch this group's next block
            pf_ok = (j + stride + sub < hi);
            if (pf_ok) pf_rank = __ldg(P.ranks + j + stride + sub);
            if (SRC == kSrcX) {
                row = p;
                wt = 1.f;
            } else {
                const uint32_t pix = p / P.D;
                const uint32_t d = p - pix * P.D;
                const uint32_t n = pix / P.HW;
                const uint32_t hw = pix - n * P.HW;
                const int64_t widx = b * P.w_bstride + (int64_t(n) * P.D + d) * P.HW + hw;
                row = pix;
                if (SRC == kSrcDist) {
                    wt = __ldg(static_cast<const float *>(P.wsrc) + widx);
                } else {
                    const float l = __bfloat162float(
                        static_cast<const __nv_bfloat16 *>(P.wsrc)[widx]);
                    wt = __expf(l - __ldg(P.lse + int64_t(b) * P.NHW + pix));
                }
            }
        } else {
            pf_ok = false;
        }
        // gather the block's rows (independent loads), then accumulate in order
        float v[U][CPL][VEC];
        uint32_t pu[U];
        float wu[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t ru = __shfl_sync(0xFFFFFFFFu, row, gbase + u);
            wu[u] = __shfl_sync(0xFFFFFFFFu, wt, gbase + u);
            pu[u] = __shfl_sync(0xFFFFFFFFu, p, gbase + u);
            const bool ok = active && (j + u < hi);
            const Elem *rp = rows + int64_t(ru) * C;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int ch = sub + q * LPP;
                if (ok && ch < nchunks) {
                    Loader<Elem, VEC>::template load<SRC == kSrcX>(rp + ch * VEC, v[u][q]);
                } else {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) v[u][q][e] = 0.f;
                }
            }
        }
        if (active) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (j + u < hi) {
#pragma unroll
                    for (int q = 0; q < CPL; ++q)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            if (IS_MAX) {
                                const Acc pv = Acc(wu[u]) * Acc(v[u][q][e]);
                                if (pv > acc[q][e]) {
                                    acc[q][e] = pv;
                                    arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = pu[u];
                                }
                            } else {
                                acc[q][e] += Acc(wu[u]) * Acc(v[u][q][e]);
                            }
                        }
                }
            }
            j += stride;
            if (j >= hi) {
                if (coop) {
                    cur = 0xFFFFFFFEu;  // share done; combined after the loop
                } else {  // interval complete: park it in the unit's tile
                    store_interval<Acc, VEC, LPP, CPL, IS_MAX>(P, s_out, acc, arg, cur, hi, cell0, b, sub, nchunks);
                    written |= 1u << static_cast<int>(int64_t(__ldg(P.icells + cur)) - cell0);
                    cur = 0xFFFFFFFFu;
                }
            }
        }
    }
    if (coop) {  // combine the NG shares (fixed xor order: deterministic)
#pragma unroll
        for (int off = LPP; off < 32; off <<= 1) {
#pragma unroll
            for (int q = 0; q < CPL; ++q)
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const Acc o = __shfl_xor_sync(0xFFFFFFFFu, acc[q][e], off);
                    if (IS_MAX) {
                        uint32_t &ma = arg[IS_MAX ? q : 0][IS_MAX ? e : 0];
                        const uint32_t oa = __shfl_xor_sync(0xFFFFFFFFu, ma, off);
                        if (o > acc[q][e] || (o == acc[q][e] && oa < ma)) {
                            acc[q][e] = o;
                            ma = oa;
                        }
                    } else {
                        acc[q][e] += o;
                    }
                }
        }
        if (g == 0) store_interval<Acc, VEC, LPP, CPL, IS_MAX>(P, s_out, acc, arg, i0, __ldg(P.starts + i0 + 1), cell0, b,
                                   sub, nchunks);
        written = 1u << static_cast<int>(int64_t(__ldg(P.icells + i0)) - cell0);
    }
    // every group's `written` bits -> the whole warp
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) written |= __shfl_xor_sync(0xFFFFFFFFu, written, off);
    __syncwarp();
    float *out = P.out + int64_t(b) * C * P.n_cells + cell0;
    const bool has = lane < ncell && ((written >> lane) & 1u);
    if (lane < ncell)
        for (int c = 0; c < C; ++c)
            out[int64_t(c) * P.n_cells + lane] = has ? s_out[c * kTilePitch + lane] : 0.f;
}

// Per-warp shared memory of pool_slice_kernel: output tile, partial slots
// (values + argmax ids) and slot interval ids.
__host__ __device__ inline size_t slice_smem_per_warp(int C, int ng) {
    return (size_t(C) * kTilePitch + size_t(ng) * 2 * C * 2 + size_t(ng) * 2) * 4;
}

// ---------------------------------------------------------------------------
// Fast (fp32) kernel: balanced slices.
//
// The unit's intervals occupy one contiguous range [J0, J1) of the sorted
// point stream.  Lane-group g reduces the slice [J0 + L*g/NG, J0 + L*(g+1)/NG)
// sequentially, U points per step, reading each point's precomputed gather
// indices (feature row, weight index) -- no division, no shuffles in the
// loop.  Intervals that start and end inside a slice go straight to the
// output tile; the (at most two) intervals cut by a slice edge leave partial
// sums in shared slots that are combined afterwards in group order, so the
// result is deterministic for a given cache.  Every group does the same
// amount of work whatever the interval lengths.
// ---------------------------------------------------------------------------
template <typename Elem, int VEC, int LPP, int CPL, bool IS_MAX, int SRC>
__global__ void __launch_bounds__(kPoolThreads)
pool_slice_kernel(const PoolParams P) {
    extern __shared__ float s_all[];
    constexpr int NG = 32 / LPP;
    constexpr int U = CPL > 5 ? 2 : 4;
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPP, sub = lane % LPP;
    const int C = P.C;
    const int nchunks = C / VEC;
    const int b = blockIdx.y;
    float *s_out = s_all + size_t(warp) * (slice_smem_per_warp(C, NG) / 4);
    float *s_part = s_out + C * kTilePitch;                                    // [NG][2][C]
    uint32_t *s_parg = reinterpret_cast<uint32_t *>(s_part + NG * 2 * C);      // [NG][2][C]
    uint32_t *s_piv = s_parg + NG * 2 * C;                                     // [NG][2]

    const int64_t k = int64_t(blockIdx.x) * kPoolWarps + warp;
    if (k >= *P.n_units) return;
    const int64_t cell0 = __ldg(P.units + 2 * k);
    const int ncell = static_cast<int>(__ldg(P.units + 2 * k + 1));
    const uint32_t i0 = __ldg(P.cell_first + cell0), i1 = __ldg(P.cell_first + cell0 + ncell);
    bool has = false;
    if (lane < ncell)
        has = __ldg(P.cell_first + cell0 + lane + 1) > __ldg(P.cell_first + cell0 + lane);

    const Elem *rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride;
    const uint32_t J0 = __ldg(P.starts + i0), J1 = __ldg(P.starts + i1);
    const uint32_t L = J1 - J0;
    if (L > 0) {
        const uint32_t ja = J0 + uint32_t((uint64_t(L) * g) / NG);
        const uint32_t jb = J0 + uint32_t((uint64_t(L) * (g + 1)) / NG);
        // interval containing ja: the unit has <= 32 intervals, one per lane
        const uint32_t nint = i1 - i0;
        const uint32_t s_l = uint32_t(lane) < nint ? __ldg(P.starts + i0 + lane) : kNone;
        uint32_t loc = 0;
#pragma unroll 1
        for (int gg = 0; gg < NG; ++gg) {
            const uint32_t x = J0 + uint32_t((uint64_t(L) * gg) / NG);
            const unsigned m = __ballot_sync(0xFFFFFFFFu, s_l <= x);
            if (g == gg) loc = __popc(m) - 1;
        }
        uint32_t iv = i0 + loc;
        uint32_t hi = __ldg(P.starts + iv + 1);
        bool cut_first = ja > __ldg(P.starts + iv);  // interval began in an earlier slice
        uint32_t piv0 = kNone, piv1 = kNone;

        float acc[CPL][VEC];
        uint32_t arg[IS_MAX ? CPL : 1][IS_MAX ? VEC : 1];
        auto reset = [&]() {
#pragma unroll
            for (int q = 0; q < CPL; ++q)
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    acc[q][e] = IS_MAX ? -INFINITY : 0.f;
                    if (IS_MAX) arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = kNone;
                }
        };
        // park the current interval: complete ones in the tile, cut ones in a slot
        auto park = [&](bool complete, int slot) {
            if (complete) {
                const int lc = static_cast<int>(int64_t(__ldg(P.icells + iv)) - cell0);
                const float inv = P.mean ? 1.f / float(hi - __ldg(P.starts + iv)) : 1.f;
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int ch = sub + q * LPP;
                    if (ch < nchunks)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            const int c = ch * VEC + e;
                            s_out[c * kTilePitch + lc] = P.mean ? acc[q][e] * inv : acc[q][e];
                            if (IS_MAX && P.argmax)
                                P.argmax[(b * P.n_int_max + iv) * C + c] =
                                    __ldg(P.ranks + arg[IS_MAX ? q : 0][IS_MAX ? e : 0]);
                        }
                }
            } else {
                float *dst = s_part + (g * 2 + slot) * C;
                uint32_t *dsta = s_parg + (g * 2 + slot) * C;
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int ch = sub + q * LPP;
                    if (ch < nchunks)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            dst[ch * VEC + e] = acc[q][e];
                            if (IS_MAX) dsta[ch * VEC + e] = arg[IS_MAX ? q : 0][IS_MAX ? e : 0];
                        }
                }
                if (slot == 0) piv0 = iv; else piv1 = iv;
            }
        };
        reset();

        const uint32_t per = (L + NG - 1) / NG;          // longest slice
        const uint32_t nstep = (per + U - 1) / U;
        uint2 mn[U];                                      // prefetched gather indices
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t jj = ja + u;
            if (SRC == kSrcX) mn[u] = make_uint2(jj < jb ? __ldg(P.ranks + jj) : 0u, 0u);
            else mn[u] = jj < jb ? __ldg(P.meta + jj) : make_uint2(0u, 0u);
        }
#pragma unroll 1
        for (uint32_t st = 0; st < nstep; ++st) {
            const uint32_t j = ja + st * U;
            uint2 m[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                m[u] = mn[u];
                const uint32_t jj = j + U + u;
                if (SRC == kSrcX) mn[u] = make_uint2(jj < jb ? __ldg(P.ranks + jj) : 0u, 0u);
                else mn[u] = jj < jb ? __ldg(P.meta + jj) : make_uint2(0u, 0u);
            }
            float w[U];
            float v[U][CPL][VEC];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = j + u < jb;
                if (SRC == kSrcX) {
                    w[u] = ok ? 1.f : 0.f;
                } else if (SRC == kSrcDist) {
                    w[u] = ok ? __ldg(static_cast<const float *>(P.wsrc) + b * P.w_bstride + m[u].y)
                              : 0.f;
                } else {
                    w[u] = ok ? __expf(__bfloat162float(static_cast<const __nv_bfloat16 *>(
                                           P.wsrc)[b * P.w_bstride + m[u].y]) -
                                       __ldg(P.lse + int64_t(b) * P.NHW + m[u].x))
                              : 0.f;
                }
                const Elem *rp = rows + size_t(m[u].x) * C;
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int ch = sub + q * LPP;
                    if (ok && ch < nchunks) {
                        Loader<Elem, VEC>::template load<SRC == kSrcX>(rp + ch * VEC, v[u][q]);
                    } else {
#pragma unroll
                        for (int e = 0; e < VEC; ++e) v[u][q][e] = 0.f;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t jj = j + u;
                if (jj < jb) {
                    if (jj == hi) {  // the slice crosses into the next interval
                        park(!cut_first, 0);
                        reset();
                        cut_first = false;
                        ++iv;
                        hi = __ldg(P.starts + iv + 1);
                    }
#pragma unroll
                    for (int q = 0; q < CPL; ++q)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            if (IS_MAX) {
                                const float pv = w[u] * v[u][q][e];
                                if (pv > acc[q][e]) {
                                    acc[q][e] = pv;
                                    // sorted position; converted to the point id
                                    // (ranks[pos]) when written out
                                    arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = jj;
                                }
                            } else {
                                acc[q][e] = fmaf(w[u], v[u][q][e], acc[q][e]);
                            }
                        }
                }
            }
        }
        if (jb > ja) park(!cut_first && jb == hi, 1);
        if (sub == 0) {
            s_piv[g * 2] = piv0;
            s_piv[g * 2 + 1] = piv1;
        }
        __syncwarp();
        // combine the cut intervals' partial sums in slice order
        for (int c = lane; c < C; c += 32) {
            uint32_t run_iv = kNone, run_arg = kNone;
            float run = 0.f;
            for (int t = 0; t < 2 * NG; ++t) {
                const uint32_t x = s_piv[t];
                if (x == kNone) continue;
                const float val = s_part[t * C + c];
                const uint32_t va = IS_MAX ? s_parg[t * C + c] : 0u;
                if (x != run_iv) {
                    if (run_iv != kNone) {
                        const int lc = static_cast<int>(int64_t(__ldg(P.icells + run_iv)) - cell0);
                        const float inv = P.mean ? 1.f / float(__ldg(P.starts + run_iv + 1) -
                                                               __ldg(P.starts + run_iv))
                                                 : 1.f;
                        s_out[c * kTilePitch + lc] = run * inv;
                        if (IS_MAX && P.argmax)
                            P.argmax[(b * P.n_int_max + run_iv) * C + c] =
                                __ldg(P.ranks + run_arg);
                    }
                    run_iv = x;
                    run = val;
                    run_arg = va;
                } else if (IS_MAX) {
                    if (val > run || (val == run && va < run_arg)) {
                        run = val;
                        run_arg = va;
                    }
                } else {
                    run += val;
                }
            }
            if (run_iv != kNone) {
                const int lc = static_cast<int>(int64_t(__ldg(P.icells + run_iv)) - cell0);
                const float inv = P.mean ? 1.f / float(__ldg(P.starts + run_iv + 1) -
                                                       __ldg(P.starts + run_iv))
                                         : 1.f;
                s_out[c * kTilePitch + lc] = run * inv;
                if (IS_MAX && P.argmax)
                    P.argmax[(b * P.n_int_max + run_iv) * C + c] = __ldg(P.ranks + run_arg);
            }
        }
    }
    __syncwarp();
    float *out = P.out + int64_t(b) * C * P.n_cells + cell0;
    if (lane < ncell)
        for (int c = 0; c < C; ++c)
            out[int64_t(c) * P.n_cells + lane] = has ? s_out[c * kTilePitch + lane] : 0.f;
}

// Lane-group shape for a row of `nchunks` 16-byte chunks: LPP lanes per
// interval, CPL chunks per lane (instantiated table in pool.cu / fused.cu).
struct LaneShape {
    int lpp, cpl;
};

inline LaneShape choose_shape(int nchunks) {
    if (nchunks <= 0) return {1, 1};
    for (int lpp : {1, 2, 4, 8, 16, 32}) {
        const int need = (nchunks + lpp - 1) / lpp;
        if (lpp == 1) {
            if (need <= 2) return {1, need};
            if (need <= 5) return {1, need <= 4 ? 4 : 5};
        } else if (need <= 5) {
            return {lpp, need <= 4 ? 4 : 5};
        }
    }
    const int need = (nchunks + 31) / 32;
    if (need <= 8) return {32, 8};
    return {0, 0};
}

#define BVP_FOR_EACH_SHAPE(X) \
    X(1, 1) X(1, 2) X(1, 4) X(1, 5) X(2, 4) X(2, 5) X(4, 4) X(4, 5) X(8, 4) X(8, 5) X(16, 4) \
    X(16, 5) X(32, 4) X(32, 5) X(32, 8)

inline int64_t pool_tiles(const PoolParams &p) { return int64_t(p.nx) * p.tiles_y; }

// pool.cu
PoolParams make_pool_params(const uint32_t *ranks, const uint32_t *starts, const uint32_t *icells,
                            const uint32_t *cell_first, const uint32_t *units, const uint32_t *point_meta,
                            const int64_t *n_units, int64_t max_units, int C, int nx, int ny,
                            float *out, int mode);
template <typename T>
void launch_to_nhwc(const T *src, int64_t NB, int A, int HW, T *dst, cudaStream_t s);

// Launch the instantiated kernel for (Acc, Elem, VEC, SRC) and the shape of
// p.C.  Defined (and explicitly instantiated) in the pool_*.cu / fused.cu
// translation units so the ~30 kernels per family compile in parallel.
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
    const LaneShape sh = choose_shape(p.C / VEC);
    BVP_REQUIRE(sh.lpp > 0, BVP_ERR_UNSUPPORTED, "channel count %d not supported", p.C);
    constexpr bool kFast = sizeof(Acc) == sizeof(float);
    const size_t smem = kFast ? kPoolWarps * slice_smem_per_warp(p.C, 32 / sh.lpp)
                              : size_t(kPoolWarps) * p.C * kTilePitch * sizeof(float);
    BVP_REQUIRE(smem <= 227 * 1024, BVP_ERR_UNSUPPORTED, "channel count %d too large", p.C);
    BVP_REQUIRE(!kFast || SRC == kSrcX || p.meta, BVP_ERR_INVALID,
                "the cache's point gather table (point_meta) is required");
    const dim3 grid(static_cast<unsigned>(ceil_div(p.max_units, kPoolWarps)),
                    static_cast<unsigned>(B));
#define BVP_LAUNCH_SHAPE(L, CP)                                                              \
    if (sh.lpp == L && sh.cpl == CP) {                                                       \
        void (*k)(const PoolParams);                                                         \
        if constexpr (kFast)                                                                 \
            k = is_max ? pool_slice_kernel<Elem, VEC, L, CP, true, SRC>                      \
                       : pool_slice_kernel<Elem, VEC, L, CP, false, SRC>;                    \
        else                                                                                 \
            k = is_max ? pool_tile_kernel<Acc, Elem, VEC, L, CP, true, SRC>                  \
                       : pool_tile_kernel<Acc, Elem, VEC, L, CP, false, SRC>;                \
        if (smem > 48 * 1024)                                                                \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        k<<<grid, kPoolThreads, smem, s>>>(p);                                               \
        return BVP_OK;                                                                       \
    }
    BVP_FOR_EACH_SHAPE(BVP_LAUNCH_SHAPE)
#undef BVP_LAUNCH_SHAPE
    set_error("no kernel instance for lpp=%d cpl=%d", sh.lpp, sh.cpl);
    return BVP_ERR_UNSUPPORTED;
}

}  // namespace bvp
