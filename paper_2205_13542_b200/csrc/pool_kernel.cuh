// pool_kernel.cuh -- the cell-tiled interval-reduction kernel (forward).
//
// Restates the reference's interval_reduce (_kernels.py:22-63) for sm_100a.
// One CTA owns BVP_TILE_CELLS = 32 consecutive BEV cells.  Its interval range
// comes from the cached tile table (tile_first), warps take the tile's
// intervals round-robin, reduce each into registers, and park the result in
// a shared [C][32] tile; the CTA then writes the (C, n_cells) output rows as
// 128-byte coalesced segments -- zeros of empty cells included, so there is
// no separate memset and exactly one non-atomic store per (channel, cell).
//
// Lane mapping inside a warp: LPP lanes cover one point's channel row with
// VEC-wide 16-byte loads (CPL chunks per lane), PPW = 32/LPP points are in
// flight per warp iteration, and a final xor-shuffle combines the PPW partial
// sums.  LPP = 32 (PPW = 1) with Acc = double is the EXACT mode: each lane
// accumulates its channels in rank order in 64 bits exactly like the
// reference (products of two fp32 are exact in fp64), so the output is
// bit-identical to interval_reduce.
//
// Sources (SRC):
//   kSrcDist  : rows = NHWC features (f32), weight = dist[n,d,h,w] (f32)
//   kSrcX     : rows = materialised frustum x[p, :] (f32), weight = 1
//   kSrcFused : rows = NHWC context (bf16), weight = exp(logit - lse[pixel])
#pragma once

#include "common.cuh"

namespace bvp {

constexpr int kPoolThreads = 128;
constexpr int kPoolWarps = kPoolThreads / 32;
constexpr int kTilePitch = kTileCells + 1;

enum { kSrcDist = 0, kSrcX = 1, kSrcFused = 2 };

struct PoolParams {
    const void *rows;        // f32 NHWC features | f32 x (P,C) | bf16 NHWC context
    const void *wsrc;        // f32 dist (N,D,H,W) | bf16 logits (N,D,H,W) | unused
    const float *lse;        // fused: per-pixel log-sum-exp (N,H,W)
    const uint32_t *ranks;
    const uint32_t *starts;  // n_int + 1 entries (sentinel = n_in)
    const uint32_t *icells;
    const uint32_t *tile_first;
    float *out;              // (B, C, n_cells)
    uint32_t *argmax;        // MAX only, optional: (B, n_int_max, C)
    int C, D, HW, NHW;
    int mean;
    int64_t n_cells, n_int_max;
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

template <typename Acc, typename Elem, int VEC, int LPP, int CPL, bool IS_MAX, int SRC>
__global__ void __launch_bounds__(kPoolThreads)
pool_tile_kernel(const PoolParams P) {
    extern __shared__ float s_out[];  // [C][kTilePitch]
    constexpr int PPW = 32 / LPP;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane / LPP, sub = lane % LPP;
    const int C = P.C;
    const int nchunks = C / VEC;
    const int tile = blockIdx.x, b = blockIdx.y;
    const int64_t cell0 = int64_t(tile) * kTileCells;

    for (int i = tid; i < C * kTilePitch; i += kPoolThreads) s_out[i] = 0.f;

    const Elem *rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride;
    const uint32_t i0 = P.tile_first[tile], i1 = P.tile_first[tile + 1];
    __syncthreads();

    for (uint32_t i = i0 + warp; i < i1; i += kPoolWarps) {
        const uint32_t lo = P.starts[i], hi = P.starts[i + 1];
        const uint32_t cell = P.icells[i];
        Acc acc[CPL][VEC];
        uint32_t arg[IS_MAX ? CPL : 1][IS_MAX ? VEC : 1];
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                acc[q][e] = IS_MAX ? Acc(-INFINITY) : Acc(0);
                if (IS_MAX) arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = 0xFFFFFFFFu;
            }

        for (uint32_t j0 = lo; j0 < hi; j0 += 32) {
            const uint32_t j = j0 + lane;
            const int cnt = min(32u, hi - j0);
            uint32_t row = 0, pid = 0;
            float wt = 0.f;
            if (j < hi) {
                const uint32_t p = __ldg(P.ranks + j);
                pid = p;
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
            }
#pragma unroll 4
            for (int k = 0; k < 32; k += PPW) {
                if (k >= cnt) break;
                const int kk = k + g;
                const uint32_t rk = __shfl_sync(0xFFFFFFFFu, row, kk);
                const float wk = __shfl_sync(0xFFFFFFFFu, wt, kk);
                const uint32_t pk = IS_MAX ? __shfl_sync(0xFFFFFFFFu, pid, kk) : 0u;
                if (kk < cnt) {
                    const Elem *rp = rows + int64_t(rk) * C;
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const int ch = sub + q * LPP;
                        if (ch < nchunks) {
                            float v[VEC];
                            Loader<Elem, VEC>::template load<SRC == kSrcX>(rp + ch * VEC, v);
#pragma unroll
                            for (int e = 0; e < VEC; ++e) {
                                if (IS_MAX) {
                                    const Acc pv = Acc(wk) * Acc(v[e]);
                                    if (pv > acc[q][e]) {
                                        acc[q][e] = pv;
                                        arg[IS_MAX ? q : 0][IS_MAX ? e : 0] = pk;
                                    }
                                } else {
                                    acc[q][e] += Acc(wk) * Acc(v[e]);
                                }
                            }
                        }
                    }
                }
            }
        }
        // combine the PPW point-groups (lanes sharing `sub`)
#pragma unroll
        for (int off = LPP; off < 32; off <<= 1) {
#pragma unroll
            for (int q = 0; q < CPL; ++q)
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const Acc o = __shfl_xor_sync(0xFFFFFFFFu, acc[q][e], off);
                    if (IS_MAX) {
                        const uint32_t oa =
                            __shfl_xor_sync(0xFFFFFFFFu, arg[IS_MAX ? q : 0][IS_MAX ? e : 0], off);
                        uint32_t &ma = arg[IS_MAX ? q : 0][IS_MAX ? e : 0];
                        if (o > acc[q][e] || (o == acc[q][e] && oa < ma)) {
                            acc[q][e] = o;
                            ma = oa;
                        }
                    } else {
                        acc[q][e] += o;
                    }
                }
        }
        if (g == 0) {
            const int lc = static_cast<int>(cell - cell0);
            const Acc inv = P.mean ? Acc(1) / Acc(hi - lo) : Acc(1);
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
                            P.argmax[(b * P.n_int_max + i) * C + c] =
                                arg[IS_MAX ? q : 0][IS_MAX ? e : 0];
                    }
                }
            }
        }
    }
    __syncthreads();
    const int64_t rem = P.n_cells - cell0;
    const int ncell_tile = rem < kTileCells ? static_cast<int>(rem) : kTileCells;
    float *out = P.out + int64_t(b) * C * P.n_cells + cell0;
    for (int c = warp; c < C; c += kPoolWarps)
        if (lane < ncell_tile) out[int64_t(c) * P.n_cells + lane] = s_out[c * kTilePitch + lane];
}

// (LPP, CPL) choice for a channel count: the instantiated table below.
struct LaneShape {
    int lpp, cpl;
};

inline LaneShape choose_shape(int nchunks, bool exact, bool bf16vec) {
    if (exact) {
        for (int cpl : {1, 2, 4, 8})
            if (32 * cpl >= nchunks) return {32, cpl};
        return {0, 0};
    }
    if (bf16vec) {  // 16-byte chunks of 8 bf16
        if (nchunks <= 1) return {1, 1};
        if (nchunks <= 2) return {2, 1};
        if (nchunks <= 10) return {2, (nchunks + 1) / 2 <= 4 ? (nchunks + 1) / 2 : 5};
    } else {
        if (nchunks <= 1) return {1, 1};
        if (nchunks <= 2) return {2, 1};
        if (nchunks <= 4) return {4, 1};
        if (nchunks <= 24) {
            int cpl = (nchunks + 3) / 4;
            if (cpl == 7) cpl = 8;
            return {4, cpl};
        }
        if (nchunks <= 32) return {4, 8};
    }
    for (int lpp : {8, 16, 32})
        if (lpp * 8 >= nchunks) return {lpp, 8};
    return {0, 0};
}

}  // namespace bvp
