// pool_group.cuh -- the fast (fp32-accumulating) interval-reduction kernel,
// sm_100a: several points per warp instruction.
//
// Restates the reference's interval_reduce (_kernels.py:22-63) for the fast
// mode (fp32 accumulation, tolerance 1e-5 against the fp64 reference; the
// bit-exact fp64 mode stays in pool_kernel.cuh, which must add in strict
// rank order).
//
// Why: profiled on B200 (profiles/r01_baseline), the one-point-per-warp
// kernel is neither HBM- nor L2-bound -- it is instruction- and
// latency-bound (44 warp instructions per point, 20 of 32 lanes busy).  Here
// a warp is split into G = 32 / L lane GROUPS; each group takes one point of
// the current interval, its L lanes holding CPL VEC-element chunks of the
// point's row (C = 80 fp32: L = 4 lanes x 5 float4, 8 points per step).  A
// step is one gather record + one weight per group and CPL vector loads per
// lane, so the per-point instruction count drops ~8x and every warp keeps
// 8 rows in flight (plus the prefetched next step).
//
// Order of the fp32 sums: group g accumulates points lo+g, lo+g+G, ... of an
// interval; at the interval's end the G partials are combined by a fixed
// xor-butterfly.  The result is deterministic (independent of timing, launch
// shape and batch), within 1e-5 of the rank-order fp64 reference.
//
// Work: the cached schedule's units (<= 8 consecutive cells of one row, a
// point budget) one per warp; cells holding more than the budget ("long"
// units) are split over the 8 warps of one CTA, placed at the front of the
// grid so they never form the tail.  Finished intervals are parked in the
// warp's [C][kUnitPitch] shared tile; the unit's output block (zeros of
// empty cells included) is written once -- no memset, one non-atomic store
// per (channel, cell).
#pragma once

#include <algorithm>
#include <cstdlib>

#include "pool_kernel.cuh"

namespace bvp {

constexpr int kGroupMaxCpl = 6;     // chunks per lane instantiated (1..6)
constexpr int kNumSms = 148;        // B200
constexpr int kGroupCtasPerSm = 8;  // persistent-grid waves x residency

template <typename Elem, int VEC>
struct ChunkLoad;
template <>
struct ChunkLoad<float, 4> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const float *p, float (&v)[4]) {
        const float4 t = STREAM ? ldg_stream_f4(p) : ldg_f4(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
};
template <>
struct ChunkLoad<float, 1> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const float *p, float (&v)[1]) { v[0] = __ldg(p); }
};
template <>
struct ChunkLoad<__nv_bfloat16, 8> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const __nv_bfloat16 *p, float (&v)[8]) {
        const uint4 t = STREAM ? ldg_stream_u4(p) : __ldg(reinterpret_cast<const uint4 *>(p));
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
};
template <>
struct ChunkLoad<__nv_bfloat16, 1> {
    template <bool STREAM>
    __device__ __forceinline__ static void load(const __nv_bfloat16 *p, float (&v)[1]) {
        v[0] = __bfloat162float(p[0]);
    }
};

// Gather records and weights of the sorted point stream, 32 points per
// "window", one point per lane.  Windows 0 and 1 (with weights) cover
// [jb, jb + 64): every step's group picks its record and weight from them by
// shuffle, so no lane waits on a dependent load inside a step.  Window 2's
// weights and window 3's records are in flight (loaded one rotation = 32
// points ahead).
template <typename Elem, int VEC, int CPL, int SRC>
struct GroupStream {
    const Elem *rows;  // batch-offset, + this lane's first chunk
    const float *wdist;
    const __nv_bfloat16 *wlog;
    const float *lse;
    const uint2 *meta;
    const uint32_t *ranks;
    uint32_t C;
    int L, li, g;
    uint32_t live;  // bit k: chunk li + k*L exists
    uint32_t jb, jend;
    uint32_t r0, r1, r2, r3;  // row index per lane of windows 0..3
    uint32_t y2, y3;          // weight index of windows 2, 3 (dist / fused)
    float w0, w1, w2;         // weights of windows 0..2

    __device__ __forceinline__ GroupStream(const PoolParams &P, int b, int L_, int lg) {
        const int lane = threadIdx.x & 31;
        L = L_;
        li = lane & (L - 1);
        g = lane >> lg;
        const int nch = P.C / VEC;
        live = 0;
#pragma unroll
        for (int k = 0; k < CPL; ++k)
            if (li + k * L < nch) live |= 1u << k;
        rows = static_cast<const Elem *>(P.rows) + b * P.rows_bstride + li * VEC;
        wdist = static_cast<const float *>(P.wsrc) + (SRC == kSrcDist ? b * P.w_bstride : 0);
        wlog = static_cast<const __nv_bfloat16 *>(P.wsrc) + (SRC == kSrcFused ? b * P.w_bstride : 0);
        lse = P.lse + (SRC == kSrcFused ? int64_t(b) * P.NHW : 0);
        meta = P.meta;
        ranks = P.ranks;
        C = static_cast<uint32_t>(P.C);
    }
    __device__ __forceinline__ void load_rec(uint32_t j, uint32_t &r, uint32_t &y) const {
        if (j >= jend) {
            r = 0u;
            y = 0u;
        } else if (SRC == kSrcX) {
            r = __ldg(ranks + j);
            y = 0u;
        } else {
            const uint2 m = __ldg(meta + j);
            r = m.x;
            y = m.y;
        }
    }
    __device__ __forceinline__ float load_w(uint32_t r, uint32_t y) const {
        if (SRC == kSrcX) return 1.f;
        if (SRC == kSrcDist) return __ldg(wdist + y);
        return __expf(__bfloat162float(wlog[y]) - __ldg(lse + r));
    }
    // stream over sorted points [J0, J1)
    __device__ __forceinline__ void start(uint32_t J0, uint32_t J1) {
        const int lane = threadIdx.x & 31;
        jb = J0;
        jend = J1;
        uint32_t y0, y1;
        load_rec(J0 + lane, r0, y0);
        load_rec(J0 + 32 + lane, r1, y1);
        load_rec(J0 + 64 + lane, r2, y2);
        load_rec(J0 + 96 + lane, r3, y3);
        w0 = load_w(r0, y0);
        w1 = load_w(r1, y1);
        w2 = load_w(r2, y2);
    }
    __device__ __forceinline__ void rotate() {
        const int lane = threadIdx.x & 31;
        r0 = r1;
        w0 = w1;
        r1 = r2;
        w1 = w2;
        r2 = r3;
        y2 = y3;
        w2 = load_w(r2, y2);
        jb += 32;
        load_rec(jb + 96 + lane, r3, y3);
    }
    // make [jb, jb + 64) cover every point below `need`
    __device__ __forceinline__ void cover(uint32_t need) {
        while (need > jb + 64) rotate();
    }
    // the group's point of the step at js (points >= hi are padding: weight
    // 0, row of the step's first point) -> weight and row chunks
    __device__ __forceinline__ void fetch(uint32_t js, uint32_t hi, float &w,
                                          float (&v)[CPL][VEC]) const {
        const uint32_t j = js + g;
        const bool ok = j < hi;
        const uint32_t off = (ok ? j : js) - jb;  // < 64
        const int src = static_cast<int>(off & 31u);
        const uint32_t ra = __shfl_sync(0xFFFFFFFFu, r0, src);
        const uint32_t rb = __shfl_sync(0xFFFFFFFFu, r1, src);
        const float wa = __shfl_sync(0xFFFFFFFFu, w0, src);
        const float wb = __shfl_sync(0xFFFFFFFFu, w1, src);
        const uint32_t r = off < 32u ? ra : rb;
        w = ok ? (off < 32u ? wa : wb) : 0.f;
        const Elem *rp = rows + r * C;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            if (k == 0 || ((live >> k) & 1u))
                ChunkLoad<Elem, VEC>::template load<SRC == kSrcX>(rp + k * L * VEC, v[k]);
            else
#pragma unroll
                for (int x = 0; x < VEC; ++x) v[k][x] = 0.f;
        }
    }
};

// ARG: track the winning point of MAX (autograd); false keeps MAX's value only
template <int CPL, int VEC, bool IS_MAX, bool ARG = IS_MAX>
__device__ __forceinline__ void gacc(float (&acc)[CPL][VEC], uint32_t (&arg)[ARG ? CPL : 1][ARG ? VEC : 1],
                                     uint32_t j, bool ok, float w, const float (&v)[CPL][VEC]) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
        for (int x = 0; x < VEC; ++x) {
            if (IS_MAX) {
                const float pv = w * v[k][x];
                if (ARG) {
                    if (ok && pv > acc[k][x]) {
                        acc[k][x] = pv;
                        arg[ARG ? k : 0][ARG ? x : 0] = j;
                    }
                } else if (ok && pv > acc[k][x]) {  // first maximum, as the reference
                    acc[k][x] = pv;
                }
            } else {
                acc[k][x] = fmaf(w, v[k][x], acc[k][x]);
            }
        }
}

template <int CPL, int VEC, bool IS_MAX, bool ARG = IS_MAX>
__device__ __forceinline__ void greset(float (&acc)[CPL][VEC], uint32_t (&arg)[ARG ? CPL : 1][ARG ? VEC : 1]) {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
#pragma unroll
        for (int x = 0; x < VEC; ++x) {
            acc[k][x] = IS_MAX ? -INFINITY : 0.f;
            if (ARG) arg[ARG ? k : 0][ARG ? x : 0] = 0xFFFFFFFFu;
        }
}

// Combine the G group partials (xor butterfly over the group bits of the
// lane id; every group ends with the full result).  MAX keeps the first
// (lowest sorted position) point attaining the maximum.
template <int CPL, int VEC, bool IS_MAX>
__device__ __forceinline__ void gcombine(float (&acc)[CPL][VEC],
                                         uint32_t (&arg)[IS_MAX ? CPL : 1][IS_MAX ? VEC : 1], int L) {
#pragma unroll 1
    for (int off = L; off < 32; off <<= 1) {
#pragma unroll
        for (int k = 0; k < CPL; ++k)
#pragma unroll
            for (int x = 0; x < VEC; ++x) {
                const float o = __shfl_xor_sync(0xFFFFFFFFu, acc[k][x], off);
                if (IS_MAX) {
                    const uint32_t oa = __shfl_xor_sync(0xFFFFFFFFu, arg[IS_MAX ? k : 0][IS_MAX ? x : 0], off);
                    uint32_t &a = arg[IS_MAX ? k : 0][IS_MAX ? x : 0];
                    if (o > acc[k][x] || (o == acc[k][x] && oa < a)) {
                        acc[k][x] = o;
                        a = oa;
                    }
                } else {
                    acc[k][x] += o;
                }
            }
    }
}

#ifndef BVP_GROUP_MIN_BLOCKS
#define BVP_GROUP_MIN_BLOCKS 2
#endif

template <typename Elem, int VEC, int CPL, bool IS_MAX, int SRC>
__global__ void __launch_bounds__(kPoolThreads, BVP_GROUP_MIN_BLOCKS)
pool_group_kernel(const PoolParams P, int L, int lg) {
    using Stream = GroupStream<Elem, VEC, CPL, SRC>;
    extern __shared__ float s_all[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.y;
    const int C = P.C;
    const uint32_t G = 32u >> lg;
    Stream st(P, b, L, lg);
    const int g = st.g;
    const int nch = C / VEC;
    float acc[CPL][VEC];
    uint32_t arg[IS_MAX ? CPL : 1][IS_MAX ? VEC : 1];
    float va[CPL][VEC], vb[CPL][VEC];
    float wa, wb;

    // Walk the sorted points [J0, J1) of consecutive intervals iv, iv+1, ...
    // (ends read from P.starts; iv_end bounds the prefetch), in steps of G
    // points that never straddle an interval; on_end(iv, lo, hi) after each
    // interval with the combined result in acc (every group holds it).
    // Rows are fetched one step ahead into the other buffer.
    auto walk = [&](uint32_t J0, uint32_t J1, uint32_t iv, uint32_t iv_end, uint32_t hi,
                    auto &&on_end) {
        st.start(J0, J1);
        uint32_t lo = J0;
        uint32_t hi2 = iv + 1 < iv_end ? __ldg(P.starts + iv + 2) : hi;
        // interval cells (prefetched one interval ahead)
        uint32_t cell = iv < iv_end ? __ldg(P.icells + iv) : 0u;
        uint32_t cell2 = iv + 1 < iv_end ? __ldg(P.icells + iv + 1) : 0u;
        uint32_t js = J0;
        greset<CPL, VEC, IS_MAX>(acc, arg);
        st.fetch(js, hi, wa, va);
        // one step: accumulate the buffered step at js, prefetch the next
        auto step = [&](float (&cur)[CPL][VEC], float wcur, float (&nxt)[CPL][VEC],
                        float &wnxt) -> bool {
            uint32_t njs = js + G, nhi = hi;
            const bool boundary = njs >= hi;
            if (boundary) {
                njs = hi;
                nhi = hi2;
            }
            const bool more = njs < J1;
            if (more) {
                st.cover(min(njs + G, nhi));
                st.fetch(njs, nhi, wnxt, nxt);
            }
            gacc<CPL, VEC, IS_MAX>(acc, arg, js + g, js + g < hi, wcur, cur);
            if (boundary) {
                gcombine<CPL, VEC, IS_MAX>(acc, arg, L);
                on_end(iv, lo, hi, cell);
                greset<CPL, VEC, IS_MAX>(acc, arg);
                ++iv;
                lo = hi;
                hi = hi2;
                cell = cell2;
                if (more) {
                    hi2 = iv + 1 < iv_end ? __ldg(P.starts + iv + 2) : hi;
                    cell2 = iv + 1 < iv_end ? __ldg(P.icells + iv + 1) : 0u;
                }
            }
            js = njs;
            return more;
        };
#pragma unroll 1
        while (step(va, wa, vb, wb) && step(vb, wb, va, wa)) {
        }
    };

    // Persistent grid: CTA-uniform tickets t = blockIdx.x, +gridDim.x, ...
    // Tickets [0, n_long) are the long cells (one CTA each, the 8 warps take
    // equal slices); the rest are blocks of 8 tasks, one per warp.
    const int64_t n_long = P.sched_counts[1], n_units = P.sched_counts[0];
    int64_t t = blockIdx.x;
#pragma unroll 1
    for (; t < n_long; t += gridDim.x) {
        const uint32_t k = __ldg(P.long_units + t);
        const int64_t cell = __ldg(P.units + 4 * size_t(k));
        const uint32_t iv = __ldg(P.units + 4 * size_t(k) + 2);
        const uint32_t lo = __ldg(P.starts + iv), hi = __ldg(P.starts + iv + 1);
        const uint32_t Ln = hi - lo;
        const uint32_t a = lo + uint32_t(uint64_t(Ln) * warp / kPoolWarps);
        const uint32_t e = lo + uint32_t(uint64_t(Ln) * (warp + 1) / kPoolWarps);
        float *s_val = s_all;  // [warps][C] partials (+ [warps][C] argmax)
        uint32_t *s_arg = reinterpret_cast<uint32_t *>(s_all + kPoolWarps * C);
        auto park_slice = [&](uint32_t, uint32_t, uint32_t, uint32_t) {
            if (g != 0) return;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int ch = st.li + q * L;
                if (ch < nch)
#pragma unroll
                    for (int x = 0; x < VEC; ++x) {
                        s_val[warp * C + ch * VEC + x] = acc[q][x];
                        if (IS_MAX) s_arg[warp * C + ch * VEC + x] = arg[IS_MAX ? q : 0][IS_MAX ? x : 0];
                    }
            }
        };
        if (e > a) {
            walk(a, e, 0u, 0u, e, park_slice);  // one "interval": the slice
        } else {
            greset<CPL, VEC, IS_MAX>(acc, arg);
            park_slice(0u, 0u, 0u, 0u);
        }
        __syncthreads();
        float *out = P.out + int64_t(b) * C * P.n_cells + cell;
        const float inv = P.mean ? 1.f / float(Ln) : 1.f;
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
        __syncthreads();  // s_val is reused by the next ticket
    }

    // ---- regular work: one TASK (a run of consecutive units, one contiguous
    // point range, units.cu) per warp, walked as one stream -------------------
    if (P.long_only) return;
    float *s_tile = s_all + warp * C * kUnitPitch;
    const int64_t n_cells = P.n_cells;
    const int64_t n_tasks = P.sched_counts[2];
    const uint2 *units2 = reinterpret_cast<const uint2 *>(P.units);  // (cell0, ncell|has|long) per 16 B
#pragma unroll 1
    for (; (t - n_long) * kPoolWarps < n_tasks; t += gridDim.x) {
        const int64_t k = (t - n_long) * kPoolWarps + warp;
        if (k >= n_tasks) break;
        const uint4 ta = __ldg(P.tasks + 2 * k), tb = __ldg(P.tasks + 2 * k + 1);
        if (ta.y & kLongUnit) continue;
        uint32_t u = ta.x;
        const uint32_t u_end = ta.x + (ta.y & 0xFFFFu);
        uint2 ur = __ldg(units2 + 2 * size_t(u));
        uint2 ur_next = u + 1 < u_end ? __ldg(units2 + 2 * size_t(u + 1)) : make_uint2(0u, 0u);
        int64_t cell0 = ur.x;
        // write the current unit's output block (zeros of empty cells) and
        // make the next unit current
        auto flush_unit = [&]() {
            const int ncell = static_cast<int>(ur.y & 0xFFu);
            const uint32_t has = (ur.y >> 8) & 0xFFu;
            __syncwarp();
            float *out = P.out + int64_t(b) * C * n_cells + cell0;
            const int x = lane & 7;
            if (x < ncell) {
                const bool h = (has >> x) & 1u;
                for (int c = lane >> 3; c < C; c += 4)
                    out[int64_t(c) * n_cells + x] = h ? s_tile[c * kUnitPitch + x] : 0.f;
            }
            __syncwarp();
            ++u;
            ur = ur_next;
            cell0 = ur.x;
            if (u + 1 < u_end) ur_next = __ldg(units2 + 2 * size_t(u + 1));
        };
        if (ta.w > ta.z) {
            auto park = [&](uint32_t iv, uint32_t lo, uint32_t hi, uint32_t cell) {
                while (int64_t(cell) >= cell0 + int64_t(ur.y & 0xFFu)) flush_unit();
                const int lc = static_cast<int>(int64_t(cell) - cell0);
                const float inv = P.mean ? 1.f / float(hi - lo) : 1.f;
                // group q % G writes chunk slot q
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const int ch = st.li + q * L;
                    if (g == int(q % G) && ch < nch)
#pragma unroll
                        for (int x = 0; x < VEC; ++x) {
                            const int c = ch * VEC + x;
                            s_tile[c * kUnitPitch + lc] = acc[q][x] * inv;
                            if (IS_MAX && P.argmax)
                                P.argmax[(b * P.n_int_max + iv) * C + c] =
                                    __ldg(P.ranks + arg[IS_MAX ? q : 0][IS_MAX ? x : 0]);
                        }
                }
            };
            walk(ta.z, ta.w, tb.x, tb.y, __ldg(P.starts + tb.x + 1), park);
        }
        while (u < u_end) flush_unit();
    }
}

// lanes per point group and chunks per lane for a row of nch chunks:
// the smallest power-of-two L with ceil(nch / L) * VEC <= budget floats.
inline bool choose_group(int nch, int vec, int &L, int &lg, int &cpl) {
    const int budget = vec == 8 ? 24 : 20;
    for (lg = 0, L = 1; L <= 32; L <<= 1, ++lg) {
        cpl = (nch + L - 1) / L;
        if (cpl * vec <= budget && cpl <= kGroupMaxCpl) return true;
    }
    return false;
}

template <typename Elem, int VEC, int SRC>
int run_pool_group(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    int L, lg, cpl;
    const int nch = p.C / VEC;
    BVP_REQUIRE(choose_group(nch, VEC, L, lg, cpl), BVP_ERR_UNSUPPORTED,
                "channel count %d too large for the group kernel", p.C);
    BVP_REQUIRE(SRC == kSrcX || p.meta, BVP_ERR_INVALID,
                "the cache's point gather table (point_meta) is required");
    BVP_REQUIRE(p.units && p.tasks && p.sched_counts, BVP_ERR_INVALID,
                "the schedule's units / tasks are required (built without units?)");
    const size_t smem = std::max(size_t(kPoolWarps) * p.C * kUnitPitch * sizeof(float),
                                 size_t(kPoolWarps) * p.C * 2 * sizeof(float));
    BVP_REQUIRE(smem <= 227 * 1024, BVP_ERR_UNSUPPORTED, "channel count %d too large", p.C);
    // persistent grid: at most kGroupCtasPerSm CTAs per SM, fewer when the
    // work is small (launch bounds are host upper bounds of the device counts)
    const int64_t tickets = p.max_long + (p.long_only ? 0 : ceil_div(p.max_tasks, kPoolWarps));
    if (tickets == 0) return BVP_OK;
    const dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(
                        tickets, int64_t(kNumSms) * kGroupCtasPerSm))),
                    static_cast<unsigned>(B));
#define BVP_GROUP_LAUNCH(CPLV)                                                               \
    if (cpl == CPLV) {                                                                       \
        auto k = is_max ? pool_group_kernel<Elem, VEC, CPLV, true, SRC>                      \
                        : pool_group_kernel<Elem, VEC, CPLV, false, SRC>;                    \
        if (smem > 48 * 1024)                                                                \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        k<<<grid, kPoolThreads, smem, s>>>(p, L, lg);                                        \
        return BVP_OK;                                                                       \
    }
    BVP_GROUP_LAUNCH(1) BVP_GROUP_LAUNCH(2) BVP_GROUP_LAUNCH(3)
    BVP_GROUP_LAUNCH(4) BVP_GROUP_LAUNCH(5) BVP_GROUP_LAUNCH(6)
#undef BVP_GROUP_LAUNCH
    set_error("no group kernel for %d chunks per lane", cpl);
    return BVP_ERR_UNSUPPORTED;
}

}  // namespace bvp

