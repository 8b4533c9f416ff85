// pool_kernel.cuh -- shared definitions of the interval kernels (sm_100a):
// the launch parameters, the fp32 lane-group accumulate of the chunk kernel
// (pool_ivl.cuh), its lane-layout choice, and the exact mode's in-order walk
// of the intervals longer than a chunk.
//
// Restates the reference's interval_reduce (_kernels.py:22-63).  Sources:
//   kSrcDist : rows = NHWC features (f32 | bf16), weight = dist[n,d,h,w] (f32)
//   kSrcX    : rows = the materialised frustum x[p, :] (f32), weight = 1
#pragma once

#include <cstdlib>

#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace bvp {

constexpr int kPoolWarps = 8;
constexpr int kPoolThreads = 32 * kPoolWarps;
constexpr int kNumSms = 148;        // B200
constexpr int kGroupMaxCpl = 6;     // chunks per lane instantiated (1..6)

enum { kSrcDist = 0, kSrcX = 1 };

struct PoolParams {
    const void *rows;        // f32 NHWC features | f32 x (P,C) | bf16 NHWC context
    const void *wsrc;        // f32 dist (N,D,H,W) | bf16 logits (N,D,H,W) | unused
    const uint32_t *ranks;
    const uint32_t *starts;  // n_int + 1 entries (sentinel = n_in)
    const uint32_t *icells;
    const uint32_t *cell_first;  // n_cells + 1: first interval with cell >= c
    const uint2 *meta;           // per sorted point: (feature row, weight index)
    float *out;              // (B, C, n_cells)
    uint32_t *argmax;        // MAX only, optional: (B, n_int_max, C)
    int C, D, HW, NHW;
    int mean;
    int nx, ny;
    int64_t n_cells, n_int_max;
    // chunk schedule (work.cu); work == nullptr: not built
    const uint4 *work;
    const uint4 *splits;
    const int64_t *work_counts;
    int64_t max_work, max_splits, chunk_partials;
    int chunk;
    void *scratch;           // caller's scratch for the split partials
    size_t scratch_bytes;
    int out_zeroed;          // the caller already zero-filled out (chunk kernel skips it)
    float *partials;         // split intervals: [B][n_chunks of splits][C] (workspace)
    uint32_t *partial_arg;   // MAX: sorted position of each partial's max
    int64_t rows_bstride;    // elements of rows per batch sample
    int64_t w_bstride;       // elements of wsrc per batch sample
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


// Exact mode: one CTA per split interval (longer than a chunk), summed in rank order
// like every other cell -- but with the gathers batched.  The cell's points
// are walked in tiles of T = kExactTile / C rows: all 256 threads load the
// next tile's rows (and weights) into registers while the channel threads
// run the current tile's sequential fp64 FMAs out of shared memory, so the
// cell costs ~L / T gather latencies instead of ~L / 4.
constexpr int kExactTile = 8192;                  // floats per staged tile
constexpr int kExactRegs = kExactTile / kPoolThreads;  // per thread (32)

// The cells are the chunk schedule's split intervals (work.cu).
template <int VEC, bool IS_MAX, bool SPLITS = true>
__global__ void __launch_bounds__(kPoolThreads)
pool_exact_long_kernel(const PoolParams P) {
    extern __shared__ float s_ex[];  // [T][C] rows, [T] weights
    const int C = P.C, tid = threadIdx.x;
    const int b = blockIdx.y;
    if (int64_t(blockIdx.x) >= P.work_counts[1]) return;
    const int T = min(128, kExactTile / C);
    float *s_rows = s_ex, *s_w = s_ex + T * C;
    int64_t cell;
    uint32_t iv;
    {
        const uint4 sp = __ldg(P.splits + blockIdx.x);  // interval, cell, slot, chunks
        iv = sp.x;
        cell = sp.y;
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
BVP_DECLARE_RUN_POOL(float, __nv_bfloat16, 8, kSrcDist)  // fused.cu (precomputed softmax)
BVP_DECLARE_RUN_POOL(float, __nv_bfloat16, 1, kSrcDist)  // fused.cu
#undef BVP_DECLARE_RUN_POOL


}  // namespace bvp
