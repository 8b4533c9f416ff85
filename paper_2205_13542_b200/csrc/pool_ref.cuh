// pool_ref.cuh -- the general interval reduction: any channel count, the
// reference's arithmetic (_kernels.py:22-63).  The fallback of the chunk
// kernel (pool_ivl.cuh) for channel widths its lane layouts do not cover.
//
// One warp per interval, lanes over channels (up to 4 per lane per pass);
// the interval's points are walked in rank order 8 at a time -- the 8 ranks,
// weights and rows are all loaded before the 8 are accumulated, so a warp
// waits one memory latency per 8 points.  fp64 accumulation of the exact
// fp32 x fp32 products, one rounding per add: bit-identical to the reference
// in every mode (SUM, MEAN = acc * (1/len), MEAN_DIV = acc / len (pool_naive),
// MAX = first maximum in rank order, with its point id for autograd).
#pragma once

#include "pool_kernel.cuh"

namespace bvp {

template <typename Elem>
__device__ __forceinline__ float ref_elem(const Elem *p) {
    if constexpr (std::is_same_v<Elem, float>)
        return __ldg(p);
    else
        return __bfloat162float(*p);
}

template <typename Elem, int SRC, bool IS_MAX, bool ARG>
__global__ void __launch_bounds__(256)
pool_ref_kernel(const PoolParams P) {
    constexpr int NB = 8;  // points in flight per warp
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    const int C = P.C;
    const int64_t n_int = __ldg(P.cell_first + P.n_cells);  // the cache's sentinel
    const Elem *rows = static_cast<const Elem *>(P.rows) + int64_t(b) * P.rows_bstride;
    const float *wsrc = SRC == kSrcDist ? static_cast<const float *>(P.wsrc) + int64_t(b) * P.w_bstride
                                        : nullptr;
    float *out = P.out + int64_t(b) * C * P.n_cells;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_int;
         i += warps) {
        const uint32_t lo = __ldg(P.starts + i), hi = __ldg(P.starts + i + 1);
        const uint32_t cell = __ldg(P.icells + i);
        for (int c0 = 0; c0 < C; c0 += 128) {
            double acc[4];
            uint32_t arg[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                acc[k] = IS_MAX ? -INFINITY : 0.0;
                arg[k] = 0u;
            }
            for (uint32_t j0 = lo; j0 < hi; j0 += NB) {
                const uint32_t n = min(uint32_t(NB), hi - j0);
                const uint32_t my_p = lane < int(n) ? __ldg(P.ranks + j0 + lane) : 0u;
                float w[NB], v[NB][4];
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    const uint32_t p = __shfl_sync(0xFFFFFFFFu, my_p, u);
                    const bool ok = u < int(n);
                    const int64_t row = SRC == kSrcX ? int64_t(p) : int64_t(p / uint32_t(P.D));
                    if (SRC == kSrcX) {
                        w[u] = 1.f;
                    } else {
                        const int64_t pix = row, nn = pix / P.HW, hw = pix - nn * P.HW;
                        const uint32_t d = p - uint32_t(row) * uint32_t(P.D);
                        w[u] = ok ? __ldg(wsrc + (nn * P.D + d) * P.HW + hw) : 0.f;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int c = c0 + lane + 32 * k;
                        v[u][k] = (ok && c < C) ? ref_elem(rows + row * C + c) : 0.f;
                    }
                }
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    if (u >= int(n)) break;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const double pv = __dmul_rn(double(w[u]), double(v[u][k]));
                        if (IS_MAX) {
                            if (pv > acc[k]) {
                                acc[k] = pv;
                                if (ARG) arg[k] = j0 + u;
                            }
                        } else {
                            acc[k] = __dadd_rn(acc[k], pv);
                        }
                    }
                }
            }
            const double len = double(hi - lo);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = c0 + lane + 32 * k;
                if (c >= C) continue;
                double r = acc[k];
                if (P.mean == 1) r = r * (1.0 / len);
                else if (P.mean == 2) r = r / len;
                out[int64_t(c) * P.n_cells + cell] = static_cast<float>(r);
                if (ARG && P.argmax) P.argmax[(b * P.n_int_max + i) * C + c] = __ldg(P.ranks + arg[k]);
            }
        }
    }
}

// Zero-fill of the map (empty cells stay 0, the reference's zeroed out) and
// the reference-order kernel over every interval.
template <typename Elem, int SRC>
int run_pool_ref(const PoolParams &p, int B, bool is_max, cudaStream_t s) {
    if (!p.out_zeroed) cudaMemsetAsync(p.out, 0, size_t(B) * p.C * p.n_cells * sizeof(float), s);
    const dim3 grid(unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.n_int_max, 8),
                                                                     int64_t(kNumSms) * 16))),
                    unsigned(B));
    if (!is_max)
        pool_ref_kernel<Elem, SRC, false, false><<<grid, 256, 0, s>>>(p);
    else if (p.argmax)
        pool_ref_kernel<Elem, SRC, true, true><<<grid, 256, 0, s>>>(p);
    else
        pool_ref_kernel<Elem, SRC, true, false><<<grid, 256, 0, s>>>(p);
    return check_launch("pool_ref");
}

}  // namespace bvp
