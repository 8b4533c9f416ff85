// refapi.cu -- entry points shaped exactly like the reference's native
// kernel and validators, for callers that hold the reference's own arrays.
//
//   bvp_interval_reduce_f32   _kernels.interval_reduce (_kernels.py:22-63):
//       the same arguments (ranks, starts, interval_cells, the NHWD weights
//       and NHWC features the reference's pool_interval makes at
//       pooling.py:215-216, out pre-zeroed (C, n_cells)), the same
//       arithmetic: per interval, fp64 products of fp32 inputs summed in rank
//       order (MAX: `v > acc` from -inf; MEAN: acc * (1 / len)), one fp32
//       store per channel.  Bit-identical to the reference; no schedule, no
//       workspace.  One warp per interval, lanes over channels.
//   bvp_depth_distribution_check  check_depth_distribution (lift.py:52-63):
//       min entry and the worst |sum_d p - 1| in fp64 (device results).
#include <algorithm>

#include "common.cuh"

namespace bvp {

__global__ void __launch_bounds__(256)
interval_reduce_ref_kernel(const uint32_t *__restrict__ ranks, const uint32_t *__restrict__ starts,
                           const uint32_t *__restrict__ icells, int64_t n_in, int64_t n_int,
                           const float *__restrict__ dist_t, const float *__restrict__ feats_t,
                           float *__restrict__ out, int64_t n_cells, int D, int C, int mode) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_int;
         i += warps) {
        const int64_t lo = __ldg(starts + i);
        const int64_t hi = i + 1 < n_int ? int64_t(__ldg(starts + i + 1)) : n_in;
        const uint32_t cell = __ldg(icells + i);
        for (int c0 = 0; c0 < C; c0 += 32 * 4) {  // up to 4 channels per lane per pass
            double acc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = mode == BVP_MAX ? -INFINITY : 0.0;
            for (int64_t j = lo; j < hi; ++j) {
                const uint32_t p = __ldg(ranks + j);
                const double wt = double(__ldg(dist_t + p));  // dist_t[n, h, w, d] = row p
                const float *f = feats_t + int64_t(p / uint32_t(D)) * C;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int c = c0 + lane + 32 * k;
                    if (c < C) {
                        const double v = __dmul_rn(wt, double(__ldg(f + c)));
                        if (mode == BVP_MAX) {
                            if (v > acc[k]) acc[k] = v;
                        } else {
                            acc[k] = __dadd_rn(acc[k], v);
                        }
                    }
                }
            }
            const double scale = mode == BVP_MEAN ? 1.0 / double(hi - lo) : 1.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = c0 + lane + 32 * k;
                if (c < C)
                    out[int64_t(c) * n_cells + cell] =
                        static_cast<float>(mode == BVP_MEAN ? acc[k] * scale : acc[k]);
            }
        }
    }
}

// One block per (n, 32-pixel tile): min over entries, max |sum_d - 1|.
__global__ void __launch_bounds__(256)
depth_check_kernel(const float *__restrict__ dist, int64_t NB, int D, int HW,
                   unsigned long long *__restrict__ stats) {
    const int tiles = (HW + 31) / 32;
    const int64_t n = blockIdx.x / tiles;
    const int hw = int(blockIdx.x - n * tiles) * 32 + (threadIdx.x & 31);
    const int warp = threadIdx.x >> 5;
    __shared__ double s_sum[8][32];
    __shared__ float s_min[8][32];
    double sum = 0.0;
    float mn = INFINITY;
    if (hw < HW)
        for (int d = warp; d < D; d += 8) {
            const float v = __ldg(dist + (n * D + d) * int64_t(HW) + hw);
            sum += double(v);
            mn = fminf(mn, v);
        }
    s_sum[warp][threadIdx.x & 31] = sum;
    s_min[warp][threadIdx.x & 31] = mn;
    __syncthreads();
    if (warp == 0 && hw < HW) {
        double t = 0.0;
        float m = INFINITY;
        for (int w = 0; w < 8; ++w) {
            t += s_sum[w][threadIdx.x];
            m = fminf(m, s_min[w][threadIdx.x]);
        }
        const double dev = fabs(t - 1.0);
        // non-negative doubles order like their bit patterns
        atomicMax(&stats[1], static_cast<unsigned long long>(__double_as_longlong(dev)));
        if (m < 0.f) atomicExch(&stats[0], 1ull);
    }
}

}  // namespace bvp

using namespace bvp;

extern "C" {

int bvp_interval_reduce_f32(const uint32_t *ranks, const uint32_t *interval_starts,
                            const uint32_t *interval_cells, int64_t n_in, int64_t n_int,
                            const float *dist_t, const float *feats_t, float *out,
                            int64_t n_cells, int H, int W, int D, int C, int mode,
                            void *stream) {
    (void)H;
    (void)W;
    BVP_REQUIRE(mode >= BVP_SUM && mode <= BVP_MAX, BVP_ERR_INVALID, "bad mode %d", mode);
    BVP_REQUIRE(n_in >= 0 && n_int >= 0 && D > 0 && C >= 0 && n_cells > 0, BVP_ERR_INVALID,
                "bad sizes");
    if (n_int == 0 || C == 0) return BVP_OK;
    BVP_REQUIRE(ranks && interval_starts && interval_cells && dist_t && feats_t && out,
                BVP_ERR_INVALID, "null pointer argument");
    const unsigned blocks =
        static_cast<unsigned>(std::min<int64_t>(ceil_div(n_int, 8), int64_t(148) * 16));
    interval_reduce_ref_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
        ranks, interval_starts, interval_cells, n_in, n_int, dist_t, feats_t, out, n_cells, D, C,
        mode);
    return check_launch("interval_reduce");
}

int bvp_depth_distribution_check(const float *dist, int NB, int D, int H, int W,
                                 unsigned long long *stats, void *stream) {
    BVP_REQUIRE(stats, BVP_ERR_INVALID, "null stats");
    cudaStream_t s = as_stream(stream);
    cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), s);
    if (NB == 0 || D == 0 || H * W == 0) return check_launch("depth_check");
    BVP_REQUIRE(dist && NB > 0 && D > 0 && H > 0 && W > 0, BVP_ERR_INVALID, "bad arguments");
    const int HW = H * W;
    const int64_t blocks = int64_t(NB) * ((HW + 31) / 32);
    depth_check_kernel<<<unsigned(blocks), 256, 0, s>>>(dist, NB, D, HW, stats);
    return check_launch("depth_check");
}

}  // extern "C"
