// prefixsum.cu -- the paper's "before": LSS-style cumsum pooling on the GPU.
//
// Restates pool_prefixsum (pooling.py:162-196): the rank-ordered point values
// of every channel are materialised, a full running sum is kept (one
// device-wide scan over the C x n_in values, 64-bit like the reference), and
// each interval is the difference of the running sum at its two ends.  The
// waste is deliberate: it reproduces the paper's aggregation
// baseline ("prefix sum -> interval reduction") on the same
// B200, next to the interval kernel.
#include <algorithm>

#include "scan.cuh"

namespace bvp {

__global__ void prefix_values_kernel(const float *__restrict__ features,
                                     const float *__restrict__ dist,
                                     const uint32_t *__restrict__ ranks, int64_t n_in, int C,
                                     int D, int HW, double *__restrict__ vals) {
    const int64_t total = n_in * C;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / n_in, j = e - c * n_in;
        const uint32_t p = __ldg(ranks + j);
        const uint32_t pix = p / D, d = p - pix * D;
        const uint32_t n = pix / HW, hw = pix - n * HW;
        const double w = __ldg(dist + (int64_t(n) * D + d) * HW + hw);
        vals[e] = w * double(__ldg(features + (int64_t(n) * C + c) * HW + hw));
    }
}

__global__ void prefix_diff_kernel(const double *__restrict__ ex, const double *__restrict__ total,
                                   const uint32_t *__restrict__ starts,
                                   const uint32_t *__restrict__ icells, int64_t n_in,
                                   int64_t n_int, int C, int64_t n_cells, int mean,
                                   float *__restrict__ out) {
    const int64_t all = n_int * C;
    const int64_t n = n_in * C;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < all;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / n_int, i = e - c * n_int;
        const int64_t lo = starts[i], hi = starts[i + 1];
        const int64_t a = c * n_in + lo, b = c * n_in + hi;
        const double run_b = b < n ? ex[b] : *total;
        double seg = run_b - ex[a];
        if (mean) seg /= double(hi - lo);
        out[c * n_cells + icells[i]] = float(seg);
    }
}

struct PrefixLayout {
    size_t off_vals, off_part, off_total, bytes;
};
static PrefixLayout prefix_layout(int64_t n_in, int C) {
    PrefixLayout L{};
    const int64_t n = n_in * C;
    L.off_vals = 0;
    L.off_part = (size_t(n) * 8 + 255) & ~size_t(255);
    L.off_total = (L.off_part + size_t(scan_partials_len<double>(n)) * 8 + 255) & ~size_t(255);
    L.bytes = L.off_total + 256;
    return L;
}

}  // namespace bvp

using namespace bvp;

extern "C" {

size_t bvp_prefixsum_workspace_bytes(int64_t n_in, int C) { return prefix_layout(n_in, C).bytes; }

int bvp_pool_prefixsum_f32(const float *features, const float *dist, const uint32_t *ranks,
                           const uint32_t *interval_starts, const uint32_t *interval_cells,
                           int64_t n_in, int64_t n_int, int N, int C, int H, int W, int D,
                           int64_t n_cells, int mode, float *out, void *workspace,
                           size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(mode == BVP_SUM || mode == BVP_MEAN, BVP_ERR_UNSUPPORTED,
                "prefix-sum cannot express max");
    BVP_REQUIRE(N >= 1 && C >= 0 && H >= 1 && W >= 1 && D >= 1 && n_cells >= 1 && n_in >= 0 &&
                    n_int >= 0,
                BVP_ERR_INVALID, "bad dims");
    const PrefixLayout L = prefix_layout(n_in, C);
    BVP_REQUIRE(workspace && workspace_bytes >= L.bytes, BVP_ERR_INVALID,
                "prefixsum workspace too small: need %zu bytes", L.bytes);
    BVP_REQUIRE(out || C == 0, BVP_ERR_INVALID, "null output");
    cudaStream_t s = as_stream(stream);
    if (C == 0) return BVP_OK;
    cudaMemsetAsync(out, 0, size_t(C) * n_cells * sizeof(float), s);
    if (n_int == 0 || C == 0) return check_launch("pool_prefixsum");
    BVP_REQUIRE(features && dist && ranks && interval_starts && interval_cells, BVP_ERR_INVALID,
                "null pointer argument");
    char *ws = static_cast<char *>(workspace);
    double *vals = reinterpret_cast<double *>(ws + L.off_vals);
    double *part = reinterpret_cast<double *>(ws + L.off_part);
    double *total = reinterpret_cast<double *>(ws + L.off_total);
    const int64_t n = n_in * C;
    const unsigned vb = static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 148 * 64));
    prefix_values_kernel<<<vb, 256, 0, s>>>(features, dist, ranks, n_in, C, D, H * W, vals);
    device_excl_scan<double>(vals, vals, n, part, total, s);
    const unsigned db = static_cast<unsigned>(std::min<int64_t>(ceil_div(n_int * C, 256), 148 * 64));
    prefix_diff_kernel<<<db, 256, 0, s>>>(vals, total, interval_starts, interval_cells, n_in, n_int,
                                          C, n_cells, mode == BVP_MEAN, out);
    return check_launch("pool_prefixsum");
}

}  // extern "C"
