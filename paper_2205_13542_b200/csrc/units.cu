// units.cu -- the work schedule of the interval kernels (part of the cached
// association; built once per rig like the ranks).
//
// A unit is a run of <= kUnitCells consecutive cells of one BEV row whose
// intervals hold <= budget in-range points.  A single cell holding more than
// the budget is a unit of its own, flagged long: the fast kernels split it
// over all warps of a CTA (pool_long_kernel), the exact kernel walks it in
// order.  Units are listed in x-major tile order.  Bounding the work per warp
// removes the long tail of dense near-camera cells; writing every cell of a
// unit (zeros included) keeps exactly one store per output element.
//
// The point gather table (point_meta) turns every sorted point's id into its
// feature row and weight index once, so the kernels never divide.
#include <algorithm>

#include "scan.cuh"

namespace bvp {

constexpr uint32_t kLongFlag = 0x80000000u;

__device__ __forceinline__ uint32_t cell_points(const uint32_t *__restrict__ starts,
                                                const uint32_t *__restrict__ cell_first,
                                                int64_t c) {
    const uint32_t a = cell_first[c], b = cell_first[c + 1];
    return b > a ? starts[a + 1] - starts[a] : 0u;  // at most one interval per cell
}

// Greedy cut of one row tile; WRITE=false counts, WRITE=true emits.
template <bool WRITE>
__global__ void units_kernel(const uint32_t *__restrict__ starts,
                             const uint32_t *__restrict__ cell_first, int nx, int ny,
                             int tiles_y, uint32_t budget, uint32_t *__restrict__ tile_units,
                             const uint32_t *__restrict__ offsets, uint32_t *__restrict__ units,
                             uint32_t *__restrict__ long_units,
                             unsigned long long *__restrict__ n_long) {
    const int64_t ntiles = int64_t(nx) * tiles_y;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int ty = static_cast<int>(t / nx), ix = static_cast<int>(t - int64_t(ty) * nx);
        const int iy0 = ty * kUnitCells;
        const int n = min(kUnitCells, ny - iy0);
        const int64_t c0 = int64_t(ix) * ny + iy0;
        uint32_t count = 0, acc = 0;
        uint32_t out = WRITE ? offsets[t] : 0u;
        int start = 0;
        auto emit = [&](int from, int to, bool is_long) {
            if (WRITE) {
                units[2 * out] = static_cast<uint32_t>(c0 + from);
                units[2 * out + 1] = static_cast<uint32_t>(to - from) | (is_long ? kLongFlag : 0u);
                if (is_long) long_units[atomicAdd(n_long, 1ull)] = out;
                ++out;
            }
            ++count;
        };
        for (int k = 0; k < n; ++k) {
            const uint32_t p = cell_points(starts, cell_first, c0 + k);
            if (p > budget) {
                if (k > start) emit(start, k, false);
                emit(k, k + 1, true);
                start = k + 1;
                acc = 0;
                continue;
            }
            if (acc > 0 && acc + p > budget) {
                emit(start, k, false);
                start = k;
                acc = 0;
            }
            acc += p;
        }
        if (start < n) emit(start, n, false);
        if (!WRITE) tile_units[t] = count;
    }
}

// Per sorted point: (feature row = pixel, weight index into (N,D,H,W)).
__global__ void point_meta_kernel(const uint32_t *__restrict__ ranks,
                                  const int64_t *__restrict__ counts, int64_t P, int D, int HW,
                                  uint2 *__restrict__ meta) {
    const int64_t n_in = counts[0];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_in && j < P;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = ranks[j];
        const uint32_t pix = p / D, d = p - pix * D;
        const uint32_t n = pix / HW, hw = pix - n * HW;
        meta[j] = make_uint2(pix, (n * D + d) * HW + hw);
    }
}

__global__ void store_counts_kernel(const uint32_t *__restrict__ total,
                                    const unsigned long long *__restrict__ n_long,
                                    int64_t *__restrict__ out) {
    out[0] = *total;
    out[1] = static_cast<int64_t>(*n_long);
}

struct UnitsLayout {
    int64_t ntiles;
    size_t off_tile, off_part, off_total, off_long, bytes;
};
static UnitsLayout units_layout(int nx, int ny) {
    UnitsLayout L{};
    L.ntiles = int64_t(nx) * ((ny + kUnitCells - 1) / kUnitCells);
    L.off_tile = 0;
    L.off_part = (size_t(L.ntiles) * 4 + 255) & ~size_t(255);
    L.off_total = (L.off_part + size_t(scan_partials_len<uint32_t>(L.ntiles)) * 4 + 255) &
                  ~size_t(255);
    L.off_long = L.off_total + 256;
    L.bytes = L.off_long + 256;
    return L;
}

}  // namespace bvp

using namespace bvp;

extern "C" {

int64_t bvp_units_capacity(int nx, int ny, int64_t n_int_max) {
    return units_layout(nx, ny).ntiles + 2 * n_int_max;
}

size_t bvp_units_workspace_bytes(int nx, int ny) { return units_layout(nx, ny).bytes; }

int bvp_point_meta(const uint32_t *ranks, const int64_t *counts, int N, int H, int W, int D,
                   uint32_t *point_meta, void *stream) {
    BVP_REQUIRE(ranks && counts && point_meta, BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(N >= 1 && H >= 1 && W >= 1 && D >= 1, BVP_ERR_INVALID, "bad dims");
    const int64_t P = int64_t(N) * H * W * D;
    const unsigned mb = static_cast<unsigned>(std::min<int64_t>(ceil_div(P, 256), 148 * 32));
    point_meta_kernel<<<mb, 256, 0, as_stream(stream)>>>(ranks, counts, P, D, H * W,
                                                         reinterpret_cast<uint2 *>(point_meta));
    return check_launch("point_meta");
}

int bvp_make_schedule(const uint32_t *ranks, const uint32_t *interval_starts,
                      const uint32_t *cell_first, const int64_t *counts, int N, int H, int W,
                      int D, int nx, int ny, int budget, uint32_t *units, uint32_t *long_units,
                      int64_t *sched_counts, uint32_t *point_meta, void *workspace,
                      size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(ranks && interval_starts && cell_first && counts && units && long_units &&
                    sched_counts,
                BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(nx >= 1 && ny >= 1 && budget >= 1 && N >= 1 && H >= 1 && W >= 1 && D >= 1,
                BVP_ERR_INVALID, "bad arguments");
    const UnitsLayout L = units_layout(nx, ny);
    BVP_REQUIRE(workspace && workspace_bytes >= L.bytes, BVP_ERR_INVALID,
                "schedule workspace too small: need %zu bytes", L.bytes);
    cudaStream_t s = as_stream(stream);
    char *ws = static_cast<char *>(workspace);
    auto *tile_units = reinterpret_cast<uint32_t *>(ws + L.off_tile);
    auto *part = reinterpret_cast<uint32_t *>(ws + L.off_part);
    auto *total = reinterpret_cast<uint32_t *>(ws + L.off_total);
    auto *n_long = reinterpret_cast<unsigned long long *>(ws + L.off_long);
    const int tiles_y = (ny + kUnitCells - 1) / kUnitCells;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(L.ntiles, 128), 4096));
    cudaMemsetAsync(n_long, 0, sizeof(unsigned long long), s);
    units_kernel<false><<<blocks, 128, 0, s>>>(interval_starts, cell_first, nx, ny, tiles_y,
                                               uint32_t(budget), tile_units, nullptr, nullptr,
                                               nullptr, nullptr);
    device_excl_scan<uint32_t>(tile_units, tile_units, L.ntiles, part, total, s);
    units_kernel<true><<<blocks, 128, 0, s>>>(interval_starts, cell_first, nx, ny, tiles_y,
                                              uint32_t(budget), nullptr, tile_units, units,
                                              long_units, n_long);
    store_counts_kernel<<<1, 1, 0, s>>>(total, n_long, sched_counts);
    if (point_meta) {
        const int rc = bvp_point_meta(ranks, counts, N, H, W, D, point_meta, stream);
        if (rc != BVP_OK) return rc;
    }
    return check_launch("make_schedule");
}

}  // extern "C"
