// fusion.cu -- the camera/LiDAR shared-BEV helpers downstream of the pooled
// map (SURVEY.md §8f, next components 2-3): LiDAR flattening and bilinear
// BEV -> BEV resampling.  Reference: fusion.py:19-53 (lidar_to_bev),
// fusion.py:70-108 (grid_resample).  Both are restated bit for bit: float64
// arithmetic in the reference's operation order, explicit round-to-nearest
// intrinsics so nvcc cannot contract or reorder.
//
// lidar_to_bev is the same segmented reduction as the camera pool, over a
// dynamic cloud: quantise every point (bevgrid.py:85-98), stable-sort by cell
// with the association's own radix sort, then one thread per occupied cell
// reduces its points in input order -- np.bincount's order, so the fp64 sums
// match the reference exactly.
#include <algorithm>

#include "common.cuh"

namespace bvp {

struct LidarGrid {
    double x_min, y_min, z_min, z_max, r;
    int nx, ny;
};

// bevgrid.py:85-98 on (x, y, z) of an (M, 4) float64 cloud
__global__ void lidar_cells_kernel(const double *__restrict__ pts, int64_t M, LidarGrid g,
                                   uint32_t *__restrict__ cells) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = pts[4 * i], y = pts[4 * i + 1], z = pts[4 * i + 2];
        const double qx = floor(__ddiv_rn(__dsub_rn(x, g.x_min), g.r));
        const double qy = floor(__ddiv_rn(__dsub_rn(y, g.y_min), g.r));
        uint32_t c = kOOR;
        if (qx >= 0.0 && qx < double(g.nx) && qy >= 0.0 && qy < double(g.ny) && z >= g.z_min &&
            z < g.z_max)
            c = static_cast<uint32_t>(static_cast<int64_t>(qx) * g.ny + static_cast<int64_t>(qy));
        cells[i] = c;
    }
}

// One thread per occupied cell: count, reduced intensity, reduced height
// (fusion.py:37-52).  out (3, n_cells) is zero-filled by the caller.
__global__ void lidar_reduce_kernel(const double *__restrict__ pts,
                                    const uint32_t *__restrict__ ranks,
                                    const uint32_t *__restrict__ starts,
                                    const uint32_t *__restrict__ icells,
                                    const int64_t *__restrict__ counts, int mode, int64_t n_cells,
                                    float *__restrict__ out) {
    const int64_t n_int = counts[1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_int;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t lo = starts[i], hi = starts[i + 1], cell = icells[i];
        double a = 0.0, h = 0.0;
        if (mode == BVP_MAX) {
            a = -INFINITY;
            h = -INFINITY;
        }
        for (uint32_t j = lo; j < hi; ++j) {
            const int64_t p = ranks[j];
            const double inten = pts[4 * p + 3], height = pts[4 * p + 2];
            if (mode == BVP_MAX) {  // np.maximum.at: keep the first of equal values
                a = a >= inten ? a : inten;
                h = h >= height ? h : height;
            } else {
                a = __dadd_rn(a, inten);
                h = __dadd_rn(h, height);
            }
        }
        const double cnt = double(hi - lo);
        if (mode == BVP_MEAN) {
            a = __ddiv_rn(a, cnt);
            h = __ddiv_rn(h, cnt);
        }
        out[cell] = static_cast<float>(cnt);
        out[n_cells + cell] = static_cast<float>(a);
        out[2 * n_cells + cell] = static_cast<float>(h);
    }
}

struct ResampleGrid {
    double x_min, y_min, r;
    int nx, ny;
};

// fusion.py:84-107, one thread per (channel, destination cell)
__global__ void grid_resample_kernel(const float *__restrict__ src, int C, ResampleGrid s,
                                     ResampleGrid d, float *__restrict__ dst) {
    const int64_t nd = int64_t(d.nx) * d.ny;
    const int64_t total = int64_t(C) * nd;
    const double eps = 1e-9;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / nd, rem = e - c * nd;
        const int ix = static_cast<int>(rem / d.ny), iy = static_cast<int>(rem - int64_t(ix) * d.ny);
        // g = (dst_min + (i + 0.5) * dst_r - src_min) / src_r - 0.5
        double gx = __dsub_rn(__ddiv_rn(__dsub_rn(__dadd_rn(d.x_min, __dmul_rn(__dadd_rn(double(ix), 0.5), d.r)),
                                                  s.x_min),
                                        s.r),
                              0.5);
        double gy = __dsub_rn(__ddiv_rn(__dsub_rn(__dadd_rn(d.y_min, __dmul_rn(__dadd_rn(double(iy), 0.5), d.r)),
                                                  s.y_min),
                                        s.r),
                              0.5);
        const bool cov = (gx >= -eps) && (gx <= __dadd_rn(double(s.nx - 1), eps)) && (gy >= -eps) &&
                         (gy <= __dadd_rn(double(s.ny - 1), eps));
        gx = fmin(fmax(gx, 0.0), double(s.nx - 1));
        gy = fmin(fmax(gy, 0.0), double(s.ny - 1));
        const double x0 = floor(gx), y0 = floor(gy);
        const int64_t i0 = static_cast<int64_t>(x0), j0 = static_cast<int64_t>(y0);
        const int64_t i1 = min(i0 + 1, int64_t(s.nx - 1)), j1 = min(j0 + 1, int64_t(s.ny - 1));
        const double fx = fmin(fmax(__dsub_rn(gx, x0), 0.0), 1.0);
        const double fy = fmin(fmax(__dsub_rn(gy, y0), 0.0), 1.0);
        const float *sc = src + c * int64_t(s.nx) * s.ny;
        const double v00 = sc[i0 * s.ny + j0], v10 = sc[i1 * s.ny + j0];
        const double v01 = sc[i0 * s.ny + j1], v11 = sc[i1 * s.ny + j1];
        const double ox = __dsub_rn(1.0, fx), oy = __dsub_rn(1.0, fy);
        double acc = __dmul_rn(__dmul_rn(v00, ox), oy);
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(v10, fx), oy));
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(v01, ox), fy));
        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(v11, fx), fy));
        acc = __dmul_rn(acc, cov ? 1.0 : 0.0);  // interp *= mask (keeps -0.0)
        dst[e] = static_cast<float>(acc);
    }
}

}  // namespace bvp

using namespace bvp;

extern "C" {

size_t bvp_lidar_workspace_bytes(int64_t n_points, int nx, int ny) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const int64_t n_cells = int64_t(nx) * ny;
    const size_t m = size_t(n_points > 0 ? n_points : 1);
    return al(m * 4) * 2 + al(size_t(n_cells + 1) * 4) * 3 + al(16) +
           bvp_sort_workspace_bytes(n_points > 0 ? n_points : 1, n_cells);
}

int bvp_lidar_to_bev(const double *points, int64_t n_points, const double *grid, int nx, int ny,
                     int mode, float *out, void *workspace, size_t workspace_bytes,
                     void *stream) {
    BVP_REQUIRE(grid && out && nx >= 1 && ny >= 1 && n_points >= 0, BVP_ERR_INVALID,
                "bad arguments");
    BVP_REQUIRE(mode >= 0 && mode <= 2, BVP_ERR_INVALID, "bad mode %d", mode);
    BVP_REQUIRE(n_points == 0 || points, BVP_ERR_INVALID, "null points");
    const size_t need = bvp_lidar_workspace_bytes(n_points, nx, ny);
    BVP_REQUIRE(workspace && workspace_bytes >= need, BVP_ERR_INVALID,
                "lidar workspace too small: need %zu bytes", need);
    cudaStream_t s = as_stream(stream);
    const int64_t n_cells = int64_t(nx) * ny;
    cudaMemsetAsync(out, 0, size_t(3) * n_cells * sizeof(float), s);
    if (n_points == 0) return check_launch("lidar_to_bev");
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char *ws = static_cast<char *>(workspace);
    const size_t m4 = al(size_t(n_points) * 4), c4 = al(size_t(n_cells + 1) * 4);
    auto *cells = reinterpret_cast<uint32_t *>(ws);
    auto *ranks = reinterpret_cast<uint32_t *>(ws + m4);
    auto *starts = reinterpret_cast<uint32_t *>(ws + 2 * m4);
    auto *icells = reinterpret_cast<uint32_t *>(ws + 2 * m4 + c4);
    auto *cfirst = reinterpret_cast<uint32_t *>(ws + 2 * m4 + 2 * c4);
    auto *counts = reinterpret_cast<int64_t *>(ws + 2 * m4 + 3 * c4);
    char *sws = ws + 2 * m4 + 3 * c4 + al(16);
    const LidarGrid g{grid[0], grid[2], grid[4], grid[5], grid[6], nx, ny};
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(n_points, 256), 4096));
    lidar_cells_kernel<<<blocks, 256, 0, s>>>(points, n_points, g, cells);
    const int rc = bvp_sort_intervals(cells, n_points, n_cells, ranks, starts, icells, cfirst,
                                      nullptr, counts, sws,
                                      bvp_sort_workspace_bytes(n_points, n_cells), stream);
    if (rc != BVP_OK) return rc;
    const int64_t n_int_max = std::min<int64_t>(n_points, n_cells);
    lidar_reduce_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n_int_max, 256), 4096)),
                          256, 0, s>>>(points, ranks, starts, icells, counts, mode, n_cells, out);
    return check_launch("lidar_to_bev");
}

int bvp_grid_resample_f32(const float *src, int C, const double *src_grid, int src_nx,
                          int src_ny, const double *dst_grid, int dst_nx, int dst_ny, float *dst,
                          void *stream) {
    BVP_REQUIRE(C >= 0 && src_nx >= 1 && src_ny >= 1 && dst_nx >= 1 && dst_ny >= 1 && src_grid &&
                    dst_grid,
                BVP_ERR_INVALID, "bad arguments");
    BVP_REQUIRE(C == 0 || (src && dst), BVP_ERR_INVALID, "null pointer argument");
    if (C == 0) return BVP_OK;
    const ResampleGrid sg{src_grid[0], src_grid[2], src_grid[6], src_nx, src_ny};
    const ResampleGrid dg{dst_grid[0], dst_grid[2], dst_grid[6], dst_nx, dst_ny};
    const int64_t total = int64_t(C) * dst_nx * dst_ny;
    grid_resample_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), 148 * 32)),
                           256, 0, as_stream(stream)>>>(src, C, sg, dg, dst);
    return check_launch("grid_resample");
}

}  // extern "C"
