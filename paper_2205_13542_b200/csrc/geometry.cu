// geometry.cu -- cold association on the GPU: frustum -> ego -> BEV cell in
// float64 with the reference's exact operation order, a stable bounded-key
// LSD radix sort of the in-range points by cell, and interval / tile tables.
//
// Reference: geometry.py:162-191 (generate_frustum), bevgrid.py:85-98
// (quantize_points), bevgrid.py:142-158 (ranks_and_intervals),
// bevgrid.py:183-203 (build_cache).  Paths relative to pkg/src/bevpool/.
#include <algorithm>
#include <cstdio>
#include <functional>

#include "common.cuh"
#include "partition.cuh"
#include "scan.cuh"

namespace bvp {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kKeysPerThread = 16;
constexpr int kSortTile = kSortThreads * kKeysPerThread;  // 4096 keys per CTA
constexpr int kMaxDigitBits = 10;
constexpr int kMaxDigits = 1 << kMaxDigitBits;
constexpr int64_t kCountSortMaxRun = 64;  // counting sort while P <= 64 * n_cells

struct GridParams {
    double x_min, y_min, z_min, z_max, r;
    int nx, ny;
    double rinv;  // RN(1/r): the quantiser's fast path (exact fallback below)
};

inline GridParams grid_params(const double *grid, int nx, int ny) {
    return GridParams{grid[0], grid[2], grid[4], grid[5], grid[6], nx, ny, 1.0 / grid[6]};
}

struct FrustumParams {
    int N, H, W, D;
    double d_min, d_step;
};

// One frustum point -> flat cell id.  Every operation is an explicit
// round-to-nearest intrinsic so nvcc cannot contract or reassociate:
//   depth = d_min + step*d                         geometry.py:95-99
//   dx = (w - cx)/fx, dy = (h - cy)/fy             geometry.py:178-179
//   p = (dx*depth, dy*depth, depth)                geometry.py:184
//   e_j = fma(R[j][2],pz, fma(R[j][1],py, R[j][0]*px)) + t_j
//        (the OpenBLAS dgemm rounding of geometry.py:185-186)
//   ix = floor((x - x_min)/r) ...                  bevgrid.py:88-96
// floor(RN(a / r)) -- numpy's floor((x - x_min) / r) -- without a division
// when possible: t = RN(a * RN(1/r)) lies within 2^-51 |t| of RN(a/r), so
// unless t is that close to an integer both floors agree; otherwise (e.g.
// quotients that are exactly integral) the IEEE division decides.
__device__ __forceinline__ double floor_div(double a, const GridParams &g) {
    const double t = __dmul_rn(a, g.rinv);
    const double k = floor(t);
    const double margin = fabs(t) * 0x1p-50 + 0x1p-1000;
    if (t - k > margin && (k + 1.0) - t > margin) return k;
    return floor(__ddiv_rn(a, g.r));
}

// Ego coordinates of frustum point (pixel ray dx, dy; depth bin d) --
// generate_frustum's rounding (geometry.py:184-186 through OpenBLAS dgemm).
__device__ __forceinline__ void ego_at(const double *__restrict__ c, const FrustumParams &f,
                                       double dx, double dy, int d, double (&e)[3]) {
    const double depth = __dadd_rn(f.d_min, __dmul_rn(f.d_step, static_cast<double>(d)));
    const double px = __dmul_rn(dx, depth), py = __dmul_rn(dy, depth), pz = depth;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double acc = __dmul_rn(__ldg(c + 4 + 3 * j), px);
        acc = __fma_rn(__ldg(c + 5 + 3 * j), py, acc);
        acc = __fma_rn(__ldg(c + 6 + 3 * j), pz, acc);
        e[j] = __dadd_rn(acc, __ldg(c + 13 + j));
    }
}

// quantize_points (bevgrid.py:85-98): flat cell id of an ego point.
__device__ __forceinline__ uint32_t quantize_ego(const double (&e)[3], const GridParams &g) {
    if (!(e[2] >= g.z_min && e[2] < g.z_max)) return kOOR;
    const double qx = floor_div(__dsub_rn(e[0], g.x_min), g);
    const double qy = floor_div(__dsub_rn(e[1], g.y_min), g);
    if (qx >= 0.0 && qx < static_cast<double>(g.nx) && qy >= 0.0 &&
        qy < static_cast<double>(g.ny))
        return static_cast<uint32_t>(static_cast<int64_t>(qx) * g.ny + static_cast<int64_t>(qy));
    return kOOR;
}

__device__ __forceinline__ uint32_t cell_at(const double *__restrict__ c, const FrustumParams &f,
                                            const GridParams &g, double dx, double dy, int d) {
    double e[3];
    ego_at(c, f, dx, dy, d, e);
    return quantize_ego(e, g);
}

// The ray of pixel (h, w) of a camera: dx = (w - cx)/fx, dy = (h - cy)/fy.
__device__ __forceinline__ void pixel_ray(const double *__restrict__ c, int h, int w, double &dx,
                                          double &dy) {
    dx = __ddiv_rn(__dsub_rn(static_cast<double>(w), __ldg(c + 2)), __ldg(c + 0));
    dy = __ddiv_rn(__dsub_rn(static_cast<double>(h), __ldg(c + 3)), __ldg(c + 1));
}

__device__ __forceinline__ uint32_t point_cell(const double *__restrict__ cams,
                                               const FrustumParams &f,
                                               const GridParams &g, int64_t p) {
    const int d = static_cast<int>(p % f.D);
    int64_t rest = p / f.D;
    const int w = static_cast<int>(rest % f.W);
    rest /= f.W;
    const int h = static_cast<int>(rest % f.H);
    const int n = static_cast<int>(rest / f.H);
    const double *c = cams + 16 * n;
    double dx, dy;
    pixel_ray(c, h, w, dx, dy);
    return cell_at(c, f, g, dx, dy, d);
}

// generate_frustum: coords[p] = ego (x, y, z) of point p, (P, 3) fp64.
__global__ void frustum_points_kernel(const double *__restrict__ cams, FrustumParams f, int64_t P,
                                      double *__restrict__ coords) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int d = static_cast<int>(p % f.D);
        int64_t rest = p / f.D;
        const int w = static_cast<int>(rest % f.W);
        rest /= f.W;
        const int h = static_cast<int>(rest % f.H);
        const int n = static_cast<int>(rest / f.H);
        const double *c = cams + 16 * n;
        double dx, dy, e[3];
        pixel_ray(c, h, w, dx, dy);
        ego_at(c, f, dx, dy, d, e);
        coords[3 * p] = e[0];
        coords[3 * p + 1] = e[1];
        coords[3 * p + 2] = e[2];
    }
}

__global__ void quantize_points_kernel(const double *__restrict__ coords, int64_t M, GridParams g,
                                       uint32_t *__restrict__ cells) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double e[3] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
        cells[i] = quantize_ego(e, g);
    }
}

__global__ void frustum_cells_kernel(const double *__restrict__ cams, FrustumParams f,
                                     GridParams g, int64_t P, uint32_t *__restrict__ cells) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x)
        cells[p] = point_cell(cams, f, g, p);
}

// Pass-0 front end of the sort: (optionally) computes the cells, counts
// points per cell, and writes the tile histogram of the first radix digit.
// Tile t covers point ids [t*kSortTile, (t+1)*kSortTile).
template <bool COMPUTE>
__global__ void __launch_bounds__(kSortThreads)
pass0_front_kernel(const double *__restrict__ cams, FrustumParams f, GridParams g,
                   int64_t P, uint32_t *__restrict__ cells, uint32_t *__restrict__ cell_count,
                   int digit_bits, uint32_t *__restrict__ hist, int64_t n_tiles) {
    __shared__ uint32_t sh[kMaxDigits];
    const int n_digits = 1 << digit_bits;
    for (int i = threadIdx.x; i < n_digits; i += kSortThreads) sh[i] = 0;
    __syncthreads();
    const int64_t base = blockIdx.x * (int64_t)kSortTile;
    const uint32_t mask = n_digits - 1;
#pragma unroll 4
    for (int k = 0; k < kKeysPerThread; ++k) {
        const int64_t p = base + k * kSortThreads + threadIdx.x;
        if (p >= P) break;
        uint32_t c;
        if (COMPUTE) {
            c = point_cell(cams, f, g, p);
            cells[p] = c;
        } else {
            c = cells[p];
        }
        if (c != kOOR) {
            atomicAdd(&cell_count[c], 1u);
            atomicAdd(&sh[c & mask], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_digits; i += kSortThreads)
        hist[(int64_t)i * n_tiles + blockIdx.x] = sh[i];
}

// Histogram of the current digit over sorted positions [0, n_valid).
__global__ void __launch_bounds__(kSortThreads)
radix_upsweep_kernel(const uint32_t *__restrict__ keys, const int64_t *__restrict__ counts,
                     int shift, int digit_bits, uint32_t *__restrict__ hist, int64_t n_tiles) {
    __shared__ uint32_t sh[kMaxDigits];
    const int n_digits = 1 << digit_bits;
    for (int i = threadIdx.x; i < n_digits; i += kSortThreads) sh[i] = 0;
    __syncthreads();
    const int64_t n_valid = counts[0];
    const int64_t base = blockIdx.x * (int64_t)kSortTile;
    const uint32_t mask = n_digits - 1;
    for (int k = 0; k < kKeysPerThread; ++k) {
        const int64_t j = base + k * kSortThreads + threadIdx.x;
        if (j >= n_valid) break;
        atomicAdd(&sh[(keys[j] >> shift) & mask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_digits; i += kSortThreads)
        hist[(int64_t)i * n_tiles + blockIdx.x] = sh[i];
}

// Stable scatter of one LSD pass.  Warp w of tile t owns the contiguous key
// range [t*kSortTile + w*512, +512) and walks it in index order 32 keys at a
// time; __match_any_sync gives each key its rank among equal digits of the
// round, per-warp running counters (exclusive across warps, seeded with the
// device-wide digit-major scan of the tile histograms) give the rest.  No
// atomics decide positions, so ties keep their input order (stability).
template <bool PASS0>
__global__ void __launch_bounds__(kSortThreads)
radix_scatter_kernel(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                     int64_t n_total, const int64_t *__restrict__ counts, int shift,
                     int digit_bits, const uint32_t *__restrict__ hist_scanned, int64_t n_tiles,
                     uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out) {
    __shared__ uint32_t wcnt[kSortWarps][kMaxDigits];
    const int n_digits = 1 << digit_bits;
    const uint32_t mask = n_digits - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_valid = PASS0 ? n_total : counts[0];
    const int64_t tile_base = blockIdx.x * (int64_t)kSortTile;
    const int64_t wbase = tile_base + warp * (32 * kKeysPerThread);
    for (int i = lane; i < n_digits; i += 32) wcnt[warp][i] = 0;
    __syncwarp();
    uint32_t key[kKeysPerThread];
    bool ok[kKeysPerThread];
#pragma unroll
    for (int r = 0; r < kKeysPerThread; ++r) {
        const int64_t j = wbase + r * 32 + lane;
        uint32_t k = kOOR;
        if (j < n_valid) k = keys_in[j];
        ok[r] = (k != kOOR);
        key[r] = k;
    }
#pragma unroll
    for (int r = 0; r < kKeysPerThread; ++r) {
        const uint32_t dg = ok[r] ? ((key[r] >> shift) & mask) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, dg);
        if (ok[r] && lane == __ffs(peers) - 1) wcnt[warp][dg] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_digits; i += kSortThreads) {
        uint32_t run = hist_scanned[(int64_t)i * n_tiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t t = wcnt[w][i];
            wcnt[w][i] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kKeysPerThread; ++r) {
        const int64_t j = wbase + r * 32 + lane;
        const uint32_t dg = ok[r] ? ((key[r] >> shift) & mask) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, dg);
        uint32_t pos = 0;
        if (ok[r]) pos = wcnt[warp][dg] + __popc(peers & lanemask_lt());
        __syncwarp();
        if (ok[r] && lane == __ffs(peers) - 1) wcnt[warp][dg] += __popc(peers);
        __syncwarp();
        if (ok[r]) {
            if (keys_out) keys_out[pos] = key[r];
            vals_out[pos] = PASS0 ? static_cast<uint32_t>(j) : vals_in[j];
        }
    }
}

// packed[c] = (count > 0) << 32 | count: one scan yields both the first
// rank of every cell (low word) and its interval index (high word).
struct PackCount {  // applied as the scan loads each cell's count
    __device__ __forceinline__ unsigned long long operator()(uint32_t k) const {
        return (static_cast<unsigned long long>(k > 0) << 32) | k;
    }
};

__global__ void make_intervals_kernel(const uint32_t *__restrict__ cell_count,
                                      const unsigned long long *__restrict__ scanned,
                                      const unsigned long long *__restrict__ total,
                                      int64_t n_cells, uint32_t *__restrict__ starts,
                                      uint32_t *__restrict__ icells,
                                      uint32_t *__restrict__ cell_first,
                                      int64_t *__restrict__ counts,
                                      uint32_t *__restrict__ long_list = nullptr,
                                      uint32_t *__restrict__ n_long = nullptr) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_cells;
         c += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long ex = scanned[c];
        const uint32_t iv = static_cast<uint32_t>(ex >> 32);
        const uint32_t k = cell_count[c];
        if (k > 0) {
            starts[iv] = static_cast<uint32_t>(ex & 0xFFFFFFFFull);
            icells[iv] = static_cast<uint32_t>(c);
            // runs longer than 256 points: seg_sort_long_kernel's
            if (long_list && k > 256u) long_list[atomicAdd(n_long, 1u)] = iv;
        }
        cell_first[c] = iv;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long t = *total;
        const uint32_t n_in = static_cast<uint32_t>(t & 0xFFFFFFFFull);
        const uint32_t n_int = static_cast<uint32_t>(t >> 32);
        starts[n_int] = n_in;
        cell_first[n_cells] = n_int;
        counts[0] = n_in;
        counts[1] = n_int;
    }
}

__global__ void interval_of_point_kernel(const uint32_t *__restrict__ cells, int64_t P,
                                         const unsigned long long *__restrict__ scanned,
                                         uint32_t *__restrict__ iop) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = cells[p];
        iop[p] = (c == kOOR) ? kOOR : static_cast<uint32_t>(scanned[c] >> 32);
    }
}

// ---- counting sort (bounded keys, short runs) ------------------------------
// Used when the mean run per key is short (frustum association: ~15 points per
// cell).  (1) count_front: cell of every point and an arrival slot in its cell
// from the per-cell counter (atomicAdd's return value); (2) the per-cell
// counts are scanned into interval tables (shared with the radix path); (3)
// count_scatter: ranks[first_rank(cell) + slot] = p; (4) seg_sort: the slots
// follow atomic arrival order, so every interval's run of point indices is
// sorted ascending -- which restores the reference's stable order (ties by
// point index, bevgrid.py:149) exactly.

// Slot of this lane's point among the warp's points of the same cell: one
// atomic per distinct cell (leader lane), ranks among peers by lane.
__device__ __forceinline__ uint32_t claim_slot(uint32_t c, uint32_t *__restrict__ cell_count) {
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, c);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (c != kOOR && (threadIdx.x & 31) == leader) base = atomicAdd(&cell_count[c], __popc(peers));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    return c != kOOR ? base + __popc(peers & lanemask_lt()) : 0u;
}

constexpr int kFrontPix = 32;    // pixels per tile (one per lane)
constexpr int kFrontDepth = 64;  // depth bins per shared-memory pass

// Tile t covers 32 consecutive pixels in column-major order q = (n*W + w)*H +
// h: lanes run down an image column, i.e. along one vertical line in 3-D.
// For a near-level camera that line projects into one or two BEV cells, so a
// warp's 32 points at one depth bin mostly share a cell: one atomic claims
// consecutive slots for all of them (in point order), and count_scatter's
// stores for them are contiguous.  The sort stays exact for any rig.
__device__ __forceinline__ uint32_t tile_pixel(const FrustumParams &f, uint32_t q) {
    const uint32_t h = q % f.H, nw = q / f.H;
    const uint32_t w = nw % f.W, n = nw / f.W;
    return (n * f.H + h) * f.W + w;
}

// Frustum points, tile by tile (warps stride the depth bins).  The ray's two
// divisions run once per pixel and warp.  Cells and slots are staged in
// shared memory and written as contiguous per-pixel runs of depth bins.
__global__ void __launch_bounds__(256)
count_front_kernel(const double *__restrict__ cams, FrustumParams f, GridParams g,
                   uint32_t *__restrict__ cells, uint32_t *__restrict__ cell_count,
                   uint32_t *__restrict__ slot) {
    __shared__ uint32_t s_cell[kFrontDepth][kFrontPix + 1], s_slot[kFrontDepth][kFrontPix + 1];
    __shared__ uint32_t s_pix[kFrontPix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t npix = static_cast<uint32_t>(f.N) * f.H * f.W;
    const uint32_t ntiles = (npix + kFrontPix - 1) / kFrontPix;
    const uint32_t D = static_cast<uint32_t>(f.D);
    // programmatic dependent launch both ways: the scan after this kernel
    // may be scheduled now (it waits for this grid's completion), and this
    // kernel's geometry runs before its wait for the zero fill ahead of it
    asm volatile("griddepcontrol.launch_dependents;");
    bool waited = false;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t q = tile * kFrontPix + lane;
        const bool valid = q < npix;
        const uint32_t h = q % f.H, nw = q / f.H;
        const uint32_t w = nw % f.W, n = valid ? nw / f.W : 0;
        if (warp == 0) s_pix[lane] = (n * f.H + h) * f.W + w;
        const double *c = cams + 16 * n;
        double dx, dy;
        pixel_ray(c, static_cast<int>(h), static_cast<int>(w), dx, dy);
        const int npx = static_cast<int>(min(npix - tile * kFrontPix, uint32_t(kFrontPix)));
        for (uint32_t d0 = 0; d0 < D; d0 += kFrontDepth) {
            const int nd = static_cast<int>(min(D - d0, uint32_t(kFrontDepth)));
            for (int dd = warp; dd < nd; dd += 8) {
                const uint32_t cc = valid ? cell_at(c, f, g, dx, dy, static_cast<int>(d0) + dd)
                                          : kOOR;
                if (!waited) {  // the counters' zero fill (PDL)
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    waited = true;
                }
                s_slot[dd][lane] = claim_slot(cc, cell_count);
                s_cell[dd][lane] = cc;
            }
            __syncthreads();
            for (int i = warp; i < npx; i += 8) {
                const uint32_t p0 = s_pix[i] * D + d0;
                for (int dd = lane; dd < nd; dd += 32) {
                    cells[p0 + dd] = s_cell[dd][i];
                    slot[p0 + dd] = s_slot[dd][i];
                }
            }
            __syncthreads();
        }
    }
}

// Given cells (no geometry): points in index order, one aggregated atomic per
// distinct cell of a warp.
__global__ void __launch_bounds__(256)
count_cells_kernel(const uint32_t *__restrict__ cells, int64_t P,
                   uint32_t *__restrict__ cell_count, uint32_t *__restrict__ slot) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < P; base += stride) {
        const int64_t p = base + threadIdx.x;
        const uint32_t cc = p < P ? cells[p] : kOOR;
        const uint32_t sl = claim_slot(cc, cell_count);
        if (p < P) slot[p] = sl;
    }
}

__device__ __forceinline__ void scatter_point(uint32_t p, uint32_t c, uint32_t sl,
                                              const unsigned long long *__restrict__ scanned,
                                              uint32_t *__restrict__ ranks, uint32_t &iv) {
    iv = kOOR;
    if (c == kOOR) return;
    const unsigned long long e = __ldg(scanned + c);
    ranks[static_cast<uint32_t>(e & 0xFFFFFFFFull) + sl] = p;
    iv = static_cast<uint32_t>(e >> 32);
}

// ranks[first(cell) + slot] = p (unsorted within a cell) and the interval of
// every point.  scanned[c] = (interval index << 32) | first rank.  Frustum
// layout: the tile of count_front_kernel read as per-pixel runs, then walked
// depth-major so a warp's stores land on neighbouring cells.
__global__ void __launch_bounds__(256)
count_scatter_kernel(const uint32_t *__restrict__ cells, const uint32_t *__restrict__ slot,
                     FrustumParams f, const unsigned long long *__restrict__ scanned,
                     uint32_t *__restrict__ ranks, uint32_t *__restrict__ iop) {
    __shared__ uint32_t s_cell[kFrontDepth][kFrontPix + 1], s_slot[kFrontDepth][kFrontPix + 1];
    __shared__ uint32_t s_pix[kFrontPix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t npix = static_cast<uint32_t>(f.N) * f.H * f.W;
    const uint32_t ntiles = (npix + kFrontPix - 1) / kFrontPix;
    const uint32_t D = static_cast<uint32_t>(f.D);
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int npx = static_cast<int>(min(npix - tile * kFrontPix, uint32_t(kFrontPix)));
        if (warp == 0 && lane < npx) s_pix[lane] = tile_pixel(f, tile * kFrontPix + lane);
        __syncthreads();
        for (uint32_t d0 = 0; d0 < D; d0 += kFrontDepth) {
            const int nd = static_cast<int>(min(D - d0, uint32_t(kFrontDepth)));
            for (int i = warp; i < npx; i += 8) {
                const uint32_t p0 = s_pix[i] * D + d0;
                for (int dd = lane; dd < nd; dd += 32) {
                    s_cell[dd][i] = cells[p0 + dd];
                    s_slot[dd][i] = slot[p0 + dd];
                }
            }
            __syncthreads();
            for (int dd = warp; dd < nd; dd += 8) {
                uint32_t iv = kOOR;
                if (lane < npx)
                    scatter_point(s_pix[lane] * D + d0 + dd, s_cell[dd][lane], s_slot[dd][lane],
                                  scanned, ranks, iv);
                s_slot[dd][lane] = iv;
            }
            __syncthreads();
            if (iop)
                for (int i = warp; i < npx; i += 8) {
                    const uint32_t p0 = s_pix[i] * D + d0;
                    for (int dd = lane; dd < nd; dd += 32) iop[p0 + dd] = s_slot[dd][i];
                }
            __syncthreads();
        }
    }
}

__global__ void count_scatter_flat_kernel(const uint32_t *__restrict__ cells,
                                          const uint32_t *__restrict__ slot, int64_t P,
                                          const unsigned long long *__restrict__ scanned,
                                          uint32_t *__restrict__ ranks,
                                          uint32_t *__restrict__ iop) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint32_t iv;
        scatter_point(static_cast<uint32_t>(p), cells[p], slot[p], scanned, ranks, iv);
        if (iop) iop[p] = iv;
    }
}

// The point gather table of the interval kernels (work.cu point_meta_kernel),
// written by the run sorts as each run's final order is known: per sorted
// point its feature row (pixel) and weight index into (N, D, H, W).
struct MetaOut {
    uint2 *meta;  // null: not wanted
    uint32_t D, HW;
    __device__ __forceinline__ void put(uint32_t j, uint32_t p) const {
        const uint32_t pix = p / D, d = p - pix * D;
        const uint32_t n = pix / HW, hw = pix - n * HW;
        meta[j] = make_uint2(pix, (n * D + d) * HW + hw);
    }
};

// Ascending bitonic sort of a run of L <= 32 K values held K per lane
// (element lane + 32 m); missing elements are +inf.  mo.meta: also the run's
// gather-table entries (r's offset in ranks is lo).
template <int K>
__device__ __forceinline__ void warp_sort_run(uint32_t *r, int L, int lane,
                                              MetaOut mo = MetaOut{nullptr, 1u, 1u},
                                              uint32_t lo = 0u) {
    uint32_t v[K];
#pragma unroll
    for (int m = 0; m < K; ++m) v[m] = lane + 32 * m < L ? r[lane + 32 * m] : 0xFFFFFFFFu;
#pragma unroll
    for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {  // partner in the same lane
#pragma unroll
                for (int m = 0; m < K; ++m) {
                    const int m2 = m ^ (j >> 5);
                    if (m2 > m) {
                        const bool up = ((32 * m) & k) == 0;
                        const uint32_t lo = min(v[m], v[m2]), hi = max(v[m], v[m2]);
                        v[m] = up ? lo : hi;
                        v[m2] = up ? hi : lo;
                    }
                }
            } else {
#pragma unroll
                for (int m = 0; m < K; ++m) {
                    const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v[m], j);
                    const bool up = ((lane + 32 * m) & k) == 0, lower = (lane & j) == 0;
                    v[m] = (lower == up) ? min(v[m], o) : max(v[m], o);
                }
            }
        }
    }
#pragma unroll
    for (int m = 0; m < K; ++m)
        if (lane + 32 * m < L) {
            r[lane + 32 * m] = v[m];
            if (mo.meta) mo.put(lo + lane + 32 * m, v[m]);
        }
}

// Ascending bitonic sort of a[0, L) by `nthreads` cooperating threads (the
// all-ascending form: a mirror compare opens each merge, half-cleaners
// follow).  Positions >= L act as +inf, so compares reaching past L are
// skipped and nothing is padded.  `sync` orders the stages.
template <typename Sync>
__device__ __forceinline__ void bitonic_sort(uint32_t *a, int L, int tid, int nthreads,
                                             Sync sync) {
    int lgn = 0;
    while ((1 << lgn) < L) ++lgn;
    const int half = 1 << (lgn - 1);
    for (int lk = 1; lk <= lgn; ++lk) {
        for (int lj = lk - 1; lj >= 0; --lj) {
            const int j = 1 << lj;
            for (int i = tid; i < half; i += nthreads) {
                const int blk = i >> lj, off = i & (j - 1);
                int lo, hi;
                if (lj == lk - 1) {  // mirror compare within blocks of 2^lk
                    lo = (blk << lk) + off;
                    hi = (blk << lk) + (1 << lk) - 1 - off;
                } else {
                    lo = (blk << (lj + 1)) + off;
                    hi = lo + j;
                }
                if (hi < L) {
                    const uint32_t x = a[lo], y = a[hi];
                    if (x > y) {
                        a[lo] = y;
                        a[hi] = x;
                    }
                }
            }
            sync();
        }
    }
}

constexpr int kSegCtaMax = 8192;   // ... by one CTA: 8 warp-sorted slices, merged by rank

__device__ __forceinline__ void warp_sort_any(uint32_t *r, int L, int lane) {
    if (L <= 32) warp_sort_run<1>(r, L, lane);
    else if (L <= 64) warp_sort_run<2>(r, L, lane);
    else if (L <= 128) warp_sort_run<4>(r, L, lane);
    else if (L <= 256) warp_sort_run<8>(r, L, lane);
    else if (L <= 512) warp_sort_run<16>(r, L, lane);
    else warp_sort_run<32>(r, L, lane);
}


// One warp per interval, runs of <= 256 points sorted in registers; longer
// runs are seg_sort_long_kernel's (a separate kernel on a forked stream, so
// this one keeps the short runs' register budget and occupancy).
__global__ void __launch_bounds__(256)
seg_sort_warp_kernel(uint32_t *__restrict__ ranks, const uint32_t *__restrict__ starts,
                     const int64_t *__restrict__ counts, MetaOut mo) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_int = counts[1];
    const int64_t nwarps = int64_t(gridDim.x) * 8;
    for (int64_t iv = int64_t(blockIdx.x) * 8 + warp; iv < n_int; iv += nwarps) {
        const uint32_t lo = __ldg(starts + iv);
        const int L = static_cast<int>(__ldg(starts + iv + 1) - lo);
        if (L <= 1) {
            if (L == 1 && mo.meta && lane == 0) mo.put(lo, ranks[lo]);
            continue;
        }
        if (L <= 32) warp_sort_run<1>(ranks + lo, L, lane, mo, lo);
        else if (L <= 64) warp_sort_run<2>(ranks + lo, L, lane, mo, lo);
        else if (L <= 128) warp_sort_run<4>(ranks + lo, L, lane, mo, lo);
        else if (L <= 256) warp_sort_run<8>(ranks + lo, L, lane, mo, lo);
        // longer runs: seg_sort_long_kernel, concurrently
    }
}

// One CTA per queued run (> 256 points): up to kSegCtaMax the run is staged
// in shared memory, each warp sorts one slice in registers, and every value
// goes straight to its
// final place = its index in its slice + the number of smaller values in each
// other slice (binary searches; the values -- point ids -- are distinct);
// beyond, an in-place bitonic sort in global memory (correct for any length;
// only degenerate grids with huge cells get there).
__global__ void __launch_bounds__(256)
seg_sort_long_kernel(uint32_t *__restrict__ ranks, const uint32_t *__restrict__ starts,
                     const uint32_t *__restrict__ long_list,
                     const uint32_t *__restrict__ n_long, MetaOut mo) {
    __shared__ uint32_t sh[kSegCtaMax];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nl = *n_long;
    for (uint32_t k = blockIdx.x; k < nl; k += gridDim.x) {
        const uint32_t iv = long_list[k];
        const uint32_t lo = starts[iv];
        const int L = static_cast<int>(starts[iv + 1] - lo);
        uint32_t *r = ranks + lo;
        if (L > kSegCtaMax) {
            bitonic_sort(r, L, threadIdx.x, blockDim.x, []() { __syncthreads(); });
            __syncthreads();
            if (mo.meta)
                for (int i = threadIdx.x; i < L; i += blockDim.x) mo.put(lo + i, r[i]);
            continue;
        }
        for (int i = threadIdx.x; i < L; i += blockDim.x) sh[i] = r[i];
        __syncthreads();
        const int cs = (L + 7) / 8;
        const int a0 = min(L, warp * cs), a1 = min(L, a0 + cs);
        if (a1 > a0) warp_sort_any(sh + a0, a1 - a0, lane);
        __syncthreads();
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
            const uint32_t x = sh[i];
            const int own = i / cs;
            int pos = i - own * cs;
            for (int b = 0; b < 8; ++b) {
                if (b == own) continue;
                int l = min(L, b * cs), h = min(L, l + cs);
                while (l < h) {  // first index in slice b with value > x
                    const int m = (l + h) >> 1;
                    if (sh[m] < x) l = m + 1;
                    else h = m;
                }
                pos += l - min(L, b * cs);
            }
            r[pos] = x;
            if (mo.meta) mo.put(lo + pos, x);
        }
        __syncthreads();
    }
}

__global__ void zero_words3_kernel(uint32_t *__restrict__ a, int64_t na, uint32_t *__restrict__ b,
                                   int64_t nb, uint32_t *__restrict__ c, int64_t nc) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < na + nb + nc; i += stride) {
        if (i < na) a[i] = 0u;
        else if (i < na + nb) b[i - na] = 0u;
        else c[i - na - nb] = 0u;
    }
}

// ---- workspace layout -------------------------------------------------------
struct SortLayout {
    int key_bits, passes, digit_bits;
    int64_t n_tiles, hist_len;
    size_t off_count, off_packed, off_keys_a, off_vals_a, off_keys_b, off_vals_b, off_hist,
        off_part64, off_part32, off_total64, off_total32, off_long, off_nlong, bytes;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static SortLayout sort_layout(int64_t P, int64_t n_cells) {
    SortLayout L{};
    int bits = 1;
    while (bits < 32 && (int64_t(1) << bits) < n_cells) ++bits;  // keys < n_cells
    L.key_bits = bits;
    L.passes = (bits + kMaxDigitBits - 1) / kMaxDigitBits;
    L.digit_bits = (bits + L.passes - 1) / L.passes;
    L.n_tiles = ceil_div(P, kSortTile);
    L.hist_len = (int64_t(1) << L.digit_bits) * L.n_tiles;
    size_t o = 0;
    L.off_count = o; o = align256(o + 4 * size_t(n_cells));
    L.off_packed = o; o = align256(o + 8 * size_t(n_cells));
    L.off_keys_a = o; o = align256(o + 4 * size_t(P));
    L.off_vals_a = o; o = align256(o + 4 * size_t(P));
    L.off_keys_b = o; o = align256(o + 4 * size_t(P));
    L.off_vals_b = o; o = align256(o + 4 * size_t(P));
    L.off_hist = o; o = align256(o + 4 * size_t(L.hist_len));
    L.off_part64 = o; o = align256(o + 8 * size_t(scan_partials_len<unsigned long long>(n_cells)));
    L.off_part32 = o; o = align256(o + 4 * size_t(scan_partials_len<uint32_t>(L.hist_len)));
    L.off_total64 = o; o = align256(o + 8);
    L.off_total32 = o; o = align256(o + 8);
    L.off_long = o; o = align256(o + 4 * size_t(n_cells));
    L.off_nlong = o; o = align256(o + 8);
    L.bytes = o;
    return L;
}

// Optional work a caller hangs on the sort: `on_tables` runs (on a forked
// stream) as soon as the interval tables exist, beside the rank scatter and
// run sorts; `on_ranks` follows the final ranks on the main stream.
using SortHook = std::function<int(cudaStream_t)>;

static int sort_impl(const double *cams, const FrustumParams *fp, const GridParams *gp,
                     uint32_t *cells, int64_t P, int64_t n_cells, uint32_t *ranks,
                     uint32_t *starts, uint32_t *icells, uint32_t *cell_first, uint32_t *iop,
                     int64_t *counts, void *ws, size_t ws_bytes, cudaStream_t s,
                     const SortHook *on_tables = nullptr, const SortHook *on_ranks = nullptr,
                     uint32_t *point_meta = nullptr) {
    const SortLayout L = sort_layout(P, n_cells);
    BVP_REQUIRE(ws != nullptr && ws_bytes >= L.bytes, BVP_ERR_INVALID,
                "sort workspace too small: need %zu bytes, got %zu", L.bytes, ws_bytes);
    BVP_REQUIRE(P > 0 && P < (int64_t(1) << 32) - 1, BVP_ERR_INVALID,
                "point count %lld outside [1, 2^32-1)", (long long)P);
    BVP_REQUIRE(n_cells > 0 && n_cells < (int64_t(1) << 32) - 1, BVP_ERR_INVALID,
                "cell count %lld outside [1, 2^32-1)", (long long)n_cells);
    char *w = static_cast<char *>(ws);
    auto *cell_count = reinterpret_cast<uint32_t *>(w + L.off_count);
    auto *packed = reinterpret_cast<unsigned long long *>(w + L.off_packed);
    uint32_t *ka = reinterpret_cast<uint32_t *>(w + L.off_keys_a);
    uint32_t *va = reinterpret_cast<uint32_t *>(w + L.off_vals_a);
    uint32_t *kb = reinterpret_cast<uint32_t *>(w + L.off_keys_b);
    uint32_t *vb = reinterpret_cast<uint32_t *>(w + L.off_vals_b);
    auto *hist = reinterpret_cast<uint32_t *>(w + L.off_hist);
    auto *part64 = reinterpret_cast<unsigned long long *>(w + L.off_part64);
    auto *part32 = reinterpret_cast<uint32_t *>(w + L.off_part32);
    auto *total64 = reinterpret_cast<unsigned long long *>(w + L.off_total64);
    auto *total32 = reinterpret_cast<uint32_t *>(w + L.off_total32);

    const unsigned cb = static_cast<unsigned>(std::min<int64_t>(ceil_div(n_cells, 256), 4096));
    if (P <= kCountSortMaxRun * n_cells) {  // counting sort: short runs per key
        uint32_t *slot = ka;
        auto *long_list = reinterpret_cast<uint32_t *>(w + L.off_long);
        auto *n_long = reinterpret_cast<uint32_t *>(w + L.off_nlong);
        size_t flag_bytes = 0;
        void *flags = scan_flags(part64, n_cells, &flag_bytes);
        // the per-cell counters, the long-run count and the scan's flags in
        // one launch (three memsets measured as three dependent launches)
        zero_words3_kernel<<<cb, 256, 0, s>>>(cell_count, n_cells, n_long, 2,
                                              static_cast<uint32_t *>(flags),
                                              int64_t(flag_bytes / 4));
        if (cams) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148 * 8);
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute at1[1];
            at1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at1[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at1;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, count_front_kernel, cams, *fp, *gp, cells, cell_count, slot);
        } else {
            count_cells_kernel<<<148 * 8, 256, 0, s>>>(cells, P, cell_count, slot);
        }
        device_excl_scan_xf<unsigned long long>(cell_count, packed, n_cells, part64, total64,
                                                PackCount{}, s, true, cams != nullptr);
        // the interval tables (and what hangs on them) on a side stream, beside
        // the rank scatter; the run sorts need both
        SideFork tables(s, 1);
        make_intervals_kernel<<<cb, 256, 0, tables.side>>>(cell_count, packed, total64, n_cells,
                                                           starts, icells, cell_first, counts,
                                                           long_list, n_long);
        cudaEvent_t tables_done = nullptr;
        if (tables.side != s) {
            cudaEventCreateWithFlags(&tables_done, cudaEventDisableTiming);
            cudaEventRecord(tables_done, tables.side);
        }
        const int rc_t = on_tables ? (*on_tables)(tables.side) : BVP_OK;
        if (cams)
            count_scatter_kernel<<<148 * 8, 256, 0, s>>>(cells, slot, *fp, packed, ranks, iop);
        else
            count_scatter_flat_kernel<<<148 * 8, 256, 0, s>>>(cells, slot, P, packed, ranks, iop);
        if (tables_done) {
            cudaStreamWaitEvent(s, tables_done, 0);
            cudaEventDestroy(tables_done);
        }
        {  // short runs and long runs side by side
            SideFork fork(s);
            // the point gather table comes with the sorted runs (cams: the
            // frustum's N, H, W, D)
            const MetaOut mo{point_meta && fp ? reinterpret_cast<uint2 *>(point_meta) : nullptr,
                             fp ? uint32_t(fp->D) : 1u, fp ? uint32_t(fp->H) * fp->W : 1u};
            seg_sort_long_kernel<<<148 * 4, 256, 0, fork.side>>>(ranks, starts, long_list, n_long,
                                                                  mo);
            seg_sort_warp_kernel<<<148 * 4, 256, 0, s>>>(ranks, starts, counts, mo);
        }
        const int rc_r = on_ranks ? (*on_ranks)(s) : BVP_OK;
        tables.join();
        if (rc_t != BVP_OK) return rc_t;
        if (rc_r != BVP_OK) return rc_r;
        return check_launch("sort_intervals");
    }
    cudaMemsetAsync(cell_count, 0, 4 * size_t(n_cells), s);
    const unsigned tiles = static_cast<unsigned>(L.n_tiles);
    if (cams)
        pass0_front_kernel<true><<<tiles, kSortThreads, 0, s>>>(
            cams, *fp, *gp, P, cells, cell_count, L.digit_bits, hist, L.n_tiles);
    else
        pass0_front_kernel<false><<<tiles, kSortThreads, 0, s>>>(
            nullptr, FrustumParams{}, GridParams{}, P, cells, cell_count, L.digit_bits, hist,
            L.n_tiles);
    // interval tables from the per-cell counts (independent of the sort)
    device_excl_scan_xf<unsigned long long>(cell_count, packed, n_cells, part64, total64,
                                            PackCount{}, s);
    make_intervals_kernel<<<cb, 256, 0, s>>>(cell_count, packed, total64, n_cells, starts,
                                             icells, cell_first, counts);
    if (iop) {
        const unsigned pb = static_cast<unsigned>(std::min<int64_t>(ceil_div(P, 256), 8192));
        interval_of_point_kernel<<<pb, 256, 0, s>>>(cells, P, packed, iop);
    }
    // LSD radix passes; pass 0 drops out-of-range points, so later passes
    // (and the final ranks) only cover the n_in in-range points.
    const uint32_t *kin = cells;
    const uint32_t *vin = nullptr;
    for (int pass = 0; pass < L.passes; ++pass) {
        const int shift = pass * L.digit_bits;
        const bool last = pass == L.passes - 1;
        uint32_t *kout = last ? nullptr : ((pass & 1) ? kb : ka);
        uint32_t *vout = last ? ranks : ((pass & 1) ? vb : va);
        if (pass > 0)
            radix_upsweep_kernel<<<tiles, kSortThreads, 0, s>>>(kin, counts, shift, L.digit_bits,
                                                                hist, L.n_tiles);
        device_excl_scan<uint32_t>(hist, hist, L.hist_len, part32, total32, s);
        if (pass == 0)
            radix_scatter_kernel<true><<<tiles, kSortThreads, 0, s>>>(
                kin, nullptr, P, counts, shift, L.digit_bits, hist, L.n_tiles, kout, vout);
        else
            radix_scatter_kernel<false><<<tiles, kSortThreads, 0, s>>>(
                kin, vin, P, counts, shift, L.digit_bits, hist, L.n_tiles, kout, vout);
        kin = kout;
        vin = vout;
    }
    if (on_tables) {
        const int rc = (*on_tables)(s);
        if (rc != BVP_OK) return rc;
    }
    if (point_meta && fp) {  // radix path: the gather table from the final ranks
        const int rc = bvp_point_meta(ranks, counts, fp->N, fp->H, fp->W, fp->D, point_meta, s);
        if (rc != BVP_OK) return rc;
    }
    if (on_ranks) {
        const int rc = (*on_ranks)(s);
        if (rc != BVP_OK) return rc;
    }
    return check_launch("sort_intervals");
}

// ---- stable partition (partition.cuh) ----------------------------------------
struct PartLayout {
    int passes, digit_bits;
    int64_t n_tiles, hist_len;
    size_t keys_a, vals_a, keys_b, vals_b, hist, part, total, bytes;
};
static PartLayout part_layout(int64_t n_max, int key_bits) {
    PartLayout L{};
    key_bits = std::max(1, key_bits);
    L.passes = (key_bits + kMaxDigitBits - 1) / kMaxDigitBits;
    L.digit_bits = (key_bits + L.passes - 1) / L.passes;
    L.n_tiles = std::max<int64_t>(1, ceil_div(n_max, kSortTile));
    L.hist_len = (int64_t(1) << L.digit_bits) * L.n_tiles;
    size_t o = 0;
    L.keys_a = o; o = align256(o + 4 * size_t(n_max));
    L.vals_a = o; o = align256(o + 4 * size_t(n_max));
    L.keys_b = o; o = align256(o + 4 * size_t(n_max));
    L.vals_b = o; o = align256(o + 4 * size_t(n_max));
    L.hist = o; o = align256(o + 4 * size_t(L.hist_len));
    L.part = o; o = align256(o + 4 * size_t(scan_partials_len<uint32_t>(L.hist_len)));
    L.total = o; o = align256(o + 8);
    L.bytes = o;
    return L;
}

size_t stable_partition_ws_bytes(int64_t n_max, int key_bits) {
    return part_layout(n_max, key_bits).bytes;
}

int stable_partition(const uint32_t *keys, const uint32_t *vals, const int64_t *count,
                     int64_t n_max, int key_bits, uint32_t *vals_out, void *ws,
                     size_t ws_bytes, cudaStream_t s) {
    const PartLayout L = part_layout(n_max, key_bits);
    BVP_REQUIRE(ws && ws_bytes >= L.bytes, BVP_ERR_INVALID,
                "partition workspace too small: need %zu bytes, got %zu", L.bytes, ws_bytes);
    char *w = static_cast<char *>(ws);
    auto *hist = reinterpret_cast<uint32_t *>(w + L.hist);
    auto *part = reinterpret_cast<uint32_t *>(w + L.part);
    auto *total = reinterpret_cast<uint32_t *>(w + L.total);
    const unsigned tiles = static_cast<unsigned>(L.n_tiles);
    const uint32_t *kin = keys, *vin = vals;
    for (int pass = 0; pass < L.passes; ++pass) {
        const int shift = pass * L.digit_bits;
        const bool last = pass == L.passes - 1;
        uint32_t *kout = last ? nullptr : reinterpret_cast<uint32_t *>(w + ((pass & 1) ? L.keys_b : L.keys_a));
        uint32_t *vout = last ? vals_out : reinterpret_cast<uint32_t *>(w + ((pass & 1) ? L.vals_b : L.vals_a));
        radix_upsweep_kernel<<<tiles, kSortThreads, 0, s>>>(kin, count, shift, L.digit_bits, hist,
                                                            L.n_tiles);
        device_excl_scan<uint32_t>(hist, hist, L.hist_len, part, total, s);
        radix_scatter_kernel<false><<<tiles, kSortThreads, 0, s>>>(
            kin, vin, n_max, count, shift, L.digit_bits, hist, L.n_tiles, kout, vout);
        kin = kout;
        vin = vout;
    }
    return check_launch("stable_partition");
}

}  // namespace bvp

using namespace bvp;

extern "C" {

int bvp_frustum_cells(const double *cams, int N, int H, int W, int D, double depth_min,
                      double depth_step, const double *grid, int nx, int ny,
                      uint32_t *cell_of_point, void *stream) {
    BVP_REQUIRE(cams && grid && cell_of_point, BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(N > 0 && H > 0 && W > 0 && D > 0 && nx > 0 && ny > 0, BVP_ERR_INVALID,
                "frustum/grid dims must be positive");
    const FrustumParams f{N, H, W, D, depth_min, depth_step};
    const GridParams g = grid_params(grid, nx, ny);
    const int64_t P = int64_t(N) * H * W * D;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(P, 256), 148 * 64));
    frustum_cells_kernel<<<blocks, 256, 0, as_stream(stream)>>>(cams, f, g, P, cell_of_point);
    return check_launch("frustum_cells");
}

int bvp_frustum_points(const double *cams, int N, int H, int W, int D, double depth_min,
                       double depth_step, double *coords, void *stream) {
    BVP_REQUIRE(cams && coords, BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(N > 0 && H > 0 && W > 0 && D > 0, BVP_ERR_INVALID, "frustum dims must be positive");
    const FrustumParams f{N, H, W, D, depth_min, depth_step};
    const int64_t P = int64_t(N) * H * W * D;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(P, 256), 148 * 64));
    frustum_points_kernel<<<blocks, 256, 0, as_stream(stream)>>>(cams, f, P, coords);
    return check_launch("frustum_points");
}

int bvp_quantize_points(const double *coords, int64_t M, const double *grid, int nx, int ny,
                        uint32_t *cells, void *stream) {
    BVP_REQUIRE(M == 0 || (coords && cells), BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(grid && nx > 0 && ny > 0, BVP_ERR_INVALID, "bad grid");
    if (M == 0) return BVP_OK;
    const GridParams g = grid_params(grid, nx, ny);
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(M, 256), 148 * 64));
    quantize_points_kernel<<<blocks, 256, 0, as_stream(stream)>>>(coords, M, g, cells);
    return check_launch("quantize_points");
}

size_t bvp_sort_workspace_bytes(int64_t n_points, int64_t n_cells) {
    return sort_layout(n_points, n_cells).bytes;
}

int bvp_sort_intervals(const uint32_t *cell_of_point, int64_t n_points, int64_t n_cells,
                       uint32_t *ranks, uint32_t *interval_starts, uint32_t *interval_cells,
                       uint32_t *cell_first, uint32_t *interval_of_point, int64_t *counts,
                       void *workspace, size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(cell_of_point && ranks && interval_starts && interval_cells && cell_first &&
                    counts,
                BVP_ERR_INVALID, "null pointer argument");
    return sort_impl(nullptr, nullptr, nullptr, const_cast<uint32_t *>(cell_of_point), n_points,
                     n_cells, ranks, interval_starts, interval_cells, cell_first,
                     interval_of_point, counts, workspace, workspace_bytes, as_stream(stream));
}

int bvp_build_cache(const double *cams, int N, int H, int W, int D, double depth_min,
                    double depth_step, const double *grid, int nx, int ny,
                    uint32_t *cell_of_point, uint32_t *ranks, uint32_t *interval_starts,
                    uint32_t *interval_cells, uint32_t *cell_first, uint32_t *interval_of_point,
                    int64_t *counts, void *workspace, size_t workspace_bytes, void *stream) {
    BVP_REQUIRE(cams && grid && cell_of_point && ranks && interval_starts && interval_cells &&
                    cell_first && counts,
                BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(N > 0 && H > 0 && W > 0 && D > 0 && nx > 0 && ny > 0, BVP_ERR_INVALID,
                "frustum/grid dims must be positive");
    const FrustumParams f{N, H, W, D, depth_min, depth_step};
    const GridParams g = grid_params(grid, nx, ny);
    return sort_impl(cams, &f, &g, cell_of_point, int64_t(N) * H * W * D, int64_t(nx) * ny,
                     ranks, interval_starts, interval_cells, cell_first, interval_of_point,
                     counts, workspace, workspace_bytes, as_stream(stream));
}

int bvp_build_association(const double *cams, int N, int H, int W, int D, double depth_min,
                          double depth_step, const double *grid, int nx, int ny,
                          uint32_t *cell_of_point, uint32_t *ranks, uint32_t *interval_starts,
                          uint32_t *interval_cells, uint32_t *cell_first,
                          uint32_t *interval_of_point, int64_t *counts, int chunk,
                          uint32_t *work, uint32_t *splits, int64_t *work_counts,
                          uint32_t *point_meta, void *workspace, size_t workspace_bytes,
                          void *work_workspace, size_t work_workspace_bytes, void *stream) {
    BVP_REQUIRE(cams && grid && cell_of_point && ranks && interval_starts && interval_cells &&
                    cell_first && counts && work && splits && work_counts && point_meta,
                BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(N > 0 && H > 0 && W > 0 && D > 0 && nx > 0 && ny > 0, BVP_ERR_INVALID,
                "frustum/grid dims must be positive");
    const FrustumParams f{N, H, W, D, depth_min, depth_step};
    const GridParams g = grid_params(grid, nx, ny);
    const int64_t P = int64_t(N) * H * W * D, n_cells = int64_t(nx) * ny;
    const int64_t n_int_max = std::min(n_cells, P);
    const SortHook tables = [&](cudaStream_t side) {
        return bvp_make_work(interval_starts, interval_cells, counts, n_int_max, P, chunk, nx, ny,
                             -1, work, splits, work_counts, work_workspace, work_workspace_bytes,
                             side);
    };
    // the point gather table is written by the run sorts themselves
    return sort_impl(cams, &f, &g, cell_of_point, P, n_cells, ranks, interval_starts,
                     interval_cells, cell_first, interval_of_point, counts, workspace,
                     workspace_bytes, as_stream(stream), &tables, nullptr, point_meta);
}

}  // extern "C"
