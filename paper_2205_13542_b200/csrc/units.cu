// units.cu -- the work schedule of the interval kernels (part of the cached
// association; built once per rig like the ranks).
//
// Units: runs of <= kUnitCells consecutive cells of one BEV row whose
// intervals hold <= budget in-range points.  A single cell holding more than
// the budget is a unit of its own, flagged long (the fast kernels split it
// over the warps of a CTA, pool_long_kernel; the exact kernel walks it in
// order).  Units are listed in cell order, so consecutive units are
// contiguous in the rank-ordered point stream; every unit records which of
// its cells own an interval (the has-mask) so its output block can be
// written without further lookups.
//
// Tasks: runs of consecutive units that one warp walks as ONE continuous
// point stream.  A task starts at unit 0, at every long unit, after every
// long unit, and wherever the cumulative in-range point count crosses a
// multiple of the task budget -- so tasks are balanced and the warp's gather
// pipeline is primed once per task, not once per unit.
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

// Greedy cut of one 8-cell row tile (tiles in cell order: t = ix*tiles_y + ty);
// WRITE=false counts, WRITE=true emits (first cell, ncell | has << 8 | long).
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
        const int ix = static_cast<int>(t / tiles_y), ty = static_cast<int>(t - int64_t(ix) * tiles_y);
        const int iy0 = ty * kUnitCells;
        const int n = min(kUnitCells, ny - iy0);
        const int64_t c0 = int64_t(ix) * ny + iy0;
        uint32_t count = 0, acc = 0, has = 0;
        uint32_t out = WRITE ? offsets[t] : 0u;
        int start = 0;
        auto emit = [&](int from, int to, bool is_long) {
            if (WRITE) {
                const uint32_t m = (has >> from) & ((1u << (to - from)) - 1u);
                const uint32_t iv0 = cell_first[c0 + from];
                units[4 * out] = static_cast<uint32_t>(c0 + from);
                units[4 * out + 1] =
                    static_cast<uint32_t>(to - from) | (m << 8) | (is_long ? kLongFlag : 0u);
                units[4 * out + 2] = iv0;
                units[4 * out + 3] = starts[iv0];
                if (is_long) long_units[atomicAdd(n_long, 1ull)] = out;
                ++out;
            }
            ++count;
        };
        for (int k = 0; k < n; ++k)
            if (cell_points(starts, cell_first, c0 + k)) has |= 1u << k;
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

__device__ __forceinline__ uint32_t unit_j0(const uint32_t *__restrict__ units,
                                            const uint32_t *__restrict__ starts,
                                            const uint32_t *__restrict__ cell_first, int64_t u) {
    return starts[cell_first[units[4 * u]]];
}

// flag[u] = 1 if unit u starts a task (see the header comment).
__global__ void task_flags_kernel(const uint32_t *__restrict__ units,
                                  const uint32_t *__restrict__ starts,
                                  const uint32_t *__restrict__ cell_first,
                                  const uint32_t *__restrict__ n_units_p, uint32_t task_budget,
                                  uint32_t *__restrict__ flag) {
    const int64_t n_units = *n_units_p;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n_units;
         u += (int64_t)gridDim.x * blockDim.x) {
        uint32_t f = 1;
        if (u > 0) {
            const bool lg = units[4 * u + 1] & kLongFlag, lg_prev = units[4 * u - 3] & kLongFlag;
            const uint32_t a = unit_j0(units, starts, cell_first, u - 1);
            const uint32_t b = unit_j0(units, starts, cell_first, u);
            f = (lg || lg_prev || (a / task_budget) != (b / task_budget)) ? 1u : 0u;
        }
        flag[u] = f;
    }
}

// tasks[8t..]: first unit, unit count (| long flag), J0, J1, first interval,
// end interval, 0, 0.
__global__ void tasks_kernel(const uint32_t *__restrict__ units,
                             const uint32_t *__restrict__ starts,
                             const uint32_t *__restrict__ cell_first,
                             const uint32_t *__restrict__ n_units_p,
                             const uint32_t *__restrict__ flag,
                             const uint32_t *__restrict__ task_of, const int64_t *__restrict__ counts,
                             uint32_t *__restrict__ tasks) {
    const int64_t n_units = *n_units_p;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n_units;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[u]) continue;
        int64_t v = u + 1;
        while (v < n_units && !flag[v]) ++v;  // next task start (tasks are short)
        const uint32_t t = task_of[u];
        const uint32_t iv0 = cell_first[units[4 * u]];
        const uint32_t iv1 = v < n_units ? cell_first[units[4 * v]] : static_cast<uint32_t>(counts[1]);
        uint32_t *r = tasks + 8 * size_t(t);
        r[0] = static_cast<uint32_t>(u);
        r[1] = static_cast<uint32_t>(v - u) | (units[4 * u + 1] & kLongFlag);
        r[2] = starts[iv0];
        r[3] = starts[iv1];
        r[4] = iv0;
        r[5] = iv1;
        r[6] = 0;
        r[7] = 0;
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

// Counts, plus the sentinel unit record at index n_units (its first interval
// and first point are the ends of the last unit: n_int, n_in).
__global__ void store_counts_kernel(const uint32_t *__restrict__ n_units,
                                    const unsigned long long *__restrict__ n_long,
                                    const uint32_t *__restrict__ n_tasks,
                                    const int64_t *__restrict__ counts,
                                    uint32_t *__restrict__ units, int64_t *__restrict__ out) {
    const uint32_t nu = *n_units;
    out[0] = nu;
    out[1] = static_cast<int64_t>(*n_long);
    out[2] = *n_tasks;
    units[4 * size_t(nu)] = 0u;
    units[4 * size_t(nu) + 1] = 0u;
    units[4 * size_t(nu) + 2] = static_cast<uint32_t>(counts[1]);
    units[4 * size_t(nu) + 3] = static_cast<uint32_t>(counts[0]);
}

struct UnitsLayout {
    int64_t ntiles, cap;
    size_t off_tile, off_part, off_total, off_long, off_flag, off_taskof, off_tpart, off_ttotal,
        bytes;
};
static UnitsLayout units_layout(int nx, int ny) {
    UnitsLayout L{};
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    L.ntiles = int64_t(nx) * ((ny + kUnitCells - 1) / kUnitCells);
    L.cap = L.ntiles + 2 * int64_t(nx) * ny;  // units <= tiles + 2 * intervals
    size_t o = 0;
    L.off_tile = o; o = al(o + size_t(L.ntiles) * 4);
    L.off_part = o; o = al(o + size_t(scan_partials_len<uint32_t>(L.ntiles)) * 4);
    L.off_total = o; o = al(o + 8);
    L.off_long = o; o = al(o + 8);
    L.off_flag = o; o = al(o + size_t(L.cap) * 4);
    L.off_taskof = o; o = al(o + size_t(L.cap) * 4);
    L.off_tpart = o; o = al(o + size_t(scan_partials_len<uint32_t>(L.cap)) * 4);
    L.off_ttotal = o; o = al(o + 8);
    L.bytes = o;
    return L;
}

}  // namespace bvp

using namespace bvp;

extern "C" {

int64_t bvp_units_capacity(int nx, int ny, int64_t n_int_max) {
    return int64_t(nx) * ((ny + kUnitCells - 1) / kUnitCells) + 2 * n_int_max;
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
                      int D, int nx, int ny, int budget, int task_budget, uint32_t *units,
                      uint32_t *long_units, uint32_t *tasks, int64_t *sched_counts,
                      uint32_t *point_meta, void *workspace, size_t workspace_bytes,
                      void *stream) {
    BVP_REQUIRE(ranks && interval_starts && cell_first && counts && units && long_units &&
                    tasks && sched_counts,
                BVP_ERR_INVALID, "null pointer argument");
    BVP_REQUIRE(nx >= 1 && ny >= 1 && budget >= 1 && task_budget >= 1 && N >= 1 && H >= 1 &&
                    W >= 1 && D >= 1,
                BVP_ERR_INVALID, "bad arguments");
    const UnitsLayout L = units_layout(nx, ny);
    BVP_REQUIRE(workspace && workspace_bytes >= L.bytes, BVP_ERR_INVALID,
                "schedule workspace too small: need %zu bytes", L.bytes);
    cudaStream_t s = as_stream(stream);
    char *ws = static_cast<char *>(workspace);
    auto *tile_units = reinterpret_cast<uint32_t *>(ws + L.off_tile);
    auto *part = reinterpret_cast<uint32_t *>(ws + L.off_part);
    auto *n_units = reinterpret_cast<uint32_t *>(ws + L.off_total);
    auto *n_long = reinterpret_cast<unsigned long long *>(ws + L.off_long);
    auto *flag = reinterpret_cast<uint32_t *>(ws + L.off_flag);
    auto *tpart = reinterpret_cast<uint32_t *>(ws + L.off_tpart);
    auto *n_tasks = reinterpret_cast<uint32_t *>(ws + L.off_ttotal);
    const int tiles_y = (ny + kUnitCells - 1) / kUnitCells;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(L.ntiles, 128), 4096));
    cudaMemsetAsync(n_long, 0, sizeof(unsigned long long), s);
    units_kernel<false><<<blocks, 128, 0, s>>>(interval_starts, cell_first, nx, ny, tiles_y,
                                               uint32_t(budget), tile_units, nullptr, nullptr,
                                               nullptr, nullptr);
    device_excl_scan<uint32_t>(tile_units, tile_units, L.ntiles, part, n_units, s);
    units_kernel<true><<<blocks, 128, 0, s>>>(interval_starts, cell_first, nx, ny, tiles_y,
                                              uint32_t(budget), nullptr, tile_units, units,
                                              long_units, n_long);
    // tasks: flags over units, scan, records (over the capacity; the kernels
    // read the device unit count)
    const unsigned ub = static_cast<unsigned>(std::min<int64_t>(ceil_div(L.cap, 256), 4096));
    cudaMemsetAsync(flag, 0, size_t(L.cap) * 4, s);
    task_flags_kernel<<<ub, 256, 0, s>>>(units, interval_starts, cell_first, n_units,
                                         uint32_t(task_budget), flag);
    auto *task_of = reinterpret_cast<uint32_t *>(ws + L.off_taskof);
    device_excl_scan<uint32_t>(flag, task_of, L.cap, tpart, n_tasks, s);
    tasks_kernel<<<ub, 256, 0, s>>>(units, interval_starts, cell_first, n_units, flag, task_of,
                                    counts, tasks);
    store_counts_kernel<<<1, 1, 0, s>>>(n_units, n_long, n_tasks, counts, units, sched_counts);
    if (point_meta) {
        const int rc = bvp_point_meta(ranks, counts, N, H, W, D, point_meta, stream);
        if (rc != BVP_OK) return rc;
    }
    return check_launch("make_schedule");
}

}  // extern "C"
