/*
 * bevpool_b200.h -- C ABI of the B200 (sm_100a) BEV-pooling library
 * (libbevpool_sm100.so).  Plain pointers and sizes only; every entry point is
 * stream-ordered on the caller's cudaStream_t (passed as void*), takes DEVICE
 * pointers allocated by the caller, never allocates, never synchronises, and
 * returns BVP_OK or an error code with a message in bvp_last_error().
 *
 * Reference interfaces replaced (paths relative to the reference's
 * pkg/src/bevpool/):
 *   bvp_frustum_points    generate_frustum (geometry.py:162-191)
 *   bvp_quantize_points   quantize_points (bevgrid.py:85-98)
 *   bvp_frustum_cells     generate_frustum + quantize_points fused
 *                         (geometry.py:162-191, bevgrid.py:85-98)
 *   bvp_interval_reduce_f32  _kernels.interval_reduce (_kernels.py:22-63),
 *                         same arguments and bit-identical results
 *   bvp_depth_distribution_check  check_depth_distribution (lift.py:52-63)
 *   bvp_sort_intervals    ranks_and_intervals (bevgrid.py:142-158)
 *   bvp_build_cache       build_cache minus the host fingerprint
 *                         (bevgrid.py:183-203)
 *   bvp_pool_forward_f32  pool_interval -> _kernels.interval_reduce
 *                         (pooling.py:206-221, _kernels.py:22-63)
 *   bvp_pool_prefixsum_f32  pool_prefixsum (pooling.py:162-196)
 *   bvp_reorder_weights   reorder_weights (pooling.py:243-261)
 *   bvp_normalize_depth   normalize_depth (lift.py:17-31)
 *   bvp_any_nonfinite     the finiteness checks of _check_inputs
 *                         (pooling.py:92-95)
 *   bvp_lift_f32 / bvp_pool_lifted_f32   the paper's materialised frustum
 *                         x = depth (x) feature, then bev_pool
 *   bvp_fused_pool_bf16   lift + pool fused (config F; no reference
 *                         counterpart, semantics normalize_depth + pool)
 *   bvp_pool_backward_f32 gather backward (config B; SPEC.md:540 lists
 *                         autograd as a reference non-goal)
 *
 * Cache layout on the device (all uint32 unless noted), from bvp_build_cache:
 *   cell_of_point[P]        flat cell id per frustum point or 0xFFFFFFFF
 *   ranks[P]                first n_in entries valid (point ids sorted by
 *                           cell, stable)
 *   interval_starts[n_cells+1]  first n_int entries as the reference, plus a
 *                           sentinel interval_starts[n_int] = n_in
 *   interval_cells[n_cells] first n_int entries valid
 *   cell_first[n_cells+1]   index of the first interval whose cell is >= c
 *                           (cell_first[n_cells] = n_int): the interval range
 *                           of any run of cells in O(1)
 *   interval_of_point[P]    interval index per point or 0xFFFFFFFF
 *   counts[2] (int64)       n_in, n_int
 * and from bvp_make_work / bvp_point_meta the chunk schedule of the interval
 * kernels (bvp_schedule below).  A whole frame can be rebuilt and pooled
 * without a host round trip.
 */
#ifndef BEVPOOL_B200_H
#define BEVPOOL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* exported even when the library is built with -fvisibility=hidden */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define BVP_ABI_VERSION 9

#define BVP_OK 0
#define BVP_ERR_INVALID 1      /* bad argument            -> ValidationError     */
#define BVP_ERR_UNSUPPORTED 2  /* shape/mode not compiled -> ConfigurationError  */
#define BVP_ERR_CUDA 3         /* CUDA runtime/launch error                      */

#define BVP_OUT_OF_RANGE 0xFFFFFFFFu
#define BVP_TILE_CELLS 32

#define BVP_SUM 0
#define BVP_MEAN 1
#define BVP_MAX 2
/* MEAN as the reference's pool_naive computes it: the fp64 sum divided by the
 * point count (pooling.py:152-156) instead of multiplied by 1/count
 * (_kernels.py:57-60); exact mode only. */
#define BVP_MEAN_DIV 3
/* or-ed into mode of bvp_pool_forward_nhwc_f32: `out` was zero-filled by
 * bvp_pool_prepare_f32 since it was last written, so the zero fill is skipped */
#define BVP_OUT_ZEROED 0x100
/* or-ed into mode of bvp_tile_pool_*: launch only the tile reduction (phase 1,
 * segment rows) or only the per-cell combine into the map (phase 2); for
 * per-kernel timing.  Neither flag: both, in order. */
#define BVP_TILE_PHASE1 0x200
#define BVP_TILE_PHASE2 0x400

/* Chunk schedule of the interval kernels (device pointers; built with the
 * cache by bvp_make_work / bvp_point_meta).
 *   point_meta  2 x uint32 per sorted point j: feature row n*H*W + h*W + w
 *               and weight index (n*D + d)*H*W + h*W + w of ranks[j]
 *   work, splits, work_counts, max_work, max_splits, max_partials, chunk
 *               the chunk list from bvp_make_work (work NULL: none -- the
 *               reference-order kernel then pools every interval): work = 4 x
 *               uint32 per chunk (first sorted point, end, destination,
 *               interval), chunks of <= `chunk` points sorted by length;
 *               splits = 4 x uint32 per interval cut into several chunks
 *               (interval, cell, first partial slot, chunk count);
 *               work_counts = device int64[3] n_work, n_splits, n_partials;
 *               max_* host bounds (>= the device counts) */
typedef struct bvp_schedule {
    const uint32_t *point_meta;
    const uint32_t *work;
    const uint32_t *splits;
    const int64_t *work_counts;
    int64_t max_work;
    int64_t max_splits;
    int64_t max_partials;
    int64_t chunk;
} bvp_schedule;

int bvp_abi_version(void);
const char *bvp_last_error(void);

/* ---- geometry precompute (cold association) -------------------------- */

/* cams: device, N x 16 float64 rows fx, fy, cx, cy, R[9] (row-major,
 * camera->ego), t[3].  grid: HOST, 7 float64 x_min, x_max, y_min, y_max,
 * z_min, z_max, r.  Writes cell_of_point[N*H*W*D]. */
int bvp_frustum_cells(const double *cams, int N, int H, int W, int D,
                      double depth_min, double depth_step, const double *grid,
                      int nx, int ny, uint32_t *cell_of_point, void *stream);

/* generate_frustum (geometry.py:162-191): coords (N*H*W*D, 3) float64,
 * device, row ((n*H + h)*W + w)*D + d, the reference's rounding (the
 * OpenBLAS dgemm FMA chain of SURVEY §8c). */
int bvp_frustum_points(const double *cams, int N, int H, int W, int D,
                       double depth_min, double depth_step, double *coords, void *stream);

/* quantize_points (bevgrid.py:85-98): coords (M, 3) float64 -> cells[M]
 * uint32 (0xFFFFFFFF out of range).  grid: HOST, 7 float64. */
int bvp_quantize_points(const double *coords, int64_t M, const double *grid, int nx, int ny,
                        uint32_t *cells, void *stream);

/* Workspace for bvp_sort_intervals / bvp_build_cache. */
size_t bvp_sort_workspace_bytes(int64_t n_points, int64_t n_cells);

/* Stable bounded-key sort of the in-range points by cell id and interval
 * detection, from an existing cell_of_point (e.g. a cache loaded from disk).
 * Outputs as in the cache layout above; interval_of_point may be NULL. */
int bvp_sort_intervals(const uint32_t *cell_of_point, int64_t n_points,
                       int64_t n_cells, uint32_t *ranks,
                       uint32_t *interval_starts, uint32_t *interval_cells,
                       uint32_t *cell_first, uint32_t *interval_of_point,
                       int64_t *counts, void *workspace, size_t workspace_bytes,
                       void *stream);

/* bvp_frustum_cells + bvp_sort_intervals. */
int bvp_build_cache(const double *cams, int N, int H, int W, int D,
                    double depth_min, double depth_step, const double *grid,
                    int nx, int ny, uint32_t *cell_of_point, uint32_t *ranks,
                    uint32_t *interval_starts, uint32_t *interval_cells,
                    uint32_t *cell_first, uint32_t *interval_of_point,
                    int64_t *counts, void *workspace, size_t workspace_bytes,
                    void *stream);

/* One call per frame (CacheBuilder, config H): bvp_build_cache, with the
 * chunk list (bvp_make_work, cell order, tile -1) built on a forked stream
 * as soon as the interval tables exist -- beside the rank scatter and run
 * sorts -- and the point gather table (bvp_point_meta's output) written by the
 * run sorts as each cell's run is ordered (no pass of its own).
 * work_workspace: bvp_work_workspace_bytes(min(n_cells, P), P, chunk, nx, ny,
 * -1) bytes, distinct from workspace. */
int bvp_build_association(const double *cams, int N, int H, int W, int D,
                          double depth_min, double depth_step, const double *grid,
                          int nx, int ny, uint32_t *cell_of_point, uint32_t *ranks,
                          uint32_t *interval_starts, uint32_t *interval_cells,
                          uint32_t *cell_first, uint32_t *interval_of_point,
                          int64_t *counts, int chunk, uint32_t *work,
                          uint32_t *splits, int64_t *work_counts,
                          uint32_t *point_meta, void *workspace,
                          size_t workspace_bytes, void *work_workspace,
                          size_t work_workspace_bytes, void *stream);

/* ---- work schedule (cached with the association) ---------------------- */

/* The point gather table alone (e.g. when a loaded cache's frustum shape is
 * only known at pooling time). */
int bvp_point_meta(const uint32_t *ranks, const int64_t *counts, int N, int H,
                   int W, int D, uint32_t *point_meta, void *stream);

/* Chunk schedule of the fast (fp32) kernels (work.cu): every interval is
 * cut into chunks of <= chunk points; chunks are listed longest first, so a
 * warp's 8 lane groups (one chunk each) finish together.  An interval cut
 * into several chunks ("split") gets one fp32 partial per chunk, combined in
 * chunk order by a second pass.  tile: 0 = longest first (cell order within
 * a length); > 0 = by tile x tile cell blocks, longest first within one;
 * -1 = cell order, no sort (per-frame rebuilds).  Capacities: work
 * n_int + n_in / chunk + 1 (bvp_work_capacity), splits n_int.  work_counts: device int64[3] receiving
 * n_work, n_splits, n_partials.  Run after the cache build. */
int64_t bvp_work_capacity(int64_t n_int_max, int64_t n_points, int chunk);
size_t bvp_work_workspace_bytes(int64_t n_int_max, int64_t n_points, int chunk,
                                int nx, int ny, int tile);
int bvp_make_work(const uint32_t *interval_starts, const uint32_t *interval_cells,
                  const int64_t *counts, int64_t n_int_max, int64_t n_points, int chunk,
                  int nx, int ny, int tile,
                  uint32_t *work, uint32_t *splits, int64_t *work_counts,
                  void *workspace, size_t workspace_bytes, void *stream);

/* ---- cached forward ---------------------------------------------------- */

/* Scratch of the fast kernels (the split intervals' partials) for B samples
 * of C channels in `mode`; 0 when the schedule has no chunk schedule. */
size_t bvp_pool_scratch_bytes(const bvp_schedule *schedule, int B, int C, int mode);

/* Workspace for bvp_pool_forward_f32: the NHWC copy of the features. */
size_t bvp_pool_workspace_bytes(int B, int N, int C, int H, int W);

/* features (B,N,C,H,W) f32, dist (B,N,D,H,W) f32 -> out (B,C,nx*ny) f32.
 * Every output element is written (empty cells 0).  mode: BVP_SUM/MEAN/MAX.
 * exact != 0: 64-bit accumulation in rank order, bit-identical to the
 * reference's interval_reduce; exact == 0: fp32 accumulation (<=1.2e-7 rel).
 * feats_nhwc: workspace of bvp_pool_workspace_bytes; left holding the
 * (B,N,H,W,C) transpose (reused by the backward).  argmax: NULL, or for
 * BVP_MAX a (B, n_int_max, C) uint32 buffer receiving the winning point id of
 * every (interval, channel). */
int bvp_pool_forward_f32(const float *features, const float *dist,
                         const uint32_t *ranks, const uint32_t *interval_starts,
                         const uint32_t *interval_cells,
                         const uint32_t *cell_first, const bvp_schedule *schedule,
                         int B, int N, int C, int H, int W, int D, int nx,
                         int ny, int64_t n_int_max, int mode, int exact,
                         float *out, float *feats_nhwc, uint32_t *argmax,
                         void *scratch, size_t scratch_bytes, void *stream);

/* (NB, C, H*W) -> (NB, H*W, C) f32 copy (the features' NHWC staging that
 * bvp_pool_forward_f32 performs first; pooling.py:215). */
int bvp_to_nhwc_f32(const float *src, int NB, int C, int HW, float *dst,
                    void *stream);

/* The first half of bvp_pool_forward_f32: the features' NHWC staging and the
 * zero fill of out (B, C, n_cells), side by side on a forked stream.  Follow
 * with bvp_pool_forward_nhwc_f32(..., mode | BVP_OUT_ZEROED, ...).  out = NULL:
 * the staging alone (the fast reduction then zeroes the empty cells beside
 * its kernels). */
int bvp_pool_prepare_f32(const float *features, int B, int N, int C, int H, int W,
                         float *feats_nhwc, float *out, int64_t n_cells, void *stream);

/* Zero fill of the cells of out (B, C, n_cells) that no interval covers
 * (cell_first[c] == cell_first[c+1]); occupied cells are untouched.  The fast
 * reduction runs it beside its kernels when out was not zero-filled
 * (bvp_pool_prepare_f32 with out = NULL stages the features alone).  No
 * reference counterpart: the reference's pool_interval allocates a zeroed
 * map (pooling.py:213). */
int bvp_zero_empty_cells(const uint32_t *cell_first, int64_t n_cells, int C, int B, float *out,
                         void *stream);

/* Same as bvp_pool_forward_f32 with the features already NHWC (B,N,H,W,C). */
int bvp_pool_forward_nhwc_f32(const float *feats_nhwc, const float *dist,
                              const uint32_t *ranks,
                              const uint32_t *interval_starts,
                              const uint32_t *interval_cells,
                              const uint32_t *cell_first,
                              const bvp_schedule *schedule, int B, int N,
                              int C, int H, int W, int D, int nx, int ny,
                              int64_t n_int_max, int mode, int exact,
                              float *out, uint32_t *argmax, void *scratch,
                              size_t scratch_bytes, void *stream);

/* w_sorted[j] = dist_t[ranks[j]] (dist given as (N,D,H,W)), j < n_in. */
int bvp_reorder_weights(const float *dist, const uint32_t *ranks, int64_t n_in,
                        int N, int D, int H, int W, float *w_sorted,
                        void *stream);

/* Softmax over D of (B*N, D, H, W) logits, 64-bit math, f32 out. */
int bvp_normalize_depth(const float *logits, int NB, int D, int H, int W,
                        float *dist, void *stream);

/* Non-finite scan of n floats; *flag (device int) set to 1 if any. */
int bvp_any_nonfinite(const float *x, int64_t n, int *flag, void *stream);

/* ---- materialised frustum (the paper's bev_pool input) ----------------- */

/* x[((n*H+h)*W+w)*D+d, c] = dist[n,d,h,w] * features[n,c,h,w], (P, C) f32. */
int bvp_lift_f32(const float *features, const float *dist, int N, int C, int H,
                 int W, int D, float *x, void *stream);

/* Interval reduction over materialised rows x (P, C) -> out (C, nx*ny). */
int bvp_pool_lifted_f32(const float *x, const uint32_t *ranks,
                        const uint32_t *interval_starts,
                        const uint32_t *interval_cells,
                        const uint32_t *cell_first,
                        const bvp_schedule *schedule, int C, int nx, int ny,
                        int mode, float *out, void *scratch, size_t scratch_bytes,
                        void *stream);

/* ---- fused lift + pool, bf16 inputs (config F) ------------------------- */

/* Workspace: per-pixel log-sum-exp (f32) + NHWC bf16 context. */
size_t bvp_fused_workspace_bytes(int B, int N, int C, int H, int W, int D);

/* logits (B,N,D,H,W) bf16, context (B,N,C,H,W) bf16 -> out (B,C,nx*ny)
 * f32 = pool(softmax_D(logits) (x) context), fp32 accumulation. */
int bvp_fused_pool_bf16(const uint16_t *logits, const uint16_t *context,
                        const uint32_t *ranks, const uint32_t *interval_starts,
                        const uint32_t *interval_cells,
                        const uint32_t *cell_first,
                        const bvp_schedule *schedule, int B, int N, int C,
                        int H, int W, int D, int nx, int ny, int mode,
                        float *out, void *workspace, size_t workspace_bytes,
                        void *scratch, size_t scratch_bytes, void *stream);

/* Backward of the fused path (SUM / MEAN): grad_out (B,C,nx*ny) f32 ->
 * grad_logits (B,N,D,H,W) and grad_context (B,N,C,H,W), bf16 like the
 * inputs.  The softmax is recomputed from the logits (fp32), the gather
 * backward gives grad_context and dL/dw, the softmax Jacobian gives
 * dL/dlogits.  No atomics; deterministic.  workspace:
 * bvp_fused_backward_workspace_bytes. */
size_t bvp_fused_backward_workspace_bytes(int B, int N, int C, int H, int W, int D,
                                          int64_t n_int_max);
int bvp_fused_backward_bf16(const float *grad_out, const uint16_t *logits, const uint16_t *context,
                            const uint32_t *interval_starts, const uint32_t *interval_cells,
                            const uint32_t *cell_first, const uint32_t *interval_of_point, int B,
                            int N, int C, int H, int W, int D, int nx, int ny, int64_t n_int_max,
                            int mode, uint16_t *grad_logits, uint16_t *grad_context,
                            void *workspace, size_t workspace_bytes, void *stream);

/* ---- gather backward (config B) ---------------------------------------- */

/* Workspace: per-interval gradient rows (B, n_int_max, C) f32. */
size_t bvp_backward_workspace_bytes(int B, int C, int64_t n_int_max);

/* grad_out (B,C,nx*ny) -> grad_features (B,N,C,H,W) and grad_dist
 * (B,N,D,H,W), both fully written.  feats_nhwc as left by the forward;
 * argmax required for BVP_MAX.  Either grad pointer may be NULL. */
int bvp_pool_backward_f32(const float *grad_out, const float *feats_nhwc,
                          const float *dist, const uint32_t *interval_starts,
                          const uint32_t *interval_cells,
                          const uint32_t *cell_first,
                          const uint32_t *interval_of_point,
                          const uint32_t *argmax, int B, int N, int C, int H,
                          int W, int D, int nx, int ny, int64_t n_int_max,
                          int mode, float *grad_features, float *grad_dist,
                          void *workspace, size_t workspace_bytes,
                          void *stream);

/* Materialised backward: grad_x[p, :] = dL/dx_p (zeros for out-of-range). */
int bvp_pool_lifted_backward_f32(const float *grad_out,
                                 const uint32_t *interval_starts,
                                 const uint32_t *interval_cells,
                                 const uint32_t *cell_first,
                                 const uint32_t *interval_of_point, int C,
                                 int64_t n_points, int nx, int ny,
                                 int64_t n_int_max, int mode, float *grad_x,
                                 void *workspace, size_t workspace_bytes,
                                 void *stream);

/* ---- the reference's native kernel, as it is called ----------------------- */

/* interval_reduce (_kernels.py:22-63) with the reference's own arguments:
 * ranks[n_in], interval_starts[n_int], interval_cells[n_int] (the
 * AssociationCache arrays), dist_t (N, H, W, D) f32 and feats_t (N, H, W, C)
 * f32 (the transposes pooling.py:215-216 makes), out (C, n_cells) f32 --
 * every interval's cell is written; other cells are left as they are (the
 * reference pre-zeroes out, pooling.py:213).  mode BVP_SUM / MEAN / MAX.
 * fp64 accumulation in rank order: bit-identical to the reference.  No
 * workspace, no schedule; stream ordered. */
int bvp_interval_reduce_f32(const uint32_t *ranks, const uint32_t *interval_starts,
                            const uint32_t *interval_cells, int64_t n_in, int64_t n_int,
                            const float *dist_t, const float *feats_t, float *out,
                            int64_t n_cells, int H, int W, int D, int C, int mode,
                            void *stream);

/* check_depth_distribution (lift.py:52-63) statistics of dist (NB, D, H, W)
 * f32: stats[0] = 1 if any entry is negative, stats[1] = the bits of the
 * worst |sum_d p - 1| as a float64 (device, 2 x uint64). */
int bvp_depth_distribution_check(const float *dist, int NB, int D, int H, int W,
                                 unsigned long long *stats, void *stream);

/* ---- pixel-column tiled pooling (the fast SUM / MEAN path) -------------- */

/* Plan of the tiled reduction (csrc/tile.cu), built on the device from
 * cell_of_point alone.  A tile is one camera column segment (n, w, up to 64
 * rows); its points are grouped by cell ("segments", 8 per group).  All
 * arrays live in one caller-allocated buffer `base` of bvp_tile_plan_bytes();
 * bvp_tile_plan_init fills the struct, bvp_build_tile_plan the buffer.
 *   n_seg           device int64: number of segments ((tile, cell) pairs),
 *                   -1 if a tile overflowed the record encoding
 *   cell_seg_first  device uint32[n_cells + 1]: first segment row of a cell
 *   cell_points     device uint32[n_cells]: in-range points per cell
 *   max_seg         host bound on n_seg: rows of the segment-row scratch */
typedef struct bvp_tile_plan {
    int N, H, W, D;
    int64_t n_cells;
    void *base;
    size_t bytes;
    int64_t max_seg;
    int tile_rows;
    int64_t n_tiles;
    const int64_t *n_seg;
    const uint32_t *cell_seg_first;
    const uint32_t *cell_points;
} bvp_tile_plan;

/* 1 when the tiled path takes this frustum / grid (D <= 8192, ...). */
int bvp_tile_plan_supported(int N, int H, int W, int D, int64_t n_cells);
size_t bvp_tile_plan_bytes(int N, int H, int W, int D, int64_t n_cells);
size_t bvp_tile_plan_workspace_bytes(int N, int H, int W, int D, int64_t n_cells);
int bvp_tile_plan_init(bvp_tile_plan *plan, int N, int H, int W, int D, int64_t n_cells,
                       void *base, size_t bytes, int64_t max_seg);
/* cell_of_point[N*H*W*D] (bevgrid.py:85-98's output) -> the plan; stream
 * ordered, no host sync.  Deterministic. */
int bvp_build_tile_plan(const uint32_t *cell_of_point, bvp_tile_plan *plan,
                        void *workspace, size_t workspace_bytes, void *stream);
/* The same plan from an association: its ranks (in-range point ids by cell,
 * ties by id; bevgrid.py:142-158) are stably sorted by tile, which lists
 * every tile's points in the plan's (cell, h, d) order without a per-tile
 * sort.  counts[0] = the number of in-range points (device).  Identical
 * plan; ~5x faster than bvp_build_tile_plan at config S. */
int bvp_build_tile_plan_ranks(const uint32_t *cell_of_point, const uint32_t *ranks,
                              const int64_t *counts, bvp_tile_plan *plan,
                              void *workspace, size_t workspace_bytes, void *stream);

/* pool_interval SUM / MEAN (pooling.py:206-221) through the plan: features
 * (B,N,C,H,W) f32, dist (B,N,D,H,W) f32 -> out (B,C,n_cells) f32, every
 * element written (empty cells 0).  fp32 accumulation (<= ~1e-6 relative of
 * the reference's fp64).  rows: scratch of B * max_seg * C floats.  C <= 128. */
int bvp_tile_pool_f32(const float *features, const float *dist, const bvp_tile_plan *plan,
                      int B, int C, int mode, float *rows, size_t rows_bytes, float *out,
                      void *stream);

/* The adjoint of bvp_tile_pool_f32 (config B training, SUM / MEAN): from
 * grad_out (B,C,n_cells) and the forward's features / dist, grad_features
 * (B,N,C,H,W) and grad_dist (B,N,D,H,W) (either may be NULL: not computed),
 * every element written once (points out of range and pixels no point of
 * which is in range get 0; with C = 0 grad_dist is all zeros).  rows: the same scratch as the forward's.
 * Deterministic; fp32 (<= ~1e-6 relative of the fp64 adjoint).  Tiles of
 * <= 32 rows (every plan bvp_tile_plan_init makes). */
int bvp_tile_backward_f32(const float *grad_out, const float *features, const float *dist,
                          const bvp_tile_plan *plan, int B, int C, int mode, float *rows,
                          size_t rows_bytes, float *grad_features, float *grad_dist,
                          void *stream);

/* Fused lift + pool (config F): logits (B,N,D,H,W) bf16 and context
 * (B,N,C,H,W) bf16 -> out (B,C,n_cells) f32 = pool(softmax_D(logits) (x)
 * context); the depth softmax of a tile's pixels is formed in shared memory
 * (fp32), nothing else is materialised. */
int bvp_tile_pool_fused_bf16(const uint16_t *logits, const uint16_t *context,
                             const bvp_tile_plan *plan, int B, int C, int mode, float *rows,
                             size_t rows_bytes, float *out, void *stream);

/* Its adjoint (config F training, SUM / MEAN): grad_logits (B,N,D,H,W) bf16
 * and grad_context (B,N,C,H,W) bf16 (either may be NULL) from grad_out
 * (B,C,n_cells) f32.  One pass per tile: the softmax is re-formed in shared
 * memory, grad_w = <context, g'> per point, grad_context = sum_d w g' per
 * pixel, and grad_logit = w (grad_w - sum_d w grad_w) -- no fp32 copy of the
 * softmax, the context or a gradient goes through global memory.  fp32
 * arithmetic, bf16 results; deterministic.  rows: as the forward's. */
int bvp_tile_fused_backward_bf16(const float *grad_out, const uint16_t *logits,
                                 const uint16_t *context, const bvp_tile_plan *plan, int B, int C,
                                 int mode, float *rows, size_t rows_bytes, uint16_t *grad_logits,
                                 uint16_t *grad_context, void *stream);

/* ---- the paper's "before": LSS prefix-sum pooling --------- */

/* pool_prefixsum (pooling.py:162-196): materialise the full running sum over
 * the rank-ordered points per channel (64-bit), subtract at interval ends.
 * SUM / MEAN only.  workspace: bvp_prefixsum_workspace_bytes. */
size_t bvp_prefixsum_workspace_bytes(int64_t n_in, int C);
int bvp_pool_prefixsum_f32(const float *features, const float *dist,
                           const uint32_t *ranks,
                           const uint32_t *interval_starts,
                           const uint32_t *interval_cells, int64_t n_in,
                           int64_t n_int, int N, int C, int H, int W, int D,
                           int64_t n_cells, int mode, float *out,
                           void *workspace, size_t workspace_bytes,
                           void *stream);

/* ---- shared-BEV fusion (reference fusion.py) ------------ */

/* Workspace for bvp_lidar_to_bev. */
size_t bvp_lidar_workspace_bytes(int64_t n_points, int nx, int ny);

/* lidar_to_bev (fusion.py:19-53): points (M, 4) float64 x, y, z, intensity
 * (device) -> out (3, nx*ny) f32: point count, reduced intensity, reduced
 * height per cell (mode BVP_SUM / MEAN / MAX; the count ignores it).  grid:
 * HOST, 7 float64 as bvp_frustum_cells.  Bit-identical to the reference. */
int bvp_lidar_to_bev(const double *points, int64_t n_points, const double *grid,
                     int nx, int ny, int mode, float *out, void *workspace,
                     size_t workspace_bytes, void *stream);

/* grid_resample (fusion.py:70-108): bilinear BEV -> BEV, float64 math,
 * src (C, src_nx, src_ny) f32 -> dst (C, dst_nx, dst_ny) f32; grids: HOST,
 * 7 float64 each.  Bit-identical to the reference. */
int bvp_grid_resample_f32(const float *src, int C, const double *src_grid,
                          int src_nx, int src_ny, const double *dst_grid,
                          int dst_nx, int dst_ny, float *dst, void *stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* BEVPOOL_B200_H */
