/*
 * bevpool_oracle.c -- CPU restatement of the reference `bevpool` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2205_13542_b200/ links,
 * loads or calls this file; it is used by tests/ (the parity checker),
 * __graft_entry__.smoke() (the checker of the smoke run) and bench.py's
 * cpu_baseline / --impl reference leg (the CPU arm that is timed beside
 * the GPU).  It is a restatement, not a copy: every function cites the
 * reference lines whose behaviour it reproduces.
 *
 * Pinned against the reference itself: tests/golden/make_golden.py imports
 * /root/reference/pkg/src/bevpool and records SHA-256 digests of
 * cell_of_point / ranks / interval_starts / interval_cells / pool_interval
 * outputs at the T, S and H configurations; tests/test_oracle.py checks this
 * file against them bit-for-bit.
 *
 * Build (see oracle/Makefile): gcc -O3 -fopenmp -ffp-contract=off -fPIC.
 * -ffp-contract=off is REQUIRED: the reference geometry is a fixed sequence
 * of IEEE operations (one explicit fma chain, everything else separately
 * rounded) and a contracted a*b+c anywhere else changes cell ids.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OOR 0xFFFFFFFFu /* bevgrid.py:24 OUT_OF_RANGE */

/* cams: N x 16 doubles = fx, fy, cx, cy, R[9] (row-major cam->ego), t[3].
 * grid: x_min, x_max, y_min, y_max, z_min, z_max, r.
 *
 * Restates geometry.py:162-191 (generate_frustum) fused with
 * bevgrid.py:85-98 (quantize_points):
 *   depth_d = d_min + step * d                       geometry.py:95-99
 *   dx = (w - cx) / fx ; dy = (h - cy) / fy          geometry.py:178-179
 *   p  = (dx*depth, dy*depth, 1.0*depth)             geometry.py:184
 *   e_j = (p @ R^T)_j + t_j                          geometry.py:185-186
 * The OpenBLAS dgemm row (geometry.py:185) rounds as
 *   fma(R[j][2], pz, fma(R[j][1], py, R[j][0] * px))
 * (measured bit-exact), then "+ t" is a separate add.
 *   ix = floor((x - x_min) / r), iy likewise         bevgrid.py:88-89
 *   in range iff 0<=ix<nx, 0<=iy<ny, z_min<=z<z_max  bevgrid.py:91-95
 *   cell = ix*ny + iy else OUT_OF_RANGE              bevgrid.py:96
 * Point order ((n*H + h)*W + w)*D + d                geometry.py:106-107
 */
void oracle_frustum_cells(const double *cams, int N, int H, int W, int D,
                          double d_min, double d_step, const double *grid,
                          int nx, int ny, uint32_t *cells)
{
    const double x_min = grid[0], y_min = grid[2];
    const double z_min = grid[4], z_max = grid[5], r = grid[6];
    #pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; ++n) {
        for (int h = 0; h < H; ++h) {
            const double *c = cams + 16 * n;
            const double fx = c[0], fy = c[1], cx = c[2], cy = c[3];
            const double *R = c + 4, *t = c + 13;
            const double dy = ((double)h - cy) / fy;
            for (int w = 0; w < W; ++w) {
                const double dx = ((double)w - cx) / fx;
                size_t base = (((size_t)n * H + h) * W + w) * (size_t)D;
                for (int d = 0; d < D; ++d) {
                    const double depth = d_min + d_step * (double)d;
                    const double px = dx * depth, py = dy * depth, pz = 1.0 * depth;
                    double e[3];
                    for (int j = 0; j < 3; ++j) {
                        double acc = R[3 * j + 0] * px;
                        acc = fma(R[3 * j + 1], py, acc);
                        acc = fma(R[3 * j + 2], pz, acc);
                        e[j] = acc + t[j];
                    }
                    const double fxq = floor((e[0] - x_min) / r);
                    const double fyq = floor((e[1] - y_min) / r);
                    uint32_t cell = OOR;
                    if (fxq >= 0.0 && fxq < (double)nx && fyq >= 0.0 &&
                        fyq < (double)ny && e[2] >= z_min && e[2] < z_max)
                        cell = (uint32_t)((int64_t)fxq * ny + (int64_t)fyq);
                    cells[base + d] = cell;
                }
            }
        }
    }
}

/* Restates bevgrid.py:142-158 (ranks_and_intervals): stable sort of the
 * in-range point indices by cell id, interval starts where the cell changes.
 * Implemented as a stable counting sort over the bounded key range
 * [0, n_cells), which yields exactly numpy's stable argsort order.
 * counts_out[0] = n_in, counts_out[1] = n_int.  Returns 0, or -1 if a cell
 * id >= n_cells is found (the reference would still sort it; callers pass
 * the grid's n_cells so this indicates a corrupt input). */
int oracle_ranks_and_intervals(const uint32_t *cells, int64_t P, int64_t n_cells,
                               uint32_t *ranks, uint32_t *starts,
                               uint32_t *icells, int64_t *counts_out)
{
    int64_t *cursor = (int64_t *)calloc((size_t)n_cells + 1, sizeof(int64_t));
    if (!cursor) return -2;
    int64_t n_in = 0;
    for (int64_t p = 0; p < P; ++p) {
        uint32_t c = cells[p];
        if (c == OOR) continue;
        if ((int64_t)c >= n_cells) { free(cursor); return -1; }
        cursor[c + 1]++;
        n_in++;
    }
    int64_t n_int = 0;
    for (int64_t c = 0; c < n_cells; ++c) {
        if (cursor[c + 1] > 0) {
            starts[n_int] = (uint32_t)cursor[c];
            icells[n_int] = (uint32_t)c;
            n_int++;
        }
        cursor[c + 1] += cursor[c];
    }
    for (int64_t p = 0; p < P; ++p) {
        uint32_t c = cells[p];
        if (c == OOR) continue;
        ranks[cursor[c]++] = (uint32_t)p;
    }
    free(cursor);
    counts_out[0] = n_in;
    counts_out[1] = n_int;
    return 0;
}

/* (N, A, H, W) -> (N, H, W, A) copy; pooling.py:215-216 ascontiguousarray
 * of transpose(0, 2, 3, 1). */
void oracle_to_nhwc(const float *src, int N, int A, int H, int W, float *dst)
{
    #pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; ++n)
        for (int h = 0; h < H; ++h)
            for (int w = 0; w < W; ++w) {
                float *o = dst + (((size_t)n * H + h) * W + w) * (size_t)A;
                for (int a = 0; a < A; ++a)
                    o[a] = src[(((size_t)n * A + a) * H + h) * W + w];
            }
}

/* Restates _kernels.py:22-63 (interval_reduce): one job per interval,
 * 64-bit accumulation in rank order, one store per (channel, cell).
 * mode 0 = SUM, 1 = MEAN (acc * (1/len)), 2 = MAX (start -inf, strict >).
 * dist_t (N,H,W,D) and feats_t (N,H,W,C) contiguous; out (C, n_cells)
 * pre-zeroed by the caller (pooling.py:213). */
void oracle_interval_reduce(const uint32_t *ranks, int64_t n_in,
                            const uint32_t *starts, const uint32_t *icells,
                            int64_t n_int, const float *dist_t,
                            const float *feats_t, float *out, int64_t n_cells,
                            int H, int W, int D, int C, int mode)
{
    (void)H;
    (void)W;
    #pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (C > 0 ? C : 1));
        #pragma omp for schedule(static)
        for (int64_t i = 0; i < n_int; ++i) {
            int64_t lo = starts[i];
            int64_t hi = (i + 1 < n_int) ? (int64_t)starts[i + 1] : n_in;
            for (int c = 0; c < C; ++c) acc[c] = (mode == 2) ? -INFINITY : 0.0;
            for (int64_t j = lo; j < hi; ++j) {
                int64_t p = ranks[j];
                int64_t pix = p / D;          /* (n*H + h)*W + w */
                double wt = (double)dist_t[p]; /* dist_t flat index == p */
                const float *f = feats_t + pix * (int64_t)C;
                if (mode == 2) {
                    for (int c = 0; c < C; ++c) {
                        double v = wt * (double)f[c];
                        if (v > acc[c]) acc[c] = v;
                    }
                } else {
                    for (int c = 0; c < C; ++c) acc[c] += wt * (double)f[c];
                }
            }
            int64_t cell = icells[i];
            if (mode == 1) {
                double inv = 1.0 / (double)(hi - lo);
                for (int c = 0; c < C; ++c) out[(int64_t)c * n_cells + cell] = (float)(acc[c] * inv);
            } else {
                for (int c = 0; c < C; ++c) out[(int64_t)c * n_cells + cell] = (float)acc[c];
            }
        }
        free(acc);
    }
}

/* Full reference pool_interval (pooling.py:206-221) on host buffers:
 * zero out, transpose features and dist to NHWC/NHWD, interval_reduce.
 * scratch must hold N*H*W*(C+D) floats.  This is the stage the CPU
 * baseline times. */
void oracle_pool_interval(const float *features, const float *dist,
                          const uint32_t *ranks, int64_t n_in,
                          const uint32_t *starts, const uint32_t *icells,
                          int64_t n_int, float *out, int64_t n_cells,
                          int N, int C, int H, int W, int D, int mode,
                          float *scratch)
{
    memset(out, 0, sizeof(float) * (size_t)C * (size_t)n_cells);
    if (n_int == 0 || C == 0) return;
    float *feats_t = scratch;
    float *dist_t = scratch + (size_t)N * H * W * C;
    oracle_to_nhwc(features, N, C, H, W, feats_t);
    oracle_to_nhwc(dist, N, D, H, W, dist_t);
    oracle_interval_reduce(ranks, n_in, starts, icells, n_int, dist_t, feats_t,
                           out, n_cells, H, W, D, C, mode);
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
