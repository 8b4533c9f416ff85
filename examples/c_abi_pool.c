/* c_abi_pool.c -- the pooling path driven from plain C through the C ABI
 * (include/bevpool_b200.h), the way a non-Python host (a TensorRT plugin,
 * a cgo/JNI binding) would: one camera, tiny config T of BASELINE.json
 * (16 x 44 features, D = 59, C = 32, 128 x 128 grid at 0.8 m).
 *
 *   per frame:  bvp_build_association  (geometry, sort, intervals, chunk list,
 *                                       point gather table; one call)
 *               bvp_normalize_depth    (fp64 softmax over D)
 *               bvp_pool_forward_f32   (fast fp32 and exact fp64)
 *   per rig:    bvp_build_tile_plan_ranks (the tiled reduction's plan, from
 *                                       the association)
 *               bvp_tile_pool_f32      (the tiled reduction: the fast path)
 *   training:   bvp_tile_backward_f32  (its adjoint, config B)
 *               bvp_tile_pool_fused_bf16 + bvp_tile_fused_backward_bf16
 *                                      (config F: bf16 logits and context,
 *                                       forward and adjoint)
 *
 * Writes the inputs, the cache's ranks / interval table, the maps and the
 * gradients to <out_dir>/<name>.bin so tests/test_c_abi.py can check them against
 * the oracle.
 *
 *   gcc -O2 examples/c_abi_pool.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2205_13542_b200 -lbevpool_sm100 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2205_13542_b200 -o /tmp/c_abi_pool
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "bevpool_b200.h"

#define CHECK_BVP(call)                                                            \
    do {                                                                           \
        int rc_ = (call);                                                          \
        if (rc_ != BVP_OK) {                                                       \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, bvp_last_error()); \
            return 1;                                                              \
        }                                                                          \
    } while (0)
#define CHECK_CUDA(call)                                                           \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));            \
            return 1;                                                              \
        }                                                                          \
    } while (0)

static void *dev_alloc(size_t bytes) {
    void *p = NULL;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return NULL;
    return p;
}

static int dump(const char *dir, const char *name, const void *dev, size_t bytes) {
    char path[1024];
    snprintf(path, sizeof path, "%s/%s.bin", dir, name);
    void *h = malloc(bytes ? bytes : 1);
    if (!h || cudaMemcpy(h, dev, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    FILE *f = fopen(path, "wb");
    if (!f) return 1;
    fwrite(h, 1, bytes, f);
    fclose(f);
    free(h);
    return 0;
}

/* fp32 -> bf16 bits, round to nearest even (finite inputs) */
static uint16_t to_bf16(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

static uint64_t lcg = 0x9E3779B97F4A7C15ull;
static float uniform(float lo, float hi) {
    lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
    return lo + (hi - lo) * (float)((lcg >> 40) * (1.0 / 16777216.0));
}

int main(int argc, char **argv) {
    const char *out_dir = argc > 1 ? argv[1] : ".";
    if (bvp_abi_version() != BVP_ABI_VERSION) {
        fprintf(stderr, "ABI mismatch: library %d, header %d\n", bvp_abi_version(), BVP_ABI_VERSION);
        return 1;
    }
    const int N = 1, H = 16, W = 44, D = 59, C = 32, nx = 128, ny = 128;
    const double d_min = 1.0, d_step = 1.0;
    const double grid[7] = {-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.8};
    const int64_t P = (int64_t)N * H * W * D, n_cells = (int64_t)nx * ny;
    const int64_t n_int_max = P < n_cells ? P : n_cells;
    const int chunk = 64;
    /* one level camera looking along +x, 1.6 m up: fx = fy = 0.8 W */
    const double cam[16] = {0.8 * W, 0.8 * W, W / 2.0, H / 2.0,
                            0, 0, 1, -1, 0, 0, 0, -1, 0, 0, 0, 1.6};

    float *h_feat = malloc(sizeof(float) * N * C * H * W);
    float *h_logit = malloc(sizeof(float) * N * D * H * W);
    for (int64_t i = 0; i < (int64_t)N * C * H * W; ++i) h_feat[i] = uniform(-1.f, 1.f);
    for (int64_t i = 0; i < (int64_t)N * D * H * W; ++i) h_logit[i] = uniform(-3.f, 3.f);

    double *d_cam = dev_alloc(sizeof cam);
    uint32_t *cells = dev_alloc(4 * P), *ranks = dev_alloc(4 * P), *iop = dev_alloc(4 * P);
    uint32_t *starts = dev_alloc(4 * (n_cells + 1)), *icells = dev_alloc(4 * n_cells);
    uint32_t *cell_first = dev_alloc(4 * (n_cells + 1));
    int64_t *counts = dev_alloc(16), *work_counts = dev_alloc(24);
    const int64_t work_cap = bvp_work_capacity(n_int_max, P, chunk);
    uint32_t *work = dev_alloc(16 * work_cap), *splits = dev_alloc(16 * n_int_max);
    uint32_t *meta = dev_alloc(8 * P);
    const size_t ws_bytes = bvp_sort_workspace_bytes(P, n_cells);
    const size_t wws_bytes = bvp_work_workspace_bytes(n_int_max, P, chunk, nx, ny, -1);
    void *ws = dev_alloc(ws_bytes), *wws = dev_alloc(wws_bytes);
    float *feat = dev_alloc(sizeof(float) * N * C * H * W);
    float *logit = dev_alloc(sizeof(float) * N * D * H * W);
    float *dist = dev_alloc(sizeof(float) * N * D * H * W);
    float *nhwc = dev_alloc(bvp_pool_workspace_bytes(1, N, C, H, W));
    float *out_fast = dev_alloc(sizeof(float) * C * n_cells);
    float *out_exact = dev_alloc(sizeof(float) * C * n_cells);
    if (!d_cam || !cells || !ranks || !iop || !starts || !icells || !cell_first || !counts ||
        !work_counts || !work || !splits || !meta || !ws || !wws || !feat || !logit || !dist ||
        !nhwc || !out_fast || !out_exact) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    CHECK_CUDA(cudaMemcpy(d_cam, cam, sizeof cam, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(feat, h_feat, sizeof(float) * N * C * H * W, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(logit, h_logit, sizeof(float) * N * D * H * W, cudaMemcpyHostToDevice));

    /* the frame: association, depth softmax, pooling (default stream) */
    CHECK_BVP(bvp_build_association(d_cam, N, H, W, D, d_min, d_step, grid, nx, ny, cells, ranks,
                                    starts, icells, cell_first, iop, counts, chunk, work, splits,
                                    work_counts, meta, ws, ws_bytes, wws, wws_bytes, NULL));
    CHECK_BVP(bvp_normalize_depth(logit, N, D, H, W, dist, NULL));
    int64_t host_counts[2], host_wc[3];
    CHECK_CUDA(cudaMemcpy(host_counts, counts, sizeof host_counts, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(host_wc, work_counts, sizeof host_wc, cudaMemcpyDeviceToHost));
    bvp_schedule sched;
    memset(&sched, 0, sizeof sched);
    sched.point_meta = meta;
    sched.work = work;
    sched.splits = splits;
    sched.work_counts = work_counts;
    sched.max_work = host_wc[0];
    sched.max_splits = host_wc[1];
    sched.max_partials = host_wc[2];
    sched.chunk = chunk;
    const size_t scratch_bytes = bvp_pool_scratch_bytes(&sched, 1, C, BVP_SUM);
    void *scratch = dev_alloc(scratch_bytes);
    CHECK_BVP(bvp_pool_forward_f32(feat, dist, ranks, starts, icells, cell_first, &sched, 1, N, C,
                                   H, W, D, nx, ny, n_int_max, BVP_SUM, 0, out_fast, nhwc, NULL,
                                   scratch, scratch_bytes, NULL));
    CHECK_BVP(bvp_pool_forward_f32(feat, dist, ranks, starts, icells, cell_first, &sched, 1, N, C,
                                   H, W, D, nx, ny, n_int_max, BVP_SUM, 1, out_exact, nhwc, NULL,
                                   scratch, scratch_bytes, NULL));
    /* the tiled reduction (csrc/tile.cu): plan from the association, then
     * the pooling; the plan is per rig, the pooling per frame */
    const size_t plan_bytes = bvp_tile_plan_bytes(N, H, W, D, n_cells);
    const size_t plan_ws_bytes = bvp_tile_plan_workspace_bytes(N, H, W, D, n_cells);
    if (plan_bytes == 0) {
        fprintf(stderr, "frustum not supported by the tile plan\n");
        return 1;
    }
    void *plan_buf = dev_alloc(plan_bytes), *plan_ws = dev_alloc(plan_ws_bytes);
    bvp_tile_plan plan;
    CHECK_BVP(bvp_tile_plan_init(&plan, N, H, W, D, n_cells, plan_buf, plan_bytes, P));
    CHECK_BVP(bvp_build_tile_plan_ranks(cells, ranks, counts, &plan, plan_ws, plan_ws_bytes, NULL));
    const size_t rows_bytes = sizeof(float) * (size_t)plan.max_seg * C;
    void *rows = dev_alloc(rows_bytes);
    float *out_tiled = dev_alloc(sizeof(float) * C * n_cells);
    CHECK_BVP(bvp_tile_pool_f32(feat, dist, &plan, 1, C, BVP_SUM, rows, rows_bytes, out_tiled,
                                NULL));

    /* training: the adjoint of the SUM map for a random grad_out (config B),
     * then config F's fused forward and adjoint on bf16 copies of the inputs */
    const size_t gmap_bytes = sizeof(float) * C * n_cells;
    float *h_g = malloc(gmap_bytes);
    for (int64_t i = 0; i < (int64_t)C * n_cells; ++i) h_g[i] = uniform(-1.f, 1.f);
    const int64_t n_feat = (int64_t)N * C * H * W, n_pt = (int64_t)N * D * H * W;
    uint16_t *h_lb = malloc(2 * n_pt), *h_cb = malloc(2 * n_feat);
    for (int64_t i = 0; i < n_pt; ++i) h_lb[i] = to_bf16(h_logit[i]);
    for (int64_t i = 0; i < n_feat; ++i) h_cb[i] = to_bf16(h_feat[i]);
    float *g = dev_alloc(gmap_bytes), *grad_feat = dev_alloc(sizeof(float) * n_feat);
    float *grad_dist = dev_alloc(sizeof(float) * n_pt), *out_fused = dev_alloc(gmap_bytes);
    uint16_t *lb = dev_alloc(2 * n_pt), *cb = dev_alloc(2 * n_feat);
    uint16_t *grad_logit = dev_alloc(2 * n_pt), *grad_ctx = dev_alloc(2 * n_feat);
    if (!h_g || !h_lb || !h_cb || !g || !grad_feat || !grad_dist || !out_fused || !lb || !cb ||
        !grad_logit || !grad_ctx) {
        fprintf(stderr, "allocation failed\n");
        return 1;
    }
    CHECK_CUDA(cudaMemcpy(g, h_g, gmap_bytes, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(lb, h_lb, 2 * n_pt, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(cb, h_cb, 2 * n_feat, cudaMemcpyHostToDevice));
    CHECK_BVP(bvp_tile_backward_f32(g, feat, dist, &plan, 1, C, BVP_SUM, rows, rows_bytes,
                                    grad_feat, grad_dist, NULL));
    CHECK_BVP(bvp_tile_pool_fused_bf16(lb, cb, &plan, 1, C, BVP_SUM, rows, rows_bytes, out_fused,
                                       NULL));
    CHECK_BVP(bvp_tile_fused_backward_bf16(g, lb, cb, &plan, 1, C, BVP_SUM, rows, rows_bytes,
                                           grad_logit, grad_ctx, NULL));
    CHECK_CUDA(cudaDeviceSynchronize());

    /* fast vs exact, the reference's tolerance metric max|a-b| / max(1,|a|) */
    const size_t map_bytes = sizeof(float) * C * n_cells;
    float *a = malloc(map_bytes), *b = malloc(map_bytes);
    CHECK_CUDA(cudaMemcpy(a, out_exact, map_bytes, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(b, out_fast, map_bytes, cudaMemcpyDeviceToHost));
    double worst = 0.0, total = 0.0;
    for (int64_t i = 0; i < (int64_t)C * n_cells; ++i) {
        const double d = fabs((double)a[i] - (double)b[i]) / fmax(1.0, fabs((double)a[i]));
        if (d > worst) worst = d;
        total += a[i];
    }
    printf("n_in=%lld n_int=%lld chunks=%lld splits=%lld sum=%.9g fast_vs_exact=%.3e\n",
           (long long)host_counts[0], (long long)host_counts[1], (long long)host_wc[0],
           (long long)host_wc[1], total, worst);
    if (dump(out_dir, "features", feat, sizeof(float) * N * C * H * W) ||
        dump(out_dir, "dist", dist, sizeof(float) * N * D * H * W) ||
        dump(out_dir, "cell_of_point", cells, 4 * P) ||
        dump(out_dir, "ranks", ranks, 4 * host_counts[0]) ||
        dump(out_dir, "interval_starts", starts, 4 * host_counts[1]) ||
        dump(out_dir, "interval_cells", icells, 4 * host_counts[1]) ||
        dump(out_dir, "out_exact", out_exact, map_bytes) ||
        dump(out_dir, "out_fast", out_fast, map_bytes) ||
        dump(out_dir, "out_tiled", out_tiled, map_bytes) ||
        dump(out_dir, "grad_out", g, gmap_bytes) ||
        dump(out_dir, "grad_features", grad_feat, sizeof(float) * n_feat) ||
        dump(out_dir, "grad_dist", grad_dist, sizeof(float) * n_pt) ||
        dump(out_dir, "logits_bf16", lb, 2 * n_pt) ||
        dump(out_dir, "context_bf16", cb, 2 * n_feat) ||
        dump(out_dir, "out_fused", out_fused, gmap_bytes) ||
        dump(out_dir, "grad_logits", grad_logit, 2 * n_pt) ||
        dump(out_dir, "grad_context", grad_ctx, 2 * n_feat)) {
        fprintf(stderr, "writing %s failed\n", out_dir);
        return 1;
    }
    return worst <= 1e-5 ? 0 : 2;
}
