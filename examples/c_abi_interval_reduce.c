/* c_abi_interval_reduce.c -- the reference's native kernel call, from C.
 *
 * A host holding the reference's own arrays (an AssociationCache's ranks /
 * interval_starts / interval_cells and the NHWD / NHWC transposes that
 * pooling.py:215-216 makes) replaces _kernels.interval_reduce
 * (_kernels.py:22-63) by one call: bvp_interval_reduce_f32.  No schedule,
 * no workspace, no other state.
 *
 *   c_abi_interval_reduce <dir> n_in n_int n_cells H W D C N
 *
 * reads <dir>/{ranks,starts,icells,dist_t,feats_t}.bin, writes
 * <dir>/out_{sum,mean,max}.bin ((C, n_cells) f32 each, pre-zeroed like the
 * reference's out).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "bevpool_b200.h"

static void *load(const char *dir, const char *name, size_t bytes) {
    char path[1024];
    snprintf(path, sizeof path, "%s/%s.bin", dir, name);
    FILE *f = fopen(path, "rb");
    void *h = malloc(bytes ? bytes : 1), *d = NULL;
    if (!f || !h || fread(h, 1, bytes, f) != bytes) return NULL;
    fclose(f);
    if (cudaMalloc(&d, bytes ? bytes : 16) != cudaSuccess) return NULL;
    cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
    free(h);
    return d;
}

int main(int argc, char **argv) {
    if (argc != 10) {
        fprintf(stderr, "usage: %s dir n_in n_int n_cells H W D C N\n", argv[0]);
        return 2;
    }
    const char *dir = argv[1];
    const int64_t n_in = atoll(argv[2]), n_int = atoll(argv[3]), n_cells = atoll(argv[4]);
    const int H = atoi(argv[5]), W = atoi(argv[6]), D = atoi(argv[7]), C = atoi(argv[8]);
    const int N = atoi(argv[9]);
    const uint32_t *ranks = load(dir, "ranks", 4 * (size_t)n_in);
    const uint32_t *starts = load(dir, "starts", 4 * (size_t)n_int);
    const uint32_t *icells = load(dir, "icells", 4 * (size_t)n_int);
    const float *dist_t = load(dir, "dist_t", 4 * (size_t)N * H * W * D);
    const float *feats_t = load(dir, "feats_t", 4 * (size_t)N * H * W * C);
    if (!ranks || !starts || !icells || !dist_t || !feats_t) {
        fprintf(stderr, "cannot load inputs\n");
        return 1;
    }
    const size_t out_bytes = 4 * (size_t)C * n_cells;
    float *out = NULL;
    if (cudaMalloc((void **)&out, out_bytes) != cudaSuccess) return 1;
    float *host = malloc(out_bytes);
    const char *names[3] = {"out_sum", "out_mean", "out_max"};
    const int modes[3] = {BVP_SUM, BVP_MEAN, BVP_MAX};
    for (int m = 0; m < 3; ++m) {
        cudaMemset(out, 0, out_bytes);  /* the reference's out = zeros((C, n_cells)) */
        int rc = bvp_interval_reduce_f32(ranks, starts, icells, n_in, n_int, dist_t, feats_t, out,
                                         n_cells, H, W, D, C, modes[m], NULL);
        if (rc != BVP_OK) {
            fprintf(stderr, "bvp_interval_reduce_f32: %s\n", bvp_last_error());
            return 1;
        }
        if (cudaMemcpy(host, out, out_bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
        char path[1024];
        snprintf(path, sizeof path, "%s/%s.bin", dir, names[m]);
        FILE *f = fopen(path, "wb");
        fwrite(host, 1, out_bytes, f);
        fclose(f);
    }
    printf("ok\n");
    return 0;
}
