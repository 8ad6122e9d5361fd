/* filter_c.c — the Filter Pipeline through the C-ABI only (no Python).
 *
 * Builds pipeline(gauss_noise, solarize, mirror) from the built-in
 * leaves, splits an H x W RGBA8 image into `parts` partitions on device 0,
 * runs it, and prints an FNV-1a checksum of the output so a test can compare
 * it with the oracle.  Input pixel i has bytes (i*7, i*13, i*29, 255) mod 256.
 * Usage: filter_c H W parts
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "marrow.h"

#define CHECK(x)                                                                       \
    do {                                                                               \
        mw_status s_ = (x);                                                            \
        if (s_ != MW_OK) {                                                             \
            fprintf(stderr, "%s: %s: %s\n", #x, mw_status_string(s_), mw_last_error(0)); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(int argc, char** argv) {
    const int64_t H = argc > 1 ? atoll(argv[1]) : 64, W = argc > 2 ? atoll(argv[2]) : 96;
    const int parts = argc > 3 ? atoi(argv[3]) : 2;
    const size_t bytes = (size_t)(H * W * 4);
    uint8_t* h = (uint8_t*)malloc(bytes);
    for (int64_t i = 0; i < H * W; ++i) {
        h[4 * i] = (uint8_t)(i * 7);
        h[4 * i + 1] = (uint8_t)(i * 13);
        h[4 * i + 2] = (uint8_t)(i * 29);
        h[4 * i + 3] = 255;
    }
    void *src, *dst;
    if (cudaMalloc(&src, bytes) != cudaSuccess || cudaMalloc(&dst, bytes) != cudaSuccess) return 2;
    cudaMemcpy(src, h, bytes, cudaMemcpyHostToDevice);

    mw_ctx* ctx;
    CHECK(mw_ctx_create(0, 0, 1, parts, NULL, 0, NULL, &ctx));
    mw_node *noise, *sol, *mir, *tree;
    CHECK(mw_kernel_gauss_noise(4, 8, &noise));
    CHECK(mw_kernel_solarize(128, &sol));
    CHECK(mw_kernel_mirror(&mir));
    mw_node* stages[3] = {noise, sol, mir};
    CHECK(mw_pipeline(stages, 3, &tree));
    mw_node_release(noise);  /* the pipeline retains its stages */
    mw_node_release(sol);
    mw_node_release(mir);

    mw_arg args[2] = {{0}};
    for (int k = 0; k < 2; ++k) {
        args[k].ptr = k ? dst : src;
        args[k].dtype = MW_DT_U8;
        args[k].ndim = 3;
        args[k].shape[0] = H;
        args[k].shape[1] = W;
        args[k].shape[2] = 4;
        args[k].mode = MW_PARTITION;
        args[k].location = MW_LOC_DEVICE;
        args[k].local_offset = 0;
        args[k].local_rows = H;
    }
    cudaStream_t s;
    cudaStreamCreate(&s);
    mw_future* f;
    CHECK(mw_run(ctx, tree, args, 2, s, &f));
    CHECK(mw_future_wait(f));
    mw_future_release(f);
    float ms[64], wall;
    CHECK(mw_last_timings(ctx, ms, 64, &wall));

    cudaMemcpy(h, dst, bytes, cudaMemcpyDeviceToHost);
    uint64_t fnv = 1469598103934665603ull;
    for (size_t i = 0; i < bytes; ++i) fnv = (fnv ^ h[i]) * 1099511628211ull;
    printf("fnv1a %016llx parts %d wall_ms %.3f\n", (unsigned long long)fnv, parts, wall);

    mw_node_release(tree);
    CHECK(mw_ctx_destroy(ctx));
    cudaFree(src);
    cudaFree(dst);
    free(h);
    return 0;
}
