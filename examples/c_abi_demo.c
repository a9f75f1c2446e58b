/*
 * Standalone C client of libarv_b200.so (no Python, no torch): the C ABI of
 * include/approxrv_b200.h is all a reference-side binding needs.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c -L paper_2012_09715_b200 -larv_b200 \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2012_09715_b200 -o c_abi_demo
 *   ./c_abi_demo <table.f32 path> <n> <out.f32 path>
 *
 * Reads a natural-layout octave x sub-interval table (f32[2][16][8], degree 1,
 * K = 16, sub_bits = 3), generates n samples of PCG32(42, 0) through
 * arv_pcg32_subdyadic_f32, and writes them to the output file.  Also exercises
 * the drop-in dyadic_eval32 entry point and the error path.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "approxrv_b200.h"

#define CHECK_CUDA(x)                                                              \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));               \
            return 2;                                                              \
        }                                                                          \
    } while (0)

int main(int argc, char **argv) {
    if (argc != 4) {
        fprintf(stderr, "usage: %s table.f32 n out.f32\n", argv[0]);
        return 1;
    }
    const int64_t n = atoll(argv[2]);
    float table[2 * 16 * 8];
    FILE *f = fopen(argv[1], "rb");
    if (!f || fread(table, sizeof(float), 256, f) != 256) {
        fprintf(stderr, "cannot read table\n");
        return 1;
    }
    fclose(f);
    if (arv_abi_version() != ARV_ABI_VERSION) return 3;

    float *d_table = NULL, *d_out = NULL;
    CHECK_CUDA(cudaMalloc((void **)&d_table, sizeof(table)));
    CHECK_CUDA(cudaMalloc((void **)&d_out, (size_t)n * sizeof(float)));
    CHECK_CUDA(cudaMemcpy(d_table, table, sizeof(table), cudaMemcpyHostToDevice));

    /* fused PCG32 -> 16x8 table, on the default stream */
    int rc = arv_pcg32_subdyadic_f32(42, 0, 0, d_table, 1, 16, 3, d_out, n, NULL);
    if (rc != ARV_OK) {
        fprintf(stderr, "arv_pcg32_subdyadic_f32: %s\n", arv_last_error());
        return 4;
    }
    /* argument validation surfaces as a code + message, not a crash */
    if (arv_pcg32_subdyadic_f32(42, 0, 0, d_table, 9, 16, 3, d_out, n, NULL) != ARV_ERR_CONFIG) return 5;

    float *h = (float *)malloc((size_t)n * sizeof(float));
    CHECK_CUDA(cudaMemcpy(h, d_out, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost));
    FILE *o = fopen(argv[3], "wb");
    fwrite(h, sizeof(float), (size_t)n, o);
    fclose(o);
    printf("ok n=%lld first=%.9g launches=%llu\n", (long long)n, h[0], (unsigned long long)arv_launch_count());
    free(h);
    cudaFree(d_out);
    cudaFree(d_table);
    return 0;
}
