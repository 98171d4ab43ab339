/*
 * bench_native.c -- the hot path timed from plain C through the C ABI (no Python, no torch):
 * an independent check of bench.py's kernel numbers.
 *
 * Inputs: BASELINE config 2 (C2, 2^28 angles U[-1e4, 1e4], seed 1) from the shared input
 * generator (inputs/gen.c, no method arithmetic), copied to the device once.  For each
 * variant and layout: W warm-up launches, then K launches back to back bracketed by CUDA
 * events on one stream; prints one JSON line with ms per launch, pairs/s and GB/s at
 * 12 B/pair.  Usage: bench_native [K=50] [W=5] [log2n=28]
 * Build: tools/bench_native.sh (gcc, links libsincos_pairs.so, libsincos_inputs.so, cudart).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../include/sincos_pairs.h"

int sincos_gen_range(int config, uint64_t start, uint64_t count, float *out, int nthreads);

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) {                                                                    \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));              \
            return 2;                                                                               \
        }                                                                                           \
    } while (0)

int main(int argc, char **argv) {
    const int K = argc > 1 ? atoi(argv[1]) : 50, W = argc > 2 ? atoi(argv[2]) : 5;
    const int lg = argc > 3 ? atoi(argv[3]) : 28;
    const size_t n = (size_t)1 << lg;
    float *h = (float *)malloc(n * sizeof(float));
    if (!h || sincos_gen_range(2, 0, n, h, 0) != 0) return 3;
    float *th, *s, *c, *io;
    CK(cudaMalloc((void **)&th, n * 4));
    CK(cudaMalloc((void **)&s, n * 4));
    CK(cudaMalloc((void **)&c, n * 4));
    CK(cudaMalloc((void **)&io, n * 8));
    CK(cudaMemcpy(th, h, n * 4, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    printf("{\"tool\": \"bench_native\", \"n\": %zu, \"steps\": %d, \"warmup\": %d, \"results\": {", n, K, W);
    const char *sep = "";
    for (int inter = 0; inter < 2; ++inter)
        for (int v = 0; v < 2; ++v) {
            for (int k = 0; k < W + K; ++k) {
                if (k == W) CK(cudaEventRecord(e0, st));
                sincos_status_t r = inter ? sincos_pairs(th, NULL, NULL, io, n, (sincos_variant_t)v, st)
                                          : sincos_pairs(th, s, c, NULL, n, (sincos_variant_t)v, st);
                if (r != SINCOS_OK) { fprintf(stderr, "%s\n", sincos_status_string(r)); return 4; }
            }
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double per = ms / K;
            printf("%s\"%s_%s\": {\"ms\": %.5f, \"pairs_per_s\": %.4e, \"GBps\": %.1f}", sep, v ? "A" : "N",
                   inter ? "interleaved" : "split", per, n / (per * 1e-3), 12.0 * n / (per * 1e-3) / 1e9);
            sep = ", ";
        }
    printf("}, \"launches\": %llu}\n", (unsigned long long)sincos_launch_count());
    return 0;
}
