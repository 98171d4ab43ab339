/*
 * abi_native.c -- the C ABI used from plain C, no Python (test driver; GPU needed).
 *
 * Allocates device buffers with the CUDA runtime, calls sincos_pairs (both variants, split
 * and interleaved, aligned and misaligned), sincos_pairs_host (pageable host buffers), the
 * phase grid, and checks every output against the C oracle (oracle/, test infrastructure)
 * by value.  Exit status 0 = all equal.  Built and run by tests/test_gpu_native.py.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/sincos_pairs.h"
#include "../../oracle/sincos_oracle.h"

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 2;                                                                  \
        }                                                                              \
    } while (0)

static int same(float a, float b) { return a == b || (isnan(a) && isnan(b)); }

static uint64_t lcg(uint64_t *s) {
    *s = *s * 6364136223846793005ull + 1442695040888963407ull;
    return *s >> 11;
}

int main(void) {
    const size_t n = (1u << 20) + 13, off = 3;
    float *th = (float *)malloc((n + off) * 4), *s = (float *)malloc(n * 4), *c = (float *)malloc(n * 4);
    float *ws = (float *)malloc(n * 4), *wc = (float *)malloc(n * 4), *io = (float *)malloc(8 * n);
    uint64_t seed = 42;
    for (size_t i = 0; i < n + off; ++i) th[i] = (float)(((double)lcg(&seed) * 0x1.0p-53 - 0.5) * 2e4);
    th[off + 5] = NAN;
    th[off + 6] = INFINITY;
    th[off + 7] = -0.0f;
    float *dth, *ds, *dc, *dio;
    CK(cudaMalloc((void **)&dth, (n + off) * 4));
    CK(cudaMalloc((void **)&ds, (n + off) * 4));
    CK(cudaMalloc((void **)&dc, (n + off) * 4));
    CK(cudaMalloc((void **)&dio, 8 * n));
    CK(cudaMemcpy(dth, th, (n + off) * 4, cudaMemcpyHostToDevice));
    int bad = 0;
    for (int v = 0; v < 2; ++v) {
        sincos_oracle(th + off, ws, wc, n, v);
        for (int shift = 0; shift < 2; ++shift) {   /* aligned, then element offset 3 (scalar head) */
            const size_t o = shift ? off : 0;
            if (shift == 0) sincos_oracle(th, ws, wc, n, v);
            else sincos_oracle(th + off, ws, wc, n, v);
            sincos_status_t st = sincos_pairs(dth + o, ds + o, dc + o, NULL, n, (sincos_variant_t)v, NULL);
            if (st != SINCOS_OK) { fprintf(stderr, "sincos_pairs: %s\n", sincos_status_string(st)); return 3; }
            CK(cudaMemcpy(s, ds + o, n * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(c, dc + o, n * 4, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < n; ++i) bad += !same(s[i], ws[i]) || !same(c[i], wc[i]);
            st = sincos_pairs(dth + o, NULL, NULL, dio, n, (sincos_variant_t)v, NULL);
            if (st != SINCOS_OK) return 3;
            CK(cudaMemcpy(io, dio, 8 * n, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < n; ++i) bad += !same(io[2 * i + 1], ws[i]) || !same(io[2 * i], wc[i]);
        }
        /* host-buffer path (pageable memory: correct, only slower) */
        void *wsp;
        size_t wsb = sincos_host_workspace_min_bytes();
        CK(cudaMalloc(&wsp, wsb));
        sincos_oracle(th + off, ws, wc, n, v);
        if (sincos_pairs_host(th + off, s, c, NULL, n, (sincos_variant_t)v, wsp, wsb, NULL) != SINCOS_OK) return 4;
        for (size_t i = 0; i < n; ++i) bad += !same(s[i], ws[i]) || !same(c[i], wc[i]);
        CK(cudaFree(wsp));
    }
    /* error conventions */
    bad += sincos_pairs(dth, ds, NULL, NULL, 16, SINCOS_NORMALIZED, NULL) != SINCOS_ERR_INVALID_ARGUMENT;
    bad += sincos_pairs(dth, ds, ds + 4, NULL, 16, SINCOS_NORMALIZED, NULL) != SINCOS_ERR_OVERLAP;
    bad += sincos_pairs(NULL, NULL, NULL, NULL, 0, SINCOS_NORMALIZED, NULL) != SINCOS_OK;
    /* phase grid, turns: 64 x 1024 grid vs the oracle's phase grid */
    {
        const size_t nf = 64, nt = 1024;
        float f[64], t[1024];
        for (size_t i = 0; i < nf; ++i) f[i] = (float)(512.0 * (double)lcg(&seed) * 0x1.0p-53);
        for (size_t j = 0; j < nt; ++j) t[j] = (float)(((double)j + (double)lcg(&seed) * 0x1.0p-53) / nt);
        float *df, *dt;
        CK(cudaMalloc((void **)&df, nf * 4));
        CK(cudaMalloc((void **)&dt, nt * 4));
        CK(cudaMemcpy(df, f, nf * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dt, t, nt * 4, cudaMemcpyHostToDevice));
        for (int v = 0; v < 2; ++v) {
            if (sincos_phase_grid(df, nf, dt, nt, ds, dc, NULL, SINCOS_TURNS, (sincos_variant_t)v, NULL) != SINCOS_OK)
                return 5;
            oracle_phase_grid(f, nf, t, nt, 1, v, ws, wc);
            CK(cudaMemcpy(s, ds, nf * nt * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(c, dc, nf * nt * 4, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < nf * nt; ++i) bad += !same(s[i], ws[i]) || !same(c[i], wc[i]);
        }
        CK(cudaFree(df));
        CK(cudaFree(dt));
    }
    CK(cudaDeviceSynchronize());
    printf("abi_native: %s, %d mismatches, %llu launches, %s\n", bad ? "FAIL" : "ok", bad,
           (unsigned long long)sincos_launch_count(), sincos_version());
    return bad ? 1 : 0;
}
