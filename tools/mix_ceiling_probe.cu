// mix_ceiling_probe.cu -- the DRAM ceiling of a streaming kernel that reads 4 B for every 4R B
// it writes, with no arithmetic: the traffic mix of the phase-grid kernels on short rows (the
// staged kernel at nt = 5 interleaved reads one f per 5 pairs = 4 B per 40 B written, R = 10;
// nt = 11 split 4 B per 88 B, R = 22), next to the hot path's mix (R = 2: 4 B in, 8 B out) and
// a write-only stream (NEXT(1)).
//
// Shape as in the product kernels: full grid of 128-thread blocks, one trip per thread; thread
// i loads the 256-bit vector i of `in` (streaming, L1 no-allocate, L2 evict-first) and writes R
// 256-bit vectors; a warp's output is contiguous (32 R vectors) and each of its R store
// instructions writes 32 consecutive vectors (1 KB of whole lines).  Write-only: the same
// stores, no load.  Each case: 3 warm-up launches, then the median of 5 rounds of 4
// back-to-back launches timed by CUDA events.  Output bytes per launch ~8.6 GB (the phase
// grid's 2^30 pairs x 8 B), inputs 1/R of that.  3 s idle before each case (burst, as the
// phase-grid measurements in tools/phase_mix_compare.py).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mix_ceiling_probe mix_ceiling_probe.cu
// Prints one JSON line per case.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));           \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

__device__ __forceinline__ void ld8(float (&r)[8], const float *p) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st8(float *p, const float (&r)[8]) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}

template <int R, bool LOAD>
__global__ void __launch_bounds__(128) mix(const float *in, float *out, size_t nvec) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nvec) return;                 // nvec is a multiple of 32: whole warps
    float x[8];
    if constexpr (LOAD) {
        ld8(x, in + 8 * i);
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = static_cast<float>(i + j);
    }
    const size_t lane = threadIdx.x & 31u, w = i - lane;     // w: the warp's first vector
#pragma unroll
    for (int r = 0; r < R; ++r) {
        x[r & 7] += 1.0f;                   // keep the stores distinct (one FADD per store)
        st8(out + 8 * (w * R + 32 * r + lane), x);
    }
}

template <int R, bool LOAD>
static void run(const char *name, const float *in, float *out, size_t out_floats) {
    const size_t nvec = out_floats / (8 * R) / 32 * 32;
    const unsigned grid = static_cast<unsigned>((nvec + 127) / 128);
    CK(cudaDeviceSynchronize());
    sleep(3);
    for (int k = 0; k < 3; ++k) mix<R, LOAD><<<grid, 128>>>(in, out, nvec);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ms;
    for (int rnd = 0; rnd < 5; ++rnd) {
        CK(cudaEventRecord(a));
        for (int k = 0; k < 4; ++k) mix<R, LOAD><<<grid, 128>>>(in, out, nvec);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float t = 0.0f;
        CK(cudaEventElapsedTime(&t, a, b));
        ms.push_back(t / 4);
    }
    std::sort(ms.begin(), ms.end());
    const double rd = LOAD ? 32.0 * nvec : 0.0, wr = 32.0 * nvec * R;
    const double t = ms[ms.size() / 2] * 1e-3;
    printf("{\"case\": \"%s\", \"R\": %d, \"load\": %s, \"ms\": %.4f, \"read_GB\": %.4f, \"write_GB\": %.4f, "
           "\"GBps_total\": %.1f, \"GBps_written\": %.1f, \"ms_min\": %.4f, \"ms_max\": %.4f}\n",
           name, R, LOAD ? "true" : "false", ms[ms.size() / 2], rd / 1e9, wr / 1e9, (rd + wr) / t / 1e9, wr / t / 1e9,
           ms.front(), ms.back());
    fflush(stdout);
    CK(cudaEventDestroy(a));
    CK(cudaEventDestroy(b));
}

int main() {
    const size_t out_floats = size_t(1) << 31;               // 8.6 GB written per launch
    float *in = nullptr, *out = nullptr;
    CK(cudaMalloc(&in, out_floats / 2 * sizeof(float) + 64));
    CK(cudaMalloc(&out, out_floats * sizeof(float) + 64));
    CK(cudaMemset(in, 0, out_floats / 2 * sizeof(float)));
    run<2, true>("hot path mix (4 B in, 8 B out)", in, out, out_floats);
    run<10, true>("staged nt=5 interleaved mix (4 B in, 40 B out)", in, out, out_floats);
    run<22, true>("staged nt=11 split mix (4 B in, 88 B out)", in, out, out_floats);
    run<8, false>("write-only", in, out, out_floats);
    run<10, true>("staged nt=5 interleaved mix (repeat)", in, out, out_floats);
    CK(cudaFree(in));
    CK(cudaFree(out));
    return 0;
}
