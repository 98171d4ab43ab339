// rw_phase_probe.cu -- does separating the read and write phases of the 4-in / 8-out stream
// raise its DRAM throughput toward the read-only / write-only ceilings (DESIGN.md section 5,
// "Where the ceiling is": 7.46 / 7.54 TB/s alone, 6.83-6.90 mixed)?
//
// No-math traffic only (outputs = copies of theta), C2 size.  Kernels:
//   ref      : the hot path's shape -- full grid, 128 threads, one 256-bit load and two 256-bit
//              stores per thread.
//   phased   : persistent (SMs x B CTAs of T threads); each thread loads E floats into
//              registers (a chunk = grid x E floats), then stores them to sin[] and cos[];
//              BAR = 0 free-running, 1 a grid barrier between the read and the write phase and
//              after the write phase (all loads of a chunk landed before any store of it).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o rw_phase_probe rw_phase_probe.cu
// Prints one JSON line per configuration.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

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
__device__ __forceinline__ void st8(float *p, const float *r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}

__global__ void __launch_bounds__(128) ref_kernel(const float *__restrict__ th, float *__restrict__ s,
                                                  float *__restrict__ c, size_t nvec) {
    size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nvec) return;
    float r[8];
    ld8(r, th + 8 * v);
    st8(s + 8 * v, r);
    st8(c + 8 * v, r);
}

__device__ unsigned int g_arrive;
__device__ unsigned int g_gen;

__device__ __forceinline__ void grid_barrier(unsigned nblocks, unsigned &gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned a = atomicAdd(&g_arrive, 1u);
        if (a == nblocks - 1) {
            g_arrive = 0;
            __threadfence();
            atomicExch(&g_gen, gen + 1);
        } else {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&g_gen));
            } while (g == gen);
        }
    }
    gen += 1;
    __syncthreads();
}

// Each thread: E/8 vectors per chunk; vector j of thread t in chunk k sits at
// k * (G * E/8) + j * G + t (G = total threads): every load and store instruction of a warp
// covers 1 KiB contiguous.
template <int E, int BAR>
__global__ void __launch_bounds__(256) phased_kernel(const float *__restrict__ th, float *__restrict__ s,
                                                     float *__restrict__ c, size_t nvec, unsigned gen0) {
    constexpr int NV = E / 8;
    const size_t G = (size_t)gridDim.x * blockDim.x;
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned gen = gen0;
    float r[NV][8];
    for (size_t base = 0; base < nvec; base += G * NV) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            size_t v = base + j * G + t;
            if (v < nvec) ld8(r[j], th + 8 * v);
        }
        if (BAR) {
            float acc = 0.f;                    // wait for every load of this thread to land
#pragma unroll
            for (int j = 0; j < NV; ++j) acc += r[j][0];
            if (acc == 1.2345e-38f) g_arrive += 0;   // never true for the probe's data
            asm volatile("" ::"f"(acc));
            grid_barrier(gridDim.x, gen);
        }
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            size_t v = base + j * G + t;
            if (v < nvec) {
                st8(s + 8 * v, r[j]);
                st8(c + 8 * v, r[j]);
            }
        }
        if (BAR) grid_barrier(gridDim.x, gen);
    }
}

template <int E, int BAR>
static void run_phased(const float *th, float *s, float *c, size_t nvec, int per_sm, int threads, int sms,
                       unsigned &gen, cudaStream_t st) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, phased_kernel<E, BAR>, threads, 0));
    int b = per_sm < occ ? per_sm : occ;
    unsigned nb = (unsigned)(b * sms);
    phased_kernel<E, BAR><<<nb, threads, 0, st>>>(th, s, c, nvec, gen);
    if (BAR) {
        size_t chunks = (nvec + (size_t)nb * threads * (E / 8) - 1) / ((size_t)nb * threads * (E / 8));
        gen += (unsigned)(2 * chunks);
    }
}

int main(int argc, char **argv) {
    size_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (1ull << 28);
    int reps = argc > 2 ? atoi(argv[2]) : 20;
    size_t nvec = n / 8;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float *th, *s, *c, *flush;
    size_t flush_bytes = 256ull << 20;
    CK(cudaMalloc(&th, n * 4));
    CK(cudaMalloc(&s, n * 4));
    CK(cudaMalloc(&c, n * 4));
    CK(cudaMalloc(&flush, flush_bytes));
    CK(cudaMemset(th, 0x3f, n * 4));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    unsigned gen = 0;
    unsigned zero = 0;
    CK(cudaMemcpyToSymbol(g_arrive, &zero, 4));
    CK(cudaMemcpyToSymbol(g_gen, &zero, 4));

    auto timeit = [&](const char *name, int e, int bar, int per_sm, auto &&launch) {
        for (int w = 0; w < 3; ++w) launch();
        CK(cudaStreamSynchronize(st));
        float tot = 0.f, best = 1e30f;
        for (int i = 0; i < reps; ++i) {
            CK(cudaMemsetAsync(flush, i & 0xff, flush_bytes, st));
            CK(cudaEventRecord(e0, st));
            launch();
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            tot += ms;
            if (ms < best) best = ms;
        }
        CK(cudaGetLastError());
        double bytes = 12.0 * (double)(nvec * 8);
        printf("{\"kernel\": \"%s\", \"E\": %d, \"bar\": %d, \"per_sm\": %d, \"ms_mean\": %.5f, \"GBps_mean\": %.1f, "
               "\"GBps_best\": %.1f}\n",
               name, e, bar, per_sm, tot / reps, bytes / (tot / reps) / 1e6, bytes / best / 1e6);
        fflush(stdout);
    };

    for (int round = 0; round < 2; ++round) {
        timeit("ref", 8, 0, 0, [&] { ref_kernel<<<(unsigned)((nvec + 127) / 128), 128, 0, st>>>(th, s, c, nvec); });
#define P(E, BAR, PS)                                                                                       \
    timeit("phased", E, BAR, PS, [&] { run_phased<E, BAR>(th, s, c, nvec, PS, 256, sms, gen, st); });
        P(8, 0, 8) P(16, 0, 4) P(32, 0, 2) P(64, 0, 2)
        P(32, 1, 2) P(64, 1, 2) P(64, 1, 1) P(128, 1, 1)
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
