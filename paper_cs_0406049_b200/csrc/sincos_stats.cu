// sincos_stats.cu -- KB5: per-shard error statistics in fp64 (verification only).
//
// The paper's metrics: combined error sqrt((c - ref_c)^2 + (s - ref_s)^2)
// and amplitude error |1 - sqrt(c^2 + s^2)|, with the reference computed "to
// double precision" -- here CUDA's fp64 sincos() of the widened
// angle.  A fixed grid (kStatsBlocks x kStatsThreads), per-thread accumulators
// in grid-stride order, a fixed-shape block tree, and a last-block pass over the
// block partials in block order make every field deterministic.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/sincos_pairs.h"
#include "sincos_launch.h"

namespace sincos_b200 {

struct Partial {
    double max_comb, sum_sq, max_amp;
    unsigned long long n, nan_count;
    float worst;
    int pad;
};

constexpr int kStatsBlocks = 1024;
constexpr int kStatsThreads = 256;

struct StatsWs {
    Partial part[kStatsBlocks];
    unsigned int done;
};

size_t stats_ws_bytes() { return sizeof(StatsWs); }

__device__ __forceinline__ void merge(Partial &a, const Partial &b) {
    if (b.max_comb > a.max_comb) {
        a.max_comb = b.max_comb;
        a.worst = b.worst;
    }
    a.sum_sq += b.sum_sq;
    a.max_amp = fmax(a.max_amp, b.max_amp);
    a.n += b.n;
    a.nan_count += b.nan_count;
}

__global__ void __launch_bounds__(kStatsThreads) sincos_stats_kernel(const float *theta, const float *so,
                                                                    const float *co, const float *io, size_t n,
                                                                    sincos_stats_t *out, StatsWs *ws) {
    Partial p{0.0, 0.0, 0.0, 0ull, 0ull, 0.0f, 0};
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += nthr) {
        const float s = io ? io[2 * e + 1] : so[e];
        const float c = io ? io[2 * e] : co[e];
        if (isnan(s) || isnan(c)) {
            p.nan_count++;
            continue;
        }
        double rs, rc;
        sincos(static_cast<double>(theta[e]), &rs, &rc);
        const double dc = static_cast<double>(c) - rc, ds = static_cast<double>(s) - rs;
        const double comb = sqrt(dc * dc + ds * ds);
        const double amp = fabs(1.0 - sqrt(static_cast<double>(c) * c + static_cast<double>(s) * s));
        p.n++;
        p.sum_sq += comb * comb;
        if (comb > p.max_comb) {
            p.max_comb = comb;
            p.worst = theta[e];
        }
        p.max_amp = fmax(p.max_amp, amp);
    }
    __shared__ Partial sh[kStatsThreads];
    sh[threadIdx.x] = p;
    __syncthreads();
    for (int w = kStatsThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) merge(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    __shared__ bool last;
    if (threadIdx.x == 0) {
        ws->part[blockIdx.x] = sh[0];
        __threadfence();
        last = (atomicAdd(&ws->done, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        Partial t = ws->part[0];
        for (unsigned b = 1; b < gridDim.x; ++b) merge(t, ws->part[b]);
        out->n = t.n;
        out->nan_count = t.nan_count;
        out->max_comb = t.max_comb;
        out->sum_sq = t.sum_sq;
        out->max_amp = t.max_amp;
        out->kernel_ms = 0.0;
        out->worst_theta = t.worst;
        out->device = 0;
        out->reserved = 0;
        ws->done = 0;  // ready for the next call on this workspace
    }
}

cudaError_t launch_stats(const float *theta, const float *so, const float *co, const float *io, size_t n,
                         sincos_stats_t *out, void *ws, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(&static_cast<StatsWs *>(ws)->done, 0, sizeof(unsigned int), stream);
    if (e != cudaSuccess) return e;
    StatsWs *w = static_cast<StatsWs *>(ws);
    void *args[] = {&theta, &so, &co, &io, &n, &out, &w};
    return cudaLaunchKernel(reinterpret_cast<const void *>(sincos_stats_kernel), dim3(kStatsBlocks),
                            dim3(kStatsThreads), args, 0, stream);
}

}  // namespace sincos_b200
