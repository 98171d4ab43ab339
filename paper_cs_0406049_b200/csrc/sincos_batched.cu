// sincos_batched.cu -- many independent arrays in ONE launch (serving many small requests).
//
// The paper's problem is "a large number" of pairs for arbitrary angles; in a serving
// setting they arrive as many separate arrays.  One launch per array costs ~2-3 us of launch
// latency each, which dominates below ~10^5 elements.  Here the host validates the items and
// passes a table (one record per item + a prefix sum of 1024-element chunks, up to
// kBatchMax items) as the kernel's own parameter block (__grid_constant__, up to 32 KB on
// sm_70+ with CUDA >= 12.1) -- no staging copy, no workspace, fully asynchronous; every block
// finds its item by binary search over the prefix (warp-uniform) and runs the same
// per-element method (sincos_math.cuh) on its chunk: 256-bit loads and stores when the item's
// theta and outputs share their alignment, one element per thread otherwise.  Numerics
// identical to sincos_pairs.
//
// Not part of the product library (SURVEY 8 does not list it): compiled into the A/B build
// (-DSINCOS_AB, libsincos_pairs_ab.so) only.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_launch.h"
#include "sincos_math.cuh"

#ifdef SINCOS_AB
namespace sincos_b200 {

constexpr int kBatchThreads = 128;
constexpr uint64_t kBatchChunk = kBatchThreads * 8;   // elements per block

template <int V>
__device__ __forceinline__ void batch_one(const BatchItem &it, uint64_t e) {
    float s, c;
    sincos_pair<V>(it.theta[e], s, c);
    if (it.io) {
        it.io[2 * e] = c;
        it.io[2 * e + 1] = s;
    } else {
        it.so[e] = s;
        it.co[e] = c;
    }
}

template <int V, int CAP>
__global__ void __launch_bounds__(kBatchThreads) sincos_batched_kernel(const __grid_constant__ BatchParamsT<CAP> p) {
    const uint64_t b = blockIdx.x;
    int lo = 0, hi = p.count;                 // the item i with prefix[i] <= b < prefix[i + 1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (p.prefix[mid] <= b) lo = mid; else hi = mid;
    }
    const BatchItem it = p.items[lo];
    const uint64_t c = b - p.prefix[lo];
    const unsigned t = threadIdx.x;
    if (!it.vec) {                            // one element per thread, 8 strided trips (coalesced)
        const uint64_t base = c * kBatchChunk;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint64_t e = base + static_cast<uint64_t>(k) * kBatchThreads + t;
            if (e < it.n) batch_one<V>(it, e);
        }
        return;
    }
    // vector body from element `head` (theta and outputs 32-B aligned there); chunk 0 also
    // covers [0, head), the last chunk the ragged tail
    if (c == 0 && t < it.head) batch_one<V>(it, t);
    const uint64_t v = c * kBatchThreads + t;
    const uint64_t e0 = it.head + 8 * v;
    if (e0 + 8 <= it.n) {
        float x[8];
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
                     : "l"(it.theta + e0));
        if (it.io) {
            float cs[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) sincos_pair<V>(x[k], cs[2 * k + 1], cs[2 * k]);
#pragma unroll
            for (int h = 0; h < 2; ++h)
                asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                             :: "l"(it.io + 2 * e0 + 8 * h), "f"(cs[8 * h]), "f"(cs[8 * h + 1]), "f"(cs[8 * h + 2]),
                                "f"(cs[8 * h + 3]), "f"(cs[8 * h + 4]), "f"(cs[8 * h + 5]), "f"(cs[8 * h + 6]),
                                "f"(cs[8 * h + 7])
                             : "memory");
        } else {
            float sv[8], cv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) sincos_pair<V>(x[k], sv[k], cv[k]);
            asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                         :: "l"(it.so + e0), "f"(sv[0]), "f"(sv[1]), "f"(sv[2]), "f"(sv[3]), "f"(sv[4]), "f"(sv[5]),
                            "f"(sv[6]), "f"(sv[7])
                         : "memory");
            asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                         :: "l"(it.co + e0), "f"(cv[0]), "f"(cv[1]), "f"(cv[2]), "f"(cv[3]), "f"(cv[4]), "f"(cv[5]),
                            "f"(cv[6]), "f"(cv[7])
                         : "memory");
        }
    } else {
        for (uint64_t e = e0; e < it.n && e < e0 + 8; ++e) batch_one<V>(it, e);   // ragged tail
    }
}

template <int CAP>
static cudaError_t launch_cap(int variant, const BatchParams &p, uint64_t blocks, cudaStream_t stream) {
    BatchParamsT<CAP> q;                      // the first `count` records, in a smaller block
    q.count = p.count;
    q.pad = 0;
    for (int i = 0; i <= p.count; ++i) q.prefix[i] = p.prefix[i];
    for (int i = 0; i < p.count; ++i) q.items[i] = p.items[i];
    const void *fn = variant == kNormalized
                         ? reinterpret_cast<const void *>(sincos_batched_kernel<kNormalized, CAP>)
                         : reinterpret_cast<const void *>(sincos_batched_kernel<kRenormalized, CAP>);
    void *args[] = {&q};
    return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(blocks)), dim3(kBatchThreads), args, 0, stream);
}

cudaError_t launch_batched(int variant, const BatchParams &p, cudaStream_t stream) {
    const uint64_t blocks = p.prefix[p.count];
    if (blocks == 0) return cudaSuccess;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    if (p.count <= 16) return launch_cap<16>(variant, p, blocks, stream);
    if (p.count <= 96) return launch_cap<96>(variant, p, blocks, stream);
    const void *fn = variant == kNormalized
                         ? reinterpret_cast<const void *>(sincos_batched_kernel<kNormalized, kBatchMax>)
                         : reinterpret_cast<const void *>(sincos_batched_kernel<kRenormalized, kBatchMax>);
    void *args[] = {const_cast<BatchParams *>(&p)};
    return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(blocks)), dim3(kBatchThreads), args, 0, stream);
}

uint64_t batched_chunks(uint64_t n, uint64_t head, bool vec) {
    if (n == 0) return 0;
    if (!vec) return (n + kBatchChunk - 1) / kBatchChunk;
    const uint64_t body = n > head ? n - head : 0;
    const uint64_t ch = (body + kBatchChunk - 1) / kBatchChunk;
    return ch > 0 ? ch : 1;
}

}  // namespace sincos_b200
#endif  // SINCOS_AB
