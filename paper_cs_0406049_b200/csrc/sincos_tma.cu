// sincos_tma.cu -- the hot path with TMA bulk loads (launch mode prefetch = 2).
//
// A persistent variant of KB1/KB2: each CTA walks tiles of kTile elements of theta
// (tile b, b + grid, b + 2*grid, ...).  One elected thread streams tiles into a ring
// of kStages shared-memory stages with cp.async.bulk (the TMA engine, global ->
// shared, completion counted in bytes on an mbarrier per stage), kStages - 1 tiles
// ahead of the consumers; every thread then takes its 8 elements from shared memory,
// evaluates the pairs and writes 2 x 256 bits to global memory directly.  The aim is
// to keep the read stream deep (up to kStages x kTile x 4 B in flight per CTA)
// independently of how long the arithmetic takes.  Numerics identical to KB1.
// Elements past the last whole tile are left to the caller (launch_tma returns how
// many it covered).
#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_launch.h"
#include "sincos_math.cuh"

namespace sincos_b200 {

constexpr int kTmaThreads = 256;
constexpr int kTile = kTmaThreads * 8;  // elements per tile (8 KB of theta)
constexpr int kStages = 5;  // 40 KB of static shared memory per CTA

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(0x12F0000000000000ull)
        : "memory");
}

__device__ __forceinline__ void st8(float *p, const float *r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}

template <int V, bool INTER>
__global__ void __launch_bounds__(kTmaThreads) sincos_tma_kernel(const float *__restrict__ theta, float *so,
                                                                 float *co, float *io, size_t ntiles) {
    __shared__ alignas(128) float buf[kStages][kTile];
    __shared__ alignas(8) uint64_t bar[kStages];
    const size_t G = gridDim.x;
    const size_t first = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // prologue: tiles 0 .. kStages-2 of this CTA
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages - 1; ++s) {
            const size_t t = first + s * G;
            if (t < ntiles) {
                mbar_expect_tx(&bar[s], kTile * 4);
                bulk_load(buf[s], theta + t * kTile, kTile * 4, &bar[s]);
            }
        }
    }
    size_t i = 0;
    for (size_t t = first; t < ntiles; t += G, ++i) {
        const int s = static_cast<int>(i % kStages);
        const uint32_t phase = static_cast<uint32_t>((i / kStages) & 1);
        // refill the stage consumed in the previous trip (all threads are past it)
        if (threadIdx.x == 0) {
            const size_t tn = t + (kStages - 1) * G;
            const int sn = static_cast<int>((i + kStages - 1) % kStages);
            if (tn < ntiles) {
                mbar_expect_tx(&bar[sn], kTile * 4);
                bulk_load(buf[sn], theta + tn * kTile, kTile * 4, &bar[sn]);
            }
        }
        mbar_wait(&bar[s], phase);
        float x[8];
        const float4 *src = reinterpret_cast<const float4 *>(&buf[s][threadIdx.x * 8]);
        const float4 a = src[0], b = src[1];
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
        x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        __syncthreads();  // every thread has its 8 values: the stage may be refilled next trip
        const size_t e0 = t * kTile + threadIdx.x * 8;
        if constexpr (INTER) {
            float cs[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) sincos_pair<V>(x[k], cs[2 * k + 1], cs[2 * k]);
            st8(io + 2 * e0, cs);
            st8(io + 2 * e0 + 8, cs + 8);
        } else {
            float sv[8], cv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) sincos_pair<V>(x[k], sv[k], cv[k]);
            st8(so + e0, sv);
            st8(co + e0, cv);
        }
    }
}

// Launch over the whole tiles of [theta, theta + n) (theta 16-B aligned, outputs 32-B
// aligned at element 0).  Returns the number of elements covered in *done.
cudaError_t launch_tma(int variant, bool inter, unsigned grid, const float *theta, float *so, float *co, float *io,
                       size_t n, size_t *done, cudaStream_t stream) {
    size_t ntiles = n / kTile;
    *done = ntiles * kTile;
    if (ntiles == 0) return cudaSuccess;
    if (grid > ntiles) grid = static_cast<unsigned>(ntiles);
    void *args[] = {&theta, &so, &co, &io, &ntiles};
    const void *fn;
    if (variant == kNormalized)
        fn = inter ? (const void *)sincos_tma_kernel<kNormalized, true> : (const void *)sincos_tma_kernel<kNormalized, false>;
    else
        fn = inter ? (const void *)sincos_tma_kernel<kRenormalized, true> : (const void *)sincos_tma_kernel<kRenormalized, false>;
    return cudaLaunchKernel(fn, dim3(grid), dim3(kTmaThreads), args, 0, stream);
}

}  // namespace sincos_b200
