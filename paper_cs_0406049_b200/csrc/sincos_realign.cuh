// sincos_realign.cuh -- eight consecutive angles from any 4-B offset, with aligned 256-bit
// loads: the re-alignment of KB3b (sincos_kernels.cu) for the kernels whose outputs fix the
// vector alignment (16-bit outputs, general methods) and the hybrid KB3c form (sincos_outshift.cu).
//
// The caller's vector v covers angles theta[head + 8v .. head + 8v + 7]; tal = theta + head - K
// is 32-B aligned, K = 1..7 the angles' float offset past that boundary (the callers run an
// aligned-load instance for K = 0).  Lane l loads a = tal[8v .. 8v+7]; the next aligned vector b comes from
// lane l+1 by warp shuffles, or from its own load for the warp's last lane and for a lane
// whose neighbour is past the end (issued together with the first load: one round trip).
// x = a[K..7] ++ b[0..K-1].
// Must be called by all 32 lanes (act = false for lanes past the end); the host sizes nvec
// so that tal[8 nvec + 7] lies inside theta when K > 0.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sincos_b200 {

__device__ __forceinline__ void ld8_stream(float (&r)[8], const float *p) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}

// the same load kept in the caches (operands re-read by many blocks, e.g. the phase grid's t)
__device__ __forceinline__ void ld8_keep(float (&r)[8], const float *p) {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}

// K (1..7) is a compile-time parameter: only the K values taken from the next lane are shuffled
// and the selection is register renaming (a run-time K with a switch over register moves was
// measured 15-20% slower).  KEEP: cache-resident loads (ld8_keep) instead of streaming ones.
template <int K, bool KEEP = false>
__device__ __forceinline__ void load8_realigned_k(const float *tal, size_t v, size_t nvec, unsigned lane, bool act,
                                                  float (&x)[8]) {
    const bool own = act && (lane == 31u || v + 1 >= nvec);
    float a[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    float bo[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    if constexpr (KEEP) {
        if (act) ld8_keep(a, tal + 8 * v);
        if (own) ld8_keep(bo, tal + 8 * v + 8);
    } else {
        if (act) ld8_stream(a, tal + 8 * v);
        if (own) ld8_stream(bo, tal + 8 * v + 8);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (j + K < 8) {
            x[j] = a[j + K];
        } else {
            const float b = __shfl_down_sync(0xFFFFFFFFu, a[j + K - 8], 1);
            x[j] = own ? bo[j + K - 8] : b;
        }
    }
}

// Host side: the aligned-angle offset K and the first vector element, for outputs whose vector
// alignment holds at element head0 and repeats every 8 elements (so K is the same at head0 + 8):
// head >= K keeps tal inside theta; nvec such that every second aligned load stays inside
// theta (K > 0).
inline void realign_plan(const float *theta, size_t n, size_t head0, int *k, size_t *head, size_t *nvec) {
    const int kk = static_cast<int>(((reinterpret_cast<uintptr_t>(theta) + 4 * head0) & 31) / 4);
    size_t h = head0;
    if (h < static_cast<size_t>(kk)) h += 8;
    if (h > n) h = n;
    size_t nv = (n - h) / 8;
    if (kk > 0) nv = n + kk >= h + 8 ? (n + kk - h - 8) / 8 : 0;   // (h - K) + 8 nvec + 7 <= n - 1
    *k = kk;
    *head = h;
    *nvec = nv;
}

}  // namespace sincos_b200
