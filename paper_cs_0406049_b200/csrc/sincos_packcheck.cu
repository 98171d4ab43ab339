// sincos_packcheck.cu -- test hook: the packed-fp32 method (sincos_math2.cuh, used by the
// fused sum) against the scalar method (sincos_math.cuh / sincos_method.cuh) over EVERY fp32
// bit pattern, in radians (x1 = RN(x / 2pi), the whole method) and in turns (x is already
// x1, the method from the reduction).  Each lane of a packed instruction must round exactly
// as the scalar instruction does; this proves it for all 2^32 inputs instead of sampled ones.
// Counts mismatching outputs (NaN matches NaN; bits otherwise, so -0 vs +0 would count).
#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_launch.h"
#include "sincos_math2.cuh"

namespace sincos_b200 {

__device__ __forceinline__ bool same_bits(float a, float b) {
    return (a != a && b != b) || __float_as_uint(a) == __float_as_uint(b);
}

// SHAPE -1: the paper's table of variant V; 0 / 1: method_from_q_exact<4,3,2,FIX> / <3,2,1,FIX>;
// -2: negative control, the scalar side uses the OTHER table (must mismatch almost everywhere)
template <int V, int SHAPE, int FIX>
__device__ __forceinline__ void scalar_from_q(const MethodParams &m, float q, float &s, float &c) {
    if constexpr (SHAPE == -2) sincos_from_q<1 - V>(q, s, c);
    else if constexpr (SHAPE < 0) sincos_from_q<V>(q, s, c);
    else if constexpr (SHAPE == 0) method_from_q_exact<4, 3, 2, FIX>(m, q, s, c);
    else method_from_q_exact<3, 2, 1, FIX>(m, q, s, c);
}
template <int V, int SHAPE, int FIX>
__device__ __forceinline__ void packed_from_q(const MethodParams &m, F2 q, F2 &s, F2 &c) {
    if constexpr (SHAPE < 0) sincos_from_q2<V>(q, s, c);   // -1 and -2
    else if constexpr (SHAPE == 0) method_from_q_exact2<4, 3, 2, FIX>(m, q, s, c);
    else method_from_q_exact2<3, 2, 1, FIX>(m, q, s, c);
}

template <int V, int SHAPE, int FIX>
__global__ void __launch_bounds__(256) packcheck_kernel(const MethodParams m, unsigned long long *mismatch) {
    const uint64_t nthr = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long bad = 0;
    for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < (1ull << 32);
         i += 2 * nthr) {
        const float x0 = __uint_as_float(static_cast<uint32_t>(i));
        const float x1 = __uint_as_float(static_cast<uint32_t>(i + 1));
#pragma unroll
        for (int turns = 0; turns < 2; ++turns) {
            const float y0 = turns ? x0 : __fmul_rn(x0, kInvTwoPi);
            const float y1 = turns ? x1 : __fmul_rn(x1, kInvTwoPi);
            float s0, c0, s1, c1;
            scalar_from_q<V, SHAPE, FIX>(m, reduce_turn(y0), s0, c0);
            scalar_from_q<V, SHAPE, FIX>(m, reduce_turn(y1), s1, c1);
            const F2 x = pk2(x0, x1);
            const F2 y = turns ? x : mul2(x, bc2(kInvTwoPi));
            F2 s, c;
            packed_from_q<V, SHAPE, FIX>(m, reduce_turn2(y), s, c);
            bad += !same_bits(s0, lo2(s)) + !same_bits(c0, lo2(c)) + !same_bits(s1, hi2(s)) +
                   !same_bits(c1, hi2(c));
        }
    }
    if (bad) atomicAdd(mismatch, bad);
}

cudaError_t launch_packcheck(int variant, int shape, int fix, const MethodParams *m, unsigned grid,
                             unsigned long long *mismatch_dev, cudaStream_t stream) {
    const MethodParams mp = m ? *m : MethodParams{};
    const void *fn;
    if (shape == -2)
        fn = reinterpret_cast<const void *>(packcheck_kernel<kNormalized, -2, 0>);
    else if (shape < 0)
        fn = variant == kNormalized ? reinterpret_cast<const void *>(packcheck_kernel<kNormalized, -1, 0>)
                                    : reinterpret_cast<const void *>(packcheck_kernel<kRenormalized, -1, 0>);
    else if (shape == 0)
        fn = fix == 0 ? reinterpret_cast<const void *>(packcheck_kernel<0, 0, 0>)
                      : reinterpret_cast<const void *>(packcheck_kernel<0, 0, 1>);
    else
        fn = fix == 0 ? reinterpret_cast<const void *>(packcheck_kernel<0, 1, 0>)
                      : reinterpret_cast<const void *>(packcheck_kernel<0, 1, 1>);
    void *args[] = {const_cast<MethodParams *>(&mp), &mismatch_dev};
    return cudaLaunchKernel(fn, dim3(grid), dim3(256), args, 0, stream);
}

}  // namespace sincos_b200
