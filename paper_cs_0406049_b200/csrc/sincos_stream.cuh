// sincos_stream.cuh -- the streaming building blocks shared by the hot-path kernels
// (sincos_kernels.cu, sincos_outshift.cu): the per-element operation of each kernel "variant"
// (the paper's two methods, the no-math ceiling, the CUDA-function context kernels), the
// 128/256-bit streaming loads and stores, and the per-vector / per-element emitters.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_math.cuh"

namespace sincos_b200 {

constexpr int kNull = 2;  // KB4: the traffic-ceiling "variant"
// Context only (bench): CUDA's own functions with the same traffic -- libm sincosf (accurate,
// Payne-Hanek slow path for large arguments) and the __sincosf intrinsic.
constexpr int kCmpSincosf = 3;
constexpr int kCmpIntrinsic = 4;

template <int V>
__device__ __forceinline__ void op(float t, float &s, float &c) {
    if constexpr (V == kNull) {
        s = t;
        c = t;
    } else if constexpr (V == kCmpSincosf) {
        sincosf(t, &s, &c);
    } else if constexpr (V == kCmpIntrinsic) {
        __sincosf(t, &s, &c);
    } else {
        sincos_pair<V>(t, s, c);
    }
}

// ---- streaming memory access ----------------------------------------------
// Cache-policy qualifiers of the 256-bit accesses (overridable at build time for the
// policy experiment in tools/hint_experiment.py; the defaults were measured best).
#ifndef SINCOS_LD8_Q
#define SINCOS_LD8_Q ".L1::no_allocate.L2::evict_first"
#endif
#ifndef SINCOS_ST8_Q
#define SINCOS_ST8_Q ".L1::no_allocate.L2::evict_first"
#endif
template <int W, bool NC> struct Mem;

template <> struct Mem<8, true> {
    static __device__ __forceinline__ void load(float (&r)[8], const float *p) {
        asm volatile("ld.global.nc" SINCOS_LD8_Q ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                     : "l"(p));
    }
};
template <> struct Mem<8, false> {
    static __device__ __forceinline__ void load(float (&r)[8], const float *p) {
        asm volatile("ld.global" SINCOS_LD8_Q ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                     : "l"(p));
    }
};
template <> struct Mem<4, true> {
    static __device__ __forceinline__ void load(float (&r)[4], const float *p) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
                     : "l"(p));
    }
};
template <> struct Mem<4, false> {
    static __device__ __forceinline__ void load(float (&r)[4], const float *p) {
        asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
                     : "l"(p));
    }
};

__device__ __forceinline__ void store8(float *p, const float *r) {
    asm volatile("st.global" SINCOS_ST8_Q ".v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}
__device__ __forceinline__ void store4(float *p, const float *r) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3])
                 : "memory");
}
template <int W>
__device__ __forceinline__ void storeW(float *p, const float *r) {
    if constexpr (W == 8) store8(p, r); else store4(p, r);
}

// Compute and store one vector of W elements whose first element is `e0`.
template <int V, bool INTER, int W>
__device__ __forceinline__ void emit(const float (&x)[W], size_t e0, float *so, float *co, float *io) {
    if constexpr (INTER) {
        float cs[2 * W];
#pragma unroll
        for (int k = 0; k < W; ++k) op<V>(x[k], cs[2 * k + 1], cs[2 * k]);
#pragma unroll
        for (int h = 0; h < 2; ++h) storeW<W>(io + 2 * e0 + h * W, cs + h * W);
    } else {
        float s[W], c[W];
#pragma unroll
        for (int k = 0; k < W; ++k) op<V>(x[k], s[k], c[k]);
        storeW<W>(so + e0, s);
        storeW<W>(co + e0, c);
    }
}

template <int V, bool INTER>
__device__ __forceinline__ void emit_scalar(const float *theta, size_t e, float *so, float *co, float *io) {
    float s, c;
    op<V>(theta[e], s, c);
    if constexpr (INTER) {
        io[2 * e] = c;
        io[2 * e + 1] = s;
    } else {
        so[e] = s;
        co[e] = c;
    }
}

}  // namespace sincos_b200
