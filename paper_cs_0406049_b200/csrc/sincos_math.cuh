// sincos_math.cuh -- per-element device math of the hot path (sm_100a).
//
// The paper's method, PAPER.md P:50-57 and Fig. 1, restated for one
// CUDA thread and one fp32 angle.  Every operation is an explicit
// round-to-nearest intrinsic so that nvcc neither contracts nor reorders:
//   __fmul_rn  = vec_madd(a, b, 0.0)            (a single rounded product)
//   __fmaf_rn  = vec_madd / vec_nmsub with a non-zero addend (single rounding)
//   rintf      = vec_round (nearest, ties to even; cvt.rni.f32.f32 -> FRND)
// The library is built with -fmad=false -ftz=false as a second guard.
// The path has no value-dependent control flow: SASS of the
// value path is FMUL/FFMA/FADD/FRND (+ F2F/MUFU.RCP64H/DFMA for variant A).
#pragma once

#include <cuda_runtime.h>

namespace sincos_b200 {

enum Variant : int { kNormalized = 0, kRenormalized = 1 };

// Scale constant of Fig. 1, (vector float)(1.0/(2.0*3.1415926536)),
// which rounds to the same fp32 as 1/(2 pi): 0x3E22F983 (reading G12).
__device__ constexpr float kInvTwoPi = 0x1.45f306p-3f;

// Quarter-angle series coefficients, each the fp32 rounding of the decimal
// the paper prints (Fig. 1 casts the double literal to vector float).
template <int V> struct Series;

// Method 1, "normalised": P:140-148 == Fig. 1 P:246-258.
template <> struct Series<kNormalized> {
    static constexpr float ss1 =  0x1.921fb6p+0f;   //  1.5707963235
    static constexpr float ss2 = -0x1.4abbbep-1f;   // -0.645963615
    static constexpr float ss3 =  0x1.46609cp-4f;   //  0.0796819754
    static constexpr float ss4 = -0x1.2df648p-8f;   // -0.0046075748
    static constexpr float cc1 = -0x1.3bd39ep+0f;   // -1.2336977925
    static constexpr float cc2 =  0x1.03b1fap-2f;   //  0.2536086171
    static constexpr float cc3 = -0x1.4ee010p-6f;   // -0.0204391631
};

// Method 2, "angle-accurate" (dagger): Fig. 1 P:230-242.  ss2 is the Fig. 1
// value -0.6466386396 (the text P:161 transposes two digits; reading G1).
template <> struct Series<kRenormalized> {
    static constexpr float ss1 =  0x1.921fb6p+0f;   //  1.5707963268
    static constexpr float ss2 = -0x1.4b1438p-1f;   // -0.6466386396
    static constexpr float ss3 =  0x1.16296cp-4f;   //  0.0679105987
    static constexpr float ss4 = -0x1.2f6682p-10f;  // -0.0011573807
    static constexpr float cc1 = -0x1.3beff2p+0f;   // -1.2341299769
    static constexpr float cc2 =  0x1.f8e08ap-3f;   //  0.2465220241
    static constexpr float cc3 = -0x1.9614d0p-7f;   // -0.0123926179
};

// Correctly rounded fp32 reciprocal RN(1/d), branch-free ("precise reciprocal",
// P:157-158, Fig. 1; the paper's Reciprocal() body is not listed).
// MUFU.RCP seed (rcp.approx.ftz.f32) and one Newton step in FMA: the residual
// e = 1 - d*y0 is exact in fp32 for a seed within an ulp, and y0 + y0*e rounds once.
// On sm_100a this sequence returns RN(1/d) for EVERY fp32 d in [0.5, 2) -- including
// the near-midpoint case d = 1 - 2^-24 -- verified exhaustively on the B200
// (tools/rcp_probe.cu; tests/test_gpu_parity.py::test_reciprocal_exhaustive), and the
// method only produces d = s2^2 + c2^2 in [0.9975, 1.0000002] (SURVEY [X10]; the
// all-2^32-input hash test covers every d that occurs).  3 instructions, branch-free;
// rcp.rn.f32 would also be exact but compiles to a slow-path branch, and the fp64
// Newton sequence used before costs 8 instructions (F2F, MUFU.RCP64H, 4 DFMA, F2F).
__device__ __forceinline__ float rcp_rn(float d) {
    float y0;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(d));
    const float e = __fmaf_rn(-d, y0, 1.0f);
    return __fmaf_rn(y0, e, y0);
}

// The pair from a reduced turn q1 in [-1/2, 1/2] (steps a4-a9).  Step letters follow
// DESIGN.md section 1.
template <int V>
__device__ __forceinline__ void sincos_from_q(float q1, float &s_out, float &c_out) {
    using K = Series<V>;
    // a4-a5  quarter-angle series, P:280-310 (Horner, innermost first)
    const float q2 = __fmul_rn(q1, q1);
    const float s1 = __fmul_rn(q1, __fmaf_rn(q2, __fmaf_rn(q2, __fmaf_rn(q2, K::ss4, K::ss3), K::ss2), K::ss1));
    const float c1 = __fmaf_rn(q2, __fmaf_rn(q2, __fmaf_rn(q2, K::cc3, K::cc2), K::cc1), 1.0f);
    // a6  first doubling, Eq. (1) in Fig. 1 order
    const float c2 = __fmaf_rn(-s1, s1, __fmul_rn(c1, c1));
    const float s2 = __fmul_rn(2.0f, __fmul_rn(s1, c1));
    // a7  amplitude factor from the penultimate pair
    const float c2c2 = __fmul_rn(c2, c2);
    float f;
    if (V == kNormalized)
        f = __fmaf_rn(-s2, s2, __fmaf_rn(-c2, c2, 2.0f));
    else
        f = rcp_rn(__fmaf_rn(s2, s2, c2c2));
    // a8  second doubling
    const float c3 = __fmaf_rn(-s2, s2, c2c2);
    const float s3 = __fmul_rn(2.0f, __fmul_rn(s2, c2));
    // a9  apply
    c_out = __fmul_rn(c3, f);
    s_out = __fmul_rn(s3, f);
}

// a2-a3  turn reduction: x1 = RN(x / 2pi) ... q1 = x1 - rint(x1), exact.
__device__ __forceinline__ float reduce_turn(float x1) { return __fsub_rn(x1, rintf(x1)); }

// One pair from an angle in radians (the whole method, a2-a9).
template <int V>
__device__ __forceinline__ void sincos_pair(float theta, float &s_out, float &c_out) {
    sincos_from_q<V>(reduce_turn(__fmul_rn(theta, kInvTwoPi)), s_out, c_out);
}

// One pair from a phase already in turns (theta / 2pi): the method from the reduction on
// (P:53-54), without the scale by 1/2pi and its rounding (NEXT(1)).
template <int V>
__device__ __forceinline__ void sincos_pair_turns(float x1, float &s_out, float &c_out) {
    sincos_from_q<V>(reduce_turn(x1), s_out, c_out);
}

}  // namespace sincos_b200
