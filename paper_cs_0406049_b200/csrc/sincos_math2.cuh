// sincos_math2.cuh -- the per-element math of sincos_math.cuh on two elements at once,
// with sm_100a's packed fp32 instructions (PTX fma/mul/add.rn.f32x2 -> SASS FFMA2 /
// FMUL2 / FADD2).
//
// Each packed instruction rounds each of its two lanes exactly as the scalar instruction
// does (IEEE RN-even, no flush-to-zero without .ftz), so every function here is
// bit-identical, lane by lane, to its scalar twin -- the same operations in the same
// order (Fig. 1).  What changes is the issue cost: one instruction per two
// elements, which matters only where the pairs are consumed in registers and the kernel
// is bound by instruction issue (the fused sum, sincos_nudft.cu), not by HBM.
// FRND (vec_round, cvt.rni) and MUFU.RCP have no packed form and stay scalar.
#pragma once

#include <stdint.h>

#include "sincos_math.cuh"
#include "sincos_method.cuh"

namespace sincos_b200 {

// Two fp32 lanes in one 64-bit register pair: lo = element 0, hi = element 1.
struct F2 {
    uint64_t v;
};

__device__ __forceinline__ F2 pk2(float lo, float hi) {
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ F2 bc2(float x) { return pk2(x, x); }
__device__ __forceinline__ float lo2(F2 a) { return __uint_as_float(static_cast<uint32_t>(a.v)); }
__device__ __forceinline__ float hi2(F2 a) { return __uint_as_float(static_cast<uint32_t>(a.v >> 32)); }
// RN(a*b + c) per lane (one rounding)
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
    F2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return d;
}
// RN(-a*b + c) per lane: the negation is written on the halves so that ptxas folds it
// into the FFMA2 operand modifier (no extra instruction)
__device__ __forceinline__ F2 nfma2(F2 a, F2 b, F2 c) {
    F2 d;
    asm("{\n\t.reg .f32 a0, a1;\n\t.reg .b64 na;\n\t"
        "mov.b64 {a0, a1}, %1;\n\tneg.f32 a0, a0;\n\tneg.f32 a1, a1;\n\t"
        "mov.b64 na, {a0, a1};\n\tfma.rn.f32x2 %0, na, %2, %3;\n\t}"
        : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return d;
}
// RN(a*b) per lane
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
    F2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}
// RN(a - b) per lane
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
    F2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
    return d;
}

// a2-a3 on two lanes: q = x1 - rint(x1) (FRND per lane, one FADD2)
__device__ __forceinline__ F2 reduce_turn2(F2 x1) { return sub2(x1, pk2(rintf(lo2(x1)), rintf(hi2(x1)))); }

// rcp_rn on two lanes: MUFU.RCP per lane, the Newton step packed (same arithmetic)
__device__ __forceinline__ F2 rcp_rn2(F2 d) {
    float y0l, y0h;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y0l) : "f"(lo2(d)));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y0h) : "f"(hi2(d)));
    const F2 y0 = pk2(y0l, y0h);
    const F2 e = nfma2(d, y0, bc2(1.0f));
    return fma2(y0, e, y0);
}

// sincos_from_q<V> on two lanes (steps a4-a9, same operations, same order)
template <int V>
__device__ __forceinline__ void sincos_from_q2(F2 q1, F2 &s_out, F2 &c_out) {
    using K = Series<V>;
    const F2 q2 = mul2(q1, q1);
    const F2 s1 = mul2(q1, fma2(q2, fma2(q2, fma2(q2, bc2(K::ss4), bc2(K::ss3)), bc2(K::ss2)), bc2(K::ss1)));
    const F2 c1 = fma2(q2, fma2(q2, fma2(q2, bc2(K::cc3), bc2(K::cc2)), bc2(K::cc1)), bc2(1.0f));
    const F2 c2 = nfma2(s1, s1, mul2(c1, c1));
    const F2 s2 = mul2(bc2(2.0f), mul2(s1, c1));
    const F2 c2c2 = mul2(c2, c2);
    F2 f;
    if (V == kNormalized)
        f = nfma2(s2, s2, nfma2(c2, c2, bc2(2.0f)));
    else
        f = rcp_rn2(fma2(s2, s2, c2c2));
    const F2 c3 = nfma2(s2, s2, c2c2);
    const F2 s3 = mul2(bc2(2.0f), mul2(s2, c2));
    c_out = mul2(c3, f);
    s_out = mul2(s3, f);
}

// method_from_q_exact<NS, NC, ND, FIX> on two lanes (compile-time shapes)
template <int NS, int NC, int ND, int FIX>
__device__ __forceinline__ void method_from_q_exact2(const MethodParams &m, F2 q1, F2 &s_out, F2 &c_out) {
    const F2 q2 = mul2(q1, q1);
    F2 ps = bc2(m.ss[NS - 1]);
#pragma unroll
    for (int i = NS - 2; i >= 0; --i) ps = fma2(q2, ps, bc2(m.ss[i]));
    F2 s = mul2(q1, ps);
    F2 c = bc2(1.0f);
    if constexpr (NC > 0) {
        F2 pc = bc2(m.cc[NC - 1]);
#pragma unroll
        for (int i = NC - 2; i >= 0; --i) pc = fma2(q2, pc, bc2(m.cc[i]));
        c = fma2(q2, pc, bc2(1.0f));
    }
    F2 f = bc2(1.0f);
    if constexpr (ND > 0) {
#pragma unroll
        for (int i = 0; i < ND - 1; ++i) {
            const F2 cn = nfma2(s, s, mul2(c, c));
            s = mul2(bc2(2.0f), mul2(s, c));
            c = cn;
        }
        const F2 cc2 = mul2(c, c);
        if constexpr (FIX == 0) f = nfma2(s, s, nfma2(c, c, bc2(2.0f)));
        if constexpr (FIX == 1) f = rcp_rn2(fma2(s, s, cc2));
        const F2 cn = nfma2(s, s, cc2);
        s = mul2(bc2(2.0f), mul2(s, c));
        c = cn;
    }
    c_out = mul2(c, f);
    s_out = mul2(s, f);
}

// method_from_q_n<NT, FIX, 2 N2> on N2 lane pairs (run-time doubling count, zero-padded
// Horner): the same operations, stage by stage, lane by lane.
template <int NT, int FIX, int N2>
__device__ __forceinline__ void method_from_q_n2(const MethodParams &m, const F2 (&q1)[N2], F2 (&s_out)[N2],
                                                 F2 (&c_out)[N2]) {
#pragma unroll
    for (int k = 0; k < N2; ++k) {
        const F2 q2 = mul2(q1[k], q1[k]);
        F2 ps = bc2(m.ss[NT - 1]);
#pragma unroll
        for (int i = NT - 2; i >= 0; --i) ps = fma2(q2, ps, bc2(m.ss[i]));
        F2 pc = bc2(m.cc[NT - 1]);
#pragma unroll
        for (int i = NT - 2; i >= 0; --i) pc = fma2(q2, pc, bc2(m.cc[i]));
        s_out[k] = mul2(q1[k], ps);
        c_out[k] = fma2(q2, pc, bc2(1.0f));
    }
    if (m.doublings > 0) {
        for (int i = 0; i < m.doublings - 1; ++i) {          // warp-uniform bound
#pragma unroll
            for (int k = 0; k < N2; ++k) {
                const F2 s = s_out[k], c = c_out[k];
                c_out[k] = nfma2(s, s, mul2(c, c));
                s_out[k] = mul2(bc2(2.0f), mul2(s, c));
            }
        }
#pragma unroll
        for (int k = 0; k < N2; ++k) {
            const F2 s = s_out[k], c = c_out[k];             // the penultimate pair
            const F2 cc2 = mul2(c, c);
            F2 f = bc2(1.0f);
            if constexpr (FIX == 0) f = nfma2(s, s, nfma2(c, c, bc2(2.0f)));
            if constexpr (FIX == 1) f = rcp_rn2(fma2(s, s, cc2));
            c_out[k] = mul2(nfma2(s, s, cc2), f);
            s_out[k] = mul2(mul2(bc2(2.0f), mul2(s, c)), f);
        }
    }
}

}  // namespace sincos_b200
