// sincos_method.cuh -- NEXT(3): one pair by a general method (any series degrees up to
// NT, any doubling count, penultimate-pair fix), for the kernels in sincos_method.cu and
// sincos_nudft.cu.  See sincos_method.cu for the reading of the paper.
#pragma once

#include "sincos_math.cuh"

namespace sincos_b200 {

struct MethodParams {
    float ss[8];      // zero-padded: fma(q2, 0, c) == c, so padding is exact
    float cc[8];
    int doublings;
};

// FIX: 0 linear (2 - s^2 - c^2), 1 exact reciprocal 1/(s^2 + c^2), 3 none -- from the
// penultimate pair (Fig. 1).  q1 is the reduced turn.
template <int NT, int FIX>
__device__ __forceinline__ void method_from_q(const MethodParams &m, float q1, float &s_out, float &c_out) {
    const float q2 = __fmul_rn(q1, q1);
    float ps = m.ss[NT - 1];
#pragma unroll
    for (int i = NT - 2; i >= 0; --i) ps = __fmaf_rn(q2, ps, m.ss[i]);
    float pc = m.cc[NT - 1];
#pragma unroll
    for (int i = NT - 2; i >= 0; --i) pc = __fmaf_rn(q2, pc, m.cc[i]);
    float s = __fmul_rn(q1, ps);
    float c = __fmaf_rn(q2, pc, 1.0f);
    float f = 1.0f;
    if (m.doublings > 0) {
        for (int i = 0; i < m.doublings - 1; ++i) {          // warp-uniform bound
            const float cn = __fmaf_rn(-s, s, __fmul_rn(c, c));
            s = __fmul_rn(2.0f, __fmul_rn(s, c));
            c = cn;
        }
        const float cc2 = __fmul_rn(c, c);                   // (s, c): the penultimate pair
        if constexpr (FIX == 0) f = __fmaf_rn(-s, s, __fmaf_rn(-c, c, 2.0f));
        if constexpr (FIX == 1) f = rcp_rn(__fmaf_rn(s, s, cc2));
        const float cn = __fmaf_rn(-s, s, cc2);
        s = __fmul_rn(2.0f, __fmul_rn(s, c));
        c = cn;
    }
    c_out = __fmul_rn(c, f);
    s_out = __fmul_rn(s, f);
}

// The same with compile-time degrees and doubling count (no padding, no loop): used for the
// specialised shapes the launcher recognises.  Bit-identical to method_from_q.
template <int NS, int NC, int ND, int FIX>
__device__ __forceinline__ void method_from_q_exact(const MethodParams &m, float q1, float &s_out, float &c_out) {
    const float q2 = __fmul_rn(q1, q1);
    float ps = m.ss[NS - 1];
#pragma unroll
    for (int i = NS - 2; i >= 0; --i) ps = __fmaf_rn(q2, ps, m.ss[i]);
    float s = __fmul_rn(q1, ps);
    float c = 1.0f;
    if constexpr (NC > 0) {
        float pc = m.cc[NC - 1];
#pragma unroll
        for (int i = NC - 2; i >= 0; --i) pc = __fmaf_rn(q2, pc, m.cc[i]);
        c = __fmaf_rn(q2, pc, 1.0f);
    }
    float f = 1.0f;
    if constexpr (ND > 0) {
#pragma unroll
        for (int i = 0; i < ND - 1; ++i) {
            const float cn = __fmaf_rn(-s, s, __fmul_rn(c, c));
            s = __fmul_rn(2.0f, __fmul_rn(s, c));
            c = cn;
        }
        const float cc2 = __fmul_rn(c, c);
        if constexpr (FIX == 0) f = __fmaf_rn(-s, s, __fmaf_rn(-c, c, 2.0f));
        if constexpr (FIX == 1) f = rcp_rn(__fmaf_rn(s, s, cc2));
        const float cn = __fmaf_rn(-s, s, cc2);
        s = __fmul_rn(2.0f, __fmul_rn(s, c));
        c = cn;
    }
    c_out = __fmul_rn(c, f);
    s_out = __fmul_rn(s, f);
}

template <int NT, int FIX>
__device__ __forceinline__ void method_pair(const MethodParams &m, float theta, float &s_out, float &c_out) {
    method_from_q<NT, FIX>(m, reduce_turn(__fmul_rn(theta, kInvTwoPi)), s_out, c_out);
}

// N pairs at once from their reduced turns, stage by stage: the run-time doubling loop runs
// once over all N (per pair it would serialise the N independent chains behind N loops).  The
// same operations on each element as method_from_q: bit-identical.
template <int NT, int FIX, int N>
__device__ __forceinline__ void method_from_q_n(const MethodParams &m, const float (&q1)[N], float (&s_out)[N],
                                                float (&c_out)[N]) {
    // s_out / c_out hold the running pair from the series on (no separate arrays live)
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const float q2 = __fmul_rn(q1[k], q1[k]);
        float ps = m.ss[NT - 1];
#pragma unroll
        for (int i = NT - 2; i >= 0; --i) ps = __fmaf_rn(q2, ps, m.ss[i]);
        float pc = m.cc[NT - 1];
#pragma unroll
        for (int i = NT - 2; i >= 0; --i) pc = __fmaf_rn(q2, pc, m.cc[i]);
        s_out[k] = __fmul_rn(q1[k], ps);
        c_out[k] = __fmaf_rn(q2, pc, 1.0f);
    }
    if (m.doublings > 0) {
        for (int i = 0; i < m.doublings - 1; ++i) {          // warp-uniform bound
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const float s = s_out[k], c = c_out[k];
                c_out[k] = __fmaf_rn(-s, s, __fmul_rn(c, c));
                s_out[k] = __fmul_rn(2.0f, __fmul_rn(s, c));
            }
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const float s = s_out[k], c = c_out[k];          // the penultimate pair
            const float cc2 = __fmul_rn(c, c);
            float f = 1.0f;
            if constexpr (FIX == 0) f = __fmaf_rn(-s, s, __fmaf_rn(-c, c, 2.0f));
            if constexpr (FIX == 1) f = rcp_rn(__fmaf_rn(s, s, cc2));
            c_out[k] = __fmul_rn(__fmaf_rn(-s, s, cc2), f);
            s_out[k] = __fmul_rn(__fmul_rn(2.0f, __fmul_rn(s, c)), f);
        }
    }
    // (no doublings: the series pair times f = 1, i.e. unchanged -- as method_from_q)
}

// Eight pairs of angles in radians (the streaming kernel's vector).
template <int NT, int FIX>
__device__ __forceinline__ void method_pair8(const MethodParams &m, const float (&theta)[8], float (&s_out)[8],
                                             float (&c_out)[8]) {
    float q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = reduce_turn(__fmul_rn(theta[k], kInvTwoPi));
    method_from_q_n<NT, FIX, 8>(m, q, s_out, c_out);
}

inline MethodParams make_params(const float *ss, int n_ss, const float *cc, int n_cc, int doublings) {
    MethodParams m;
    for (int i = 0; i < 8; ++i) {
        m.ss[i] = i < n_ss ? ss[i] : 0.0f;
        m.cc[i] = i < n_cc ? cc[i] : 0.0f;
    }
    m.doublings = doublings;
    return m;
}

}  // namespace sincos_b200
