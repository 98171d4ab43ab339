// sincos_method.cu -- NEXT(3): the method with any series degrees and doubling count.
//
// Eq. (1) doublings keep the angle error and square the amplitude, so any
// number n of doublings works with series fitted for the angle 2 pi x / 2^n, by either
// fitting method (P:120-126 normalised, P:152-154 angle-accurate).  The coefficients
// come from the caller (e.g. paper_cs_0406049_b200.coeff_fit) and sit in the kernel's
// parameter (constant) bank.  Series are evaluated with a fixed-length Horner over
// zero-padded coefficients: fma(q2, 0, c) == c exactly, so padding leaves the result
// bit-identical to the unpadded Horner of the method's own degree and keeps the
// per-element code branch-free (the doubling count is a warp-uniform loop bound).
#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_launch.h"
#include "sincos_method.cuh"
#include "sincos_realign.cuh"
#include "sincos_storeshift.cuh"

namespace sincos_b200 {

template <int NT, int FIX, bool INTER>
__device__ __forceinline__ void method_scalar(const MethodParams &m, const float *theta, size_t e, float *so,
                                              float *co, float *io) {
    float s, c;
    method_pair<NT, FIX>(m, theta[e], s, c);
    if constexpr (INTER) {
        io[2 * e] = c;
        io[2 * e + 1] = s;
    } else {
        so[e] = s;
        co[e] = c;
    }
}

__device__ __forceinline__ void st8m(float *p, const float *r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}

// Full grid, eight angles per thread over [head, head + 8 nvec); scalar head/tail.
// K = 0: theta shares the outputs' 32-B alignment (one aligned 256-bit load per thread).
// K = 1..7 (a template parameter): theta sits K floats off it and is re-aligned in registers
// (sincos_realign.cuh), with warp-uniform trips for the shuffles.
// SH (split only): cos[] sits kc = 1..7 floats off sin[]'s 32-B frame and is written as whole
// 32-B blocks re-aligned by warp shuffles (KB3c's store_realigned, sincos_storeshift.cuh).
// vec == false: every element scalar (interleaved pairs only 4-B aligned).
template <int NT, int FIX, bool INTER, int K, bool SH>
__global__ void __launch_bounds__(128) method_kernel(const MethodParams m, const float *theta, float *so,
                                                     float *co, float *io, size_t head, size_t nvec, size_t n,
                                                     bool vec, int k, int kc) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (!vec) {
        for (size_t e = tid; e < n; e += nthr) method_scalar<NT, FIX, INTER>(m, theta, e, so, co, io);
        return;
    }
    const size_t tail0 = head + 8 * nvec;
    if (tid < head) method_scalar<NT, FIX, INTER>(m, theta, tid, so, co, io);
    if (tid < n - tail0) method_scalar<NT, FIX, INTER>(m, theta, tail0 + tid, so, co, io);
    const unsigned lane = threadIdx.x & 31u;
    const float *tal = theta + head - k;
    constexpr bool RE = K > 0;
    constexpr bool WU = RE || SH;          // warp-uniform trips: the shuffles need all 32 lanes
    for (size_t w0 = WU ? tid - lane : tid; w0 < nvec; w0 += nthr) {
        const size_t v = WU ? w0 + lane : w0;
        const bool act = v < nvec;
        float x[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        if constexpr (RE) {
            load8_realigned_k<(K > 0 ? K : 1)>(tal, v, nvec, lane, act, x);
            if (!SH && !act) continue;
        } else if constexpr (SH) {
            if (act) ld8_stream(x, theta + head + 8 * v);
        } else {
            ld8_stream(x, theta + head + 8 * v);
        }
        const size_t e0 = head + 8 * v;
        float sv[8], cv[8];
        method_pair8<NT, FIX>(m, x, sv, cv);
        if constexpr (INTER) {
            float cs[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                cs[2 * k] = cv[k];
                cs[2 * k + 1] = sv[k];
            }
            if constexpr (SH) {
                // pairs only 4-B aligned: theta's frame, the pairs kc = 1/3/5/7 floats off it
                const bool last = act && (lane == 31u || v + 1 >= nvec);
                switch (kc) {
                case 1: store_realigned<16, 1>(io, 2 * e0, cs, 1, lane, act, last); break;
                case 3: store_realigned<16, 3>(io, 2 * e0, cs, 3, lane, act, last); break;
                case 5: store_realigned<16, 5>(io, 2 * e0, cs, 5, lane, act, last); break;
                default: store_realigned<16, 7>(io, 2 * e0, cs, 7, lane, act, last); break;
                }
            } else {
                st8m(io + 2 * e0, cs);
                st8m(io + 2 * e0 + 8, cs + 8);
            }
        } else if constexpr (SH) {
            const bool last = act && (lane == 31u || v + 1 >= nvec);
            if (act) st8m(so + e0, sv);
            switch (kc) {
            case 1: store_realigned<8, 1>(co, e0, cv, 1, lane, act, last); break;
            case 2: store_realigned<8, 2>(co, e0, cv, 2, lane, act, last); break;
            case 3: store_realigned<8, 3>(co, e0, cv, 3, lane, act, last); break;
            case 4: store_realigned<8, 4>(co, e0, cv, 4, lane, act, last); break;
            case 5: store_realigned<8, 5>(co, e0, cv, 5, lane, act, last); break;
            case 6: store_realigned<8, 6>(co, e0, cv, 6, lane, act, last); break;
            default: store_realigned<8, 7>(co, e0, cv, 7, lane, act, last); break;
            }
        } else {
            st8m(so + e0, sv);
            st8m(co + e0, cv);
        }
    }
}

template <int NT, int FIX, int K>
static const void *pick_mr(bool inter, bool sh) {
    if (inter)
        return sh ? reinterpret_cast<const void *>(method_kernel<NT, FIX, true, 0, true>)
                  : reinterpret_cast<const void *>(method_kernel<NT, FIX, true, K, false>);
    return sh ? reinterpret_cast<const void *>(method_kernel<NT, FIX, false, K, true>)
              : reinterpret_cast<const void *>(method_kernel<NT, FIX, false, K, false>);
}
template <int NT, int FIX>
static const void *pick_m(bool inter, int k, bool sh) {
    switch (k) {
    case 0: return pick_mr<NT, FIX, 0>(inter, sh);
    case 1: return pick_mr<NT, FIX, 1>(inter, sh);
    case 2: return pick_mr<NT, FIX, 2>(inter, sh);
    case 3: return pick_mr<NT, FIX, 3>(inter, sh);
    case 4: return pick_mr<NT, FIX, 4>(inter, sh);
    case 5: return pick_mr<NT, FIX, 5>(inter, sh);
    case 6: return pick_mr<NT, FIX, 6>(inter, sh);
    default: return pick_mr<NT, FIX, 7>(inter, sh);
    }
}

// fix: 0 linear (penultimate), 1 reciprocal (penultimate), 3 none.  Terms <= 4 use the
// 4-term Horner, otherwise the 8-term one.
cudaError_t launch_method(const float *ss, int n_ss, const float *cc, int n_cc, int doublings, int fix, bool inter,
                          bool vec, unsigned grid, const float *theta, float *so, float *co, float *io, size_t head,
                          size_t nvec, size_t n, int k, cudaStream_t stream) {
    MethodParams m = make_params(ss, n_ss, cc, n_cc, doublings);
    const bool small = n_ss <= 4 && n_cc <= 4;
    const void *fn;
    const int kk = vec ? k : 0;
    // split: cos[]'s float offset from sin[]'s 32-B frame at the vector elements; interleaved
    // pairs only 4-B aligned: their float offset from theta's frame (odd)
    int kc = !vec ? 0
             : inter ? (reinterpret_cast<uintptr_t>(io) & 7 ? static_cast<int>(((reinterpret_cast<uintptr_t>(io) + 8 * head) & 31) / 4) : 0)
                     : static_cast<int>(((reinterpret_cast<uintptr_t>(co) + 4 * head) & 31) / 4);
    const bool sh = kc != 0;
    if (small)
        fn = fix == 0 ? pick_m<4, 0>(inter, kk, sh) : fix == 1 ? pick_m<4, 1>(inter, kk, sh) : pick_m<4, 3>(inter, kk, sh);
    else
        fn = fix == 0 ? pick_m<8, 0>(inter, kk, sh) : fix == 1 ? pick_m<8, 1>(inter, kk, sh) : pick_m<8, 3>(inter, kk, sh);
    void *args[] = {&m, &theta, &so, &co, &io, &head, &nvec, &n, &vec, &k, &kc};
    return cudaLaunchKernel(fn, dim3(grid), dim3(128), args, 0, stream);
}

}  // namespace sincos_b200
