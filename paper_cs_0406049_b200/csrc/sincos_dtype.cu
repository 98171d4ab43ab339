// sincos_dtype.cu -- NEXT(4): other output dtypes and SoA <-> AoS adapters.
//
// Half-width outputs: the pair is evaluated by the method in fp32 exactly as in
// sincos_pairs and then rounded once to IEEE binary16 or bfloat16 (round to nearest
// even).  Traffic drops from 12 to 8 bytes per pair (4 in, 2 x 2 out), so the same HBM
// roofline gives 1.5x the pairs per second.  The adapters convert between the split
// (sin[], cos[]) and interleaved ({cos, sin} float2) fp32 layouts.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_launch.h"
#include "sincos_math.cuh"
#include "sincos_realign.cuh"

namespace sincos_b200 {

template <int DT> __device__ __forceinline__ uint16_t to16(float x);
template <> __device__ __forceinline__ uint16_t to16<1>(float x) { return __half_as_ushort(__float2half_rn(x)); }
template <> __device__ __forceinline__ uint16_t to16<2>(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

__device__ __forceinline__ uint32_t pack2(uint16_t lo, uint16_t hi) {
    return static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
}

__device__ __forceinline__ void st4u(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// cos[] when it does not share sin[]'s 16-B offset (split outputs): the eight values at a
// position whose alignment `cw` is the same for every vector (16 / 8 / 4 / 2 bytes: one 128-bit
// store, two 64-bit, four 32-bit or eight 16-bit ones -- warp-uniform; each warp instruction still
// covers its 32 threads' neighbouring blocks, which L2 merges into whole sectors).
__device__ __forceinline__ void st8x16(uint16_t *p, const uint16_t (&c)[8], int cw) {
    if (cw == 16) {
        st4u(p, pack2(c[0], c[1]), pack2(c[2], c[3]), pack2(c[4], c[5]), pack2(c[6], c[7]));
    } else if (cw == 8) {
#pragma unroll
        for (int h = 0; h < 8; h += 4)
            asm volatile("st.global.L1::no_allocate.v2.b32 [%0], {%1,%2};" ::"l"(p + h), "r"(pack2(c[h], c[h + 1])),
                         "r"(pack2(c[h + 2], c[h + 3]))
                         : "memory");
    } else if (cw == 4) {
#pragma unroll
        for (int h = 0; h < 8; h += 2)
            asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" ::"l"(p + h), "r"(pack2(c[h], c[h + 1])) : "memory");
    } else {
#pragma unroll
        for (int h = 0; h < 8; ++h)
            asm volatile("st.global.L1::no_allocate.b16 [%0], %1;" ::"l"(p + h), "h"(c[h]) : "memory");
    }
}

// Halfwords [A, B) of a 16-B block from r[0 .. B - A), as naturally aligned pieces (2 / 4 / 8 B).
template <int A, int B>
__device__ __forceinline__ void store16_range(uint16_t *blk, const uint16_t *r) {
    if constexpr (A < B) {
        constexpr int al = (A & 1) ? 1 : (A & 2) ? 2 : 4;             // alignment of position A, halfwords
        constexpr int m = al <= (B - A) ? al : ((B - A) >= 2 ? 2 : 1);
        if constexpr (m == 4)
            asm volatile("st.global.L1::no_allocate.v2.b32 [%0], {%1,%2};" ::"l"(blk + A), "r"(pack2(r[0], r[1])),
                         "r"(pack2(r[2], r[3]))
                         : "memory");
        else if constexpr (m == 2)
            asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" ::"l"(blk + A), "r"(pack2(r[0], r[1])) : "memory");
        else
            asm volatile("st.global.L1::no_allocate.b16 [%0], %1;" ::"l"(blk + A), "h"(r[0]) : "memory");
        store16_range<A + m, B>(blk, r + m);
    }
}

// cos[] O halfwords (1..7) past sin[]'s 16-B frame, written as whole aligned 16-B blocks built
// from the neighbouring lane's values -- the output re-alignment of KB3c (sincos_outshift.cu)
// on 16-bit elements: O <= 4 the block at e0 - O takes the previous lane's last O values
// (shuffled up), O > 4 the block at e0 + 8 - O the next lane's first 8 - O (shuffled down);
// the warp's lane 0 and last active lane store their partial blocks as aligned pieces.  All 32
// lanes call it.
template <int O>
__device__ __forceinline__ void store16_shift(uint16_t *x, size_t e0, const uint16_t (&c)[8], unsigned lane, bool act,
                                              bool last) {
    uint16_t *blk0 = x + e0 - O;
    if constexpr (O <= 4) {
        uint16_t prev[O];
#pragma unroll
        for (int j = 0; j < O; ++j)
            prev[j] = static_cast<uint16_t>(__shfl_up_sync(0xFFFFFFFFu, static_cast<unsigned>(c[8 - O + j]), 1));
        if (!act) return;
        if (lane > 0) {
            uint16_t b[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = j < O ? prev[j] : c[j - O];
            st4u(blk0, pack2(b[0], b[1]), pack2(b[2], b[3]), pack2(b[4], b[5]), pack2(b[6], b[7]));
        } else {
            store16_range<O, 8>(blk0, c);
        }
        if (last) store16_range<0, O>(blk0 + 8, c + 8 - O);
    } else {
        constexpr int D = 8 - O;
        uint16_t next[D];
#pragma unroll
        for (int j = 0; j < D; ++j)
            next[j] = static_cast<uint16_t>(__shfl_down_sync(0xFFFFFFFFu, static_cast<unsigned>(c[j]), 1));
        if (!act) return;
        if (lane == 0) store16_range<O, 8>(blk0, c);
        if (last) {
            store16_range<0, O>(blk0 + 8, c + D);
        } else {
            uint16_t b[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = j < O ? c[D + j] : next[j - O];
            st4u(blk0 + 8, pack2(b[0], b[1]), pack2(b[2], b[3]), pack2(b[4], b[5]), pack2(b[6], b[7]));
        }
    }
}

template <int V, int DT, bool INTER>
__device__ __forceinline__ void emit16_scalar(const float *theta, size_t e, uint16_t *so, uint16_t *co,
                                              uint16_t *io) {
    float s, c;
    sincos_pair<V>(theta[e], s, c);
    if constexpr (INTER) {
        io[2 * e] = to16<DT>(c);
        io[2 * e + 1] = to16<DT>(s);
    } else {
        so[e] = to16<DT>(s);
        co[e] = to16<DT>(c);
    }
}

// Full grid, eight angles per thread; outputs: split 2 x 128-bit, interleaved 256-bit.
// K = 0: theta shares the outputs' vector alignment (one aligned 256-bit load per thread, 32
// registers: full occupancy).  K = 1..7 (a template parameter): theta sits K floats off it and is
// re-aligned in registers (sincos_realign.cuh), with warp-uniform trips for the shuffles.
template <int V, int DT, bool INTER, int K, bool SH>
__global__ void __launch_bounds__(128) sincos16_kernel(const float *theta, uint16_t *so, uint16_t *co, uint16_t *io,
                                                       size_t head, size_t nvec, size_t n, int k, int cw) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t tail0 = head + 8 * nvec;
    if (tid < head) emit16_scalar<V, DT, INTER>(theta, tid, so, co, io);
    if (tid < n - tail0) emit16_scalar<V, DT, INTER>(theta, tail0 + tid, so, co, io);
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
        uint16_t s16[8], c16[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float s, c;
            sincos_pair<V>(x[k], s, c);
            s16[k] = to16<DT>(s);
            c16[k] = to16<DT>(c);
        }
        if constexpr (INTER) {
            uint32_t w[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) w[k] = pack2(c16[k], s16[k]);
            asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                         ::"l"(io + 2 * e0), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]),
                         "r"(w[6]), "r"(w[7])
                         : "memory");
        } else if constexpr (SH) {
            // cw: cos[]'s halfword offset O (1..7) at the vector elements
            const bool last = act && (lane == 31u || v + 1 >= nvec);
            if (act)
                st4u(so + e0, pack2(s16[0], s16[1]), pack2(s16[2], s16[3]), pack2(s16[4], s16[5]),
                     pack2(s16[6], s16[7]));
            switch (cw) {
            case 1: store16_shift<1>(co, e0, c16, lane, act, last); break;
            case 2: store16_shift<2>(co, e0, c16, lane, act, last); break;
            case 3: store16_shift<3>(co, e0, c16, lane, act, last); break;
            case 4: store16_shift<4>(co, e0, c16, lane, act, last); break;
            case 5: store16_shift<5>(co, e0, c16, lane, act, last); break;
            case 6: store16_shift<6>(co, e0, c16, lane, act, last); break;
            default: store16_shift<7>(co, e0, c16, lane, act, last); break;
            }
        } else {
            st4u(so + e0, pack2(s16[0], s16[1]), pack2(s16[2], s16[3]), pack2(s16[4], s16[5]), pack2(s16[6], s16[7]));
            st8x16(co + e0, c16, cw);
        }
    }
}

// cos[] re-aligned by shuffles (SH) unless it shares sin[]'s 16-B offset or sits 8 B off it
// (there two 64-bit stores per vector run at the aligned rate); cw = 16 / 8 / halfword offset
#ifndef SINCOS_16_SHIFT
#define SINCOS_16_SHIFT 1                    // 0: the 4-/2-B piece stores instead (A/B)
#endif
template <int V, int DT, int K>
static const void *pick16r(bool inter, bool sh) {
    if (inter) return reinterpret_cast<const void *>(sincos16_kernel<V, DT, true, K, false>);
    return sh ? reinterpret_cast<const void *>(sincos16_kernel<V, DT, false, K, true>)
              : reinterpret_cast<const void *>(sincos16_kernel<V, DT, false, K, false>);
}
template <int V, int DT>
static const void *pick16i(bool inter, int k, bool sh) {
    switch (k) {
    case 0: return pick16r<V, DT, 0>(inter, sh);
    case 1: return pick16r<V, DT, 1>(inter, sh);
    case 2: return pick16r<V, DT, 2>(inter, sh);
    case 3: return pick16r<V, DT, 3>(inter, sh);
    case 4: return pick16r<V, DT, 4>(inter, sh);
    case 5: return pick16r<V, DT, 5>(inter, sh);
    case 6: return pick16r<V, DT, 6>(inter, sh);
    default: return pick16r<V, DT, 7>(inter, sh);
    }
}

cudaError_t launch_pairs16(int variant, int dtype, bool inter, unsigned grid, const float *theta, void *so, void *co,
                           void *io, size_t head, size_t nvec, size_t n, int k, int cw, cudaStream_t stream) {
    const void *fn;
    // cw: cos[]'s alignment in bytes at the vector elements (16, 8, 4, 2)
    const bool sh = SINCOS_16_SHIFT && !inter && cw != 16 && cw != 8;
    if (sh) cw = static_cast<int>(((reinterpret_cast<uintptr_t>(co) + 2 * head) & 15) / 2);   // halfword offset
    if (variant == kNormalized)
        fn = dtype == 1 ? pick16i<kNormalized, 1>(inter, k, sh) : pick16i<kNormalized, 2>(inter, k, sh);
    else
        fn = dtype == 1 ? pick16i<kRenormalized, 1>(inter, k, sh) : pick16i<kRenormalized, 2>(inter, k, sh);
    uint16_t *s = static_cast<uint16_t *>(so), *c = static_cast<uint16_t *>(co), *i = static_cast<uint16_t *>(io);
    void *args[] = {&theta, &s, &c, &i, &head, &nvec, &n, &k, &cw};
    return cudaLaunchKernel(fn, dim3(grid), dim3(128), args, 0, stream);
}

// ---- adapters: split <-> interleaved (fp32) ---------------------------------------------------
// Vector body when sin, cos and the pairs are 16-B aligned: a thread moves 4 elements -- two
// 128-bit loads and two 128-bit stores (whole sectors per warp instruction); any other alignment
// and the ragged tail one element per thread.  Grid-stride.
__global__ void __launch_bounds__(256) interleave_kernel(const float *__restrict__ s, const float *__restrict__ c,
                                                         float2 *__restrict__ io, size_t n) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(c) |
                       reinterpret_cast<uintptr_t>(io)) & 15) == 0;
    const size_t nv = vec ? n / 4 : 0;
    for (size_t v = tid; v < nv; v += nthr) {
        const float4 sv = __ldcs(reinterpret_cast<const float4 *>(s) + v);
        const float4 cv = __ldcs(reinterpret_cast<const float4 *>(c) + v);
        float4 *o = reinterpret_cast<float4 *>(io + 4 * v);
        __stcs(o, make_float4(cv.x, sv.x, cv.y, sv.y));
        __stcs(o + 1, make_float4(cv.z, sv.z, cv.w, sv.w));
    }
    for (size_t e = 4 * nv + tid; e < n; e += nthr) io[e] = make_float2(__ldcs(c + e), __ldcs(s + e));
}

__global__ void __launch_bounds__(256) deinterleave_kernel(const float2 *__restrict__ io, float *__restrict__ s,
                                                           float *__restrict__ c, size_t n) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(c) |
                       reinterpret_cast<uintptr_t>(io)) & 15) == 0;
    const size_t nv = vec ? n / 4 : 0;
    for (size_t v = tid; v < nv; v += nthr) {
        const float4 *p = reinterpret_cast<const float4 *>(io + 4 * v);
        const float4 a = __ldcs(p), b = __ldcs(p + 1);
        __stcs(reinterpret_cast<float4 *>(c) + v, make_float4(a.x, a.z, b.x, b.z));
        __stcs(reinterpret_cast<float4 *>(s) + v, make_float4(a.y, a.w, b.y, b.w));
    }
    for (size_t e = 4 * nv + tid; e < n; e += nthr) {
        const float2 v = __ldcs(io + e);
        __stcs(c + e, v.x);
        __stcs(s + e, v.y);
    }
}

// All three buffers 32-B aligned: eight elements per thread with 256-bit streaming accesses
// (L1 no-allocate, L2 evict-first) in the full grid of 128-thread blocks, like the hot path --
// every warp access covers whole lines (the 128-bit form ran 5.98 / 6.06 TB/s).
__device__ __forceinline__ void ld8_nc(float (&r)[8], const float *p) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st8_nc(float *p, const float *r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}

#ifndef SINCOS_ADAPTER_MINB
#define SINCOS_ADAPTER_MINB 8      // 64 registers, 8 blocks/SM: 6.95-6.97 TB/s (1: 72 regs, 5.82-5.87; 12: 6.85)
#endif
__global__ void __launch_bounds__(128, SINCOS_ADAPTER_MINB) interleave8_kernel(const float *__restrict__ s, const float *__restrict__ c,
                                                          float *__restrict__ io, size_t n) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nv = n / 8;
    for (size_t v = tid; v < nv; v += nthr) {
        float sv[8], cv[8], o[16];
        ld8_nc(sv, s + 8 * v);
        ld8_nc(cv, c + 8 * v);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            o[2 * k] = cv[k];
            o[2 * k + 1] = sv[k];
        }
        st8_nc(io + 16 * v, o);
        st8_nc(io + 16 * v + 8, o + 8);
    }
    for (size_t e = 8 * nv + tid; e < n; e += nthr) {
        io[2 * e] = c[e];
        io[2 * e + 1] = s[e];
    }
}

__global__ void __launch_bounds__(128, SINCOS_ADAPTER_MINB) deinterleave8_kernel(const float *__restrict__ io, float *__restrict__ s,
                                                            float *__restrict__ c, size_t n) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nv = n / 8;
    for (size_t v = tid; v < nv; v += nthr) {
        float a[8], b[8], sv[8], cv[8];
        ld8_nc(a, io + 16 * v);
        ld8_nc(b, io + 16 * v + 8);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            cv[k] = a[2 * k];
            sv[k] = a[2 * k + 1];
            cv[4 + k] = b[2 * k];
            sv[4 + k] = b[2 * k + 1];
        }
        st8_nc(s + 8 * v, sv);
        st8_nc(c + 8 * v, cv);
    }
    for (size_t e = 8 * nv + tid; e < n; e += nthr) {
        c[e] = io[2 * e];
        s[e] = io[2 * e + 1];
    }
}

cudaError_t launch_interleave(bool to_inter, unsigned grid, const float *s, const float *c, float *io, size_t n,
                              cudaStream_t stream) {
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(io)) & 31) ==
        0) {
        size_t g = (n / 8 + 127) / 128;
        const size_t tail = n % 8;
        if (g < (tail + 127) / 128) g = (tail + 127) / 128;
        if (g < 1) g = 1;
        if (g > 0x7FFFFFFFu) g = 0x7FFFFFFFu;                               // grid-strides past it
        float *ss = const_cast<float *>(s), *cc = const_cast<float *>(c);
        void *args[] = {to_inter ? reinterpret_cast<void *>(&ss) : reinterpret_cast<void *>(&io),
                        to_inter ? reinterpret_cast<void *>(&cc) : reinterpret_cast<void *>(&ss),
                        to_inter ? reinterpret_cast<void *>(&io) : reinterpret_cast<void *>(&cc), &n};
        return cudaLaunchKernel(to_inter ? reinterpret_cast<const void *>(interleave8_kernel)
                                         : reinterpret_cast<const void *>(deinterleave8_kernel),
                                dim3(static_cast<unsigned>(g)), dim3(128), args, 0, stream);
    }
    if (to_inter) {
        float2 *o = reinterpret_cast<float2 *>(io);
        void *args[] = {&s, &c, &o, &n};
        return cudaLaunchKernel(reinterpret_cast<const void *>(interleave_kernel), dim3(grid), dim3(256), args, 0,
                                stream);
    }
    const float2 *i = reinterpret_cast<const float2 *>(io);
    float *ss = const_cast<float *>(s), *cc = const_cast<float *>(c);
    void *args[] = {&i, &ss, &cc, &n};
    return cudaLaunchKernel(reinterpret_cast<const void *>(deinterleave_kernel), dim3(grid), dim3(256), args, 0,
                            stream);
}

}  // namespace sincos_b200
