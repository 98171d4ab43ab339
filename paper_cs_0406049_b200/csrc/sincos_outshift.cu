// sincos_outshift.cu -- KB3c, the output-realigning form of the hot path,
// in its own translation unit: its 64 compile-time (sin, cos) offset pairs per variant build in
// parallel with the rest of the library.
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "sincos_launch.h"
#include "sincos_stream.cuh"

namespace sincos_b200 {

// KB3c: the outputs are what does not share theta's alignment (split: sin and cos at
// different offsets mod 16 B; interleaved: only 4-B aligned pairs).  The frame is theta's:
// thread v loads the aligned 256-bit theta[head + 8v ..] and computes its eight pairs; each
// output stream X sits K_X floats past a 32-B boundary at that frame and is written as
// whole aligned vectors anyway -- the block of X that thread v stores holds the last K_X values
// of thread v-1 (one warp shuffle up) and its own first values.  A warp's lane 0 has no
// predecessor in the warp and stores its own part one float at a time; the warp's last
// active lane stores the K_X values that spill into the next warp's frame the same way, so
// every element is written exactly once.  K_X is warp-uniform at run time (a switch over
// register moves).  Head [0, head) and tail one element per thread.  Same numerics.
template <int K, int W>
__device__ __forceinline__ void shift_block(const float (&prev)[W], const float (&val)[W], float (&blk)[W]) {
#pragma unroll
    for (int j = 0; j < W; ++j) blk[j] = j < K ? prev[W - K + j] : val[j - K];
}

// Store the W values `val` (W = 8 or 16) of floats [f0, f0 + W) of stream x, whose aligned
// 8-float (32-B) blocks start k floats (0..7) before f0.  All 32 lanes call it (shuffles).
// KC >= 0: k known at compile time (== KC); KC < 0: k at run time (a switch over register moves).
template <int W, int KC>
__device__ __forceinline__ void store_realigned(float *x, size_t f0, const float (&val)[W], int k_rt, unsigned lane,
                                                bool act, bool last) {
    const int k = KC >= 0 ? KC : k_rt;
    if (k == 0) {
        if (act) {
#pragma unroll
            for (int h = 0; h < W; h += 8) store8(x + f0 + h, val + h);
        }
        return;
    }
    // only the predecessor's last k <= 7 values are ever used: shuffle those (7, or K)
    constexpr int NS = KC > 0 ? KC : 7;
    float prev[W];
#pragma unroll
    for (int j = 0; j < W; ++j) prev[j] = j >= W - NS ? __shfl_up_sync(0xFFFFFFFFu, val[j], 1) : 0.0f;
    if (!act) return;
    if (lane > 0) {
        float blk[W];
        if constexpr (KC > 0) {
            shift_block<(KC > 0 ? KC : 1), W>(prev, val, blk);
        } else {
            switch (k) {
            case 1: shift_block<1, W>(prev, val, blk); break;
            case 2: shift_block<2, W>(prev, val, blk); break;
            case 3: shift_block<3, W>(prev, val, blk); break;
            case 4: shift_block<4, W>(prev, val, blk); break;
            case 5: shift_block<5, W>(prev, val, blk); break;
            case 6: shift_block<6, W>(prev, val, blk); break;
            default: shift_block<7, W>(prev, val, blk); break;
            }
        }
#pragma unroll
        for (int h = 0; h < W; h += 8) store8(x + f0 - k + h, blk + h);
    } else {
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j < W - k) x[f0 + j] = val[j];
    }
    if (last) {
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j >= W - k) x[f0 + j] = val[j];
    }
}

// KI: the interleaved stream's offset at compile time (1, 3, 5, 7: pairs only 4-B aligned), or
// for split outputs KI = 8 * KS + KC with both offsets at compile time (0..63), or -1 (both at
// run time)
template <int V, bool INTER, int KI>
__global__ void __launch_bounds__(512) sincos_outshift_kernel(const float *theta, float *so, float *co, float *io,
                                                              size_t head, size_t nvec, size_t n, int ks, int kc) {
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + nvec * 8;
    if (tid < head) emit_scalar<V, INTER>(theta, tid, so, co, io);
    if (tid < n - tail0) emit_scalar<V, INTER>(theta, tail0 + tid, so, co, io);
    const unsigned lane = threadIdx.x & 31u;
    for (size_t w0 = tid - lane; w0 < nvec; w0 += nthr) {   // warp-uniform trips
        const size_t v = w0 + lane;
        const bool act = v < nvec;
        const bool last = act && (lane == 31u || v + 1 >= nvec);
        float x[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        if (act) Mem<8, true>::load(x, theta + head + 8 * v);
        const size_t e0 = head + 8 * v;
        if constexpr (INTER) {
            float cs[16];
#pragma unroll
            for (int j = 0; j < 8; ++j) op<V>(x[j], cs[2 * j + 1], cs[2 * j]);
            store_realigned<16, KI>(io, 2 * e0, cs, ks, lane, act, last);
        } else {
            float sv[8], cv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) op<V>(x[j], sv[j], cv[j]);
            store_realigned<8, (KI >= 0 ? KI / 8 : -1)>(so, e0, sv, ks, lane, act, last);
            store_realigned<8, (KI >= 0 ? KI % 8 : -1)>(co, e0, cv, kc, lane, act, last);
        }
    }
}

template <int V, int... K>
static const void *pick_split(int k, std::integer_sequence<int, K...>) {
    const void *fn = reinterpret_cast<const void *>(sincos_outshift_kernel<V, false, -1>);
    ((k == K ? (fn = reinterpret_cast<const void *>(sincos_outshift_kernel<V, false, K>), 0) : 0), ...);
    return fn;
}

template <int V>
static const void *pick_outshift(bool inter, int ks, int kc) {
    if (!inter) {
        if constexpr (V == kNull) return reinterpret_cast<const void *>(sincos_outshift_kernel<V, false, -1>);
        else return pick_split<V>(8 * ks + kc, std::make_integer_sequence<int, 64>{});
    }
    switch (ks) {
    case 1: return reinterpret_cast<const void *>(sincos_outshift_kernel<V, true, 1>);
    case 3: return reinterpret_cast<const void *>(sincos_outshift_kernel<V, true, 3>);
    case 5: return reinterpret_cast<const void *>(sincos_outshift_kernel<V, true, 5>);
    case 7: return reinterpret_cast<const void *>(sincos_outshift_kernel<V, true, 7>);
    default: return reinterpret_cast<const void *>(sincos_outshift_kernel<V, true, -1>);
    }
}

cudaError_t launch_outshift(int variant, bool inter, int ks, int kc, unsigned grid, unsigned threads,
                            const float *theta, float *so, float *co, float *io, size_t head, size_t nvec, size_t n,
                            cudaStream_t stream) {
    const void *fn = variant == kNormalized     ? pick_outshift<kNormalized>(inter, ks, kc)
                     : variant == kRenormalized ? pick_outshift<kRenormalized>(inter, ks, kc)
                                                : pick_outshift<kNull>(inter, ks, kc);
    void *args[] = {&theta, &so, &co, &io, &head, &nvec, &n, &ks, &kc};
    return cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, 0, stream);
}

// KB3b, 256-bit form: theta K = 1..7 floats past a 32-B boundary where the outputs take
// 256-bit stores (split: sin and cos at one offset mod 32 B; interleaved: 8-B aligned pairs).
// Lane l loads a = tal[8v .. 8v+7] (aligned 256-bit); b = the next vector from lane l+1 (only
// its first K values, K shuffles), or the lane's own load when it has no right-hand neighbour
// (issued with the first: one round trip).  K is a template parameter: the selection is
// register renaming.  Head and tail one element per thread.
template <int V, bool INTER, int K>
__global__ void __launch_bounds__(512) sincos_shift8_kernel(const float *theta, float *so, float *co, float *io,
                                                            size_t head, size_t nvec, size_t n) {
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + nvec * 8;
    if (tid < head) emit_scalar<V, INTER>(theta, tid, so, co, io);
    if (tid < n - tail0) emit_scalar<V, INTER>(theta, tail0 + tid, so, co, io);
    const float *tal = theta + head - K;           // 32-B aligned (host guarantees head >= K)
    const unsigned lane = threadIdx.x & 31u;
    for (size_t w0 = tid - lane; w0 < nvec; w0 += nthr) {   // warp-uniform trips
        const size_t v = w0 + lane;
        const bool act = v < nvec;
        const bool own = act && (lane == 31u || v + 1 >= nvec);
        float a[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        float bo[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        if (act) Mem<8, true>::load(a, tal + 8 * v);
        if (own) Mem<8, true>::load(bo, tal + 8 * v + 8);
        float x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j + K < 8) {
                x[j] = a[j + K];
            } else {
                const float b = __shfl_down_sync(0xFFFFFFFFu, a[j + K - 8], 1);
                x[j] = own ? bo[j + K - 8] : b;
            }
        }
        if (act) emit<V, INTER, 8>(x, head + 8 * v, so, co, io);
    }
}

template <int V, bool INTER>
static const void *pick_shift8(int k) {
    switch (k) {
    case 1: return reinterpret_cast<const void *>(sincos_shift8_kernel<V, INTER, 1>);
    case 2: return reinterpret_cast<const void *>(sincos_shift8_kernel<V, INTER, 2>);
    case 3: return reinterpret_cast<const void *>(sincos_shift8_kernel<V, INTER, 3>);
    case 4: return reinterpret_cast<const void *>(sincos_shift8_kernel<V, INTER, 4>);
    case 5: return reinterpret_cast<const void *>(sincos_shift8_kernel<V, INTER, 5>);
    case 6: return reinterpret_cast<const void *>(sincos_shift8_kernel<V, INTER, 6>);
    default: return reinterpret_cast<const void *>(sincos_shift8_kernel<V, INTER, 7>);
    }
}

cudaError_t launch_shift8(int variant, bool inter, int k, unsigned grid, unsigned threads, const float *theta,
                          float *so, float *co, float *io, size_t head, size_t nvec, size_t n, cudaStream_t stream) {
    const void *fn;
    switch (variant) {
    case kNormalized: fn = inter ? pick_shift8<kNormalized, true>(k) : pick_shift8<kNormalized, false>(k); break;
    case kRenormalized: fn = inter ? pick_shift8<kRenormalized, true>(k) : pick_shift8<kRenormalized, false>(k); break;
    default: fn = inter ? pick_shift8<kNull, true>(k) : pick_shift8<kNull, false>(k); break;
    }
    void *args[] = {&theta, &so, &co, &io, &head, &nvec, &n};
    return cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, 0, stream);
}

}  // namespace sincos_b200
