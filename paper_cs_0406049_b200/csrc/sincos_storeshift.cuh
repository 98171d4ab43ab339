// sincos_storeshift.cuh -- the output re-alignment of KB3c: a stream whose
// 32-B blocks do not line up with the thread's eight values is written as whole aligned blocks
// built from the neighbouring lane's values (warp shuffles), the warp's edge blocks as aligned
// pieces.  Used by the KB3c / hybrid kernels (sincos_outshift.cu) and the general-method kernel
// (sincos_method.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_stream.cuh"

namespace sincos_b200 {

template <int K, int W>
__device__ __forceinline__ void shift_block(const float (&prev)[W], const float (&val)[W], float (&blk)[W]) {
#pragma unroll
    for (int j = 0; j < W; ++j) blk[j] = j < K ? prev[W - K + j] : val[j - K];
}

__device__ __forceinline__ void st_piece(float *p, const float *r, int m) {
    if (m == 4)
        asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                     :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]) : "memory");
    else if (m == 2)
        asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1,%2};"
                     :: "l"(p), "f"(r[0]), "f"(r[1]) : "memory");
    else
        asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" :: "l"(p), "f"(r[0]) : "memory");
}

// Floats [A, B) of the 32-B block at `blk` from r[0 .. B - A), as naturally aligned pieces
// (largest first at each position): at most three stores.
template <int A, int B>
__device__ __forceinline__ void store_range(float *blk, const float *r) {
    if constexpr (A < B) {
        constexpr int al = (A & 1) ? 1 : (A & 2) ? 2 : (A & 4) ? 4 : 8;   // alignment of position A
        constexpr int m = al < (B - A) ? al : ((B - A) >= 4 ? 4 : (B - A) >= 2 ? 2 : 1);
        constexpr int mm = m > 4 ? 4 : m;
        st_piece(blk + A, r, mm);
        store_range<A + mm, B>(blk, r + mm);
    }
}

// Store the W values `val` (W = 8 or 16) of floats [f0, f0 + W) of stream x, whose aligned
// 8-float (32-B) blocks start k floats (0..7) before f0.  All 32 lanes call it (shuffles).
// KC >= 0: k known at compile time (== KC); KC < 0: k at run time.
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
    if constexpr (KC > 4) {
        // k > 4: the blocks the thread stores start 8 - k floats into its own values and end with
        // the successor's first 8 - k (shuffled down: 8 - k < 4 shuffles instead of k)
        constexpr int D = 8 - KC;
        float next[W];
#pragma unroll
        for (int j = 0; j < W; ++j) next[j] = j < D ? __shfl_down_sync(0xFFFFFFFFu, val[j], 1) : 0.0f;
        if (!act) return;
        if (lane == 0) store_range<KC, 8>(x + f0 - KC, val);          // its head: floats [k, 8) of a block
        if constexpr (W == 16) store8(x + f0 + D, val + D);              // its own whole block
        if (last) {
            store_range<0, KC>(x + f0 + W - KC, val + W - KC);         // no successor: a partial block
        } else {
            float blk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) blk[j] = j < KC ? val[W - KC + j] : next[j - KC];
            store8(x + f0 + W - KC, blk);
        }
        return;
    }
    // k <= 4 (or at run time): only the predecessor's last k values are used: shuffle those
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
        // lane 0: floats [k, 8) of its first block, then (W = 16) its one whole block
        if constexpr (KC > 0) {
            store_range<KC, 8>(x + f0 - KC, val);
            if constexpr (W == 16) store8(x + f0 + 8 - KC, val + 8 - KC);
        } else {
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (j < W - k) x[f0 + j] = val[j];
        }
    }
    if (last) {
        // floats [0, k) of the block after the thread's last one
        if constexpr (KC > 0) {
            store_range<0, KC>(x + f0 + W - KC, val + W - KC);
        } else {
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (j >= W - k) x[f0 + j] = val[j];
        }
    }
}

}  // namespace sincos_b200
