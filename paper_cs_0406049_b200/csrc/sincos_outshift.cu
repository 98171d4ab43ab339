// sincos_outshift.cu -- KB3c, the output-realigning form of the hot path,
// in its own translation unit: its 64 compile-time (sin, cos) offset pairs per variant build in
// parallel with the rest of the library.
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "sincos_launch.h"
#include "sincos_realign.cuh"
#include "sincos_storeshift.cuh"
#include "sincos_stream.cuh"

namespace sincos_b200 {

// KB3c: the outputs are what does not share theta's alignment (split: sin and cos at
// different offsets mod 16 B; interleaved: only 4-B aligned pairs).  The frame is theta's:
// thread v loads the aligned 256-bit theta[head + 8v ..] and computes its eight pairs; each
// output stream X sits k_X floats past a 32-B boundary at that frame and is written as
// whole aligned 32-B blocks anyway -- the block of X that thread v stores holds the last k_X
// values of thread v-1 (warp shuffles up) and its own first values; for k_X > 4, mirrored, its
// own last values and the first 8 - k_X of thread v+1 (shuffles down: never more than four
// shuffles per stream; with seven, k = 7 ran 10% slower than k = 1).  A warp's lane 0 has no
// predecessor in the warp: it stores the part of its first block that is its own (floats
// [k, 8) of that block) and the warp's last active lane the k values that spill into the next
// warp's frame (floats [0, k) of the next block) -- each as at most three naturally aligned
// pieces (16 / 8 / 4 B) when k is a compile-time constant (the first form stored these one
// float at a time: 8 scalar stores per stream and warp, 16 for interleaved pairs; ncu: issue
// slots 65-69% busy against the aligned kernel's 48%).  Every element is written exactly once.
// (A form that let the previous warp store the whole edge block through shared memory needed
// a CTA barrier per trip and ran 15-20% slower: the barrier couples the warps' HBM latencies.)
// k_X is a template parameter (KC >= 0) for the cases that occur, else warp-uniform at run time
// (a switch over register moves, single-float edge stores).  Head [0, head) and tail one
// element per thread.  Same numerics as every other path.  (The store helpers:
// sincos_storeshift.cuh.)
//
// KI: the interleaved stream's offset at compile time (1, 3, 5, 7: pairs only 4-B aligned), or
// for split outputs KI = 8 * KS + KC with both offsets at compile time (0..63), or -1 (both at
// run time)
// Register budget.  Uncapped, most instances take 34-48 registers: 10-12 resident 128-thread
// blocks per SM.  Capped at 32 (16 blocks, full occupancy, a few bytes of spill) they run
// faster where the kernel waits on HBM (sin+2 cos+5: 6.46 -> 6.67 TB/s; tools/ab_layouts.py,
// profiles/r02) -- as long as the spill stays small, which the store order below arranges.
//
// Which stream to store first (split).  Both streams' eight values are live until the first
// one is stored, so the first stream's re-alignment sets the register peak; at 32 registers
// ptxas spills (bytes; sm_100a, nvcc 12.9, both variants) when the stream at offset a goes
// first while offset b's values wait: a = 0, 1, 7: 0; a = 2, 5: 4; a = 3: 8 (12 if b = 0);
// a = 4: 16-24; a = 6: 4 (12 if b is odd).  Storing the cheaper one first keeps every split
// instance at <= 8 bytes, so all of them are capped.  Sin first throughout (the first round-2
// form) spilled up to 24 bytes at sin offset 4, where those instances ran uncapped at 40-48
// registers: 5.70-6.54 TB/s, now 6.45-6.79 (all 64 pairs timed both orders, both variants:
// profiles/r02/ab_layouts_order*.jsonl, ab_layouts_flip*.jsonl, ab_all_new_v*.jsonl).
//
// Interleaved pairs at k = 3, 5, 7 floats: two trips per thread (half the blocks), the next
// trip's theta vector loaded before this trip's pairs are computed and stored, at 40 registers
// (12 resident blocks) -- 6.54-6.81 TB/s against 5.80-6.54 with one trip per thread (variant A
// lost most, at 48-56 registers uncapped); k = 1 fits 32 registers and runs at 6.88-6.91
// without it (prefetching there cost 1-2%).  profiles/r02/ab_inter_pf_v*.jsonl.
#ifndef SINCOS_OUTSHIFT_PF
#define SINCOS_OUTSHIFT_PF 1                 // 0: one trip per thread everywhere (A/B)
#endif
template <bool INTER, int KI>
__host__ __device__ constexpr bool outshift_pf() {
    return SINCOS_OUTSHIFT_PF && INTER && (KI == 3 || KI == 5 || KI == 7);
}
#ifndef SINCOS_OUTSHIFT_ORDER
#define SINCOS_OUTSHIFT_ORDER 1          // 0: sin first, 2: the other order (A/B builds only)
#endif
__host__ __device__ constexpr int spill_first(int a, int b) {
    return a == 4 ? 16 : a == 3 ? (b == 0 ? 12 : 8) : a == 6 ? (b % 2 ? 12 : 4) : (a == 2 || a == 5) ? 4 : 0;
}
template <int KI>
__host__ __device__ constexpr bool cos_first() {
    if constexpr (KI < 0 || SINCOS_OUTSHIFT_ORDER == 0) return false;
    else if constexpr (SINCOS_OUTSHIFT_ORDER == 2) return !(spill_first(KI % 8, KI / 8) < spill_first(KI / 8, KI % 8));
    else return spill_first(KI % 8, KI / 8) < spill_first(KI / 8, KI % 8);
}
template <bool INTER, int KI>
constexpr int outshift_min_blocks() {
    if constexpr (INTER) {
        return outshift_pf<INTER, KI>() ? 12 : KI >= 0 && KI <= 4 ? 16 : 1;
    } else {
        if constexpr (SINCOS_OUTSHIFT_ORDER == 0) {
            constexpr int ks = KI / 8, kc = KI % 8;
            return KI < 0 || ks == 4 || (ks == 6 && kc % 2 == 1) || (ks == 3 && kc == 0) ? 1 : 16;
        } else {
            return KI < 0 ? 1 : 16;
        }
    }
}
template <bool INTER, int KI>
constexpr int outshift_max_threads() { return outshift_min_blocks<INTER, KI>() > 1 ? 128 : 512; }

template <int V, bool INTER, int KI>
__global__ void __launch_bounds__(outshift_max_threads<INTER, KI>(), outshift_min_blocks<INTER, KI>())
sincos_outshift_kernel(const float *theta, float *so, float *co, float *io,
                                                              size_t head, size_t nvec, size_t n, int ks, int kc) {
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + nvec * 8;
    if (tid < head) emit_scalar<V, INTER>(theta, tid, so, co, io);
    if (tid < n - tail0) emit_scalar<V, INTER>(theta, tail0 + tid, so, co, io);
    const unsigned lane = threadIdx.x & 31u;
    constexpr bool PF = outshift_pf<INTER, KI>();
    float xn[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    if (PF && tid < nvec) Mem<8, true>::load(xn, theta + head + 8 * tid);
    for (size_t w0 = tid - lane; w0 < nvec; w0 += nthr) {   // warp-uniform trips
        const size_t v = w0 + lane;
        const bool act = v < nvec;
        const bool last = act && (lane == 31u || v + 1 >= nvec);
        float x[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        if constexpr (PF) {
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = xn[j];
            if (v + nthr < nvec) Mem<8, true>::load(xn, theta + head + 8 * (v + nthr));
        } else {
            if (act) Mem<8, true>::load(x, theta + head + 8 * v);
        }
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
            if constexpr (cos_first<KI>()) {
                store_realigned<8, (KI >= 0 ? KI % 8 : -1)>(co, e0, cv, kc, lane, act, last);
                store_realigned<8, (KI >= 0 ? KI / 8 : -1)>(so, e0, sv, ks, lane, act, last);
            } else {
                store_realigned<8, (KI >= 0 ? KI / 8 : -1)>(so, e0, sv, ks, lane, act, last);
                store_realigned<8, (KI >= 0 ? KI % 8 : -1)>(co, e0, cv, kc, lane, act, last);
            }
        }
    }
}

// Split layouts with BOTH streams off theta's frame (ks, kc != 0, ks != kc).  Re-aligning one
// output stream costs ~1% (sin+0 cos+k: 6.79-6.81 TB/s against 6.86 aligned) and re-aligning
// theta onto the outputs' frame about as little (KB3b: 6.80-6.89), while re-aligning both
// output streams cost 3-9% (6.2-6.7; profiles/r02/ab_all_rot_v*.jsonl).  So most of these
// layouts take the frame of one output stream ("direct": plain 256-bit stores), theta re-aligned
// onto it from the next lane as in KB3b (KT = 8 - k_direct floats, sincos_realign.cuh) and only
// the other stream re-aligned by store_realigned (KX = k_other - k_direct mod 8).  The vectors
// start at hb + KT (scalar head below that); the last lane's second theta vector must lie
// inside theta, so one vector fewer than KB3c's, the tail one element per thread.
// Measured over all 42 such layouts, both variants, three boxes (tools/ab_layouts.py,
// profiles/r02/ab_hyb*.jsonl; per-layout results reproduced to ~0.3%): the direct stream is the
// one further past its 32-B boundary (the other choice lost 2-5% nearly everywhere); the
// hybrid gains 0.5-3.8% in 28 layouts and loses 0.4-2.8% where the offsets are {1,2}, {1,3},
// {1,4}, {1,6}, {2,3}, {2,4} or {4,7}, which keep both streams re-aligned on theta's frame.
// (Fewer theta shuffles for KT > 4 -- each lane loading the second vector and taking the
// first 8 - KT values from its predecessor -- changed nothing: the shuffle count is not what
// costs here.)
#ifndef SINCOS_OUTSHIFT_HYB
#define SINCOS_OUTSHIFT_HYB 1        // 0: every such layout on theta's frame (A/B)
#endif
__host__ __device__ constexpr bool hyb_pair(int a, int b) {   // unordered offsets {a, b}, a < b
    return !((a == 1 && (b == 2 || b == 3 || b == 4 || b == 6)) || (a == 2 && (b == 3 || b == 4)) ||
             (a == 4 && b == 7));
}
template <int KI>
__host__ __device__ constexpr bool hyb_applies() {
    constexpr int ks = KI / 8, kc = KI % 8;
    return SINCOS_OUTSHIFT_HYB != 0 && KI >= 0 && ks != 0 && kc != 0 && ks != kc &&
           hyb_pair(ks < kc ? ks : kc, ks < kc ? kc : ks);
}
// the direct stream: the one further past its 32-B boundary
template <int KI>
__host__ __device__ constexpr bool hyb_sin_direct() { return KI / 8 > KI % 8; }

template <int V, int KI>
__global__ void __launch_bounds__(128, 16)
sincos_outshift_hyb_kernel(const float *theta, float *so, float *co, float *io, size_t hb, size_t nvec, size_t n,
                           int, int) {
    (void)io;
    constexpr bool SD = hyb_sin_direct<KI>();
    constexpr int kd = SD ? KI / 8 : KI % 8, kx = SD ? KI % 8 : KI / 8;
    constexpr int KT = 8 - kd;              // theta's float offset at the direct stream's frame (1..7)
    constexpr int KX = (kx - kd + 8) % 8;   // the other stream's offset there (1..7)
    const size_t head = hb + KT < n ? hb + KT : n;
    const size_t nv = nvec > 0 ? nvec - 1 : 0;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + nv * 8;
    if (tid < head) emit_scalar<V, false>(theta, tid, so, co, nullptr);
    if (tid < n - tail0) emit_scalar<V, false>(theta, tail0 + tid, so, co, nullptr);
    const float *tal = theta + hb;          // 32-B aligned: theta + head - KT
    float *dst = SD ? so : co;
    float *oth = SD ? co : so;
    const unsigned lane = threadIdx.x & 31u;
    for (size_t w0 = tid - lane; w0 < nv; w0 += nthr) {   // warp-uniform trips
        const size_t v = w0 + lane;
        const bool act = v < nv;
        const bool last = act && (lane == 31u || v + 1 >= nv);
        float x[8];
        load8_realigned_k<KT>(tal, v, nv, lane, act, x);
        float d[8], o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (SD) op<V>(x[j], d[j], o[j]);
            else op<V>(x[j], o[j], d[j]);
        }
        if (act) store8(dst + head + 8 * v, d);
        store_realigned<8, KX>(oth, head + 8 * v, o, KX, lane, act, last);
    }
}

template <int V, int K>
static const void *split_fn() {
    if constexpr (hyb_applies<K>()) return reinterpret_cast<const void *>(sincos_outshift_hyb_kernel<V, K>);
    else return reinterpret_cast<const void *>(sincos_outshift_kernel<V, false, K>);
}

template <int V, int... K>
static const void *pick_split(int k, std::integer_sequence<int, K...>) {
    const void *fn = reinterpret_cast<const void *>(sincos_outshift_kernel<V, false, -1>);
    ((k == K ? (fn = split_fn<V, K>(), 0) : 0), ...);
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
    if (SINCOS_OUTSHIFT_PF && inter && (ks == 3 || ks == 5 || ks == 7)) grid = (grid + 1) / 2;   // two trips each
    if (threads > 128) {            // (A/B block sizes) the register-capped instances take 128 at most
        grid = static_cast<unsigned>((static_cast<size_t>(grid) * threads + 127) / 128);
        threads = 128;
    }
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
