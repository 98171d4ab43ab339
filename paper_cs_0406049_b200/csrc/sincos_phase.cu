// sincos_phase.cu -- NEXT(1): sine-cosine pairs of phases generated in the kernel.
//
// The paper's application computes phase factors of optical paths for Huygens'
// principle; its problem statement is angles "in random order, or for
// non-uniformly spaced values".  BASELINE configs[3] is such a set: the
// phases theta_ij = 2 pi f_i t_j of a non-uniform grid.  Instead of reading a
// materialised theta array (4 B/pair) the kernel forms each phase from its factors,
//   p_ij = RN(f_i * t_j)                                  (one fp32 rounding)
// and evaluates the method on it: as radians (the whole pipeline) or, with
// units = turns, from the reduction on -- which also removes the 1/2pi
// rounding of large phases.  Output: the nf x nt grid, row-major (row = f_i), split
// or interleaved {cos, sin}.  Traffic: 8 B written per pair; f and t (nf + nt floats)
// stay in L1/L2.  Write-bound: the roofline is the write bandwidth of HBM.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_launch.h"
#include "sincos_math.cuh"
#include "sincos_math2.cuh"
#include "sincos_realign.cuh"
#include "sincos_storeshift.cuh"

namespace sincos_b200 {

constexpr int kPhaseThreads = 128;

template <int V, bool TURNS>
__device__ __forceinline__ void phase_pair(float f, float t, float &s, float &c) {
    const float p = __fmul_rn(f, t);
    if constexpr (TURNS)
        sincos_pair_turns<V>(p, s, c);
    else
        sincos_pair<V>(p, s, c);
}

// Eight pairs of one row: p_k = RN(f t_k).  SINCOS_PACKED_PHASE (default): two at a time in
// packed fp32 (FMUL2/FFMA2, sincos_math2.cuh; each lane rounds as the scalar instruction) --
// identical values, half the FP32 instructions issued.  The write-only grid runs into the
// board's power cap within ~0.1 s; packed: 1.18-1.21 J per 2^30-pair launch vs 1.33-1.43 J
// and 6.57 vs 6.35-6.39 TB/s sustained, the same 7.55-7.58 TB/s burst (tools/ab_phase.py
// sustain, profiles/ab_phase_rows_r01.jsonl).
#ifndef SINCOS_PACKED_PHASE
#define SINCOS_PACKED_PHASE 1
#endif
template <int V, bool TURNS>
__device__ __forceinline__ void phase8f(const float (&fv)[8], const float (&tv)[8], float (&sv)[8], float (&cv)[8]) {
    if constexpr (SINCOS_PACKED_PHASE) {
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            F2 x = mul2(pk2(fv[k], fv[k + 1]), pk2(tv[k], tv[k + 1]));
            if constexpr (!TURNS) x = mul2(x, bc2(kInvTwoPi));
            F2 s2, c2;
            sincos_from_q2<V>(reduce_turn2(x), s2, c2);
            sv[k] = lo2(s2);
            sv[k + 1] = hi2(s2);
            cv[k] = lo2(c2);
            cv[k + 1] = hi2(c2);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) phase_pair<V, TURNS>(fv[k], tv[k], sv[k], cv[k]);
    }
}

template <int V, bool TURNS>
__device__ __forceinline__ void phase8(float fi, const float (&tv)[8], float (&sv)[8], float (&cv)[8]) {
    if constexpr (SINCOS_PACKED_PHASE) {
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            F2 x = mul2(bc2(fi), pk2(tv[k], tv[k + 1]));
            if constexpr (!TURNS) x = mul2(x, bc2(kInvTwoPi));
            F2 s2, c2;
            sincos_from_q2<V>(reduce_turn2(x), s2, c2);
            sv[k] = lo2(s2);
            sv[k + 1] = hi2(s2);
            cv[k] = lo2(c2);
            cv[k + 1] = hi2(c2);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) phase_pair<V, TURNS>(fi, tv[k], sv[k], cv[k]);
    }
}

__device__ __forceinline__ void st8_stream(float *p, const float *r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}

// Vector path: nt % 8 == 0, t and the outputs 32-B aligned.  Block (x, y) covers 128
// vectors of 8 t-values of rows y, y + gridDim.y, ...: every thread loads one 256-bit
// vector of t (L1-cached, reused by every row) and its row's f once per row.
// Interleaved output with nt % 256 == 0: a lane's two 256-bit stores go to pairs 4l..4l+3 and
// 128+4l..+3 of its warp's 256 (t loaded as two 128-bit vectors), so each warp store instruction
// writes 1 KB of whole lines instead of alternating 32-B halves of 2 KB: +1-2% burst, +3% in
// the board's power cap (6.36 -> 6.55 TB/s sustained at nt = 2^15; profiles/r02/ab_phase_inter_halves*.jsonl).
#ifndef SINCOS_PHASE_INTER_HALVES
#define SINCOS_PHASE_INTER_HALVES 1
#endif
template <int V, bool INTER, bool TURNS>
__global__ void __launch_bounds__(kPhaseThreads) phase_grid_vec(const float *__restrict__ f,
                                                               const float *__restrict__ t, size_t nf,
                                                               size_t nt, float *so, float *co, float *io) {
    const size_t nt8 = nt / 8;
    const size_t v = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= nt8) return;
#if SINCOS_PHASE_INTER_HALVES
    // interleaved, nt % 256 == 0: lane l of a warp takes pairs 4l..4l+3 and 128+4l..+3 of the
    // warp's 256, so each 256-bit store instruction covers 1 KB contiguous (whole lines)
    if constexpr (INTER) {
        if (nt % 256 == 0) {
            const unsigned lane = threadIdx.x & 31u;
            const size_t w0 = (v - lane) * 8;                         // the warp's first pair of the row
            const size_t j0 = w0 + 4 * lane, j1 = w0 + 128 + 4 * lane;
            float tt[8];
            const float4 a = __ldg(reinterpret_cast<const float4 *>(t + j0));
            const float4 b = __ldg(reinterpret_cast<const float4 *>(t + j1));
            tt[0] = a.x; tt[1] = a.y; tt[2] = a.z; tt[3] = a.w; tt[4] = b.x; tt[5] = b.y; tt[6] = b.z; tt[7] = b.w;
            for (size_t i = blockIdx.y; i < nf; i += gridDim.y) {
                const float fi = __ldg(f + i);
                float sv[8], cv[8];
                phase8<V, TURNS>(fi, tt, sv, cv);
                float cs[16];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    cs[2 * k] = cv[k];
                    cs[2 * k + 1] = sv[k];
                }
                st8_stream(io + 2 * (i * nt + j0), cs);
                st8_stream(io + 2 * (i * nt + j1), cs + 8);
            }
            return;
        }
    }
#endif
    float tt[8];
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(tt[0]), "=f"(tt[1]), "=f"(tt[2]), "=f"(tt[3]), "=f"(tt[4]), "=f"(tt[5]), "=f"(tt[6]),
                   "=f"(tt[7])
                 : "l"(t + 8 * v));
    for (size_t i = blockIdx.y; i < nf; i += gridDim.y) {
        const float fi = __ldg(f + i);
        const size_t e0 = i * nt + 8 * v;
        float sv[8], cv[8];
        phase8<V, TURNS>(fi, tt, sv, cv);
        if constexpr (INTER) {
            float cs[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                cs[2 * k] = cv[k];
                cs[2 * k + 1] = sv[k];
            }
            st8_stream(io + 2 * e0, cs);
            st8_stream(io + 2 * e0 + 8, cs + 8);
        } else {
            st8_stream(so + e0, sv);
            st8_stream(co + e0, cv);
        }
    }
}

// Any shape / alignment: one element per thread.
template <int V, bool INTER, bool TURNS>
__global__ void __launch_bounds__(kPhaseThreads) phase_grid_scalar(const float *__restrict__ f,
                                                                  const float *__restrict__ t, size_t nf,
                                                                  size_t nt, float *so, float *co, float *io) {
    const size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= nt) return;
    const float tj = t[j];
    for (size_t i = blockIdx.y; i < nf; i += gridDim.y) {
        float s, c;
        phase_pair<V, TURNS>(f[i], tj, s, c);
        const size_t e = i * nt + j;
        if constexpr (INTER) {
            io[2 * e] = c;
            io[2 * e + 1] = s;
        } else {
            so[e] = s;
            co[e] = c;
        }
    }
}

// Flat path (any nt, outputs with whole-sector stores): the nf x nt grid as one row-major
// array of n pairs; thread v owns pairs [head + 8v, head + 8v + 8) and writes them with 256-bit
// streaming stores, like the hot path.  (i, j) of its first pair come from one fp64 quotient
// estimate corrected to the exact integer divmod; the next seven advance j and wrap rows (any
// nt >= 1, rows shorter than 8 included).  f and t are read through the read-only cache.
// Pairs [0, head) and [head + 8 nvec, n) go one per thread.
__device__ __forceinline__ void divmod_nt(size_t e, size_t nt, double inv_nt, size_t &i, size_t &j) {
    size_t q = static_cast<size_t>(static_cast<double>(e) * inv_nt);
    // the estimate is within a few units of e / nt for e < 2^53: correct it exactly
    while (q * nt > e) --q;
    while ((q + 1) * nt <= e) ++q;
    i = q;
    j = e - q * nt;
}

template <int V, bool INTER, bool TURNS>
__device__ __forceinline__ void phase_one(const float *__restrict__ f, const float *__restrict__ t, size_t nt,
                                          double inv_nt, size_t e, float *so, float *co, float *io) {
    size_t i, j;
    divmod_nt(e, nt, inv_nt, i, j);
    float s, c;
    phase_pair<V, TURNS>(__ldg(f + i), __ldg(t + j), s, c);
    if constexpr (INTER) {
        io[2 * e] = c;
        io[2 * e + 1] = s;
    } else {
        so[e] = s;
        co[e] = c;
    }
}

template <int R>
__device__ __forceinline__ void select_t(const float (&w)[12], float (&tv)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) tv[k] = w[R + k];
}

// The eight pairs e0 .. e0 + 7 of the flat mapping (pair e = i nt + j), into sv / cv.
template <int V, bool TURNS>
__device__ __forceinline__ void flat_pairs8(const float *__restrict__ f, const float *__restrict__ t, size_t nt,
                                            double inv_nt, bool t_al16, size_t e0, float (&sv)[8], float (&cv)[8]) {
    size_t i, j;
    divmod_nt(e0, nt, inv_nt, i, j);
    if (j + 8 <= nt) {
        // the common case: the eight pairs lie in one row -- one f and t[j .. j+7]: with t
        // 16-B aligned, three aligned 128-bit loads from t[j - r] (r = j mod 4, uniform along
        // a row) and a register selection; else eight loads at immediate offsets
        const float fi = __ldg(f + i);
        float tv[8];
        const size_t r = j & 3;
        if (t_al16 && j - r + 12 <= nt) {
            const float4 *tq = reinterpret_cast<const float4 *>(t + (j - r));
            const float4 q0 = __ldg(tq), q1 = __ldg(tq + 1), q2 = __ldg(tq + 2);
            const float w[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
            switch (r) {
            case 0: select_t<0>(w, tv); break;
            case 1: select_t<1>(w, tv); break;
            case 2: select_t<2>(w, tv); break;
            default: select_t<3>(w, tv); break;
            }
        } else {
            const float *tp = t + j;
#pragma unroll
            for (int k = 0; k < 8; ++k) tv[k] = __ldg(tp + k);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) phase_pair<V, TURNS>(fi, tv[k], sv[k], cv[k]);
    } else if (nt >= 8) {
        // one row boundary inside the vector: rows i and i+1, branch-free per pair
        const float f0 = __ldg(f + i), f1 = __ldg(f + i + 1);   // row i+1 exists: reached
        const size_t kw = nt - j;                                // first pair of row i+1
        float tv[8], fv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const bool next = static_cast<size_t>(k) >= kw;
            tv[k] = __ldg(t + (next ? k - kw : j + k));
            fv[k] = next ? f1 : f0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) phase_pair<V, TURNS>(fv[k], tv[k], sv[k], cv[k]);
    } else {
        // rows shorter than a vector: walk the pairs
        float fi = __ldg(f + i);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            phase_pair<V, TURNS>(fi, __ldg(t + j), sv[k], cv[k]);
            if (++j == nt && k < 7) {      // next row (only when a pair of it follows)
                j = 0;
                fi = __ldg(f + ++i);
            }
        }
    }
}

template <int V, bool INTER, bool TURNS>
__global__ void __launch_bounds__(kPhaseThreads) phase_grid_flat(const float *__restrict__ f,
                                                                const float *__restrict__ t, size_t nf,
                                                                size_t nt, float *so, float *co, float *io,
                                                                size_t head, size_t nvec, size_t n,
                                                                double inv_nt) {
    const bool t_al16 = (reinterpret_cast<uintptr_t>(t) & 15) == 0;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + 8 * nvec;
    if (tid < head) phase_one<V, INTER, TURNS>(f, t, nt, inv_nt, tid, so, co, io);
    if (tid < n - tail0) phase_one<V, INTER, TURNS>(f, t, nt, inv_nt, tail0 + tid, so, co, io);
    for (size_t v = tid; v < nvec; v += nthr) {
        const size_t e0 = head + 8 * v;
        float sv[8], cv[8];
        flat_pairs8<V, TURNS>(f, t, nt, inv_nt, t_al16, e0, sv, cv);
        if constexpr (INTER) {
            float cs[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                cs[2 * k] = cv[k];
                cs[2 * k + 1] = sv[k];
            }
            st8_stream(io + 2 * e0, cs);
            st8_stream(io + 2 * e0 + 8, cs + 8);
        } else {
            st8_stream(so + e0, sv);
            st8_stream(co + e0, cv);
        }
    }
}

// Unshared output alignment (split: cos[] off sin[]'s 32-B offset; interleaved: pairs only
// 4-B aligned), any row length: the flat mapping in sin[]'s 32-B frame (interleaved: any
// frame), sin[] stored as 256-bit vectors and the re-aligned stream -- cos[], or the pairs --
// written as whole 32-B blocks built by warp shuffles (KB3c's store_realigned, kc = its float
// offset at the vector elements), warp-uniform trips.  Before it these layouts ran one pair
// per thread (0.4-3.7 TB/s).
template <int V, bool INTER, bool TURNS>
__global__ void __launch_bounds__(kPhaseThreads) phase_grid_flat_sh(const float *__restrict__ f,
                                                                   const float *__restrict__ t, size_t nf,
                                                                   size_t nt, float *so, float *co, float *io,
                                                                   size_t head, size_t nvec, size_t n,
                                                                   double inv_nt, int kc) {
    const bool t_al16 = (reinterpret_cast<uintptr_t>(t) & 15) == 0;
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + 8 * nvec;
    if (tid < head) phase_one<V, INTER, TURNS>(f, t, nt, inv_nt, tid, so, co, io);
    if (tid < n - tail0) phase_one<V, INTER, TURNS>(f, t, nt, inv_nt, tail0 + tid, so, co, io);
    const unsigned lane = threadIdx.x & 31u;
    for (size_t w0 = tid - lane; w0 < nvec; w0 += nthr) {
        const size_t v = w0 + lane;
        const bool act = v < nvec;
        const bool last = act && (lane == 31u || v + 1 >= nvec);
        const size_t e0 = head + 8 * v;
        float sv[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        float cv[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
        if (act) flat_pairs8<V, TURNS>(f, t, nt, inv_nt, t_al16, e0, sv, cv);
        if constexpr (INTER) {
            float cs[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                cs[2 * k] = cv[k];
                cs[2 * k + 1] = sv[k];
            }
            switch (kc) {
            case 1: store_realigned<16, 1>(io, 2 * e0, cs, 1, lane, act, last); break;
            case 3: store_realigned<16, 3>(io, 2 * e0, cs, 3, lane, act, last); break;
            case 5: store_realigned<16, 5>(io, 2 * e0, cs, 5, lane, act, last); break;
            default: store_realigned<16, 7>(io, 2 * e0, cs, 7, lane, act, last); break;
            }
        } else {
            if (act) st8_stream(so + e0, sv);
            switch (kc) {
            case 1: store_realigned<8, 1>(co, e0, cv, 1, lane, act, last); break;
            case 2: store_realigned<8, 2>(co, e0, cv, 2, lane, act, last); break;
            case 3: store_realigned<8, 3>(co, e0, cv, 3, lane, act, last); break;
            case 4: store_realigned<8, 4>(co, e0, cv, 4, lane, act, last); break;
            case 5: store_realigned<8, 5>(co, e0, cv, 5, lane, act, last); break;
            case 6: store_realigned<8, 6>(co, e0, cv, 6, lane, act, last); break;
            default: store_realigned<8, 7>(co, e0, cv, 7, lane, act, last); break;
            }
        }
    }
}

template <int V, bool INTER, bool TURNS>
static const void *pick_flat_sh() {
    return reinterpret_cast<const void *>(phase_grid_flat_sh<V, INTER, TURNS>);
}

cudaError_t launch_phase_flat_sh(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                                 size_t nt, float *so, float *co, float *io, size_t head, size_t nvec,
                                 unsigned grid, int kc, cudaStream_t stream) {
    const void *fn;
    if (variant == kNormalized)
        fn = inter ? (turns ? pick_flat_sh<kNormalized, true, true>() : pick_flat_sh<kNormalized, true, false>())
                   : (turns ? pick_flat_sh<kNormalized, false, true>() : pick_flat_sh<kNormalized, false, false>());
    else
        fn = inter ? (turns ? pick_flat_sh<kRenormalized, true, true>() : pick_flat_sh<kRenormalized, true, false>())
                   : (turns ? pick_flat_sh<kRenormalized, false, true>()
                            : pick_flat_sh<kRenormalized, false, false>());
    size_t n = nf * nt;
    double inv_nt = 1.0 / static_cast<double>(nt);
    void *args[] = {&f, &t, &nf, &nt, &so, &co, &io, &head, &nvec, &n, &inv_nt, &kc};
    return cudaLaunchKernel(fn, dim3(grid), dim3(kPhaseThreads), args, 0, stream);
}

// Row path (nt % 8 != 0 or t not 32-B aligned; nt >= kPhaseRowsMinNt): the vector kernel's
// structure -- a thread keeps eight t-values in registers and writes them for several rows --
// with the rows' changing alignment taken care of by the row stride.  Output row i's first
// 32-B aligned pair is j = a_i = (h0 - i nt) mod 8 (h0: the first aligned pair of the output
// array), which depends on i mod 8 only; a row slot (lx threads) takes rows q, q + S, ... with
// the slot count S a multiple of 8, so every row of a slot starts its vectors at the same
// column `head` and reads the same t windows t[head + 8v .. head + 8v + 7].  Those are loaded
// once per slot from aligned 256-bit vectors re-aligned by warp shuffles (load8_realigned_k,
// compile-time offset K = the window's float offset past a 32-B boundary, warp-uniform: one
// switch over the load only, so that the slots of different row classes share one copy of the
// row loop in the instruction cache).  Pairs before head and after the last vector (<= 14
// each) go one per lane in the slot's first warp of block column 0.  f comes 32 rows at a
// time, one per lane, broadcast by shuffles.
template <int K>
__device__ __forceinline__ void rows_window(const float *__restrict__ t, size_t head, size_t v, size_t nvec,
                                            unsigned lane, bool act, float (&tv)[8]) {
    if constexpr (K == 0) {
        if (act) ld8_keep(tv, t + head + 8 * v);
    } else {
        load8_realigned_k<K, true>(t + head - K, v, nvec, lane, act, tv);
    }
}

template <int V, bool INTER, bool TURNS>
__global__ void __launch_bounds__(kPhaseThreads) phase_grid_rows(const float *__restrict__ f,
                                                                const float *__restrict__ t, size_t nf,
                                                                size_t nt, float *so, float *co, float *io,
                                                                unsigned h0, unsigned lx) {
    // the block's 128 threads: 128 / lx row slots of lx threads (lx = 32, 64, 128: short rows
    // keep every warp busy); slot q = blockIdx.y * (128 / lx) + ty takes rows q, q + S, q + 2S
    // ... with S = gridDim.y * (128 / lx) a multiple of 8: one row class per slot
    const unsigned ty = threadIdx.x / lx, tx = threadIdx.x % lx;
    const size_t by = kPhaseThreads / lx;
    const size_t q = static_cast<size_t>(blockIdx.y) * by + ty;
    const size_t gy = static_cast<size_t>(gridDim.y) * by;
    // the slot's row class: a = first aligned column of its rows, then the realign plan of t
    // from column a (as realign_plan): head >= K keeps the aligned loads inside t
    const unsigned ri = static_cast<unsigned>((q & 7u) * (nt & 7u)) & 7u;            // i nt mod 8
    const size_t a = (h0 + 8u - ri) & 7u;
    const int K = static_cast<int>(((reinterpret_cast<uintptr_t>(t) + 4 * a) & 31) / 4);
    const size_t head = a < static_cast<size_t>(K) ? a + 8 : a;
    const size_t nvec = K > 0 ? (nt + K - head - 8) / 8 : (nt - head) / 8;   // nt >= kPhaseRowsMinNt >= 64: no underflow
    const unsigned lane = threadIdx.x & 31u;
    const size_t v = static_cast<size_t>(blockIdx.x) * lx + tx;
    const bool edge = blockIdx.x == 0 && tx < 32;                          // the row ends' warp
    if (v - lane >= nvec && !edge) return;                                 // whole warp idle
    const bool act = v < nvec;
    // rows i = q + r gy, 32 at a time: lane l loads f of the chunk's row l (issued first, with
    // the row-end t and the t windows, so the three latencies overlap), the row loop takes it
    // by a shuffle one row ahead
    size_t i0 = q;
    float fl = i0 + lane * gy < nf ? __ldg(f + i0 + lane * gy) : 0.0f;
    // row-end pair of this lane: lanes 0..15 the head columns, 16..31 the tail columns
    const size_t je = lane < 16 ? lane : head + 8 * nvec + (lane - 16);
    const bool has_e = edge && (lane < 16 ? je < head : je < nt);
    const float te = has_e ? __ldg(t + je) : 0.0f;
    float tv[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    switch (K) {
    case 0: rows_window<0>(t, head, v, nvec, lane, act, tv); break;
    case 1: rows_window<1>(t, head, v, nvec, lane, act, tv); break;
    case 2: rows_window<2>(t, head, v, nvec, lane, act, tv); break;
    case 3: rows_window<3>(t, head, v, nvec, lane, act, tv); break;
    case 4: rows_window<4>(t, head, v, nvec, lane, act, tv); break;
    case 5: rows_window<5>(t, head, v, nvec, lane, act, tv); break;
    case 6: rows_window<6>(t, head, v, nvec, lane, act, tv); break;
    default: rows_window<7>(t, head, v, nvec, lane, act, tv); break;
    }
    for (; i0 < nf; i0 += 32 * gy) {
        if (i0 != q) {
            const size_t il = i0 + lane * gy;
            fl = il < nf ? __ldg(f + il) : 0.0f;
        }
        const size_t rows = (nf - i0 + gy - 1) / gy;                       // rows of this block left
        const int nr = rows < 32 ? static_cast<int>(rows) : 32;
        float fi = __shfl_sync(0xFFFFFFFFu, fl, 0);
        for (int r = 0; r < nr; ++r) {
            const float fn = __shfl_sync(0xFFFFFFFFu, fl, (r + 1) & 31);
            const size_t r0 = (i0 + r * gy) * nt;
            if (has_e) {
                float s, c;
                phase_pair<V, TURNS>(fi, te, s, c);
                if constexpr (INTER) {
                    io[2 * (r0 + je)] = c;
                    io[2 * (r0 + je) + 1] = s;
                } else {
                    so[r0 + je] = s;
                    co[r0 + je] = c;
                }
            }
            if (act) {
                const size_t e0 = r0 + head + 8 * v;
                float sv[8], cv[8];
                phase8<V, TURNS>(fi, tv, sv, cv);
                if constexpr (INTER) {
                    float cs[16];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        cs[2 * k] = cv[k];
                        cs[2 * k + 1] = sv[k];
                    }
                    st8_stream(io + 2 * e0, cs);
                    st8_stream(io + 2 * e0 + 8, cs + 8);
                } else {
                    st8_stream(so + e0, sv);
                    st8_stream(co + e0, cv);
                }
            }
            fi = fn;
        }
    }
}

template <int V, bool INTER, bool TURNS>
static const void *pick_rows() {
    return reinterpret_cast<const void *>(phase_grid_rows<V, INTER, TURNS>);
}

cudaError_t launch_phase_rows(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, unsigned h0, int sms,
                              cudaStream_t stream) {
    static_assert(kPhaseRowsMinNt >= 64, "row path: every row class needs whole vectors");
    if (nt < kPhaseRowsMinNt || h0 > 7) return cudaErrorInvalidValue;
    const void *fn;
    if (variant == kNormalized)
        fn = inter ? (turns ? pick_rows<kNormalized, true, true>() : pick_rows<kNormalized, true, false>())
                   : (turns ? pick_rows<kNormalized, false, true>() : pick_rows<kNormalized, false, false>());
    else
        fn = inter ? (turns ? pick_rows<kRenormalized, true, true>() : pick_rows<kRenormalized, true, false>())
                   : (turns ? pick_rows<kRenormalized, false, true>() : pick_rows<kRenormalized, false, false>());
    // lx threads per row slot (a warp for rows of <= 32 vectors), 128 / lx slots per block;
    // S = row slots in all: a multiple of 8 (one row class per slot), kPhaseRowsPerBlock rows
    // per slot (the set-up -- t windows, row ends -- amortised over a few rows; 1-2 rows per
    // slot and 16-32 measured slower: tools/ab_phase.py), but >= 8 blocks per SM in all
    const size_t nv8 = nt / 8;                                            // >= nvec of every class
    const unsigned lx = nv8 <= 32 ? 32u : nv8 <= 64 ? 64u : 128u;
    const size_t by = kPhaseThreads / lx;
    const size_t gx = (nv8 + lx - 1) / lx;
    const size_t fill = (static_cast<size_t>(sms > 0 ? sms : 148) * 8 + gx - 1) / gx * by;
    size_t slots = (nf + kPhaseRowsPerBlock - 1) / kPhaseRowsPerBlock;
    if (slots < fill) slots = fill;
    slots = (slots + 7) / 8 * 8;
    const size_t rows8 = (nf + 7) / 8 * 8;
    if (slots > rows8) slots = rows8;
    if (slots > 65528 * by) slots = 65528 * by;
    const size_t gy = (slots + by - 1) / by;                               // slots is a multiple of by (<= 4)
    if (gx == 0 || gx > 0x7FFFFFFFu) return cudaErrorInvalidValue;
    void *args[] = {&f, &t, &nf, &nt, &so, &co, &io, &h0, const_cast<unsigned *>(&lx)};
    return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), dim3(kPhaseThreads),
                            args, 0, stream);
}

// Short rows (1 <= nt < kPhaseRowsMinNt = 1024): the flat kernel's mapping (8 consecutive pairs of the
// row-major grid per thread) with one code path for every vector -- a warp spans several short
// rows, and the flat kernel's separate in-row / row-boundary forms ran both in most warps (17 of
// 32 lanes active per instruction).
// t comes from shared memory: four copies ts[r][m] = t[(m + r) mod nt], so that the window
// t[(j .. j+7) mod nt] (wrapping into the next row's first t-values) is ts[j & 3][(j & ~3) ..]:
// two aligned 128-bit loads and no selection; each pair takes f_i or f_{i+1} by a select
// (SMALL, nt < 8: f_{i + (j + k) / nt}, the row offsets from a 16-entry table).
// The grid strides by a fixed number of pairs, 8 x (threads in the grid) = step_q nt + step_r
// (host-computed), so a thread advances its (row, column) by integer adds and one compare per
// vector -- only its first vector needs the fp64 quotient -- and the f values of its next
// vector are loaded before this one's arithmetic: the f fetch latency, which bound the first
// form of this kernel (per-vector fp64 divmod -> dependent f load: ncu 10.8 long-scoreboard
// stalls per issue), overlaps the method.
// 16.6 KB of shared memory per block; phase_short_blocks_per_sm(nt) blocks per SM, grid-striding.
constexpr int kShortNtMax = static_cast<int>(kPhaseRowsMinNt);
constexpr int kShortStride = kShortNtMax + 16;                              // floats per copy (16-B rows)
static_assert(4 * kShortStride * sizeof(float) + 16 <= 48 * 1024,
              "short-row kernel: four t copies must fit static shared memory (kPhaseRowsMinNt too large)");
static_assert(kShortStride % 4 == 0, "short-row kernel: copies must start 16-B aligned");

// the f values of the vector whose first pair is (i, j): f0 = f_i, f1 = f_{i+1} when the row ends
// inside the vector (nt >= 8); SMALL (nt < 8): fr[k] = f_{i + (j + k) / nt}
template <bool SMALL>
__device__ __forceinline__ void short_f(const float *__restrict__ f, size_t i, unsigned j, unsigned ntu,
                                        const unsigned char *rowoff, float (&fr)[8]) {
    if constexpr (SMALL) {
#pragma unroll
        for (int k = 0; k < 8; ++k) fr[k] = __ldg(f + i + rowoff[j + k]);
    } else {
        fr[0] = __ldg(f + i);
        fr[1] = ntu - j < 8u ? __ldg(f + i + 1) : fr[0];        // row i+1 exists when reached
    }
}

// Register cap: the interleaved rows-of->=8 instances at 32 registers (16 resident blocks; 42-48
// uncapped) ran 1-2% faster, the split ones 3-6% slower and the nt < 8 ones ~30% slower (spills)
// -- profiles/r02/ab_phase_short_minb.jsonl; so only the first are capped.
template <bool INTER, bool SMALL>
constexpr int short_min_blocks() { return INTER && !SMALL ? 16 : 1; }
template <int V, bool INTER, bool TURNS, bool SMALL>
__global__ void __launch_bounds__(kPhaseThreads, short_min_blocks<INTER, SMALL>()) phase_grid_short(const float *__restrict__ f,
                                                                 const float *__restrict__ t, size_t nf,
                                                                 size_t nt, float *so, float *co, float *io,
                                                                 size_t head, size_t nvec, size_t n,
                                                                 double inv_nt, size_t step_q, unsigned step_r) {
    __shared__ __align__(16) float ts[4][kShortStride];
    __shared__ unsigned char rowoff[16];                                  // m / nt (nt < 8)
    const unsigned ntu = static_cast<unsigned>(nt);
    if (threadIdx.x < 16) rowoff[threadIdx.x] = static_cast<unsigned char>(threadIdx.x / ntu);
    for (unsigned q = threadIdx.x; q < 4u * (ntu + 8u); q += blockDim.x) {
        const unsigned r = q / (ntu + 8u), m = q % (ntu + 8u);
        ts[r][m] = __ldg(t + (m + r) % ntu);
    }
    __syncthreads();
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + 8 * nvec;
    if (tid < head) phase_one<V, INTER, TURNS>(f, t, nt, inv_nt, tid, so, co, io);
    if (tid < n - tail0) phase_one<V, INTER, TURNS>(f, t, nt, inv_nt, tail0 + tid, so, co, io);
    size_t v = tid;
    if (v >= nvec) return;
    size_t i, j0;
    divmod_nt(head + 8 * v, nt, inv_nt, i, j0);
    unsigned j = static_cast<unsigned>(j0);
    float fr[8];
    short_f<SMALL>(f, i, j, ntu, rowoff, fr);
    for (;;) {
        const size_t e0 = head + 8 * v;
        // the next vector: (i, j) + step pairs, and its f values issued now
        const size_t vn = v + nthr;
        size_t in = i + step_q;
        unsigned jn = j + step_r;
        if (jn >= ntu) {
            jn -= ntu;
            ++in;
        }
        float gr[8];
        if (vn < nvec) short_f<SMALL>(f, in, jn, ntu, rowoff, gr);
        const unsigned r = j & 3u;
        const float4 *w = reinterpret_cast<const float4 *>(&ts[r][j - r]);
        const float4 w0 = w[0], w1 = w[1];
        const float tv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        float fv[8];
        if constexpr (SMALL) {
#pragma unroll
            for (int k = 0; k < 8; ++k) fv[k] = fr[k];
        } else {
            const unsigned kw = ntu - j;                                  // first pair of row i+1
#pragma unroll
            for (int k = 0; k < 8; ++k) fv[k] = static_cast<unsigned>(k) >= kw ? fr[1] : fr[0];
        }
        float sv[8], cv[8];
        phase8f<V, TURNS>(fv, tv, sv, cv);
        if constexpr (INTER) {
            float cs[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                cs[2 * k] = cv[k];
                cs[2 * k + 1] = sv[k];
            }
            st8_stream(io + 2 * e0, cs);
            st8_stream(io + 2 * e0 + 8, cs + 8);
        } else {
            st8_stream(so + e0, sv);
            st8_stream(co + e0, cv);
        }
        if (vn >= nvec) break;
        v = vn;
        i = in;
        j = jn;
#pragma unroll
        for (int k = 0; k < 8; ++k) fr[k] = gr[k];
    }
}

// Tiny rows (nt = NT = 1..7, a compile-time parameter; outputs 32-B aligned at pair 0): a
// thread owns a group of 8 rows -- 8 NT consecutive pairs of the row-major grid, NT whole
// 8-pair vectors -- so every pair's (row, column) inside the group is a constant: pair 8m + q
// is f[8g + (8m + q) / NT] x t[(8m + q) % NT].  One 256-bit load of the group's eight f values
// (f 32-B aligned; else eight scalar loads), the NT t values in registers once per thread, no
// selects and no division; NT vectors of 256-bit streaming stores.  f is read once, so these
// grids move 4 / NT B of f per pair besides the 8 B written.  Against the short-row kernel
// (per-pair f selects, row-offset table): nt = 1 4.59 / 4.64 TB/s written vs 4.41 / 4.13
// (split / interleaved), nt = 2, 3 split 5.47 / 5.60 vs 5.19 / 5.28; but a lane's stores are
// 8 NT pairs apart, so one warp store spans NT times more lines, and from nt = 4 on (and for
// interleaved nt = 2, 3) it is slower (profiles/r02/ab_phase_tiny.jsonl): the ABI takes it for
// nt = 1, and for nt = 2, 3 split.  Rows past the last whole group: one pair per thread.
template <int V, bool INTER, bool TURNS, int NT>
__global__ void __launch_bounds__(kPhaseThreads) phase_grid_tiny(const float *__restrict__ f,
                                                                const float *__restrict__ t, size_t nf,
                                                                float *so, float *co, float *io, size_t ngroups,
                                                                bool f_al32) {
    const size_t gid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    // rows past the last whole group (< 8 of them): one pair per thread
    const size_t rem0 = 8 * ngroups * NT, rem = nf * NT - rem0;
    if (gid < rem) {
        const size_t e = rem0 + gid;
        float sr, cr;
        phase_pair<V, TURNS>(__ldg(f + e / NT), __ldg(t + e % NT), sr, cr);
        if constexpr (INTER) {
            io[2 * e] = cr;
            io[2 * e + 1] = sr;
        } else {
            so[e] = sr;
            co[e] = cr;
        }
    }
    float tt[NT];
#pragma unroll
    for (int b = 0; b < NT; ++b) tt[b] = __ldg(t + b);
    for (size_t g = gid; g < ngroups; g += nthr) {
        float fr[8];
        if (f_al32) {
            ld8_stream(fr, f + 8 * g);
        } else {
#pragma unroll
            for (int a = 0; a < 8; ++a) fr[a] = __ldg(f + 8 * g + a);
        }
        const size_t e0 = 8 * NT * g;
#pragma unroll
        for (int m = 0; m < NT; ++m) {
            float fv[8], tv[8], sv[8], cv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                fv[q] = fr[(8 * m + q) / NT];
                tv[q] = tt[(8 * m + q) % NT];
            }
            phase8f<V, TURNS>(fv, tv, sv, cv);
            const size_t e = e0 + 8 * m;
            if constexpr (INTER) {
                float cs[16];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    cs[2 * k] = cv[k];
                    cs[2 * k + 1] = sv[k];
                }
                st8_stream(io + 2 * e, cs);
                st8_stream(io + 2 * e + 8, cs + 8);
            } else {
                st8_stream(so + e, sv);
                st8_stream(co + e, cv);
            }
        }
    }
}

template <int V, bool INTER, bool TURNS>
static const void *pick_tiny(size_t nt) {
    switch (nt) {
    case 1: return reinterpret_cast<const void *>(phase_grid_tiny<V, INTER, TURNS, 1>);
    case 2: return reinterpret_cast<const void *>(phase_grid_tiny<V, INTER, TURNS, 2>);
    case 3: return reinterpret_cast<const void *>(phase_grid_tiny<V, INTER, TURNS, 3>);
    case 4: return reinterpret_cast<const void *>(phase_grid_tiny<V, INTER, TURNS, 4>);
    case 5: return reinterpret_cast<const void *>(phase_grid_tiny<V, INTER, TURNS, 5>);
    case 6: return reinterpret_cast<const void *>(phase_grid_tiny<V, INTER, TURNS, 6>);
    default: return reinterpret_cast<const void *>(phase_grid_tiny<V, INTER, TURNS, 7>);
    }
}

cudaError_t launch_phase_tiny(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, cudaStream_t stream) {
    if (nt < 1 || nt > 7) return cudaErrorInvalidValue;
    const void *fn;
    if (variant == kNormalized)
        fn = inter ? (turns ? pick_tiny<kNormalized, true, true>(nt) : pick_tiny<kNormalized, true, false>(nt))
                   : (turns ? pick_tiny<kNormalized, false, true>(nt) : pick_tiny<kNormalized, false, false>(nt));
    else
        fn = inter ? (turns ? pick_tiny<kRenormalized, true, true>(nt) : pick_tiny<kRenormalized, true, false>(nt))
                   : (turns ? pick_tiny<kRenormalized, false, true>(nt)
                            : pick_tiny<kRenormalized, false, false>(nt));
    size_t ngroups = nf / 8;
    const size_t rem = (nf - 8 * ngroups) * nt;                       // < 56 tail pairs
    size_t work = ngroups > rem ? ngroups : rem;
    size_t grid = (work + kPhaseThreads - 1) / kPhaseThreads;
    if (grid < 1) grid = 1;
    if (grid > 0x7FFFFFFFu) grid = 0x7FFFFFFFu;                        // grid-strides past it
    bool f_al32 = (reinterpret_cast<uintptr_t>(f) & 31) == 0;
    void *args[] = {&f, &t, &nf, &so, &co, &io, &ngroups, &f_al32};
    return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(kPhaseThreads), args, 0, stream);
}

// Staged short rows (round 2): rows of NT = 4..14 pairs (split) or 2..15 pairs (interleaved),
// outputs 16-B aligned at pair 0.  The tiny-row kernel's lane stores are 8 NT pairs apart, so
// its warp store instructions scatter over NT x more lines; here a warp computes a region of
// 128 whole rows (lane l: rows 4l..4l+3, one 128-bit load of their f, every (row, column)
// a compile-time constant as in the tiny kernel), stages the region's 128 NT pairs in shared
// memory and writes it back as 128-bit stores of 512 B contiguous per warp instruction (longer
// rows: 2 rows per lane, regions of 64 rows; staged_rows below).  Lane l
// writes its chunks (16 B) S l + q (S = chunks per lane: NT split, 2 NT interleaved), the
// write-back reads chunks 32 j + l; chunk c is kept at c ^ ((c >> z) & 7), z = the number of
// trailing zero bits of S (odd S: unswizzled), which makes both conflict-free for every S here
// (a quarter-warp's eight 16-B accesses hit eight distinct bank groups; an unswizzled S = 12
// was 4-way on the writes and cost interleaved nt = 6 16%).  Rows past the last whole region:
// one pair per thread.
__host__ __device__ constexpr int ctz_c(int s) { return s % 2 ? 0 : 1 + ctz_c(s / 2); }
template <int S>
__device__ __forceinline__ int stage_chunk(int c) {
    constexpr int z = ctz_c(S);
    if constexpr (z == 0) return c;
    else return c ^ ((c >> z) & 7);
}
// Rows per lane: 4 (rows of 2-7 pairs, and split rows of 8-13), 2 for interleaved rows of 8-15
// pairs and split rows of 14 (half the staging: 128-thread blocks, registers capped at 72; with
// 4 rows per lane these ran no faster than the short-row kernel).  Against the short-row
// kernel, burst: interleaved 9-15 +1-4% (14 in variant A -1.3%, 8 equal), split 14 +5%
// (profiles/r02/ab_phase_r2_v*.jsonl).
__host__ __device__ constexpr int staged_rows(bool inter, int nt) { return nt <= 7 || (!inter && nt <= 13) ? 4 : 2; }
// A warp stages 256 R NT bytes: 128-thread blocks up to R NT = 44 (44 KB of static shared
// memory), 64 above (<= 48 KB)
__host__ __device__ constexpr int staged_threads(bool inter, int nt) {
    return staged_rows(inter, nt) * nt <= 44 ? 128 : 64;
}
// Rows of 8-13 pairs: registers capped at 72.  Without the cap they took 134-214 and ran 20-40%
// slower; at 64 some instances spill (profiles/r02/ab_phase_mid8b_v*.jsonl).  Rows of 2-7
// pairs keep ptxas's own choice (32-72): any explicit minimum blocks per SM -- even 1 -- let
// it spend more registers there, and the 7-pair rows lost up to 22%.
#ifndef SINCOS_PHASE_STAGED_REGS
#define SINCOS_PHASE_STAGED_REGS 72
#endif
__host__ __device__ constexpr int staged_min_blocks(bool inter, int nt) {
    return 65536 / (staged_threads(inter, nt) * SINCOS_PHASE_STAGED_REGS);
}
__device__ __forceinline__ void st_shared4(const float4 *p, float a, float b, float c, float d) {
    const unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" :: "r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ float4 ld_shared4(const float4 *p) {
    const unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(p));
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_global4(float *p, float4 v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
}

// K pairs (K even) of the lane's rows, pairs K0 .. K0 + K - 1 in row-major order of its R x NT
template <int V, bool TURNS, int NT, int R, int K, int K0>
__device__ __forceinline__ void staged_pairs(const float (&fr)[R], const float (&tt)[NT], float (&sv)[K],
                                             float (&cv)[K]) {
#pragma unroll
    for (int k = 0; k < K; k += 2) {
        if constexpr (SINCOS_PACKED_PHASE) {
            F2 x = mul2(pk2(fr[(K0 + k) / NT], fr[(K0 + k + 1) / NT]), pk2(tt[(K0 + k) % NT], tt[(K0 + k + 1) % NT]));
            if constexpr (!TURNS) x = mul2(x, bc2(kInvTwoPi));
            F2 s2, c2;
            sincos_from_q2<V>(reduce_turn2(x), s2, c2);
            sv[k] = lo2(s2);
            sv[k + 1] = hi2(s2);
            cv[k] = lo2(c2);
            cv[k + 1] = hi2(c2);
        } else {
            phase_pair<V, TURNS>(fr[(K0 + k) / NT], tt[(K0 + k) % NT], sv[k], cv[k]);
            phase_pair<V, TURNS>(fr[(K0 + k + 1) / NT], tt[(K0 + k + 1) % NT], sv[k + 1], cv[k + 1]);
        }
    }
}

// Chunks (16 B) per lane and stream: split R NT / 4, interleaved R NT / 2 (whole chunks: R NT is
// a multiple of 4, resp. 2, for every instance).
template <bool INTER, int NT, int R>
__host__ __device__ constexpr int staged_stride() { return INTER ? R * NT / 2 : R * NT / 4; }

// compute pairs [K0, K0 + K) and stage them: split -> chunk K0/4 .. of the lane's sin / cos runs,
// interleaved -> chunks K0/2 .. of its {cos, sin} run
template <int V, bool INTER, bool TURNS, int NT, int R, int K, int K0>
__device__ __forceinline__ void stage_batch(const float (&fr)[R], const float (&tt)[NT], float4 *ws, unsigned lane) {
    float sv[K], cv[K];
    staged_pairs<V, TURNS, NT, R, K, K0>(fr, tt, sv, cv);
    constexpr int S = staged_stride<INTER, NT, R>();
    if constexpr (INTER) {
#pragma unroll
        for (int h = 0; h < K / 2; ++h) {
            const int c = static_cast<int>(lane) * S + K0 / 2 + h;
            st_shared4(ws + stage_chunk<S>(c), cv[2 * h], sv[2 * h], cv[2 * h + 1], sv[2 * h + 1]);
        }
    } else {
#pragma unroll
        for (int h = 0; h < K / 4; ++h) {
            const int c = static_cast<int>(lane) * S + K0 / 4 + h;
            st_shared4(ws + stage_chunk<S>(c), sv[4 * h], sv[4 * h + 1], sv[4 * h + 2], sv[4 * h + 3]);
            st_shared4(ws + 32 * S + stage_chunk<S>(c), cv[4 * h], cv[4 * h + 1], cv[4 * h + 2], cv[4 * h + 3]);
        }
    }
}

// the lane's R NT pairs: batches of 8 from pair K0 on, then the rest (2, 4 or 6)
template <int V, bool INTER, bool TURNS, int NT, int R, int K0>
__device__ __forceinline__ void stage_all(const float (&fr)[R], const float (&tt)[NT], float4 *ws, unsigned lane) {
    if constexpr (R * NT - K0 >= 8) {
        stage_batch<V, INTER, TURNS, NT, R, 8, K0>(fr, tt, ws, lane);
        stage_all<V, INTER, TURNS, NT, R, K0 + 8>(fr, tt, ws, lane);
    } else if constexpr (R * NT - K0 > 0) {
        stage_batch<V, INTER, TURNS, NT, R, R * NT - K0, K0>(fr, tt, ws, lane);
    }
}

// A warp's region: 32 R whole rows = 32 R NT pairs, R rows per lane (R = 4, 2).
template <int V, bool INTER, bool TURNS, int NT, int R>
__device__ __forceinline__ void staged_body(const float *__restrict__ f, const float *__restrict__ t, size_t nf,
                                            float *so, float *co, float *io, size_t nregions, bool f_al) {
    constexpr int S = staged_stride<INTER, NT, R>();
    static_assert((INTER ? R * NT % 2 : R * NT % 4) == 0, "whole 16-B chunks per lane");
    __shared__ float4 stage[staged_threads(INTER, NT) / 32][INTER ? 32 * S : 64 * S];   // 256 R NT B per warp
    const size_t gid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t rem0 = 32 * R * NT * nregions, rem = nf * NT - rem0;   // rows past the last region
    for (size_t i = gid; i < rem; i += nthr) {
        const size_t e = rem0 + i;
        float sr, cr;
        phase_pair<V, TURNS>(__ldg(f + e / NT), __ldg(t + e % NT), sr, cr);
        if constexpr (INTER) {
            io[2 * e] = cr;
            io[2 * e + 1] = sr;
        } else {
            so[e] = sr;
            co[e] = cr;
        }
    }
    const unsigned lane = threadIdx.x & 31u;
    float4 *ws = stage[threadIdx.x >> 5];
    float tt[NT];
#pragma unroll
    for (int b = 0; b < NT; ++b) tt[b] = __ldg(t + b);
    const size_t nwarps = nthr / 32;
    for (size_t r = gid / 32; r < nregions; r += nwarps) {   // warp-uniform: one region per trip
        const size_t row0 = 32 * R * r + R * lane;
        float fr[R];
        if constexpr (R == 4) {
            if (f_al) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(f + row0));
                fr[0] = v.x;
                fr[1] = v.y;
                fr[2] = v.z;
                fr[3] = v.w;
            } else {
#pragma unroll
                for (int a = 0; a < 4; ++a) fr[a] = __ldg(f + row0 + a);
            }
        } else {
            if (f_al) {
                const float2 v = __ldg(reinterpret_cast<const float2 *>(f + row0));
                fr[0] = v.x;
                fr[1] = v.y;
            } else {
#pragma unroll
                for (int a = 0; a < R; ++a) fr[a] = __ldg(f + row0 + a);
            }
        }
        stage_all<V, INTER, TURNS, NT, R, 0>(fr, tt, ws, lane);
        __syncwarp();
        if constexpr (INTER) {
            float *dst = io + 2 * 32 * R * NT * r;
#pragma unroll
            for (int j = 0; j < S; ++j) {              // 32 S chunks = 32 R NT pairs
                const int c = 32 * j + static_cast<int>(lane);
                st_global4(dst + 4 * c, ld_shared4(ws + stage_chunk<S>(c)));
            }
        } else {
            float *ds = so + 32 * R * NT * r, *dc = co + 32 * R * NT * r;
#pragma unroll
            for (int j = 0; j < S; ++j) {              // 32 S chunks per stream
                const int c = 32 * j + static_cast<int>(lane);
                st_global4(ds + 4 * c, ld_shared4(ws + stage_chunk<S>(c)));
                st_global4(dc + 4 * c, ld_shared4(ws + 32 * S + stage_chunk<S>(c)));
            }
        }
        __syncwarp();
    }
}

// rows of 2-7 pairs: ptxas's own register choice (32-72); longer rows: capped at 72
template <int V, bool INTER, bool TURNS, int NT, int R>
__global__ void __launch_bounds__(staged_threads(INTER, NT)) phase_grid_staged(const float *__restrict__ f,
                                                                       const float *__restrict__ t, size_t nf,
                                                                       float *so, float *co, float *io,
                                                                       size_t nregions, bool f_al) {
    staged_body<V, INTER, TURNS, NT, R>(f, t, nf, so, co, io, nregions, f_al);
}
template <int V, bool INTER, bool TURNS, int NT, int R>
__global__ void __launch_bounds__(staged_threads(INTER, NT), staged_min_blocks(INTER, NT))
phase_grid_staged_wide(const float *__restrict__ f, const float *__restrict__ t, size_t nf, float *so, float *co,
                       float *io, size_t nregions, bool f_al) {
    staged_body<V, INTER, TURNS, NT, R>(f, t, nf, so, co, io, nregions, f_al);
}

template <int V, bool INTER, bool TURNS>
static const void *pick_staged(size_t nt) {
#define STG(N) reinterpret_cast<const void *>(phase_grid_staged<V, INTER, TURNS, N, 4>)
#define WIDE(N) reinterpret_cast<const void *>(phase_grid_staged_wide<V, INTER, TURNS, N, staged_rows(INTER, N)>)
    switch (nt) {
    case 2: return STG(2);
    case 3: return STG(3);
    case 4: return STG(4);
    case 5: return STG(5);
    case 6: return STG(6);
    default: break;
    }
    if constexpr (!INTER) {                // split rows of 8-13 pairs (R = 4)
        if constexpr (SINCOS_PHASE_STAGED_MAX_NT >= 8) {
            switch (nt) {
            case 8: return WIDE(8);
            case 9: return WIDE(9);
            case 10: return WIDE(10);
            case 11: return WIDE(11);
            case 12: return WIDE(12);
            case 13: return WIDE(13);
            default: break;
            }
        }
        if constexpr (SINCOS_PHASE_STAGED_MAX_NT >= 14) {
            if (nt == 14) return WIDE(14);
        }
    } else if constexpr (SINCOS_PHASE_STAGED_MAX_NT_INTER >= 8) {   // interleaved rows of 8-15 (R = 2)
        switch (nt) {
        case 8: return WIDE(8);
        case 9: return WIDE(9);
        case 10: return WIDE(10);
        case 11: return WIDE(11);
        case 12: return WIDE(12);
        case 13: return WIDE(13);
        case 14: return WIDE(14);
        case 15: return WIDE(15);
        default: break;
        }
    }
    return STG(7);
#undef STG
#undef WIDE
}

cudaError_t launch_phase_staged(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                                size_t nt, float *so, float *co, float *io, size_t max_grid, cudaStream_t stream) {
    if (!phase_staged_ok(inter, nt)) return cudaErrorInvalidValue;
    const void *fn;
    if (variant == kNormalized)
        fn = inter ? (turns ? pick_staged<kNormalized, true, true>(nt) : pick_staged<kNormalized, true, false>(nt))
                   : (turns ? pick_staged<kNormalized, false, true>(nt) : pick_staged<kNormalized, false, false>(nt));
    else
        fn = inter ? (turns ? pick_staged<kRenormalized, true, true>(nt) : pick_staged<kRenormalized, true, false>(nt))
                   : (turns ? pick_staged<kRenormalized, false, true>(nt)
                            : pick_staged<kRenormalized, false, false>(nt));
    const int R = staged_rows(inter, static_cast<int>(nt));
    size_t nregions = nf / (32 * R);
    const size_t rem = (nf - 32 * R * nregions) * nt;                 // < 32 R rows of tail pairs
    const unsigned threads = staged_threads(inter, static_cast<int>(nt));
    const size_t warps_per_block = threads / 32;
    size_t grid = (nregions + warps_per_block - 1) / warps_per_block;
    const size_t grid_rem = (rem + threads - 1) / threads;
    if (grid < grid_rem) grid = grid_rem;
    if (max_grid > 0 && grid > max_grid) grid = max_grid;               // (A/B: grid-stride)
    if (grid < 1) grid = 1;
    if (grid > 0x7FFFFFFFu / 4) grid = 0x7FFFFFFFu / 4;                // grid-strides past it
    bool f_al = (reinterpret_cast<uintptr_t>(f) & (4 * R - 1)) == 0;
    void *args[] = {&f, &t, &nf, &so, &co, &io, &nregions, &f_al};
    return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(threads), args, 0, stream);
}

template <int V, bool INTER, bool TURNS>
static const void *pick_short(bool small) {
    return small ? reinterpret_cast<const void *>(phase_grid_short<V, INTER, TURNS, true>)
                 : reinterpret_cast<const void *>(phase_grid_short<V, INTER, TURNS, false>);
}

#ifdef SINCOS_AB
template <int V, bool INTER, bool TURNS>
static const void *pick_flat() {
    return reinterpret_cast<const void *>(phase_grid_flat<V, INTER, TURNS>);
}
#endif

cudaError_t launch_phase_flat(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, size_t head, size_t nvec,
                              unsigned grid, bool short_rows, cudaStream_t stream) {
    const void *fn;
    const bool small = nt < 8;
    if (short_rows && nt >= 1 && nt < kPhaseRowsMinNt) {                  // phase_grid_short
        if (variant == kNormalized)
            fn = inter ? (turns ? pick_short<kNormalized, true, true>(small) : pick_short<kNormalized, true, false>(small))
                       : (turns ? pick_short<kNormalized, false, true>(small)
                                : pick_short<kNormalized, false, false>(small));
        else
            fn = inter ? (turns ? pick_short<kRenormalized, true, true>(small)
                                : pick_short<kRenormalized, true, false>(small))
                       : (turns ? pick_short<kRenormalized, false, true>(small)
                                : pick_short<kRenormalized, false, false>(small));
        size_t n = nf * nt;
        double inv_nt = 1.0 / static_cast<double>(nt);
        const size_t step = 8 * static_cast<size_t>(grid) * kPhaseThreads;   // pairs per grid stride
        size_t step_q = step / nt;
        unsigned step_r = static_cast<unsigned>(step % nt);
        void *args[] = {&f, &t, &nf, &nt, &so, &co, &io, &head, &nvec, &n, &inv_nt, &step_q, &step_r};
        return cudaLaunchKernel(fn, dim3(grid), dim3(kPhaseThreads), args, 0, stream);
    } else {
#ifdef SINCOS_AB
        if (variant == kNormalized)
            fn = inter ? (turns ? pick_flat<kNormalized, true, true>() : pick_flat<kNormalized, true, false>())
                       : (turns ? pick_flat<kNormalized, false, true>() : pick_flat<kNormalized, false, false>());
        else
            fn = inter ? (turns ? pick_flat<kRenormalized, true, true>() : pick_flat<kRenormalized, true, false>())
                       : (turns ? pick_flat<kRenormalized, false, true>()
                                : pick_flat<kRenormalized, false, false>());
#else
        return cudaErrorInvalidValue;        // the flat kernel is an A/B-build form
#endif
    }
    size_t n = nf * nt;
    double inv_nt = 1.0 / static_cast<double>(nt);
    void *args[] = {&f, &t, &nf, &nt, &so, &co, &io, &head, &nvec, &n, &inv_nt};
    return cudaLaunchKernel(fn, dim3(grid), dim3(kPhaseThreads), args, 0, stream);
}

template <int V, bool INTER, bool TURNS>
static const void *pick_phase(bool vec) {
    return vec ? reinterpret_cast<const void *>(phase_grid_vec<V, INTER, TURNS>)
               : reinterpret_cast<const void *>(phase_grid_scalar<V, INTER, TURNS>);
}

template <int V>
static const void *pick_phase_v(bool inter, bool turns, bool vec) {
    if (inter) return turns ? pick_phase<V, true, true>(vec) : pick_phase<V, true, false>(vec);
    return turns ? pick_phase<V, false, true>(vec) : pick_phase<V, false, false>(vec);
}

cudaError_t launch_phase_grid(int variant, bool inter, bool turns, bool vec, const float *f, size_t nf,
                              const float *t, size_t nt, float *so, float *co, float *io, cudaStream_t stream) {
    const void *fn = variant == kNormalized ? pick_phase_v<kNormalized>(inter, turns, vec)
                                            : pick_phase_v<kRenormalized>(inter, turns, vec);
    const size_t cols = vec ? nt / 8 : nt;
    const size_t gx = (cols + kPhaseThreads - 1) / kPhaseThreads;
    const size_t gy = nf < 65535 ? nf : 65535;
    if (gx == 0 || gx > 0x7FFFFFFFu) return cudaErrorInvalidValue;
    void *args[] = {&f, &t, &nf, &nt, &so, &co, &io};
    return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), dim3(kPhaseThreads),
                            args, 0, stream);
}

}  // namespace sincos_b200
