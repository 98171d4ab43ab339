// sincos_nudft.cu -- NEXT(2): the consumer of the pairs, fused.
//
// "The author has been applying this method to the rapid computation of optical
// diffraction patterns via Huygens' principle": a sum of many unit
// phasors of non-uniformly spaced phases weighted by complex amplitudes,
//     F_k = sum_j a_j (cos p_kj + i sin p_kj),     p_kj = RN(f_k * t_j),
// i.e. a direct non-uniform Fourier sum.  The pairs are evaluated by the paper's
// method in registers and consumed at once -- none reaches HBM -- so the kernel is
// bound by the FP32 pipe, not by memory: per term 1 FMUL (the phase) + the method
// (~23 FP32-pipe ops + FRND, N) + 4 FFMA (complex multiply-accumulate).
//
// Layout: block (x, y) owns kKPerBlock frequencies (kKPerThread per thread, strided by
// the block size so the partial stores coalesce) and segment y of consecutive terms j
// (nudft_segment: about 8192 blocks in all, a fixed count, so the arithmetic does not
// depend on the device).  The segment's (t_j, a_j) are staged through shared memory in
// tiles and read by all threads as broadcasts.  Each thread sums its kKPerThread complex
// sums in fp32 over runs of nudft_chunk(nt) consecutive terms (sequential FMAs), adds each
// run into fp64 accumulators, writes the segment's fp64 partial to the workspace, and a
// second kernel adds the segments' partials in fp64 in order (deterministic) and rounds to
// complex64.  The error bound needs only the fp32 run length, whatever the segment length.
#include <cuda_runtime.h>
#include <stdint.h>


#include "sincos_launch.h"
#include "sincos_math2.cuh"
#include "sincos_method.cuh"

namespace sincos_b200 {

constexpr int kNuThreads = 128;
#ifndef SINCOS_NUDFT_KPT
#define SINCOS_NUDFT_KPT 4
#endif
constexpr int kKPerThread = SINCOS_NUDFT_KPT;
// Terms per trip of the inner loop.  Unrolled by 8 the loop's own instructions (index, compare,
// branch, shared-memory address) leave the issue stream and the compiler may interleave
// consecutive terms' chains; outputs bit-identical, 56 registers, no spill.  Gain: +3-7% over
// the rolled loop in the libraries A/B (C4 shape, packed; tools/ab_nudft.py,
// profiles/r02/ab_nudft_unroll*.json; 4 and 16 within 1% of 8), but only 0-1% in the bench
// line against earlier bench lines (bench_r02/c2_final12.json vs c2_final11.json) and -1.8% /
// +0.2% in kernel time under ncu (radians / turns) -- the rolled loop read lower in the A/B
// tool's context than in the bench's.  Kept: never slower.
#ifndef SINCOS_NUDFT_UNROLL
#define SINCOS_NUDFT_UNROLL 8
#endif
constexpr int kNuUnroll = SINCOS_NUDFT_UNROLL;
constexpr int kKPerBlock = kNuThreads * kKPerThread;
constexpr int kTileJ = 256;

// Comparison "variants" for the bench only (not the paper's method): CUDA's libm
// sincosf (accurate, with a slow path for large arguments) and the __sincosf intrinsic.
constexpr int kLibmSincosf = 3;
constexpr int kIntrinsicSincosf = 4;
// NEXT(3) general methods: V = kMethodBase + (NT == 8 ? 4 : 0) + FIX, FIX in {0, 1, 3}.
constexpr int kMethodBase = 16;
// Specialised general-method shapes: V = kMethodExactBase + 4 * spec + FIX.
constexpr int kMethodExactBase = 32;

template <int V, bool TURNS>
__device__ __forceinline__ void term_pair(const MethodParams &mp, float f, float t, float &s, float &c) {
    const float p = __fmul_rn(f, t);
    if constexpr (V >= kMethodExactBase) {
        // specialised shapes: spec 0 = (n_ss 4, n_cc 3, 2 doublings), spec 1 = (3, 2, 1)
        constexpr int SPEC = (V - kMethodExactBase) / 4;
        constexpr int FIX = (V - kMethodExactBase) % 4;
        constexpr int NS = SPEC == 0 ? 4 : 3, NC = SPEC == 0 ? 3 : 2, ND = SPEC == 0 ? 2 : 1;
        const float x = TURNS ? p : __fmul_rn(p, kInvTwoPi);
        method_from_q_exact<NS, NC, ND, FIX>(mp, reduce_turn(x), s, c);
    } else if constexpr (V >= kMethodBase) {
        constexpr int NT = (V - kMethodBase) >= 4 ? 8 : 4;
        constexpr int FIX = (V - kMethodBase) % 4;
        if constexpr (TURNS) method_from_q<NT, FIX>(mp, reduce_turn(p), s, c);
        else method_pair<NT, FIX>(mp, p, s, c);
    } else if constexpr (V == kLibmSincosf) {
        if constexpr (TURNS) sincospif(2.0f * p, &s, &c); else sincosf(p, &s, &c);
    } else if constexpr (V == kIntrinsicSincosf) {
        __sincosf(TURNS ? 6.28318530717958647692f * p : p, &s, &c);
    } else if constexpr (TURNS) {
        sincos_pair_turns<V>(p, s, c);
    } else {
        sincos_pair<V>(p, s, c);
    }
}

// Two frequencies of one term at once (packed fp32, sincos_math2.cuh): the same
// operations as term_pair for lanes m and m+1, bit-identical, half the FP32 issue slots.
template <int V>
constexpr bool kPackable = V == kNormalized || V == kRenormalized || V >= kMethodBase;

template <int V, bool TURNS>
__device__ __forceinline__ void term_pair2(const MethodParams &mp, F2 f, float t, F2 &s, F2 &c) {
    const F2 p = mul2(f, bc2(t));
    const F2 x = TURNS ? p : mul2(p, bc2(kInvTwoPi));
    if constexpr (V >= kMethodExactBase) {
        constexpr int SPEC = (V - kMethodExactBase) / 4;
        constexpr int FIX = (V - kMethodExactBase) % 4;
        constexpr int NS = SPEC == 0 ? 4 : 3, NC = SPEC == 0 ? 3 : 2, ND = SPEC == 0 ? 2 : 1;
        method_from_q_exact2<NS, NC, ND, FIX>(mp, reduce_turn2(x), s, c);
    } else {
        sincos_from_q2<V>(reduce_turn2(x), s, c);
    }
}

template <int V, bool TURNS, bool PACK>
__global__ void __launch_bounds__(kNuThreads, 9) nudft_partial(const float *__restrict__ f, size_t nf,
                                                            const float *__restrict__ t,
                                                            const float2 *__restrict__ a, size_t nt,
                                                            size_t seg, size_t chunk, double2 *__restrict__ part,
                                                            const MethodParams mp) {
    __shared__ float4 sj[kTileJ];    // {t_j, re a_j, im a_j, 0}: one 128-bit broadcast load per term
    // the thread's fp64 accumulators live in shared memory (touched once per chunk), keeping
    // the registers -- and so the occupancy -- of the fp32 inner loop
    __shared__ double2 acc[kKPerThread][kNuThreads];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // let nudft_reduce be scheduled
    const size_t k0 = static_cast<size_t>(blockIdx.x) * kKPerBlock + threadIdx.x;
    const size_t j0 = static_cast<size_t>(blockIdx.y) * seg;
    const size_t j1 = j0 + seg < nt ? j0 + seg : nt;
    float fk[kKPerThread], re[kKPerThread], im[kKPerThread];
#pragma unroll
    for (int m = 0; m < kKPerThread; ++m) {
        const size_t k = k0 + m * kNuThreads;
        fk[m] = k < nf ? f[k] : 0.0f;
        re[m] = 0.0f;
        im[m] = 0.0f;
        acc[m][threadIdx.x] = make_double2(0.0, 0.0);
    }
    const unsigned tiles_per_chunk = static_cast<unsigned>(chunk / kTileJ);
    unsigned tiles = 0;
    for (size_t jt = j0; jt < j1; jt += kTileJ) {
        // every `chunk` terms (a multiple of the tile) the fp32 sums move into fp64
        if (tiles++ == tiles_per_chunk) {
            tiles = 1;
#pragma unroll
            for (int m = 0; m < kKPerThread; ++m) {
                double2 d = acc[m][threadIdx.x];
                d.x += re[m];
                d.y += im[m];
                acc[m][threadIdx.x] = d;
                re[m] = 0.0f;
                im[m] = 0.0f;
            }
        }
        const int len = static_cast<int>(j1 - jt < kTileJ ? j1 - jt : kTileJ);
        __syncthreads();
        for (int q = threadIdx.x; q < len; q += kNuThreads) {
            const float2 aq = a[jt + q];
            sj[q] = make_float4(t[jt + q], aq.x, aq.y, 0.0f);
        }
        __syncthreads();
#pragma unroll kNuUnroll
        for (int q = 0; q < len; ++q) {
            const float4 v = sj[q];
            const float tj = v.x;
            const float2 aj = make_float2(v.y, v.z);
            if constexpr (PACK && V >= kMethodBase && V < kMethodExactBase) {
                // general methods, packed: all the thread's frequencies stage by stage
                constexpr int NT = (V - kMethodBase) >= 4 ? 8 : 4;
                constexpr int FIX = (V - kMethodBase) % 4;
                constexpr int N2 = kKPerThread / 2;
                F2 q[N2], sv[N2], cv[N2];
#pragma unroll
                for (int m = 0; m < N2; ++m) {
                    const F2 p = mul2(pk2(fk[2 * m], fk[2 * m + 1]), bc2(tj));
                    q[m] = reduce_turn2(TURNS ? p : mul2(p, bc2(kInvTwoPi)));
                }
                method_from_q_n2<NT, FIX, N2>(mp, q, sv, cv);
                const F2 ar = bc2(aj.x), ai = bc2(aj.y);
#pragma unroll
                for (int m = 0; m < N2; ++m) {
                    F2 r = pk2(re[2 * m], re[2 * m + 1]), i = pk2(im[2 * m], im[2 * m + 1]);
                    r = fma2(ar, cv[m], r);
                    r = nfma2(ai, sv[m], r);
                    i = fma2(ar, sv[m], i);
                    i = fma2(ai, cv[m], i);
                    re[2 * m] = lo2(r);
                    re[2 * m + 1] = hi2(r);
                    im[2 * m] = lo2(i);
                    im[2 * m + 1] = hi2(i);
                }
            } else if constexpr (PACK) {
                const F2 ar = bc2(aj.x), ai = bc2(aj.y);
#pragma unroll
                for (int m = 0; m < kKPerThread; m += 2) {
                    F2 s, c;
                    term_pair2<V, TURNS>(mp, pk2(fk[m], fk[m + 1]), tj, s, c);
                    // the scalar loop's four FMAs, lanes m and m+1
                    F2 r = pk2(re[m], re[m + 1]), i = pk2(im[m], im[m + 1]);
                    r = fma2(ar, c, r);
                    r = nfma2(ai, s, r);
                    i = fma2(ar, s, i);
                    i = fma2(ai, c, i);
                    re[m] = lo2(r);
                    re[m + 1] = hi2(r);
                    im[m] = lo2(i);
                    im[m + 1] = hi2(i);
                }
            } else if constexpr (V >= kMethodBase && V < kMethodExactBase) {
                // general methods: all the thread's frequencies stage by stage (method_from_q_n)
                constexpr int NT = (V - kMethodBase) >= 4 ? 8 : 4;
                constexpr int FIX = (V - kMethodBase) % 4;
                float q[kKPerThread], sv[kKPerThread], cv[kKPerThread];
#pragma unroll
                for (int m = 0; m < kKPerThread; ++m) {
                    const float p = __fmul_rn(fk[m], tj);
                    q[m] = reduce_turn(TURNS ? p : __fmul_rn(p, kInvTwoPi));
                }
                method_from_q_n<NT, FIX, kKPerThread>(mp, q, sv, cv);
#pragma unroll
                for (int m = 0; m < kKPerThread; ++m) {
                    re[m] = __fmaf_rn(aj.x, cv[m], re[m]);
                    re[m] = __fmaf_rn(-aj.y, sv[m], re[m]);
                    im[m] = __fmaf_rn(aj.x, sv[m], im[m]);
                    im[m] = __fmaf_rn(aj.y, cv[m], im[m]);
                }
            } else {
#pragma unroll
                for (int m = 0; m < kKPerThread; ++m) {
                    float s, c;
                    term_pair<V, TURNS>(mp, fk[m], tj, s, c);
                    // (ar + i ai)(c + i s) accumulated with single-rounding FMAs
                    re[m] = __fmaf_rn(aj.x, c, re[m]);
                    re[m] = __fmaf_rn(-aj.y, s, re[m]);
                    im[m] = __fmaf_rn(aj.x, s, im[m]);
                    im[m] = __fmaf_rn(aj.y, c, im[m]);
                }
            }
        }
    }
#pragma unroll
    for (int m = 0; m < kKPerThread; ++m) {
        const size_t k = k0 + m * kNuThreads;
        const double2 d = acc[m][threadIdx.x];
        if (k < nf) part[static_cast<size_t>(blockIdx.y) * nf + k] = make_double2(d.x + re[m], d.y + im[m]);
    }
}

__global__ void __launch_bounds__(256) nudft_reduce(const double2 *__restrict__ part, size_t nf, size_t nseg,
                                                    float2 *__restrict__ out) {
    // launched as a programmatic dependent of nudft_partial: scheduled while the partial sums
    // drain, it waits here for their completion (and visibility) before reading them
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nf) return;
    double re = 0.0, im = 0.0;
    for (size_t c = 0; c < nseg; ++c) {
        const double2 p = part[c * nf + k];
        re += p.x;
        im += p.y;
    }
    out[k] = make_float2(__double2float_rn(re), __double2float_rn(im));
}

// The fp32 summation length: terms summed in fp32, in order, before they move into fp64 (the
// error bound's "chunk").  256 for short sums, else 1024.
size_t nudft_chunk(size_t nt) { return nt < 4096 ? static_cast<size_t>(kTileJ) : 1024; }

// Terms per block row (grid.y = segments): a multiple of the chunk, short enough that the grid
// has about kNudftTargetBlocks blocks (a fixed count, so the arithmetic is the same on every
// device), and at most 65535 segments.
constexpr size_t kNudftTargetBlocks = 8192;
size_t nudft_segment(size_t nf, size_t nt) {
    const size_t chunk = nudft_chunk(nt);
    size_t gx = (nf + kKPerBlock - 1) / kKPerBlock;
    if (gx < 1) gx = 1;                                                // nf == 0: any (unused) value
    size_t want = (kNudftTargetBlocks + gx - 1) / gx;                 // segments wanted
    if (want < 1) want = 1;
    size_t seg = (nt + want - 1) / want;
    const size_t min_seg = (nt + 65534) / 65535;
    if (seg < min_seg) seg = min_seg;
    seg = (seg + chunk - 1) / chunk * chunk;
    return seg > 0 ? seg : chunk;
}

size_t nudft_ws_bytes(size_t nf, size_t nt) {
    const size_t seg = nudft_segment(nf, nt);
    const size_t nseg = (nt + seg - 1) / seg;
    return nseg * nf * sizeof(double2);
}

// Packed fp32 for the paper's tables and the specialised method shapes; their scalar twins
// (bit-identical) exist in the A/B build only, for the comparison.  Kernels that are not
// packable (comparison functions, general method shapes) have only the scalar form.
#ifdef SINCOS_AB
constexpr bool kScalarTwins = true;
#else
constexpr bool kScalarTwins = false;
#endif

template <int V>
static const void *pick_nudft(bool turns, bool packed) {
    if constexpr (kPackable<V> && kKPerThread % 2 == 0) {
        if constexpr (kScalarTwins) {
            if (!packed)
                return turns ? reinterpret_cast<const void *>(nudft_partial<V, true, false>)
                             : reinterpret_cast<const void *>(nudft_partial<V, false, false>);
        }
        return turns ? reinterpret_cast<const void *>(nudft_partial<V, true, true>)
                     : reinterpret_cast<const void *>(nudft_partial<V, false, true>);
    } else {
        (void)packed;
        return turns ? reinterpret_cast<const void *>(nudft_partial<V, true, false>)
                     : reinterpret_cast<const void *>(nudft_partial<V, false, false>);
    }
}

cudaError_t launch_nudft(int variant, bool turns, const float *f, size_t nf, const float *t, const float *a,
                         size_t nt, float *out, void *ws, cudaStream_t stream, const MethodParams *method,
                         int method_nt, int method_fix, int method_spec, bool packed) {
    size_t chunk = nudft_chunk(nt);
    size_t seg = nudft_segment(nf, nt);
    const size_t nchunks = (nt + seg - 1) / seg;                       // segments (grid.y)
    const size_t gx = (nf + kKPerBlock - 1) / kKPerBlock;
    if (gx > 0x7FFFFFFFu || nchunks > 65535) return cudaErrorInvalidValue;
    const void *fn;
    switch (variant) {
    case kNormalized: fn = pick_nudft<kNormalized>(turns, packed); break;
    case kRenormalized: fn = pick_nudft<kRenormalized>(turns, packed); break;
    case kLibmSincosf: fn = pick_nudft<kLibmSincosf>(turns, packed); break;
    case kIntrinsicSincosf: fn = pick_nudft<kIntrinsicSincosf>(turns, packed); break;
    default:
        if (method == nullptr) return cudaErrorInvalidValue;
        if (method_spec >= 0 && method_fix != 3)
            fn = method_spec == 0 ? (method_fix == 0 ? pick_nudft<kMethodExactBase + 0>(turns, packed)
                                                     : pick_nudft<kMethodExactBase + 1>(turns, packed))
                                  : (method_fix == 0 ? pick_nudft<kMethodExactBase + 4>(turns, packed)
                                                     : pick_nudft<kMethodExactBase + 5>(turns, packed));
        else if (method_nt <= 4)
            fn = method_fix == 0 ? pick_nudft<kMethodBase + 0>(turns, packed)
                 : method_fix == 1 ? pick_nudft<kMethodBase + 1>(turns, packed) : pick_nudft<kMethodBase + 3>(turns, packed);
        else
            fn = method_fix == 0 ? pick_nudft<kMethodBase + 4>(turns, packed)
                 : method_fix == 1 ? pick_nudft<kMethodBase + 5>(turns, packed) : pick_nudft<kMethodBase + 7>(turns, packed);
        break;
    }
    MethodParams mp = method ? *method : MethodParams{};
    const float2 *a2 = reinterpret_cast<const float2 *>(a);
    double2 *part = static_cast<double2 *>(ws);
    void *args[] = {&f, &nf, &t, &a2, &nt, &seg, &chunk, &part, &mp};
    cudaError_t e = cudaLaunchKernel(fn, dim3(static_cast<unsigned>(gx), static_cast<unsigned>(nchunks)),
                                     dim3(kNuThreads), args, 0, stream);
    if (e != cudaSuccess) return e;
    float2 *o = reinterpret_cast<float2 *>(out);
    size_t nch = nchunks;
    void *rargs[] = {&part, &nf, &nch, &o};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((nf + 255) / 256));
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(nudft_reduce), rargs);
}

}  // namespace sincos_b200
