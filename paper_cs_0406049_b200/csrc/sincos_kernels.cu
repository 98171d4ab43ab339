// sincos_kernels.cu -- sm_100a kernels of the hot path and their launchers.
//
// KB1/KB2  sincos_vec_kernel<V, INTER, W, U, NC>
//          grid-stride streaming kernel; each thread moves W floats of theta per
//          access (W = 8: one 256-bit LDG; W = 4: one 128-bit LDG), U accesses in
//          flight per loop trip (the GPU form of "computes two vectors at a
//          time"), and writes 8 B of output per element with 256-bit
//          (or 128-bit) streaming stores: split sin[]/cos[] (INTER = false) or
//          interleaved {cos, sin} pairs (INTER = true).  Loads bypass L1 and
//          are L2 evict-first; stores too -- no element is touched twice.
//          The scalar head (to reach alignment) and tail (n mod W) are done by
//          the first threads of the grid with the same math.
// KB3      sincos_scalar_kernel<V, INTER>: any 4-B alignment, one element per
//          thread, identical numerics (A/B build only: the product re-aligns instead).
// KB4      V = kNull: the traffic ceiling (same access pattern, no math).
// KB5      sincos_stats_kernel: fp64 error statistics (verification only).
//
// HBM-bound by design: 12 algorithmic bytes per pair (4 in, 8 out) against
// ~30 issued instructions per pair, i.e. ~2.5 instr/B while a B200 issues
// ~5.7 lane-instr per HBM byte.  No shared memory, no
// tensor cores (not a contraction).
#include <cuda_runtime.h>
#include <stdint.h>

#include "sincos_launch.h"
#include "sincos_stream.cuh"

namespace sincos_b200 {

// KB1/KB2.  Elements [0, head) and [head + nvec*W, n) scalar; the body is nvec
// vectors of W elements starting at element `head` (aligned by the host).
// Programmatic dependent launch (sm_90+): let the next kernel on the stream be scheduled as soon
// as every block of this one has started, and wait -- before touching global memory -- until
// the previous kernel has completed and its writes are visible.  Stream order is unchanged
// (nothing is read or written before the wait); only launch latency and block scheduling of
// back-to-back launches overlap.  Without the launch attribute both are no-ops.
// Only the 256-bit (W = 8) instances carry it: in the 128-bit instances, with twice the blocks,
// the per-block PREEXIT / ACQBULK cost 15% even on plain launches (measured); launch_vec uses
// the PDL attribute only for W = 8 (a kernel launched with it must wait before any access).
template <int W>
__device__ __forceinline__ void pdl_enter() {
    if constexpr (W == 8) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
}

template <int V, bool INTER, int W, int U, bool NC, bool PF>
__global__ void __launch_bounds__(512) sincos_vec_kernel(const float *theta, float *so, float *co, float *io,
                                                         size_t head, size_t nvec, size_t n) {
    pdl_enter<W>();
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + nvec * W;
    if (tid < head) emit_scalar<V, INTER>(theta, tid, so, co, io);
    if (tid < n - tail0) emit_scalar<V, INTER>(theta, tail0 + tid, so, co, io);

    const float *tb = theta + head;
    size_t v = tid;
    if constexpr (PF) {
        // Software pipeline: the U loads of trip k+1 are issued before trip k computes and
        // stores, so every warp keeps loads in flight while it does arithmetic.
        const size_t step = U * nthr;
        bool have = v + (U - 1) * nthr < nvec;
        float x[U][W];
        if (have) {
#pragma unroll
            for (int u = 0; u < U; ++u) Mem<W, NC>::load(x[u], tb + (v + u * nthr) * W);
        }
        while (have) {
            const size_t nv = v + step;
            const bool more = nv + (U - 1) * nthr < nvec;
            float y[U][W];
            if (more) {
#pragma unroll
                for (int u = 0; u < U; ++u) Mem<W, NC>::load(y[u], tb + (nv + u * nthr) * W);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) emit<V, INTER, W>(x[u], head + (v + u * nthr) * W, so, co, io);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < W; ++k) x[u][k] = y[u][k];
            v = nv;
            have = more;
        }
    } else if constexpr (U > 1) {
        for (; v + (U - 1) * nthr < nvec; v += U * nthr) {
            float x[U][W];
#pragma unroll
            for (int u = 0; u < U; ++u) Mem<W, NC>::load(x[u], tb + (v + u * nthr) * W);
#pragma unroll
            for (int u = 0; u < U; ++u) emit<V, INTER, W>(x[u], head + (v + u * nthr) * W, so, co, io);
        }
    }
    for (; v < nvec; v += nthr) {
        float x[W];
        Mem<W, NC>::load(x, tb + v * W);
        emit<V, INTER, W>(x, head + v * W, so, co, io);
    }
}

// KB3b: theta and the outputs do not share an alignment.  The outputs keep whole-sector
// stores -- split: 128-bit stores to sin[] and cos[] (a warp instruction covers whole 32-B
// sectors); interleaved: ONE 256-bit store of the four {cos, sin} pairs (two 128-bit stores
// would each write half of every sector) -- and theta, K = 0..3 floats past a 16-B boundary
// there, is read as ALIGNED float4 vectors and re-aligned in registers: lane l holds a =
// theta_al[4v .. 4v+3] and takes the next vector b from lane l+1 with warp shuffles (the
// warp's last lane, or a lane whose neighbour is past the end, loads b itself), then its four
// angles are a[K..3] ++ b[0..K-1] -- a static register selection, K being a template
// parameter (K = 0: no shuffle).  Every loop trip is warp-uniform (all lanes shuffle).
// Elements [0, head) and [head + 4 nvec, n) are done one per thread; the host sizes nvec so
// that every b load stays inside theta.  Same numerics as every other path.
template <int V, bool INTER, int K>
__global__ void __launch_bounds__(512) sincos_shift_kernel(const float *theta, float *so, float *co, float *io,
                                                           size_t head, size_t nvec, size_t n) {
    const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tail0 = head + nvec * 4;
    if (tid < head) emit_scalar<V, INTER>(theta, tid, so, co, io);
    if (tid < n - tail0) emit_scalar<V, INTER>(theta, tail0 + tid, so, co, io);

    const float *tal = theta + head - K;           // 16-B aligned (host guarantees head >= K)
    const unsigned lane = threadIdx.x & 31u;
    for (size_t w0 = tid - lane; w0 < nvec; w0 += nthr) {   // warp-uniform trips
        const size_t v = w0 + lane;
        const bool act = v < nvec;
        float a[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        float x[4];
        if constexpr (K == 0) {
            if (act) Mem<4, true>::load(a, tal + 4 * v);
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = a[j];
        } else {
            // the lanes without a neighbour issue their own second load together with the first,
            // so the warp waits for one memory round trip, not two
            const bool own = act && (lane == 31u || v + 1 >= nvec);
            float bo[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            if (act) Mem<4, true>::load(a, tal + 4 * v);
            if (own) Mem<4, true>::load(bo, tal + 4 * v + 4);
            float b[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = __shfl_down_sync(0xFFFFFFFFu, a[j], 1);
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = own ? bo[j] : b[j];
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = j + K < 4 ? a[j + K] : b[j + K - 4];
        }
        if (!act) continue;
        const size_t e0 = head + 4 * v;
        if constexpr (INTER) {
            float cs[8];
#pragma unroll
            for (int j = 0; j < 4; ++j) op<V>(x[j], cs[2 * j + 1], cs[2 * j]);
            store8(io + 2 * e0, cs);
        } else {
            emit<V, false, 4>(x, e0, so, co, io);
        }
    }
}

// KB3: any alignment.
template <int V, bool INTER>
__global__ void __launch_bounds__(512) sincos_scalar_kernel(const float *theta, float *so, float *co, float *io,
                                                            size_t n) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += nthr)
        emit_scalar<V, INTER>(theta, e, so, co, io);
}

__global__ void __launch_bounds__(512) rcp_kernel(const float *d, float *out, size_t n) {
    const size_t nthr = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += nthr)
        out[e] = rcp_rn(d[e]);
}

// ---- dispatch -----------------------------------------------------------------
using VecFn = void (*)(const float *, float *, float *, float *, size_t, size_t, size_t);
using ScalarFn = void (*)(const float *, float *, float *, float *, size_t);

// The product instantiates U = 1 without software prefetch only (measured best, DESIGN.md
// section 5); the A/B build adds U = 2, 4 and the prefetching forms.
template <int V, bool INTER, int W, bool NC, bool PF>
static VecFn pick_u(int unroll) {
#ifdef SINCOS_AB
    switch (unroll) {
    case 1: return sincos_vec_kernel<V, INTER, W, 1, NC, PF>;
    case 2: return sincos_vec_kernel<V, INTER, W, 2, NC, PF>;
    default: return sincos_vec_kernel<V, INTER, W, 4, NC, PF>;
    }
#else
    (void)unroll;
    return sincos_vec_kernel<V, INTER, W, 1, NC, false>;
#endif
}

template <int V, bool INTER, int W, bool NC>
static VecFn pick_pf(int unroll, bool pf) {
#ifdef SINCOS_AB
    return pf ? pick_u<V, INTER, W, NC, true>(unroll) : pick_u<V, INTER, W, NC, false>(unroll);
#else
    (void)pf;
    return pick_u<V, INTER, W, NC, false>(unroll);
#endif
}

template <int V, bool INTER>
static VecFn pick_vec(int w, int unroll, bool nc, bool pf) {
    if (w == 8) return nc ? pick_pf<V, INTER, 8, true>(unroll, pf) : pick_pf<V, INTER, 8, false>(unroll, pf);
    return nc ? pick_pf<V, INTER, 4, true>(unroll, pf) : pick_pf<V, INTER, 4, false>(unroll, pf);
}

template <int V>
static VecFn pick_inter(bool inter, int w, int unroll, bool nc, bool pf) {
    return inter ? pick_vec<V, true>(w, unroll, nc, pf) : pick_vec<V, false>(w, unroll, nc, pf);
}

VecFn vec_kernel(int variant, bool inter, int w, int unroll, bool nc, bool pf) {
    switch (variant) {
    case kNormalized: return pick_inter<kNormalized>(inter, w, unroll, nc, pf);
    case kRenormalized: return pick_inter<kRenormalized>(inter, w, unroll, nc, pf);
    default: return pick_inter<kNull>(inter, w, unroll, nc, pf);
    }
}

#ifdef SINCOS_AB
ScalarFn scalar_kernel(int variant, bool inter) {
    switch (variant) {
    case kNormalized: return inter ? sincos_scalar_kernel<kNormalized, true> : sincos_scalar_kernel<kNormalized, false>;
    case kRenormalized: return inter ? sincos_scalar_kernel<kRenormalized, true> : sincos_scalar_kernel<kRenormalized, false>;
    default: return inter ? sincos_scalar_kernel<kNull, true> : sincos_scalar_kernel<kNull, false>;
    }
}

#endif  // SINCOS_AB

cudaError_t launch_vec(int variant, bool inter, int w, int unroll, bool nc, bool pf, bool pdl, unsigned grid,
                       unsigned threads, const float *theta, float *so, float *co, float *io, size_t head,
                       size_t nvec, size_t n, cudaStream_t stream) {
    VecFn fn = vec_kernel(variant, inter, w, unroll, nc, pf);
    void *args[] = {&theta, &so, &co, &io, &head, &nvec, &n};
    // inside a CUDA graph capture the plain launch is kept: graph replay already removes the
    // launch latency, and the programmatic edges measured slower for small graphed kernels
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (!pdl || w != 8 || cudaStreamIsCapturing(stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return cudaLaunchKernel(reinterpret_cast<const void *>(fn), dim3(grid), dim3(threads), args, 0, stream);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(fn), args);
}

#ifdef SINCOS_AB
cudaError_t launch_scalar(int variant, bool inter, unsigned grid, unsigned threads, const float *theta, float *so,
                          float *co, float *io, size_t n, cudaStream_t stream) {
    ScalarFn fn = scalar_kernel(variant, inter);
    void *args[] = {&theta, &so, &co, &io, &n};
    return cudaLaunchKernel(reinterpret_cast<const void *>(fn), dim3(grid), dim3(threads), args, 0, stream);
}
#endif

#ifdef SINCOS_AB   // the 128-bit theta re-alignment: A/B build only (the product routes those layouts to KB3c)
template <int V, bool INTER>
static VecFn pick_shift(int k) {
    switch (k) {
    case 0: return sincos_shift_kernel<V, INTER, 0>;
    case 1: return sincos_shift_kernel<V, INTER, 1>;
    case 2: return sincos_shift_kernel<V, INTER, 2>;
    default: return sincos_shift_kernel<V, INTER, 3>;
    }
}

cudaError_t launch_shift(int variant, bool inter, int k, unsigned grid, unsigned threads, const float *theta,
                         float *so, float *co, float *io, size_t head, size_t nvec, size_t n, cudaStream_t stream) {
    VecFn fn;
    switch (variant) {
    case kNormalized: fn = inter ? pick_shift<kNormalized, true>(k) : pick_shift<kNormalized, false>(k); break;
    case kRenormalized: fn = inter ? pick_shift<kRenormalized, true>(k) : pick_shift<kRenormalized, false>(k); break;
    default: fn = inter ? pick_shift<kNull, true>(k) : pick_shift<kNull, false>(k); break;
    }
    void *args[] = {&theta, &so, &co, &io, &head, &nvec, &n};
    return cudaLaunchKernel(reinterpret_cast<const void *>(fn), dim3(grid), dim3(threads), args, 0, stream);
}
#endif

cudaError_t launch_rcp(unsigned grid, unsigned threads, const float *d, float *out, size_t n, cudaStream_t stream) {
    void *args[] = {&d, &out, &n};
    return cudaLaunchKernel(reinterpret_cast<const void *>(rcp_kernel), dim3(grid), dim3(threads), args, 0, stream);
}

// Context kernels (kCmpSincosf / kCmpIntrinsic): the default launch shape only (256-bit, U = 1).
cudaError_t launch_compare(int which, bool inter, unsigned grid, unsigned threads, const float *theta, float *so,
                           float *co, float *io, size_t nvec, size_t n, cudaStream_t stream) {
    VecFn fn;
    if (which == kCmpSincosf)
        fn = inter ? sincos_vec_kernel<kCmpSincosf, true, 8, 1, true, false>
                   : sincos_vec_kernel<kCmpSincosf, false, 8, 1, true, false>;
    else
        fn = inter ? sincos_vec_kernel<kCmpIntrinsic, true, 8, 1, true, false>
                   : sincos_vec_kernel<kCmpIntrinsic, false, 8, 1, true, false>;
    size_t head = 0;
    void *args[] = {&theta, &so, &co, &io, &head, &nvec, &n};
    return cudaLaunchKernel(reinterpret_cast<const void *>(fn), dim3(grid), dim3(threads), args, 0, stream);
}

}  // namespace sincos_b200
