// sincos_launch.h -- internal launch interface between the C ABI and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/sincos_pairs.h"

namespace sincos_b200 {

// variant: 0 = N, 1 = A, 2 = null (traffic ceiling); w = 4 or 8 floats per access;
// unroll = 1, 2 or 4; nc = read-only (non-coherent) loads, false when theta aliases an output.
// pf = software-pipelined loads (trip k+1 in flight while trip k computes).
cudaError_t launch_vec(int variant, bool inter, int w, int unroll, bool nc, bool pf, unsigned grid,
                       unsigned threads, const float *theta, float *so, float *co, float *io, size_t head,
                       size_t nvec, size_t n, cudaStream_t stream);
// Context kernels for the bench (3 = CUDA sincosf, 4 = __sincosf), 32-B aligned buffers, head 0.
cudaError_t launch_compare(int which, bool inter, unsigned grid, unsigned threads, const float *theta, float *so,
                           float *co, float *io, size_t nvec, size_t n, cudaStream_t stream);
// KB3b: outputs 16-B aligned from element `head`, theta K = k floats past a 16-B boundary there.
cudaError_t launch_shift(int variant, bool inter, int k, unsigned grid, unsigned threads, const float *theta,
                         float *so, float *co, float *io, size_t head, size_t nvec, size_t n, cudaStream_t stream);
// KB3b, 256-bit form (sincos_outshift.cu): outputs 32-B aligned from `head`, theta k = 1..7 floats
// past a 32-B boundary there.
cudaError_t launch_shift8(int variant, bool inter, int k, unsigned grid, unsigned threads, const float *theta,
                          float *so, float *co, float *io, size_t head, size_t nvec, size_t n, cudaStream_t stream);
// KB3c: theta 32-B aligned from element `head`; outputs re-aligned (ks / kc: sin / cos float
// offsets past a 32-B boundary there; interleaved: ks = the pairs' float offset past 32 B).
cudaError_t launch_outshift(int variant, bool inter, int ks, int kc, unsigned grid, unsigned threads,
                            const float *theta, float *so, float *co, float *io, size_t head, size_t nvec, size_t n,
                            cudaStream_t stream);
// Many arrays in one launch (sincos_batched.cu): one record per item in device memory.
struct BatchItem {
    const float *theta;
    float *so, *co, *io;
    uint64_t n, head;      // head: elements before the 32-B aligned vector body (vec == 1)
    uint32_t vec, pad;     // 1: 256-bit body from `head`; 0: one element per thread
};
constexpr int kBatchMax = 480;   // items per launch: the table fits the 32 KB parameter block
// The table travels in the kernel's parameter block; the launch copies the whole struct, so it
// comes in three capacities (the smallest that holds the batch is launched).
template <int CAP>
struct BatchParamsT {
    int count;
    int pad;
    uint64_t prefix[CAP + 1];   // cumulative 1024-element chunks (blocks)
    BatchItem items[CAP];
};
using BatchParams = BatchParamsT<kBatchMax>;
static_assert(sizeof(BatchParams) <= 32764, "kernel parameter block limit");
uint64_t batched_chunks(uint64_t n, uint64_t head, bool vec);
cudaError_t launch_batched(int variant, const BatchParams &p, cudaStream_t stream);
// Programmatic dependent launch of the vector kernel: 1 = on (default), 0 = plain launches.
int set_pdl(int on);
cudaError_t launch_scalar(int variant, bool inter, unsigned grid, unsigned threads, const float *theta, float *so,
                          float *co, float *io, size_t n, cudaStream_t stream);
cudaError_t launch_rcp(unsigned grid, unsigned threads, const float *d, float *out, size_t n, cudaStream_t stream);
// Persistent TMA bulk-load pipeline over the whole 2048-element tiles of [theta, theta+n);
// *done = elements covered (the caller finishes the rest).
cudaError_t launch_tma(int variant, bool inter, unsigned grid, const float *theta, float *so, float *co, float *io,
                       size_t n, size_t *done, cudaStream_t stream);
// NEXT(1) phase grid (sincos_phase.cu); vec = 256-bit path (nt % 8 == 0, 32-B aligned t/outputs).
cudaError_t launch_phase_grid(int variant, bool inter, bool turns, bool vec, const float *f, size_t nf,
                              const float *t, size_t nt, float *so, float *co, float *io, cudaStream_t stream);
// NEXT(1) flat path for any nt: pairs [head, head + 8 nvec) as 256-bit stores (outputs 32-B
// aligned at `head`), the rest one per thread; grid-stride over `grid` blocks.  short_rows:
// for nt < kPhaseRowsMinNt the one-path kernel with t in shared memory.
cudaError_t launch_phase_flat(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, size_t head, size_t nvec,
                              unsigned grid, bool short_rows, cudaStream_t stream);
// NEXT(1) row path for nt % 8 != 0 or unaligned t (nt >= kPhaseRowsMinNt): h0 = the first
// pair at which the outputs are 32-B aligned (0..7); t any 4-B alignment.
#ifndef SINCOS_PHASE_ROWS_MIN_NT
#define SINCOS_PHASE_ROWS_MIN_NT 1024
#endif
constexpr size_t kPhaseRowsMinNt = SINCOS_PHASE_ROWS_MIN_NT;   // shorter rows: the short-row kernel (t in shared memory; measured faster below ~1000)
#ifndef SINCOS_PHASE_ROWS_PER_BLOCK
#define SINCOS_PHASE_ROWS_PER_BLOCK 8
#endif
constexpr size_t kPhaseRowsPerBlock = SINCOS_PHASE_ROWS_PER_BLOCK;   // target rows per row slot
#ifndef SINCOS_PHASE_VEC_MIN_NT
#define SINCOS_PHASE_VEC_MIN_NT 256
#endif
constexpr size_t kPhaseVecMinNt = SINCOS_PHASE_VEC_MIN_NT;     // aligned rows shorter: the short-row kernel
#ifndef SINCOS_PHASE_SHORT_BPS
#define SINCOS_PHASE_SHORT_BPS 256
#endif
constexpr size_t kPhaseShortBlocksPerSm = SINCOS_PHASE_SHORT_BPS;     // short-row kernel grid, per SM
cudaError_t launch_phase_rows(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, unsigned h0, int sms,
                              cudaStream_t stream);
// NEXT(2) fused non-uniform Fourier sum (sincos_nudft.cu); variant 3/4 = comparison sincosf.
size_t nudft_chunk(size_t nt);
size_t nudft_ws_bytes(size_t nf, size_t nt);
struct MethodParams;
// variant 5 = the general method `method` (max series terms method_nt, fix 0/1/3); method_spec
// >= 0 selects a compile-time shape (0 = n_ss 4 / n_cc 3 / 2 doublings, 1 = 3 / 2 / 1).
cudaError_t launch_nudft(int variant, bool turns, const float *f, size_t nf, const float *t, const float *a,
                         size_t nt, float *out, void *ws, cudaStream_t stream, const MethodParams *method = nullptr,
                         int method_nt = 4, int method_fix = 0, int method_spec = -1);
// Test hook (sincos_packcheck.cu): packed vs scalar method over all 2^32 inputs; shape -1 = the
// paper's table of `variant`, 0 / 1 = method shapes (4,3,2) / (3,2,1) with fix 0/1.
cudaError_t launch_packcheck(int variant, int shape, int fix, const MethodParams *m, unsigned grid,
                             unsigned long long *mismatch_dev, cudaStream_t stream);
// Packed fp32 (FFMA2) kernels for the fused sum: 1 = on (default), 0 = scalar; -1 on bad value.
int set_nudft_packed(int on);
int get_nudft_packed();
// NEXT(3) general method (sincos_method.cu).
// k = theta's float offset past the 32-B boundary at element head - k (0 = aligned).
cudaError_t launch_method(const float *ss, int n_ss, const float *cc, int n_cc, int doublings, int fix, bool inter,
                          bool vec, unsigned grid, const float *theta, float *so, float *co, float *io, size_t head,
                          size_t nvec, size_t n, int k, cudaStream_t stream);
// NEXT(4) 16-bit outputs (dtype 1 = fp16, 2 = bf16) and fp32 layout adapters (sincos_dtype.cu).
cudaError_t launch_pairs16(int variant, int dtype, bool inter, unsigned grid, const float *theta, void *so, void *co,
                           void *io, size_t head, size_t nvec, size_t n, int k, cudaStream_t stream);
cudaError_t launch_interleave(bool to_inter, unsigned grid, const float *s, const float *c, float *io, size_t n,
                              cudaStream_t stream);
const void *vec_kernel_ptr(int variant, bool inter, int w, int unroll, bool nc, bool pf);

size_t stats_ws_bytes();
cudaError_t launch_stats(const float *theta, const float *so, const float *co, const float *io, size_t n,
                         sincos_stats_t *out, void *ws, cudaStream_t stream);

}  // namespace sincos_b200
