// sincos_launch.h -- internal launch interface between the C ABI and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/sincos_pairs.h"

namespace sincos_b200 {

// Kernel selection.  The product library has ONE configuration: these defaults, the one every
// measurement in DESIGN.md was taken with (a sweep on the B200 found them best, section 5), and
// nothing in it is settable -- no process-global state changes what another caller gets.  The
// A/B build (-DSINCOS_AB -> libsincos_pairs_ab.so, loaded only by tests/ and tools/) makes each
// field settable through sincos_ab_set (csrc/sincos_ab.h) to measure the alternatives.
struct Tuning {
    int threads = 128;       // threads per block of the streaming kernels (128, 256, 512)
    int blocks_per_sm = 0;   // 0: the full grid, one trip per thread; > 0: grid-stride, SMs x this
    int vec = 8;             // floats per thread access: 8 (256-bit) or 4 (128-bit)
    int unroll = 1;          // independent vectors per thread and trip (1, 2, 4)
    int prefetch = 0;        // 1: software-pipelined loads (trip k+1 in flight while trip k computes)
    int realign = 1;         // 1: register re-alignment of unshared alignments; 0: one element per
                             // thread; 2: its 128-bit form only; 3: ragged phase rows via the flat kernel
    int pdl = 1;             // programmatic dependent launch of the 256-bit vector kernel
    int nudft_packed = 1;    // fused sum on packed fp32 (FFMA2) rather than its scalar twin
};
#ifdef SINCOS_AB
Tuning tuning();                                         // sincos_abi.cu: the A/B settings
#else
__host__ inline constexpr Tuning tuning() { return Tuning{}; }
#endif

// variant: 0 = N, 1 = A, 2 = null (traffic ceiling); w = 4 or 8 floats per access;
// unroll = 1, 2 or 4; nc = read-only (non-coherent) loads, false when theta aliases an output.
// pf = software-pipelined loads (trip k+1 in flight while trip k computes).  unroll != 1 and pf
// exist in the A/B build only.  pdl: programmatic dependent launch (256-bit instances).
cudaError_t launch_vec(int variant, bool inter, int w, int unroll, bool nc, bool pf, bool pdl, unsigned grid,
                       unsigned threads, const float *theta, float *so, float *co, float *io, size_t head,
                       size_t nvec, size_t n, cudaStream_t stream);
// Context kernels for the bench (3 = CUDA sincosf, 4 = __sincosf), 32-B aligned buffers, head 0.
cudaError_t launch_compare(int which, bool inter, unsigned grid, unsigned threads, const float *theta, float *so,
                           float *co, float *io, size_t nvec, size_t n, cudaStream_t stream);
// KB3b, 128-bit form (A/B build only): outputs 16-B aligned from element `head`, theta K = k
// floats past a 16-B boundary there.
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
#ifdef SINCOS_AB
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
// KB3, one element per thread (the A/B build's realign = 0).
cudaError_t launch_scalar(int variant, bool inter, unsigned grid, unsigned threads, const float *theta, float *so,
                          float *co, float *io, size_t n, cudaStream_t stream);
#endif  // SINCOS_AB
cudaError_t launch_rcp(unsigned grid, unsigned threads, const float *d, float *out, size_t n, cudaStream_t stream);
// NEXT(1) phase grid (sincos_phase.cu); vec = 256-bit path (nt % 8 == 0, 32-B aligned t/outputs).
cudaError_t launch_phase_grid(int variant, bool inter, bool turns, bool vec, const float *f, size_t nf,
                              const float *t, size_t nt, float *so, float *co, float *io, cudaStream_t stream);
// NEXT(1) flat path for any nt: pairs [head, head + 8 nvec) as 256-bit stores (outputs 32-B
// aligned at `head`), the rest one per thread; grid-stride over `grid` blocks.  short_rows:
// for nt < kPhaseRowsMinNt the one-path kernel with t in shared memory (the product's only
// form; short_rows = false, the flat kernel, exists in the A/B build only).
cudaError_t launch_phase_flat(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, size_t head, size_t nvec,
                              unsigned grid, bool short_rows, cudaStream_t stream);
// unshared output alignment (split cos[] off sin[]'s 32-B offset, or interleaved pairs only
// 4-B aligned): the flat mapping with the re-aligned stream written by warp shuffles
cudaError_t launch_phase_flat_sh(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                                 size_t nt, float *so, float *co, float *io, size_t head, size_t nvec,
                                 unsigned grid, int kc, cudaStream_t stream);
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
#ifndef SINCOS_PHASE_STAGED_MAX_NT
#define SINCOS_PHASE_STAGED_MAX_NT 14    // longest rows (pairs) of the staged short-row kernel, split
#endif
#ifndef SINCOS_PHASE_STAGED_MAX_NT_INTER
#define SINCOS_PHASE_STAGED_MAX_NT_INTER 15  // ... and interleaved
#endif
static_assert(SINCOS_PHASE_STAGED_MAX_NT <= 14 && SINCOS_PHASE_STAGED_MAX_NT_INTER <= 15,
              "staged instances exist for split rows of 2-14 pairs and interleaved rows of 2-15");
// Row lengths with a staged instance, up to the maxima above (the product routes split rows of
// 2-3 pairs to the tiny-row kernel instead).  Longer rows (16-31 pairs, 2 rows per lane) were
// measured: within the run-to-run spread of the short-row kernel, +-5% by shape and variant
// (profiles/r02/ab_phase_m16_v*.jsonl) -- not kept.
inline bool phase_staged_ok(bool inter, size_t nt) {
    return nt >= 2 && nt <= static_cast<size_t>(inter ? SINCOS_PHASE_STAGED_MAX_NT_INTER : SINCOS_PHASE_STAGED_MAX_NT);
}
#ifndef SINCOS_PHASE_VEC_MIN_NT
#define SINCOS_PHASE_VEC_MIN_NT 256
#endif
constexpr size_t kPhaseVecMinNt = SINCOS_PHASE_VEC_MIN_NT;     // aligned rows shorter: the short-row kernel
// Short-row kernel grid, blocks per SM (grid-striding): rows of >= 256 pairs 64 (nt = 1001
// interleaved: 6.37 vs 6.05 TB/s at 256), shorter rows 256 (nt = 2..9: 3% ahead of 64;
// tools/ab_phase.py, profiles/r02/ab_phase_short.jsonl).
#ifndef SINCOS_PHASE_SHORT_BPS
#define SINCOS_PHASE_SHORT_BPS 256
#endif
#ifndef SINCOS_PHASE_SHORT_BPS_LONG
#define SINCOS_PHASE_SHORT_BPS_LONG 64
#endif
constexpr size_t phase_short_blocks_per_sm(size_t nt) {
    return nt >= 256 ? SINCOS_PHASE_SHORT_BPS_LONG : SINCOS_PHASE_SHORT_BPS;
}
// NEXT(1) tiny rows (1 <= nt <= 7), outputs 32-B aligned at pair 0: groups of 8 rows per thread,
// the row length a compile-time parameter.
cudaError_t launch_phase_staged(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                                size_t nt, float *so, float *co, float *io, size_t max_grid, cudaStream_t stream);
cudaError_t launch_phase_tiny(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, cudaStream_t stream);
cudaError_t launch_phase_rows(int variant, bool inter, bool turns, const float *f, size_t nf, const float *t,
                              size_t nt, float *so, float *co, float *io, unsigned h0, int sms,
                              cudaStream_t stream);
// NEXT(2) fused non-uniform Fourier sum (sincos_nudft.cu); variant 3/4 = comparison sincosf.
size_t nudft_chunk(size_t nt);
size_t nudft_ws_bytes(size_t nf, size_t nt);
struct MethodParams;
// variant 5 = the general method `method` (max series terms method_nt, fix 0/1/3); method_spec
// >= 0 selects a compile-time shape (0 = n_ss 4 / n_cc 3 / 2 doublings, 1 = 3 / 2 / 1).
// packed: the FFMA2 kernels (the product's only form; false, their scalar twins, in the A/B build).
cudaError_t launch_nudft(int variant, bool turns, const float *f, size_t nf, const float *t, const float *a,
                         size_t nt, float *out, void *ws, cudaStream_t stream, const MethodParams *method = nullptr,
                         int method_nt = 4, int method_fix = 0, int method_spec = -1, bool packed = true);
// Test hook (sincos_packcheck.cu): packed vs scalar method over all 2^32 inputs; shape -1 = the
// paper's table of `variant`, 0 / 1 = method shapes (4,3,2) / (3,2,1) with fix 0/1.
cudaError_t launch_packcheck(int variant, int shape, int fix, const MethodParams *m, unsigned grid,
                             unsigned long long *mismatch_dev, cudaStream_t stream);
// NEXT(3) general method (sincos_method.cu).
// k = theta's float offset past the 32-B boundary at element head - k (0 = aligned).
cudaError_t launch_method(const float *ss, int n_ss, const float *cc, int n_cc, int doublings, int fix, bool inter,
                          bool vec, unsigned grid, const float *theta, float *so, float *co, float *io, size_t head,
                          size_t nvec, size_t n, int k, cudaStream_t stream);
// NEXT(4) 16-bit outputs (dtype 1 = fp16, 2 = bf16) and fp32 layout adapters (sincos_dtype.cu).
cudaError_t launch_pairs16(int variant, int dtype, bool inter, unsigned grid, const float *theta, void *so, void *co,
                           void *io, size_t head, size_t nvec, size_t n, int k, int cw, cudaStream_t stream);
cudaError_t launch_interleave(bool to_inter, unsigned grid, const float *s, const float *c, float *io, size_t n,
                              cudaStream_t stream);

size_t stats_ws_bytes();
cudaError_t launch_stats(const float *theta, const float *so, const float *co, const float *io, size_t n,
                         sincos_stats_t *out, void *ws, cudaStream_t stream);

}  // namespace sincos_b200
