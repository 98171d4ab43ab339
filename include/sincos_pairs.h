/*
 * sincos_pairs.h -- C ABI of libsincos_pairs.so, the B200 (sm_100a) hot path of
 *
 *   M. H. Mendenhall, "A Fast, Vectorizable Algorithm for Producing
 *   Single-Precision Sine-Cosine Pairs", arXiv cs/0406049.
 *
 * Problem statement: sine-cosine pairs "in random order, or for
 * non-uniformly spaced values", a large number of them at once.  For every
 * fp32 angle theta[i] (radians) the library computes the fp32 pair
 * (sin theta[i], cos theta[i]) by the paper's method (Fig. 1
 * P:262-362):
 *   1. scale by 1/2pi and reduce onto [-1/2, 1/2] by rounding and subtraction
 *      (round half to even, reading G4),
 *   2. evaluate the quarter-angle series for (sin, cos)(pi q / 2) (P:72-75,
 *      coefficients P:140-148 / P:159-167, Horner order of Fig. 1),
 *   3. two angle doublings with Eq. (1): s' = 2sc, c' = c^2 - s^2,
 *   4. the amplitude handling of the chosen variant, computed from the
 *      penultimate pair (Fig. 1).
 * Arithmetic: IEEE fp32, round-to-nearest-even, fused multiply-add exactly
 * where Fig. 1 has vec_madd / vec_nmsub with a non-zero addend, no flush to
 * zero.  Results are bit-identical to the paper's algorithm as restated in
 * DESIGN.md (signed zeros and NaN payloads aside).  Every entry point is
 * thread-safe and reentrant; none allocates device memory except where stated,
 * none keeps a pointer after it returns.
 *
 * All pointers named *_dev are device pointers (cudaMalloc / torch CUDA
 * tensors) of the CURRENT device; *_host are host pointers (page-locked
 * memory recommended).  `stream` is a cudaStream_t (CUstream) passed as
 * void*; NULL means the legacy default stream.  Work is enqueued
 * asynchronously unless stated otherwise.
 */
#ifndef SINCOS_PAIRS_H
#define SINCOS_PAIRS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SINCOS_API __attribute__((visibility("default")))
#else
#define SINCOS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Amplitude handling (the paper's two methods). */
typedef enum {
    /* Method 1: least-squares series for sin and cos, then the
     * linear magnitude fix f = 2 - s2^2 - c2^2 of the penultimate pair
     * (Fig. 1 FASTER_SINCOS). */
    SINCOS_NORMALIZED = 0,
    /* Method 2: series fitted to the angle (coefficients marked
     * "dagger"; ss2 = -0.6466386396 of Fig. 1, reading G1), then the
     * exact reciprocal f = RN(1/(s2^2 + c2^2)) of the penultimate pair's
     * squared magnitude (Fig. 1; "precise reciprocal"). */
    SINCOS_RENORMALIZED = 1
} sincos_variant_t;

typedef enum {
    SINCOS_OK = 0,
    SINCOS_ERR_INVALID_ARGUMENT = 1, /* NULL where a buffer is needed, both or neither output
                                        form, unknown variant, misaligned (not 4-B) pointer  */
    SINCOS_ERR_OVERLAP = 2,          /* outputs overlap each other or the input (other than
                                        theta == sin_out or theta == cos_out exactly)        */
    SINCOS_ERR_CUDA = 3,             /* a CUDA call failed; see sincos_last_cuda_error()      */
    SINCOS_ERR_NCCL = 4              /* an NCCL call failed (sincos_pairs_sharded_stats only);
                                        see sincos_last_nccl_error()                         */
} sincos_status_t;

/*
 * sincos_pairs -- the hot path (one kernel launch).
 *
 *   theta_dev        n fp32 angles in radians, contiguous.
 *   sin_dev, cos_dev split output: sin_dev[i], cos_dev[i]  (both non-NULL), or
 *   inter_dev        interleaved output: inter_dev[2i] = cos, inter_dev[2i+1] = sin,
 *                    i.e. one complex64 e^{i theta} per element (struct phase {c, s},
 *                    P:262; reading G13).  Exactly one form must be given.
 *   n                element count; 0 is a no-op (pointers may then be NULL).
 *
 * Any 4-B aligned pointers are accepted; every path has identical numerics.
 * When theta and the outputs share their 32-B alignment the body runs 256-bit
 * vector loads/stores; otherwise, if the outputs can take 256-bit stores at a
 * common element (split: sin and cos at one offset mod 32 B; interleaved: 8-B
 * aligned), theta is read as aligned vectors and re-aligned in registers (warp
 * shuffles); otherwise the outputs are re-aligned instead (theta's 256-bit frame,
 * whole 32-B output blocks from neighbouring lanes) -- or, for most split layouts
 * with both sin and cos off theta's frame, theta is re-aligned onto one output's
 * frame and only the other output re-aligned.  (Exact in-place always
 * keeps the aliased output at theta's alignment.)
 * A scalar head and tail cover the ragged ends.  The kernel configuration (block
 * size, grid, vector width) is fixed per path -- a full grid of 128-thread blocks,
 * half of it with two trips per thread for interleaved pairs 4-B aligned at an odd
 * offset of 3, 5 or 7 floats -- and there is no tuning state.
 * theta_dev == sin_dev or
 * theta_dev == cos_dev (exact in-place) is allowed.  Validation happens
 * before any CUDA call; the return value reports validation and the launch
 * status only (the kernel itself cannot fail short of invalid addresses).
 */
SINCOS_API sincos_status_t sincos_pairs(const float *theta_dev, float *sin_dev, float *cos_dev,
                             float *inter_dev, size_t n, sincos_variant_t variant, void *stream);

/*
 * sincos_pairs_host -- the same computation on HOST buffers, end to end:
 * chunked host->device copies, the kernel and device->host copies pipelined
 * over three internal streams (created once per device), so the copy engines
 * run both directions while the kernel computes; chunks grow from 2^16 elements
 * to the workspace's slot size, so the first device->host copy starts early.
 * Synchronous: returns when the outputs are in host memory -- also on an error
 * after work was queued (the internal streams are drained first, so nothing of
 * the call still uses the caller's buffers).  Ordered after prior work on `stream`.
 * Concurrent calls from several host threads on one device are serialised
 * (the internal streams are shared); calls on different devices run in parallel.
 *
 *   dev_ws, ws_bytes  caller-owned device workspace of the current device
 *                     (>= sincos_host_workspace_min_bytes(); more = larger chunks).
 */
SINCOS_API sincos_status_t sincos_pairs_host(const float *theta_host, float *sin_host, float *cos_host,
                                  float *inter_host, size_t n, sincos_variant_t variant,
                                  void *dev_ws, size_t ws_bytes, void *stream);
SINCOS_API size_t sincos_host_workspace_min_bytes(void);

/*
 * NEXT(4): other output dtypes and layout adapters.
 *
 * sincos_pairs_dtype: the hot path with the pair rounded once (to nearest even) from the
 * method's fp32 result to out_dtype -- IEEE binary16 or bfloat16 (2 B per value; 8 B per
 * pair of traffic instead of 12) -- or fp32 (= sincos_pairs).  Outputs are 2-B aligned
 * uint16 arrays (split) or n {cos, sin} 16-bit pairs (interleaved); theta must not overlap
 * them.  Vector path always (8 pairs per thread; 128-bit split / 256-bit interleaved
 * stores in the frame of sin[] / the pairs), theta read as one aligned 256-bit vector or
 * re-aligned in registers when it sits off that frame; a split cos[] at another offset mod
 * 16 B is written as two 64-bit stores per vector (8 B off) or as whole 16-B blocks re-aligned
 * by warp shuffles (any other offset); head and tail one element per thread; identical values.
 *
 * sincos_interleave / sincos_deinterleave: fp32 split (sin[], cos[]) <-> interleaved
 * ({cos, sin} float2) copies; no overlap allowed.
 */
typedef enum { SINCOS_F32 = 0, SINCOS_F16 = 1, SINCOS_BF16 = 2 } sincos_dtype_t;
SINCOS_API sincos_status_t sincos_pairs_dtype(const float *theta_dev, void *sin_dev, void *cos_dev, void *inter_dev,
                                              size_t n, sincos_variant_t variant, sincos_dtype_t out_dtype,
                                              void *stream);
SINCOS_API sincos_status_t sincos_interleave(const float *sin_dev, const float *cos_dev, float *inter_dev, size_t n,
                                             void *stream);
SINCOS_API sincos_status_t sincos_deinterleave(const float *inter_dev, float *sin_dev, float *cos_dev, size_t n,
                                               void *stream);

/*
 * sincos_pairs_method -- NEXT(3): the method with caller-supplied series and doubling
 * count ("after n iterations ... two options for computing the raw pair.
 * These options differ in the fitting algorithm used to find the coefficients").
 *   s1 = RN(q * (ss[0] + q2 (ss[1] + ... q2 ss[n_ss-1])))   Horner, innermost first
 *   c1 = 1 + q2 (cc[0] + q2 (cc[1] + ... q2 cc[n_cc-1]))     (1 when n_cc == 0)
 * with q the reduced turn (steps a2-a3 unchanged), then `doublings` Eq. (1) doublings and
 * the amplitude handling `fix` taken from the penultimate pair: 0 = linear
 * f = 2 - s^2 - c^2 (method 1), 1 = exact reciprocal 1/(s^2 + c^2) (method 2; exact
 * for penultimate magnitudes^2 in [0.5, 2), i.e. any usable fit), 3 = none.
 * The paper's two methods are {its coefficients, n_ss 4, n_cc 3, doublings 2, fix 0/1}
 * and give bit-identical results to sincos_pairs.  Same buffers, alignment and error
 * conventions as sincos_pairs (in-place not supported); vector path (256-bit stores in the
 * frame of sin[] / the pairs; split cos[] at another offset mod 32 B re-aligned by warp
 * shuffles into whole 32-B blocks; interleaved pairs 8-B aligned), theta re-aligned in
 * registers when needed; interleaved pairs only 4-B aligned: theta's 32-B frame with the
 * pairs re-aligned by shuffles.
 * `method` is a host pointer, read before return.
 */
typedef struct {
    float ss[8];
    int n_ss;        /* 1..8 */
    float cc[8];
    int n_cc;        /* 0..8 */
    int doublings;   /* 0..8; fix requires >= 1 */
    int fix;         /* 0 linear, 1 reciprocal, 3 none */
} sincos_method_t;
SINCOS_API sincos_status_t sincos_pairs_method(const float *theta_dev, float *sin_dev, float *cos_dev,
                                               float *inter_dev, size_t n, const sincos_method_t *method,
                                               void *stream);

/*
 * sincos_phase_grid -- NEXT(1): pairs of phases generated inside the kernel.
 *
 * The paper's use case is phase factors for optical diffraction by Huygens'
 * principle -- many non-uniformly spaced phases, e.g. the
 * products of a frequency axis and a jittered time axis (BASELINE configs[3]).
 * For every i < nf, j < nt the phase is one rounded fp32 product
 *     p_ij = RN(f_dev[i] * t_dev[j])
 * and the output element (i, j), at index i*nt + j (row-major, row = f_i), is
 *     units == SINCOS_RADIANS: (sin p_ij, cos p_ij), the whole method;
 *     units == SINCOS_TURNS:   (sin 2 pi p_ij, cos 2 pi p_ij): p_ij is already in
 *                              turns, the method starts at the reduction
 *                              and skips the 1/2pi scaling and its rounding.
 * Outputs as in sincos_pairs (split sin/cos of nf*nt floats each, or interleaved
 * {cos, sin}).  Only 8 B per pair are written (no theta array is read); f and t
 * must not overlap the outputs.  Paths, identical numerics: nt % 8 == 0, nt >= 256, with
 * 32-B aligned t and outputs -- 256-bit vectors per row; any other nt / alignment with
 * outputs that can take 256-bit stores (split: sin and cos at the same offset mod
 * 32 B; interleaved: 8-B aligned) -- for nt >= 1024 the row path (each thread keeps
 * eight t-values, re-aligned by warp shuffles to the rows' output alignment, and
 * writes them for the rows of one alignment class), for nt < 1024 (and whole-vector
 * rows shorter than 256) the short-row path (8 consecutive pairs of the row-major grid
 * per thread, t from shared memory) -- except rows of 1 pair, or 2-3 pairs split, with
 * outputs 32-B aligned at pair 0: the tiny-row path (8 whole rows per thread), and rows
 * of 4-14 pairs split or 2-15 interleaved with outputs 16-B aligned at pair 0: the staged
 * path (4 or 2 whole rows per thread, a warp's 128 or 64 rows staged in shared memory and
 * written back as contiguous 512-B stores); outputs that cannot take 256-bit stores at a
 * common element (split: sin and cos at different offsets mod 32 B; interleaved: pairs
 * only 4-B aligned): 8 consecutive pairs per thread in sin[]'s 32-B frame, the other
 * stream re-aligned into whole 32-B blocks by warp shuffles.  Returns as sincos_pairs;
 * nf*nt == 0 is a no-op.
 */
typedef enum { SINCOS_RADIANS = 0, SINCOS_TURNS = 1 } sincos_units_t;
SINCOS_API sincos_status_t sincos_phase_grid(const float *f_dev, size_t nf, const float *t_dev, size_t nt,
                                             float *sin_dev, float *cos_dev, float *inter_dev,
                                             sincos_units_t units, sincos_variant_t variant, void *stream);

/*
 * sincos_nudft -- NEXT(2): the pairs' consumer fused with them, a direct
 * non-uniform Fourier / Huygens sum (the diffraction application of P:203-206):
 *     out[k] = sum_{j < nt} a[j] * (cos p_kj + i sin p_kj),   p_kj = RN(f[k] * t[j]),
 * p in radians or turns as in sincos_phase_grid, pairs bit-identical to it.
 *   a_dev    nt complex64 amplitudes, interleaved {re, im} (8-B aligned)
 *   out_dev  nf complex64 results, interleaved {re, im} (8-B aligned)
 *   ws_dev   device workspace of >= sincos_nudft_workspace_bytes(nf, nt) bytes
 *            (16-B aligned), not overlapping anything else
 * Arithmetic: complex products and sums in fp32 with FMA over runs ("chunks") of
 * sincos_nudft_chunk(nt) consecutive terms (256 for nt < 4096, else 1024), summed in
 * order; each run's sum is added into fp64, the terms split into segments for
 * parallelism (a fixed rule, the same on every device) whose fp64 partials are added in
 * segment order; one final rounding to fp32: deterministic.  Workspace: 16 B per
 * frequency per segment (a few MB at 2^15 x 2^15).  Error bound
 * against the exact sum of the same pairs:
 *   |out[k] - F_k| <= (chunk + 2) * 2^-24 * sum_j |a_j| + 2^-24 |F_k|.
 * Two launches (partials, reduction).  nf == 0 is a no-op; nt == 0 zeroes out.
 * variant: SINCOS_NORMALIZED / SINCOS_RENORMALIZED, or -- for comparison only --
 * 3 = CUDA libm sincosf (sincospif in turns), 4 = the __sincosf intrinsic.
 */
SINCOS_API size_t sincos_nudft_chunk(size_t nt);
SINCOS_API size_t sincos_nudft_workspace_bytes(size_t nf, size_t nt);
SINCOS_API sincos_status_t sincos_nudft(const float *f_dev, size_t nf, const float *t_dev, const float *a_dev,
                                        size_t nt, float *out_dev, sincos_units_t units, int variant,
                                        void *ws_dev, size_t ws_bytes, void *stream);
/* The same sum with the pairs of a general method (NEXT(3), sincos_method_t above);
 * pairs bit-identical to sincos_pairs_method, same bound and conventions. */
SINCOS_API sincos_status_t sincos_nudft_method(const float *f_dev, size_t nf, const float *t_dev,
                                               const float *a_dev, size_t nt, float *out_dev,
                                               sincos_units_t units, const sincos_method_t *method,
                                               void *ws_dev, size_t ws_bytes, void *stream);

/*
 * Host-side sharding: element ranges [lo, hi) of shard g of
 * nshards, contiguous, every shard start a multiple of 8 elements (32-B
 * aligned in any aligned array); the last shard takes the remainder.  Pure
 * function, no CUDA.  Returns 0, or -1 for nshards < 1 or g outside [0, nshards).
 */
SINCOS_API int sincos_shard_range(size_t n, int nshards, int g, size_t *lo, size_t *hi);

/* One shard resident on one device. */
typedef struct {
    int device;              /* CUDA device ordinal owning the buffers     */
    const float *theta_dev;
    float *sin_dev, *cos_dev, *inter_dev;
    size_t n;
    void *stream;            /* stream of that device (NULL = its legacy default) */
} sincos_shard_t;

/* Launch every shard on its own device (single process, many devices); no data
 * crosses devices.  Every shard is validated, and every device ordinal checked
 * against cudaGetDeviceCount (else INVALID_ARGUMENT), before anything is launched.
 * With shards on several devices, one host thread per device (created on first use,
 * kept for the process) launches that device's shards, so the devices start together
 * rather than one launch latency apart each; shards on one device launch in order from
 * the calling thread.  Returns the first failing shard's status (its CUDA error in
 * sincos_last_cuda_error of the calling thread); the other shards may have been
 * launched.  The caller's current device is unchanged.  (Test hook: the environment variable
 * SINCOS_SHARDED_WORKERS=1, read once, routes single-device calls through the worker threads too.) */
SINCOS_API sincos_status_t sincos_pairs_sharded(const sincos_shard_t *shards, int nshards,
                                     sincos_variant_t variant);

/*
 * Per-shard error statistics (verification, not the hot path): for each element,
 * the paper's metrics against an fp64 reference computed on the
 * device: combined error sqrt((c - cos)^2 + (s - sin)^2), amplitude error
 * |1 - sqrt(c^2 + s^2)|.  A 64-byte record, small enough to gather over NCCL.
 * Reductions are deterministic (fixed grid, fixed order).
 */
typedef struct {
    uint64_t n;            /* elements measured (finite outputs)          */
    uint64_t nan_count;    /* output pairs holding a NaN                  */
    double   max_comb;     /* max combined error                          */
    double   sum_sq;       /* sum of combined error squared               */
    double   max_amp;      /* max amplitude error                         */
    double   kernel_ms;    /* filled in by the caller (timing), else 0     */
    float    worst_theta;  /* an argument at max_comb                     */
    uint32_t device;       /* filled in by the caller                     */
    uint64_t reserved;
} sincos_stats_t;

/*
 * sincos_pairs_sharded_stats -- the whole single-process multi-device run:
 * launch every shard on its own device (one shard per device, distinct devices), reduce
 * each shard's error statistics (below) and kernel time (CUDA events around its launch)
 * into its 64-byte record, and all-gather the records over NCCL (ncclCommInitAll over the
 * shards' devices, ncclAllGather inside a group) -- the only collective of the path, 64 B
 * per rank.  gathered: host array of nshards records, shard order.  Synchronous (every
 * stream it used is drained before it returns, on success and on error).  NCCL is bound at
 * run time (dlopen "libnccl.so.2"); without it returns INVALID_ARGUMENT (see
 * sincos_nccl_available).  Device ordinals are checked before any launch.  The
 * communicator and small per-device buffers (stats workspace, records, events) are created
 * on the first call for a device list and kept for the process: later calls on the same
 * devices reuse them.  A failing NCCL call returns SINCOS_ERR_NCCL (its ncclResult_t in
 * sincos_last_nccl_error), a failing CUDA call SINCOS_ERR_CUDA.
 */
SINCOS_API sincos_status_t sincos_pairs_sharded_stats(const sincos_shard_t *shards, int nshards,
                                                      sincos_variant_t variant, sincos_stats_t *gathered);
SINCOS_API int sincos_nccl_available(void);
SINCOS_API int sincos_last_nccl_error(void);     /* ncclResult_t of the last SINCOS_ERR_NCCL in this thread */

SINCOS_API size_t sincos_stats_workspace_bytes(void);
/* stats_dev: device pointer to one sincos_stats_t (8-B aligned); ws_dev: device workspace
 * of sincos_stats_workspace_bytes() (8-B aligned), not shared by concurrent calls.
 * Outputs as in sincos_pairs (split or interleaved, 4-B aligned).  Asynchronous. */
SINCOS_API sincos_status_t sincos_error_stats(const float *theta_dev, const float *sin_dev,
                                   const float *cos_dev, const float *inter_dev, size_t n,
                                   sincos_stats_t *stats_dev, void *ws_dev, void *stream);

/* Traffic-ceiling kernel (bench only): same access pattern and launch as
 * sincos_pairs, no arithmetic (writes theta to both outputs). */
SINCOS_API sincos_status_t sincos_null_4in8out(const float *theta_dev, float *sin_dev, float *cos_dev,
                                    float *inter_dev, size_t n, void *stream);

/* Context kernels (bench only, not the paper's method): the same 4-in / 8-out streaming
 * kernel with CUDA's own functions -- which = 3: libm sincosf (accurate; Payne-Hanek slow
 * path for large |theta|), 4: the __sincosf intrinsic.  Buffers 32-B aligned (else
 * INVALID_ARGUMENT), no in-place; otherwise as sincos_pairs. */
SINCOS_API sincos_status_t sincos_compare_cuda(const float *theta_dev, float *sin_dev, float *cos_dev,
                                               float *inter_dev, size_t n, int which, void *stream);

/* Test hook: the packed-fp32 form of the method (sm_100a FFMA2/FMUL2/FADD2, used by the
 * fused sum) against the scalar form, for EVERY one of the 2^32 fp32 inputs, in radians and
 * in turns.  method == NULL: the paper's table of `variant`; else a specialised method shape
 * (n_ss/n_cc/doublings 4/3/2 or 3/2/1, fix 0 or 1; variant ignored).  Asynchronous on
 * `stream`: *mismatch_dev (device, 8-B aligned) is zeroed, then receives the number of
 * differing output components (NaN equals NaN; otherwise bit patterns).  0 is expected.
 * variant == -1 (method NULL) is the negative control: packed method 1 against scalar
 * method 2, which must differ wherever their pairs do (proves the check can fail). */
SINCOS_API sincos_status_t sincos_debug_packed_check(int variant, const sincos_method_t *method,
                                                     unsigned long long *mismatch_dev, void *stream);

/* Test hook: the kernel's reciprocal sequence alone, out[i] = RN(1/d[i]). */
SINCOS_API sincos_status_t sincos_debug_reciprocal(const float *d_dev, float *out_dev, size_t n,
                                        void *stream);

SINCOS_API const char *sincos_status_string(sincos_status_t s);
SINCOS_API int sincos_last_cuda_error(void);      /* cudaError_t of the last SINCOS_ERR_CUDA in this thread */
SINCOS_API const char *sincos_version(void);
/* Number of kernel launches this process has issued through the library. */
SINCOS_API uint64_t sincos_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SINCOS_PAIRS_H */
