/*
 * sincos_oracle.h -- ORACLE (test infrastructure only).
 *
 * Plain, slow, obviously-correct CPU transcription of the algorithm of
 * M. H. Mendenhall, "A Fast, Vectorizable Algorithm for Producing
 * Single-Precision Sine-Cosine Pairs", arXiv cs/0406049.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load or call anything in oracle/.  The product
 * path (paper_cs_0406049_b200/) never includes this header and never links
 * this library; the two share no code, headers, tables or constants.
 *
 * Citation keys: P:n = PAPER.md line n (section / equation / Fig. 1).
 */
#ifndef SINCOS_ORACLE_H
#define SINCOS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One coefficient set: ss1..ss4 (odd series), cc1..cc3 (even series),
 * P:140-148 (method 1), P:159-167 (method 2), Fig. 1 P:228-258. */
typedef struct {
    float ss1, ss2, ss3, ss4;
    float cc1, cc2, cc3;
} oracle_coeffs_t;

/* Which amplitude handling ends the pipeline. */
typedef enum {
    ORACLE_FIX_LINEAR_PENULTIMATE = 0, /* Fig. 1 FASTER_SINCOS: f = 2 - s2^2 - c2^2 */
    ORACLE_FIX_RECIPROCAL = 1,         /* Fig. 1 #else branch: f = 1/(s2^2 + c2^2) */
    ORACLE_FIX_TEXT_FINAL = 2,         /* test-only: text form P:131-134, (3 - s^2 - c^2)/2 on final pair */
    ORACLE_FIX_NONE = 3,               /* test-only: no amplitude handling */
    ORACLE_FIX_EXACT_FINAL = 4         /* test-only: final pair times fl32(1/sqrt(s^2+c^2)) in double
                                          (the exact renormalisation P:131-132 "divide the function
                                          pair by sqrt(1+alpha)"; used with Eq. (2) in the pins) */
} oracle_fix_t;

/* Which doubling recursion. */
typedef enum {
    ORACLE_DOUBLING_EQ1 = 0, /* Eq. (1): s'=2sc, c'=c^2-s^2 (the method) */
    ORACLE_DOUBLING_EQ2 = 1  /* Eq. (2): s'=2sc, c'=1-2s^2 (rejected; test-only) */
} oracle_doubling_t;

/* Full pipeline options.  The paper's two shipped methods are
 *   variant 0 (N): coeffs N,       EQ1, doublings 2, FIX_LINEAR_PENULTIMATE
 *   variant 1 (A): coeffs A(Fig1), EQ1, doublings 2, FIX_RECIPROCAL
 * Everything else is a test-only alternative used by the pins. */
typedef struct {
    oracle_coeffs_t coeffs;
    oracle_fix_t fix;
    oracle_doubling_t doubling;
    int doublings;   /* n in P:116-117; the shipped coefficients need n = 2 */
} oracle_opts_t;

/* Named variants (the same numbering as the product ABI's enum, restated here). */
enum {
    ORACLE_VARIANT_N = 0,       /* method 1, "normalised" (Fig. 1 FASTER_SINCOS)         */
    ORACLE_VARIANT_A = 1,       /* method 2, "angle-accurate", Fig. 1 ss2 = -0.6466386396 */
    ORACLE_VARIANT_A_TEXT = 2,  /* test-only: method 2 with the text ss2 = -0.6466386936  */
    ORACLE_VARIANT_N_TEXTFIX = 3,/* test-only: method 1 with the text's final-pair fix    */
    ORACLE_VARIANT_N_NOFIX = 4, /* test-only: method 1 without amplitude handling         */
    ORACLE_VARIANT_A_NOFIX = 5, /* test-only: method 2 without amplitude handling         */
    ORACLE_VARIANT_A_LINFIX = 6,/* test-only: method-2 coeffs with the method-1 linear fix */
    ORACLE_VARIANT_COUNT = 7
};

/* Fill *o with the options of a named variant.  Returns 0, or -1 if unknown. */
int oracle_variant_opts(int variant, oracle_opts_t *o);

/* ---- the algorithm, step by step (each in the paper's order) ---------- */

/* Turn reduction, Fig. 1: x1 = theta * (1/2pi);
 * q1 = x1 - round_half_even(x1), exact. */
float oracle_reduce_turns(float theta);

/* Quarter-angle series (Horner, innermost first), Fig. 1 P:284-310:
 * (s, c) ~ (sin, cos)(pi q / 2). */
void oracle_poly_quarter(float q1, const oracle_coeffs_t *k, float *s, float *c);

/* One doubling, Eq. (1) P:77-79 in Fig. 1's operation order P:314-318
 * (or Eq. (2) when doubling == ORACLE_DOUBLING_EQ2, test-only). */
void oracle_double_angle(float s, float c, oracle_doubling_t form, float *s_out, float *c_out);

/* The whole pipeline on one angle from its reduced turn q (kernel-only),
 * or from theta.  Returns (s, c). */
void oracle_pair_from_q(float q1, const oracle_opts_t *o, float *s, float *c);
void oracle_pair(float theta, const oracle_opts_t *o, float *s, float *c);

/* Array form: s_out[i], c_out[i] for theta[i], i < n.  Plain loop.
 * Returns 0, or -1 for an unknown variant. */
int sincos_oracle(const float *theta, float *s_out, float *c_out, size_t n, int variant);
int sincos_oracle_opts(const float *theta, float *s_out, float *c_out, size_t n,
                       const oracle_opts_t *o);

/* ---- NEXT(3): the method with any series degrees and doubling count --------
 * "the form of (1) produces a pair (after n iterations) ... there are two
 * options for computing the raw pair. These options differ in the fitting algorithm
 * used to find the coefficients".  Series (Horner, innermost first, as Fig. 1):
 *   s1 = RN(q * (ss[0] + q2 (ss[1] + ... q2 ss[n_ss-1])))        (n_ss >= 1)
 *   c1 = 1 + q2 (cc[0] + q2 (cc[1] + ... q2 cc[n_cc-1]))          (n_cc >= 0; 1 if 0)
 * then `doublings` Eq. (1) doublings, the fix from the penultimate pair (Fig. 1
 * order; needs doublings >= 1) or none.  For n_ss = 4, n_cc = 3, doublings = 2 it
 * is exactly oracle_pair_from_q with the same coefficients. */
#define ORACLE_MAX_TERMS 8
typedef struct {
    float ss[ORACLE_MAX_TERMS];
    int n_ss;
    float cc[ORACLE_MAX_TERMS];
    int n_cc;
    int doublings;    /* 0 .. 8 */
    int fix;          /* ORACLE_FIX_LINEAR_PENULTIMATE, ORACLE_FIX_RECIPROCAL or ORACLE_FIX_NONE */
} oracle_method_t;

/* Returns 0, or -1 for an invalid method. */
int oracle_method_pair_from_q(float q1, const oracle_method_t *m, float *s, float *c);
int oracle_method_sincos(const float *theta, float *s_out, float *c_out, size_t n,
                         const oracle_method_t *m);

/* ---- NEXT(1): pairs of generated phases f*t -------
 * units 0: RN(f*t) is an angle in radians (the full method);
 * units 1: RN(f*t) is in turns (theta/2pi): the method from the reduction on.
 * Returns 0, or -1 for an unknown variant or units. */
void oracle_phase_pair(float f, float t, int units, const oracle_opts_t *o, float *s, float *c);
int oracle_phase_points(const float *f, const float *t, size_t m, int units, int variant,
                        float *s_out, float *c_out);
/* element (i, j) at i*nt + j */
int oracle_phase_grid(const float *f, size_t nf, const float *t, size_t nt, int units, int variant,
                      float *s_out, float *c_out);

/* ---- NEXT(2): direct non-uniform Fourier / Huygens sum ------
 * out[k] = sum_j a_j * (cos p_kj + i sin p_kj), p_kj = RN(f_k t_j) (units as
 * above); a: nt interleaved {re, im} floats; out: nf interleaved {re, im}
 * doubles, products and sums in double.  Returns 0 or -1. */
int oracle_nudft(const float *f, size_t nf, const float *t, const float *a, size_t nt, int units,
                 int variant, double *out);

/* ---- error metrics, P:135-139 (accuracy.c) -------------------------- */

typedef struct {
    uint64_t count;        /* finite elements measured                              */
    uint64_t nan_count;    /* elements whose output pair holds a NaN                */
    double   sum_sq;       /* sum of combined error^2 (sequential order)             */
    double   max_comb;     /* max sqrt((c-rc)^2 + (s-rs)^2)                          */
    double   max_amp;      /* max |1 - sqrt(c^2 + s^2)| (signed value in amp_signed) */
    double   amp_signed;   /* the 1 - sqrt(c^2+s^2) value at max |.|               */
    double   sum_s;        /* sum of s outputs (sequential order)                    */
    double   sum_c;        /* sum of c outputs (sequential order)                    */
    float    worst_x;      /* theta (or q) at max_comb                               */
    uint32_t worst_bits;
} oracle_stats_t;

/* Reference kinds. */
enum { ORACLE_REF_DOUBLE = 0, ORACLE_REF_LONGDOUBLE = 1 };

/* Stats of given outputs (s[i], c[i]) against sin/cos(theta[i]) in double
 * (the paper's reference) or long double.  Sequential. */
void oracle_error_stats(const float *theta, const float *s, const float *c, size_t n,
                        int ref_kind, oracle_stats_t *st);

/* Same for interleaved {cos, sin} float2 outputs. */
void oracle_error_stats_interleaved(const float *theta, const float *cs, size_t n,
                                    int ref_kind, oracle_stats_t *st);

/* Stats of the oracle itself over the grid
 *   theta_k = (float)(-pi + ((2 pi) * (double)k) / (double)m),  k < m.
 * Sequential (so the sums are reproducible bit for bit). */
void oracle_grid_stats(const oracle_opts_t *o, uint64_t m, int ref_kind, oracle_stats_t *st);

/* Exhaustive stats over every fp32 bit pattern u in [lo_bits, hi_bits]
 * interpreted as theta (mode 0) or as q, kernel-only, reference sin/cos(2 pi q)
 * (mode 1).  Parallel over nthreads; max with lowest-index argmax; sums are
 * combined per fixed chunk in index order, so results do not depend on
 * nthreads. */
void oracle_sweep_bits(const oracle_opts_t *o, int mode, uint32_t lo_bits, uint32_t hi_bits,
                       int nthreads, oracle_stats_t *st);

/* NEXT(3): kernel-only stats of a general method over q = bits(lo_bits + k*stride) <= hi_bits,
 * against sin/cos(2 pi q) in double. */
void oracle_method_sweep_q(const oracle_method_t *m, uint32_t lo_bits, uint32_t hi_bits, uint32_t stride,
                           int nthreads, oracle_stats_t *st);

/* Whole-input-space transcription hash over u in [lo_bits, hi_bits]:
 *   H = sum_u mix64(((s_bits << 32) | c_bits) ^ (u * 0xD6E8FEB86659FD93)) mod 2^64
 * with NaN canonicalised to 0x7FC00000 and +-0 to 0.
 * Also counts NaN pairs and exact (0, 1) pairs. */
void oracle_hash_bits(const oracle_opts_t *o, uint32_t lo_bits, uint32_t hi_bits, int nthreads,
                      uint64_t *hash, uint64_t *nan_pairs, uint64_t *exact_01);

/* Same hash over given outputs (split or interleaved), for the product's
 * outputs copied back to the host: u = first_bits + i. */
uint64_t oracle_hash_outputs(const float *s, const float *c, const float *cs,
                             size_t n, uint32_t first_bits);

#ifdef __cplusplus
}
#endif
#endif /* SINCOS_ORACLE_H */
