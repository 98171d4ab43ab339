/*
 * sincos_oracle.c -- ORACLE (test infrastructure only; see sincos_oracle.h).
 *
 * A scalar C99 transcription of Mendenhall, arXiv cs/0406049, following the
 * paper's Fig. 1 listing operation by operation.  Each
 * AltiVec operation is restated with the C99 operation that has the same
 * single-rounding semantics:
 *
 *   vec_madd(a, b, c)   = RN(a*b + c)        -> fmaf(a, b, c)
 *   vec_nmsub(a, b, c)  = -RN(a*b - c)       -> fmaf(-a, b, c)   (RN is odd-symmetric)
 *   vec_round(x)        = nearest, ties even -> rintf(x) in the default mode
 *
 * (SURVEY.md 8(c) readings G4 tie rule, G5 fused semantics.)  Must be built
 * with -ffp-contract=off and without -ffast-math so that the compiler adds or
 * removes no rounding.  No blocking, fusion or reordering beyond Fig. 1.
 *
 * Parity status: pinned (tests/test_oracle_pins.py); see DESIGN.md "Oracle".
 */
#include "sincos_oracle.h"

#include <math.h>
#include <string.h>

/* ---- coefficients ------------------------------------------------------
 * Restated from the paper as the same decimal strings, converted exactly as
 * Fig. 1 does: a double literal cast to (vector float), i.e. (float)(double). */

/* method 1, "normalised": P:140-148 and Fig. 1 P:244-258 (identical digits). */
static const oracle_coeffs_t COEFFS_N = {
    (float)1.5707963235, (float)-0.645963615, (float)0.0796819754, (float)-0.0046075748,
    (float)-1.2336977925, (float)0.2536086171, (float)-0.0204391631};

/* method 2, "angle-accurate" (dagger): Fig. 1 P:228-242.  ss2 is the Fig. 1
 * value -0.6466386396; the text P:161 prints -0.6466386936.  Reading
 * G1 in DESIGN.md: Fig. 1 wins; the text value is kept as VARIANT_A_TEXT. */
static const oracle_coeffs_t COEFFS_A = {
    (float)1.5707963268, (float)-0.6466386396, (float)0.0679105987, (float)-0.0011573807,
    (float)-1.2341299769, (float)0.2465220241, (float)-0.0123926179};

static const oracle_coeffs_t COEFFS_A_TEXT = {
    (float)1.5707963268, (float)-0.6466386936, (float)0.0679105987, (float)-0.0011573807,
    (float)-1.2341299769, (float)0.2465220241, (float)-0.0123926179};

int oracle_variant_opts(int variant, oracle_opts_t *o)
{
    o->doubling = ORACLE_DOUBLING_EQ1;
    o->doublings = 2; /* "use 2 angle-doublings" */
    switch (variant) {
    case ORACLE_VARIANT_N:        o->coeffs = COEFFS_N;      o->fix = ORACLE_FIX_LINEAR_PENULTIMATE; return 0;
    case ORACLE_VARIANT_A:        o->coeffs = COEFFS_A;      o->fix = ORACLE_FIX_RECIPROCAL;         return 0;
    case ORACLE_VARIANT_A_TEXT:   o->coeffs = COEFFS_A_TEXT; o->fix = ORACLE_FIX_RECIPROCAL;         return 0;
    case ORACLE_VARIANT_N_TEXTFIX:o->coeffs = COEFFS_N;      o->fix = ORACLE_FIX_TEXT_FINAL;         return 0;
    case ORACLE_VARIANT_N_NOFIX:  o->coeffs = COEFFS_N;      o->fix = ORACLE_FIX_NONE;               return 0;
    case ORACLE_VARIANT_A_NOFIX:  o->coeffs = COEFFS_A;      o->fix = ORACLE_FIX_NONE;               return 0;
    case ORACLE_VARIANT_A_LINFIX: o->coeffs = COEFFS_A;      o->fix = ORACLE_FIX_LINEAR_PENULTIMATE; return 0;
    default: return -1;
    }
}

/* ---- A1: turn reduction, P:53-54 ---------------------------------------
 * "the angle is first scaled by 1/2pi and reduced modulo 1 onto [-1/2,1/2)
 * by rounding and subtraction".  Fig. 1 P:270-278:
 *   x1 = vec_madd(v, (vector float)(1.0/(2.0*3.1415926536)), 0.0)
 *   q1 = vec_nmsub(vec_round(x1), 1.0, x1)                                  */
float oracle_reduce_turns(float theta)
{
    const float k = (float)(1.0 / (2.0 * 3.1415926536)); /* P:270, reading G12 */
    float x1 = fmaf(theta, k, 0.0f);
    float q1 = fmaf(-rintf(x1), 1.0f, x1);
    return q1;
}

/* ---- A2: quarter-angle series, P:72-75, P:140-167 -------------------------
 * sin(2 pi x / 4) = x (ss1 + ss2 x^2 + ss3 x^4 + ss4 x^6)
 * cos(2 pi x / 4) = 1 + cc1 x^2 + cc2 x^4 + cc3 x^6
 * Horner, innermost first, Fig. 1 P:280-310.                               */
void oracle_poly_quarter(float q1, const oracle_coeffs_t *k, float *s, float *c)
{
    float q2 = fmaf(q1, q1, 0.0f);
    float ps = fmaf(q2, fmaf(q2, fmaf(q2, k->ss4, k->ss3), k->ss2), k->ss1);
    *s = fmaf(q1, ps, 0.0f);
    *c = fmaf(q2, fmaf(q2, fmaf(q2, k->cc3, k->cc2), k->cc1), 1.0f);
}

/* ---- A3: one angle doubling ----------------------------------------------
 * Eq. (1):  sin 2t = 2 sin t cos t,  cos 2t = cos^2 t - sin^2 t
 * in Fig. 1's order, P:314-318:
 *   c' = vec_nmsub(s, s, vec_madd(c, c, 0))
 *   s' = vec_madd(2.0, vec_madd(s, c, 0), 0)
 * Eq. (2), P:89-91 (rejected, test-only): cos 2t = 1 - 2 sin^2 t.          */
void oracle_double_angle(float s, float c, oracle_doubling_t form, float *s_out, float *c_out)
{
    if (form == ORACLE_DOUBLING_EQ1)
        *c_out = fmaf(-s, s, fmaf(c, c, 0.0f));
    else
        *c_out = fmaf(-2.0f * s, s, 1.0f);
    *s_out = fmaf(2.0f, fmaf(s, c, 0.0f), 0.0f);
}

/* ---- A3 + A6/A7: doublings and amplitude handling -------------------------
 * Fig. 1 P:312-360 for n = 2: one doubling gives the penultimate pair
 * (s2, c2); the factor fixmag1 is taken from it; the second
 * doubling gives the final pair, which is multiplied by fixmag1.
 * For general n ("after n iterations") the penultimate pair is the
 * one after n-1 doublings.                                                  */
void oracle_pair_from_q(float q1, const oracle_opts_t *o, float *s_out, float *c_out)
{
    float s, c, fix = 1.0f;
    oracle_poly_quarter(q1, &o->coeffs, &s, &c);

    for (int i = 0; i < o->doublings; ++i) {
        if (i == o->doublings - 1) {
            /* (s, c) is the penultimate pair here. */
            if (o->fix == ORACLE_FIX_LINEAR_PENULTIMATE)
                fix = fmaf(-s, s, fmaf(-c, c, 2.0f));
            else if (o->fix == ORACLE_FIX_RECIPROCAL)
                fix = 1.0f / fmaf(s, s, fmaf(c, c, 0.0f));     /* IEEE RN divide, reading G3 */
        }
        oracle_double_angle(s, c, o->doubling, &s, &c);
    }

    if (o->fix == ORACLE_FIX_TEXT_FINAL) {
        /* multiply the final pair by 1 - alpha/2 = (3 - s^2 - c^2)/2. */
        fix = fmaf(-s, s, fmaf(-c, c, 3.0f)) * 0.5f;
    } else if (o->fix == ORACLE_FIX_EXACT_FINAL) {
        /* divide the pair by sqrt(1 + alpha), alpha from the final pair. */
        fix = (float)(1.0 / sqrt((double)s * (double)s + (double)c * (double)c));
    }
    *c_out = fmaf(c, fix, 0.0f);
    *s_out = fmaf(s, fix, 0.0f);
}

void oracle_pair(float theta, const oracle_opts_t *o, float *s, float *c)
{
    oracle_pair_from_q(oracle_reduce_turns(theta), o, s, c);
}

int sincos_oracle_opts(const float *theta, float *s_out, float *c_out, size_t n,
                       const oracle_opts_t *o)
{
    for (size_t i = 0; i < n; ++i)
        oracle_pair(theta[i], o, &s_out[i], &c_out[i]);
    return 0;
}

int sincos_oracle(const float *theta, float *s_out, float *c_out, size_t n, int variant)
{
    oracle_opts_t o;
    if (oracle_variant_opts(variant, &o) != 0)
        return -1;
    return sincos_oracle_opts(theta, s_out, c_out, n, &o);
}

/* ---- NEXT(3): any series degrees and doubling count ------------- */
static int method_valid(const oracle_method_t *m)
{
    if (m->n_ss < 1 || m->n_ss > ORACLE_MAX_TERMS || m->n_cc < 0 || m->n_cc > ORACLE_MAX_TERMS)
        return 0;
    if (m->doublings < 0 || m->doublings > 8)
        return 0;
    if (m->fix == ORACLE_FIX_NONE)
        return 1;
    return (m->fix == ORACLE_FIX_LINEAR_PENULTIMATE || m->fix == ORACLE_FIX_RECIPROCAL) && m->doublings >= 1;
}

int oracle_method_pair_from_q(float q1, const oracle_method_t *m, float *s_out, float *c_out)
{
    if (!method_valid(m))
        return -1;
    float q2 = fmaf(q1, q1, 0.0f);
    float ps = m->ss[m->n_ss - 1];                       /* Horner, innermost first */
    for (int i = m->n_ss - 2; i >= 0; --i)
        ps = fmaf(q2, ps, m->ss[i]);
    float s = fmaf(q1, ps, 0.0f);
    float c = 1.0f;
    if (m->n_cc > 0) {
        float pc = m->cc[m->n_cc - 1];
        for (int i = m->n_cc - 2; i >= 0; --i)
            pc = fmaf(q2, pc, m->cc[i]);
        c = fmaf(q2, pc, 1.0f);
    }
    float fix = 1.0f;
    for (int i = 0; i < m->doublings; ++i) {
        if (i == m->doublings - 1) {                     /* the penultimate pair */
            if (m->fix == ORACLE_FIX_LINEAR_PENULTIMATE)
                fix = fmaf(-s, s, fmaf(-c, c, 2.0f));
            else if (m->fix == ORACLE_FIX_RECIPROCAL)
                fix = 1.0f / fmaf(s, s, fmaf(c, c, 0.0f));
        }
        oracle_double_angle(s, c, ORACLE_DOUBLING_EQ1, &s, &c);
    }
    *c_out = fmaf(c, fix, 0.0f);
    *s_out = fmaf(s, fix, 0.0f);
    return 0;
}

int oracle_method_sincos(const float *theta, float *s_out, float *c_out, size_t n,
                         const oracle_method_t *m)
{
    if (!method_valid(m))
        return -1;
    for (size_t i = 0; i < n; ++i)
        oracle_method_pair_from_q(oracle_reduce_turns(theta[i]), m, &s_out[i], &c_out[i]);
    return 0;
}

/* ---- NEXT(1): phases generated from their factors ----
 * The pair for the phase of frequency f and time t.  The phase is formed as
 * one rounded fp32 product p = RN(f * t).  units == 0: p is the angle in
 * radians and the whole method runs (A1 onwards).  units == 1: p is
 * already in turns (theta / 2pi), so the method enters at the reduction
 * "reduced modulo 1 onto [-1/2,1/2) by rounding and subtraction" and
 * skips the scale by 1/2pi (Fig. 1) and its rounding. */
void oracle_phase_pair(float f, float t, int units, const oracle_opts_t *o, float *s, float *c)
{
    float p = fmaf(f, t, 0.0f);
    if (units == 0) {
        oracle_pair(p, o, s, c);
    } else {
        float q1 = fmaf(-rintf(p), 1.0f, p);
        oracle_pair_from_q(q1, o, s, c);
    }
}

int oracle_phase_points(const float *f, const float *t, size_t m, int units, int variant,
                        float *s_out, float *c_out)
{
    oracle_opts_t o;
    if (oracle_variant_opts(variant, &o) != 0 || (units != 0 && units != 1))
        return -1;
    for (size_t k = 0; k < m; ++k)
        oracle_phase_pair(f[k], t[k], units, &o, &s_out[k], &c_out[k]);
    return 0;
}

/* ---- NEXT(2): the consumer of the pairs -- a direct non-uniform Fourier / Huygens sum
 * ("rapid computation of optical diffraction patterns via Huygens'
 * principle"):
 *     F_k = sum_j a_j (cos p_kj + i sin p_kj),   p_kj = RN(f_k t_j)
 * with the pairs of oracle_phase_pair (radians or turns) and the complex products
 * and the sum in double (the plain definition; a = interleaved {re, im} float
 * pairs, out = interleaved {re, im} doubles). */
int oracle_nudft(const float *f, size_t nf, const float *t, const float *a, size_t nt, int units,
                 int variant, double *out)
{
    oracle_opts_t o;
    if (oracle_variant_opts(variant, &o) != 0 || (units != 0 && units != 1))
        return -1;
    for (size_t k = 0; k < nf; ++k) {
        double re = 0.0, im = 0.0;
        for (size_t j = 0; j < nt; ++j) {
            float s, c;
            oracle_phase_pair(f[k], t[j], units, &o, &s, &c);
            const double ar = a[2 * j], ai = a[2 * j + 1];
            re += ar * (double)c - ai * (double)s;
            im += ar * (double)s + ai * (double)c;
        }
        out[2 * k] = re;
        out[2 * k + 1] = im;
    }
    return 0;
}

/* Row-major grid: element (i, j) at i*nt + j is the pair of phase f[i] * t[j]. */
int oracle_phase_grid(const float *f, size_t nf, const float *t, size_t nt, int units, int variant,
                      float *s_out, float *c_out)
{
    oracle_opts_t o;
    if (oracle_variant_opts(variant, &o) != 0 || (units != 0 && units != 1))
        return -1;
    for (size_t i = 0; i < nf; ++i)
        for (size_t j = 0; j < nt; ++j)
            oracle_phase_pair(f[i], t[j], units, &o, &s_out[i * nt + j], &c_out[i * nt + j]);
    return 0;
}
