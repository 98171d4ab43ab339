/*
 * accuracy.c -- ORACLE error metrics and sweeps (test infrastructure only).
 *
 * The error metrics are the paper's, P:135-139:
 *   combined  = sqrt((cos - ref_cos)^2 + (sin - ref_sin)^2)
 *   amplitude = 1 - sqrt(cos^2 + sin^2)
 * "where the reference functions are computed to double precision using the
 * standard system library calls".  A long-double reference
 * (sinl/cosl) is offered as the stricter cross-check BASELINE.json asks for.
 *
 * The sweeps and the whole-input-space hash are test drivers around
 * oracle_pair(); they parallelise over fixed chunks (OpenMP) and combine the
 * chunks in index order so results never depend on the thread count.
 */
#include "sincos_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void stats_init(oracle_stats_t *st)
{
    memset(st, 0, sizeof(*st));
}

static inline uint32_t f2u(float f)
{
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

static inline float u2f(uint32_t u)
{
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* Accumulate one element.  x is the argument reported as worst_x. */
static inline void stats_add(oracle_stats_t *st, float x, float s, float c, double rs, double rc,
                             long double rsl, long double rcl, int ref_kind)
{
    if (isnan(s) || isnan(c)) {
        st->nan_count++;
        return;
    }
    double comb;
    if (ref_kind == ORACLE_REF_LONGDOUBLE) {
        long double dc = (long double)c - rcl, ds = (long double)s - rsl;
        comb = (double)sqrtl(dc * dc + ds * ds);
    } else {
        double dc = (double)c - rc, ds = (double)s - rs;
        comb = sqrt(dc * dc + ds * ds);
    }
    double amp = 1.0 - sqrt((double)c * (double)c + (double)s * (double)s);
    st->count++;
    st->sum_sq += comb * comb;
    st->sum_s += (double)s;
    st->sum_c += (double)c;
    if (comb > st->max_comb) {
        st->max_comb = comb;
        st->worst_x = x;
        st->worst_bits = f2u(x);
    }
    if (fabs(amp) > st->max_amp) {
        st->max_amp = fabs(amp);
        st->amp_signed = amp;
    }
}

/* Reference pair for argument a (radians) in the requested precision. */
static inline void ref_pair(double a, long double al, int ref_kind, double *rs, double *rc,
                            long double *rsl, long double *rcl)
{
    if (ref_kind == ORACLE_REF_LONGDOUBLE) {
        *rsl = sinl(al);
        *rcl = cosl(al);
        *rs = (double)*rsl;
        *rc = (double)*rcl;
    } else {
        *rs = sin(a);
        *rc = cos(a);
        *rsl = *rs;
        *rcl = *rc;
    }
}

void oracle_error_stats(const float *theta, const float *s, const float *c, size_t n,
                        int ref_kind, oracle_stats_t *st)
{
    stats_init(st);
    for (size_t i = 0; i < n; ++i) {
        double rs, rc;
        long double rsl, rcl;
        ref_pair((double)theta[i], (long double)theta[i], ref_kind, &rs, &rc, &rsl, &rcl);
        stats_add(st, theta[i], s[i], c[i], rs, rc, rsl, rcl, ref_kind);
    }
}

void oracle_error_stats_interleaved(const float *theta, const float *cs, size_t n,
                                    int ref_kind, oracle_stats_t *st)
{
    stats_init(st);
    for (size_t i = 0; i < n; ++i) {
        double rs, rc;
        long double rsl, rcl;
        ref_pair((double)theta[i], (long double)theta[i], ref_kind, &rs, &rc, &rsl, &rcl);
        stats_add(st, theta[i], cs[2 * i + 1], cs[2 * i], rs, rc, rsl, rcl, ref_kind);
    }
}

void oracle_grid_stats(const oracle_opts_t *o, uint64_t m, int ref_kind, oracle_stats_t *st)
{
    stats_init(st);
    for (uint64_t k = 0; k < m; ++k) {
        float theta = (float)(-M_PI + ((2 * M_PI) * (double)k) / (double)m);
        float s, c;
        oracle_pair(theta, o, &s, &c);
        double rs, rc;
        long double rsl, rcl;
        ref_pair((double)theta, (long double)theta, ref_kind, &rs, &rc, &rsl, &rcl);
        stats_add(st, theta, s, c, rs, rc, rsl, rcl, ref_kind);
    }
}

/* Merge b into a; a covers lower indices than b (lowest-index argmax wins). */
static void stats_merge(oracle_stats_t *a, const oracle_stats_t *b)
{
    a->count += b->count;
    a->nan_count += b->nan_count;
    a->sum_sq += b->sum_sq;
    a->sum_s += b->sum_s;
    a->sum_c += b->sum_c;
    if (b->max_comb > a->max_comb) {
        a->max_comb = b->max_comb;
        a->worst_x = b->worst_x;
        a->worst_bits = b->worst_bits;
    }
    if (b->max_amp > a->max_amp) {
        a->max_amp = b->max_amp;
        a->amp_signed = b->amp_signed;
    }
}

#define SWEEP_CHUNK (1u << 20)

void oracle_sweep_bits(const oracle_opts_t *o, int mode, uint32_t lo_bits, uint32_t hi_bits,
                       int nthreads, oracle_stats_t *st)
{
    uint64_t total = (uint64_t)hi_bits - lo_bits + 1;
    uint64_t nchunks = (total + SWEEP_CHUNK - 1) / SWEEP_CHUNK;
    oracle_stats_t *part = (oracle_stats_t *)calloc(nchunks, sizeof(oracle_stats_t));
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t ch = 0; ch < (int64_t)nchunks; ++ch) {
        oracle_stats_t *p = &part[ch];
        stats_init(p);
        uint64_t b0 = (uint64_t)lo_bits + (uint64_t)ch * SWEEP_CHUNK;
        uint64_t b1 = b0 + SWEEP_CHUNK;
        if (b1 > (uint64_t)hi_bits + 1)
            b1 = (uint64_t)hi_bits + 1;
        for (uint64_t b = b0; b < b1; ++b) {
            float x = u2f((uint32_t)b);
            float s, c;
            double rs, rc;
            long double rsl, rcl;
            if (mode == 0) {
                oracle_pair(x, o, &s, &c);
                ref_pair((double)x, (long double)x, ORACLE_REF_DOUBLE, &rs, &rc, &rsl, &rcl);
            } else {
                /* kernel-only: the pipeline from q, vs sin/cos(2 pi q) */
                oracle_pair_from_q(x, o, &s, &c);
                ref_pair(2.0 * M_PI * (double)x, 0.0L, ORACLE_REF_DOUBLE, &rs, &rc, &rsl, &rcl);
            }
            stats_add(p, x, s, c, rs, rc, rsl, rcl, ORACLE_REF_DOUBLE);
        }
    }
    stats_init(st);
    for (uint64_t ch = 0; ch < nchunks; ++ch)
        stats_merge(st, &part[ch]);
    free(part);
}

/* NEXT(3): kernel-only stats of a general method over fp32 q = bits(u), u = lo, lo+stride, ...
 * <= hi, vs sin/cos(2 pi q) in double.  Fixed chunks merged in order (thread-count independent). */
void oracle_method_sweep_q(const oracle_method_t *m, uint32_t lo_bits, uint32_t hi_bits, uint32_t stride,
                           int nthreads, oracle_stats_t *st)
{
    if (stride == 0)
        stride = 1;
    uint64_t total = ((uint64_t)hi_bits - lo_bits) / stride + 1;
    uint64_t nchunks = (total + SWEEP_CHUNK - 1) / SWEEP_CHUNK;
    oracle_stats_t *part = (oracle_stats_t *)calloc(nchunks, sizeof(oracle_stats_t));
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t ch = 0; ch < (int64_t)nchunks; ++ch) {
        oracle_stats_t *p = &part[ch];
        stats_init(p);
        uint64_t k0 = (uint64_t)ch * SWEEP_CHUNK, k1 = k0 + SWEEP_CHUNK;
        if (k1 > total)
            k1 = total;
        for (uint64_t k = k0; k < k1; ++k) {
            float x = u2f((uint32_t)(lo_bits + k * stride));
            float s, c;
            double rs, rc;
            long double rsl, rcl;
            oracle_method_pair_from_q(x, m, &s, &c);
            ref_pair(2.0 * M_PI * (double)x, 0.0L, ORACLE_REF_DOUBLE, &rs, &rc, &rsl, &rcl);
            stats_add(p, x, s, c, rs, rc, rsl, rcl, ORACLE_REF_DOUBLE);
        }
    }
    stats_init(st);
    for (uint64_t ch = 0; ch < nchunks; ++ch)
        stats_merge(st, &part[ch]);
    free(part);
}

/* SplitMix64 finalizer with its additive pre-step (SURVEY 8(c) hash definition). */
static inline uint64_t hash_mix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint32_t canon_bits(float f)
{
    if (isnan(f))
        return 0x7FC00000u;
    if (f == 0.0f)
        return 0u;
    return f2u(f);
}

static inline uint64_t hash_term(uint64_t u, float s, float c)
{
    uint64_t key = ((uint64_t)canon_bits(s) << 32) | (uint64_t)canon_bits(c);
    return hash_mix64(key ^ (u * 0xD6E8FEB86659FD93ull));
}

void oracle_hash_bits(const oracle_opts_t *o, uint32_t lo_bits, uint32_t hi_bits, int nthreads,
                      uint64_t *hash, uint64_t *nan_pairs, uint64_t *exact_01)
{
    uint64_t h = 0, nn = 0, ex = 0;
    int64_t lo = lo_bits, hi = hi_bits;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static) reduction(+ : h, nn, ex)
#endif
    for (int64_t b = lo; b <= hi; ++b) {
        float s, c;
        oracle_pair(u2f((uint32_t)b), o, &s, &c);
        h += hash_term((uint64_t)b, s, c);
        nn += (isnan(s) || isnan(c)) ? 1 : 0;
        ex += (s == 0.0f && c == 1.0f) ? 1 : 0;
    }
    *hash = h;
    *nan_pairs = nn;
    *exact_01 = ex;
}

uint64_t oracle_hash_outputs(const float *s, const float *c, const float *cs, size_t n,
                             uint32_t first_bits)
{
    uint64_t h = 0;
    for (size_t i = 0; i < n; ++i) {
        float si = cs ? cs[2 * i + 1] : s[i];
        float ci = cs ? cs[2 * i] : c[i];
        h += hash_term((uint64_t)first_bits + i, si, ci);
    }
    return h;
}
