/*
 * libm_baseline.c -- context for the CPU baseline (SURVEY 8(d) optional row
 * "libm-baseline"): glibc's sincosf over an array, the same input/output traffic as the
 * method.  Not the paper's method and not the oracle; bench.py times it beside the oracle.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stddef.h>

void libm_sincosf_array(const float *theta, float *s, float *c, size_t n) {
    for (size_t i = 0; i < n; ++i) sincosf(theta[i], &s[i], &c[i]);
}
