/*
 * gen.c -- seeded synthetic input generators for the five BASELINE.json
 * configs.
 *
 * This module is shared by the oracle side (tests) and the product side
 * (bench, GPU tests) and therefore holds NONE of the method's arithmetic:
 * only a counter-based random number generator and the configs' value
 * distributions.  Every element is a pure function of (config, index), so
 * any index range or index sample can be generated independently and the
 * result never depends on the thread count.
 *
 *   mix64(x)          = SplitMix64 finalizer with the 0x9E3779B97F4A7C15 pre-add
 *   u(seed, stream, i) = (mix64(seed<<48 ^ stream<<40 ^ i) >> 11) * 2^-53  in [0, 1)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline double urand(uint64_t seed, uint64_t stream, uint64_t i)
{
    return (double)(mix64((seed << 48) ^ (stream << 40) ^ i) >> 11) * 0x1.0p-53;
}

static inline float bits2f(uint32_t u)
{
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static inline uint32_t f2bits(float f)
{
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

static inline float with_sign(float x, double u)
{
    return u < 0.5 ? -x : x;
}

/* Config ids: 1..5 = BASELINE.json configs[0..4]; 0 = raw fp32 bit patterns
 * (theta_i = bits(i), for whole-input-space sweeps). */
static inline float gen_one(int config, uint64_t i)
{
    switch (config) {
    case 0:
        return bits2f((uint32_t)i);
    case 1: /* C1: U[-pi, pi), seed 0 */
        return (float)(-M_PI + 2.0 * M_PI * urand(0, 0, i));
    case 2: /* C2: U[-1e4, 1e4], seed 1 */
        return (float)(-1e4 + 2e4 * urand(1, 0, i));
    case 3: { /* C3: edge / stress set, seed 2; 16 categories interleaved by index */
        int k = (int)(16.0 * urand(2, 0, i));
        double u1 = urand(2, 1, i), u2 = urand(2, 2, i), u3 = urand(2, 3, i);
        if (k <= 1) { /* exact multiples of pi/2 (as rounded to fp32) */
            double m = floor(u1 * 80001.0) - 40000.0;
            return (float)(m * (M_PI / 2.0));
        }
        if (k == 2) { /* multiples of pi */
            double m = floor(u1 * 40001.0) - 20000.0;
            return (float)(m * M_PI);
        }
        if (k <= 6) { /* within 64 ulp of (2n+1) pi, n <= 1e4: the wrap seam */
            double n = floor(u1 * 10001.0);
            float base = (float)((2.0 * n + 1.0) * M_PI);
            int32_t off = (int32_t)floor(u2 * 129.0) - 64;
            return with_sign(bits2f((uint32_t)((int32_t)f2bits(base) + off)), u3);
        }
        if (k == 7) /* signed zeros */
            return with_sign(0.0f, u3);
        if (k <= 9) { /* subnormals */
            uint32_t b = 1u + (uint32_t)(u1 * 8388607.0);
            return with_sign(bits2f(b), u3);
        }
        /* log-uniform magnitudes in [1e-30, 2^20) */
        double lo = log(1e-30), hi = log(1048576.0);
        return with_sign((float)exp(lo + (hi - lo) * u1), u3);
    }
    case 4: { /* C4: NUFFT-style phases theta_ij = 2 pi f_i t_j, 2^15 x 2^15, seed 3 */
        uint64_t r = i >> 15, j = i & 0x7FFFu;
        double f = 512.0 * urand(3, 0, r);
        double t = ((double)j + urand(3, 1, j)) * 0x1.0p-15;
        return (float)((2.0 * M_PI * f) * t);
    }
    case 5: { /* C5: normal, mean 0, sigma 100 rad (Box-Muller), seed 4 */
        double z = sqrt(-2.0 * log(1.0 - urand(4, 0, i))) * cos(2.0 * M_PI * urand(4, 1, i));
        return (float)(100.0 * z);
    }
    default:
        return NAN;
    }
}

/* Number of elements of each config (BASELINE.json configs). */
uint64_t sincos_gen_size(int config)
{
    switch (config) {
    case 0: return 1ull << 32;
    case 1: return 1ull << 20;
    case 2: return 1ull << 28;
    case 3: return 1ull << 24;
    case 4: return 1ull << 30;
    case 5: return 1ull << 32;
    default: return 0;
    }
}

/* out[k] = element (start + k) of `config`, k < count.  Returns 0 or -1. */
int sincos_gen_range(int config, uint64_t start, uint64_t count, float *out, int nthreads)
{
    if (config < 0 || config > 5)
        return -1;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t k = 0; k < (int64_t)count; ++k)
        out[k] = gen_one(config, start + (uint64_t)k);
    return 0;
}

/* out[k] = element idx[k] of `config`, k < m.  Returns 0 or -1. */
int sincos_gen_at(int config, const uint64_t *idx, uint64_t m, float *out)
{
    if (config < 0 || config > 5)
        return -1;
    for (uint64_t k = 0; k < m; ++k)
        out[k] = gen_one(config, idx[k]);
    return 0;
}

/* The raw generator, exposed for its own tests. */
double sincos_gen_urand(uint64_t seed, uint64_t stream, uint64_t i)
{
    return urand(seed, stream, i);
}
