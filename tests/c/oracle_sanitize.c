/*
 * oracle_sanitize.c -- the host C code (the oracle and the input generators) under
 * AddressSanitizer + UndefinedBehaviorSanitizer (sanitizers; test driver, CPU).
 *
 * Calls every oracle entry point and every input generator on small buffers sized exactly
 * (so an overrun is an ASan report), including the degenerate shapes (n = 0, nt = 0, one
 * element) and special values (NaN, +-Inf, +-0, subnormals, huge), and checks a few
 * closed forms.  Exit 0 and no sanitizer report = pass.  Built and run by
 * tests/test_sanitize_host.py with -fsanitize=address,undefined -fno-sanitize-recover=all.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../oracle/sincos_oracle.h"

uint64_t sincos_gen_size(int config);
int sincos_gen_range(int config, uint64_t start, uint64_t count, float *out, int nthreads);
int sincos_gen_at(int config, const uint64_t *idx, uint64_t m, float *out);

static float *fbuf(size_t n) { return (float *)malloc(n ? n * sizeof(float) : 1); }

int main(void) {
    int fails = 0;
    const float special[] = {0.0f, -0.0f, 1e-45f, -1e-40f, 1e-30f, 0.5f, 3.14159265f, 1e4f, 2.6e8f, 1e30f,
                             3.4e38f, INFINITY, -INFINITY, NAN};
    const size_t ns = sizeof special / sizeof special[0];
    for (int v = 0; v < 7; ++v) {
        float *s = fbuf(ns), *c = fbuf(ns);
        if (sincos_oracle(special, s, c, ns, v) != 0) { fprintf(stderr, "variant %d\n", v); ++fails; }
        free(s);
        free(c);
        oracle_opts_t o;
        if (oracle_variant_opts(v, &o) != 0) continue;
        float s1, c1;
        oracle_pair(0.0f, &o, &s1, &c1);
        if (!(s1 == 0.0f && c1 == 1.0f)) { fprintf(stderr, "pair(0) v=%d\n", v); ++fails; }
        for (size_t i = 0; i < ns; ++i) oracle_pair_from_q(oracle_reduce_turns(special[i]), &o, &s1, &c1);
    }
    if (sincos_oracle(special, NULL, NULL, 0, 0) != 0) ++fails;            /* n = 0 */
    /* general method */
    oracle_method_t m;
    memset(&m, 0, sizeof m);
    m.ss[0] = 1.5707963f; m.ss[1] = -0.6459636f; m.ss[2] = 0.0796820f; m.ss[3] = -0.0046076f; m.n_ss = 4;
    m.cc[0] = -1.2336978f; m.cc[1] = 0.2536086f; m.cc[2] = -0.0204392f; m.n_cc = 3;
    m.doublings = 2; m.fix = 0;
    {
        float *s = fbuf(ns), *c = fbuf(ns);
        if (oracle_method_sincos(special, s, c, ns, &m) != 0) ++fails;
        m.n_ss = 8; m.n_cc = 8; m.doublings = 8; m.fix = 1;
        if (oracle_method_sincos(special, s, c, ns, &m) != 0) ++fails;
        m.n_ss = 9;
        if (oracle_method_sincos(special, s, c, ns, &m) == 0) ++fails;  /* invalid: rejected */
        free(s);
        free(c);
    }
    /* phase pairs, grid, fused sum (nt = 0 and 1 included) */
    {
        const float f[] = {0.0f, 1.0f, 3.25f, 511.9f, NAN};
        const float t[] = {0.0f, 0.25f, 0.5f, 0.999f, 1e-40f, -2.0f, INFINITY};
        const size_t nf = 5, nt = 7;
        float *s = fbuf(nf * nt), *c = fbuf(nf * nt);
        for (int units = 0; units < 2; ++units)
            for (int v = 0; v < 2; ++v) {
                if (oracle_phase_grid(f, nf, t, nt, units, v, s, c) != 0) ++fails;
                if (oracle_phase_points(f, t, nf, units, v, s, c) != 0) ++fails;
                float *a = fbuf(2 * nt);
                for (size_t j = 0; j < 2 * nt; ++j) a[j] = (float)(j % 3) - 1.0f;
                double *out = (double *)malloc(2 * nf * sizeof(double));
                if (oracle_nudft(f, nf, t, a, nt, units, v, out) != 0) ++fails;
                if (oracle_nudft(f, nf, t, a, 0, units, v, out) != 0) ++fails;
                if (out[0] != 0.0 || out[1] != 0.0) ++fails;                  /* empty sum */
                if (oracle_nudft(f, nf, t, a, 1, units, v, out) != 0) ++fails;
                free(a);
                free(out);
            }
        free(s);
        free(c);
    }
    /* error statistics, hashes, sweeps (small ranges) */
    {
        float *s = fbuf(ns), *c = fbuf(ns), *cs = fbuf(2 * ns);
        sincos_oracle(special, s, c, ns, 0);
        for (size_t i = 0; i < ns; ++i) { cs[2 * i] = c[i]; cs[2 * i + 1] = s[i]; }
        oracle_stats_t st;
        oracle_error_stats(special, s, c, ns, 0, &st);
        oracle_error_stats(special, s, c, ns, 1, &st);
        oracle_error_stats_interleaved(special, cs, ns, 0, &st);
        oracle_error_stats(special, s, c, 0, 0, &st);
        if (oracle_hash_outputs(s, c, NULL, ns, 0u) != oracle_hash_outputs(NULL, NULL, cs, ns, 0u)) ++fails;
        oracle_opts_t o;
        oracle_variant_opts(0, &o);
        oracle_grid_stats(&o, 4096, 0, &st);
        oracle_sweep_bits(&o, 0, 0x3F000000u, 0x3F000FFFu, 2, &st);
        oracle_sweep_bits(&o, 1, 0x3E000000u, 0x3E000FFFu, 2, &st);
        uint64_t h, nn, ex;
        oracle_hash_bits(&o, 0x7F7FFF00u, 0x7FFFFFFFu, 2, &h, &nn, &ex);   /* top range: inf/NaN */
        m.n_ss = 4; m.n_cc = 3; m.doublings = 2; m.fix = 0;
        oracle_method_sweep_q(&m, 0x3E000000u, 0x3E00FFFFu, 17, 2, &st);
        free(s);
        free(c);
        free(cs);
    }
    /* input generators: every config, exact-size buffers, ranges and gathers */
    for (int cfg = 1; cfg <= 5; ++cfg) {
        const uint64_t n = 1000;
        float *x = fbuf(n);
        if (sincos_gen_range(cfg, sincos_gen_size(cfg) - n, n, x, 2) != 0) ++fails;   /* the last n */
        if (sincos_gen_range(cfg, 0, 0, x, 1) != 0) ++fails;
        uint64_t idx[3] = {0, 12345, sincos_gen_size(cfg) - 1};
        if (sincos_gen_at(cfg, idx, 3, x) != 0) ++fails;
        free(x);
    }
    if (fails) fprintf(stderr, "%d failures\n", fails);
    printf("oracle_sanitize: %s\n", fails ? "FAIL" : "ok");
    return fails ? 1 : 0;
}
