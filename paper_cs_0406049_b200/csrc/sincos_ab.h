/*
 * sincos_ab.h -- the extra entry points of the A/B build, libsincos_pairs_ab.so (built from
 * the same sources with -DSINCOS_AB; loaded by tests/ and tools/ only).  NOT part of the
 * product library's ABI (include/sincos_pairs.h): the product has one kernel configuration,
 * fixed, and no process-global state that changes what another caller gets.
 *
 * sincos_ab_set(knob, value): select a kernel form or launch shape for the measurements and
 * parity tests of the alternatives; process-global; returns the previous
 * value, or -1 for an unknown knob or unsupported value.  sincos_ab_get(knob): the value (-1
 * for an unknown knob).  Defaults = the product's configuration (sincos_launch.h Tuning).
 *
 * sincos_pairs_batched: many independent arrays in one launch (the item table in the kernel's
 * parameter block, one launch per 480 items); numerics identical to sincos_pairs.  Outside
 * kept for measurement, not shipped.
 */
#ifndef SINCOS_AB_H
#define SINCOS_AB_H

#include "../../include/sincos_pairs.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SINCOS_AB_THREADS = 0,       /* 128, 256, 512                                              */
    SINCOS_AB_BLOCKS_PER_SM = 1, /* 0 = full grid; 1..4096 = grid-stride grid of SMs x this    */
    SINCOS_AB_VEC = 2,           /* 4 or 8 floats per access                                   */
    SINCOS_AB_UNROLL = 3,        /* 1, 2, 4                                                    */
    SINCOS_AB_PREFETCH = 4,      /* 0, 1                                                       */
    SINCOS_AB_REALIGN = 5,       /* 1 re-align; 0 one per thread; 2 128-bit form; 3 flat phase */
    SINCOS_AB_PDL = 6,           /* 0, 1                                                       */
    SINCOS_AB_NUDFT_PACKED = 7,  /* 0 (scalar twins), 1                                        */
    SINCOS_AB_KNOBS = 8
} sincos_ab_knob_t;

SINCOS_API int sincos_ab_set(int knob, int value);
SINCOS_API int sincos_ab_get(int knob);

typedef struct {
    const float *theta_dev;
    float *sin_dev, *cos_dev, *inter_dev;
    uint64_t n;
} sincos_item_t;
SINCOS_API sincos_status_t sincos_pairs_batched(const sincos_item_t *items, int count, sincos_variant_t variant,
                                                void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SINCOS_AB_H */
