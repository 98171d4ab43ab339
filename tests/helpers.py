"""Test helpers: the threaded oracle runner and value-equality comparison."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle

ULP4 = 4 * 2.0 ** -23   # north_star tolerance: |delta| <= 4 fp32 ulp of 1.0 per component


def oracle_threaded(theta: np.ndarray, variant: int, threads: int | None = None, chunk: int = 1 << 22):
    """The oracle over a large array, chunked over host threads (ctypes releases the GIL;
    numerics are per element, so identical to one plain call)."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    s = np.empty_like(theta)
    c = np.empty_like(theta)
    n = theta.size
    threads = threads or os.cpu_count() or 1
    spans = [(i, min(i + chunk, n)) for i in range(0, n, chunk)]
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda ab: oracle.sincos_into(theta[ab[0]:ab[1]], s[ab[0]:ab[1]], c[ab[0]:ab[1]], variant),
                    spans))
    return s, c


def same_values(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """Element-wise equality by value (+0 == -0), NaN matching NaN (payloads differ)."""
    return (got == want) | (np.isnan(got) & np.isnan(want))


def assert_parity(got_s, got_c, want_s, want_c, what=""):
    """Bit-exact by value, and (the north_star bound) |delta| <= 4 ulp of 1.0 per component."""
    for g, w, comp in ((got_s, want_s, "sin"), (got_c, want_c, "cos")):
        ok = same_values(g, w)
        if not ok.all():
            bad = np.flatnonzero(~ok)
            i = bad[0]
            raise AssertionError(f"{what} {comp}: {bad.size} mismatches, first at {i}: got {g[i]!r} want {w[i]!r}")
        fin = np.isfinite(w)
        if fin.any():
            assert np.max(np.abs(g[fin].astype(np.float64) - w[fin])) <= ULP4
