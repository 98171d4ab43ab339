"""NEXT(3): regenerate quarter-angle series coefficients for any doubling count and degree.

The paper fits its coefficients two ways:
  method 1 ("normalised"): least-squares series for sine and cosine directly, so the raw
           pair has a small magnitude error, later fixed linearly;
  method 2 ("angle-accurate", dagger): fit the *angle* arctan(S/C) of the raw pair to the
           input angle; the magnitude is then divided out exactly.
With n doublings the series must approximate the angle 2 pi x / 2^n for the
reduced turn x in [-1/2, 1/2] (n = 2: pi x / 2, "theta/4").  Series form (Fig. 1):
  S(x) = x (ss[0] + ss[1] x^2 + ... ),  C(x) = 1 + x^2 (cc[0] + cc[1] x^2 + ...).
The paper states neither grid nor weighting (reading in DESIGN.md section 11): here a
uniform grid on [0, 1/2] (both series have a symmetry) and least squares in double; the
fitted coefficients are returned in double and rounded to fp32 by the caller.

This module only computes coefficients (host-side numpy); the method itself runs in the
library's kernel (sincos_pairs_method), and the fitted tables are inputs to it.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Fit:
    ss: np.ndarray          # odd-series coefficients (double)
    cc: np.ndarray          # even-series coefficients (double), constant 1 implied
    doublings: int
    kind: str               # "normalized" or "angle"
    residual_rms: float     # rms of the fit objective on the grid

    def fp32(self):
        return self.ss.astype(np.float32), self.cc.astype(np.float32)


def _grid(points: int):
    return np.linspace(0.0, 0.5, points)


def fit_normalized(doublings: int = 2, n_ss: int = 4, n_cc: int = 3, points: int = 4097,
                   weight: str = "uniform") -> Fit:
    """Method 1: independent linear least squares for sin and cos of the scaled
    angle a = 2 pi x / 2^n.  weight = "uniform" (absolute error) or "relative" (sine error
    relative to sin a)."""
    x = _grid(points)[1:]
    a = 2 * np.pi * x / 2 ** doublings
    # odd series: x * sum ss_i x^{2i} ~ sin a
    A = np.stack([x ** (2 * i + 1) for i in range(n_ss)], axis=1)
    b = np.sin(a)
    if weight == "relative":
        w = 1 / np.abs(b)
        A, b = A * w[:, None], b * w
    ss = np.linalg.lstsq(A, b, rcond=None)[0]
    # even series: x^2 * sum cc_i x^{2i} ~ cos a - 1
    B = np.stack([x ** (2 * i + 2) for i in range(n_cc)], axis=1)
    d = np.cos(a) - 1
    cc = np.linalg.lstsq(B, d, rcond=None)[0] if n_cc else np.zeros(0)
    res = np.concatenate([A @ ss - b, (B @ cc - d) if n_cc else d])
    return Fit(ss, cc, doublings, "normalized", float(np.sqrt(np.mean(res ** 2))))


def angle_residual(ss, cc, doublings: int, x: np.ndarray) -> np.ndarray:
    """atan2(S(x), C(x)) - 2 pi x / 2^n: the method-2 objective."""
    x2 = x * x
    S = x * np.polyval(np.asarray(ss, dtype=np.float64)[::-1], x2)
    C = 1 + x2 * np.polyval(np.asarray(cc, dtype=np.float64)[::-1], x2) if len(cc) else np.ones_like(x)
    return np.arctan2(S, C) - 2 * np.pi * x / 2 ** doublings


def fit_angle(doublings: int = 2, n_ss: int = 4, n_cc: int = 3, points: int = 4097, iters: int = 100,
              tol: float = 1e-15, free=None, start: Fit | None = None) -> Fit:
    """Method 2: Gauss-Newton on the angle residual, seeded from method 1.
    `free` optionally restricts which coefficients move: a list of ("ss"|"cc", index)."""
    x = _grid(points)[1:]
    seed = start or fit_normalized(doublings, n_ss, n_cc, points)
    ss, cc = seed.ss.copy(), seed.cc.copy()
    params = [("ss", i) for i in range(n_ss)] + [("cc", i) for i in range(n_cc)]
    if free is not None:
        params = list(free)
    x2 = x * x
    prev = None
    for _ in range(iters):
        S = x * np.polyval(ss[::-1], x2)
        C = 1 + x2 * np.polyval(cc[::-1], x2) if n_cc else np.ones_like(x)
        r = np.arctan2(S, C) - 2 * np.pi * x / 2 ** doublings
        den = S * S + C * C
        cols = []
        for kind, i in params:
            if kind == "ss":
                cols.append((C / den) * x ** (2 * i + 1))       # d atan2 / dS * dS / dss_i
            else:
                cols.append((-S / den) * x ** (2 * i + 2))      # d atan2 / dC * dC / dcc_i
        J = np.stack(cols, axis=1)
        step = np.linalg.lstsq(J, -r, rcond=None)[0]
        for (kind, i), dv in zip(params, step):
            (ss if kind == "ss" else cc)[i] += dv
        obj = float(np.sqrt(np.mean(r ** 2)))
        if prev is not None and abs(prev - obj) < tol:
            break
        prev = obj
    r = angle_residual(ss, cc, doublings, x)
    return Fit(ss, cc, doublings, "angle", float(np.sqrt(np.mean(r ** 2))))
