"""ORACLE -- test infrastructure only.

A plain, slow, obviously-correct CPU transcription (C99, ``sincos_oracle.c``)
of Mendenhall, arXiv cs/0406049, plus the paper's error metrics
(``accuracy.c``), wrapped with ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_cs_0406049_b200``) never imports it and shares no code
with it.  Parity status per function: see DESIGN.md "Oracle and its pins"
(all functions pinned; the paper's exact *max* figures are sampling-dependent,
reading G11).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, f) for f in ("sincos_oracle.c", "accuracy.c")]
_HDR = os.path.join(_HERE, "sincos_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

VARIANT_N = 0          # method 1, "normalised", Fig. 1 FASTER_SINCOS
VARIANT_A = 1          # method 2, "angle-accurate", Fig. 1 ss2
VARIANT_A_TEXT = 2     # test-only: method 2 with the text's ss2
VARIANT_N_TEXTFIX = 3  # test-only: method 1 with the text's final-pair fix
VARIANT_N_NOFIX = 4    # test-only
VARIANT_A_NOFIX = 5    # test-only
VARIANT_A_LINFIX = 6   # test-only

FIX_LINEAR_PENULTIMATE, FIX_RECIPROCAL, FIX_TEXT_FINAL, FIX_NONE, FIX_EXACT_FINAL = range(5)
DOUBLING_EQ1, DOUBLING_EQ2 = 0, 1
REF_DOUBLE, REF_LONGDOUBLE = 0, 1


def _cflags():
    flags = ["-O2", "-std=c99", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
             "-fopenmp", "-fPIC", "-shared"]
    # fmaf()/rintf() are exact IEEE operations either way; with these flags gcc
    # emits the instructions instead of calling libm (same results).
    try:
        cpu = open("/proc/cpuinfo").read()
        if " fma " in cpu and " sse4_1 " in cpu:
            flags += ["-mfma", "-msse4.1"]
    except OSError:
        pass
    return flags


_build_lock = threading.Lock()
_load_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile the oracle (gcc) if missing or stale: to a temporary file renamed into place, under
    a lock, so concurrent first uses (threads, processes) never load a half-written library."""
    with _build_lock:
        newest = max(os.path.getmtime(p) for p in _SRCS + [_HDR])
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
            tmp = f"{_LIB}.{os.getpid()}.{threading.get_ident()}.tmp"
            subprocess.check_call(["gcc", *_cflags(), "-o", tmp, *_SRCS, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


class Coeffs(ctypes.Structure):
    _fields_ = [(n, ctypes.c_float) for n in ("ss1", "ss2", "ss3", "ss4", "cc1", "cc2", "cc3")]


class Opts(ctypes.Structure):
    _fields_ = [("coeffs", Coeffs), ("fix", ctypes.c_int), ("doubling", ctypes.c_int),
                ("doublings", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint64), ("nan_count", ctypes.c_uint64),
                ("sum_sq", ctypes.c_double), ("max_comb", ctypes.c_double),
                ("max_amp", ctypes.c_double), ("amp_signed", ctypes.c_double),
                ("sum_s", ctypes.c_double), ("sum_c", ctypes.c_double),
                ("worst_x", ctypes.c_float), ("worst_bits", ctypes.c_uint32)]

    @property
    def rms(self) -> float:
        return float(np.sqrt(self.sum_sq / self.count)) if self.count else 0.0

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["rms"] = self.rms
        return d


class Method(ctypes.Structure):
    """oracle_method_t (NEXT(3)): any series degrees, doubling count and fix."""
    _fields_ = [("ss", ctypes.c_float * 8), ("n_ss", ctypes.c_int), ("cc", ctypes.c_float * 8),
                ("n_cc", ctypes.c_int), ("doublings", ctypes.c_int), ("fix", ctypes.c_int)]


def make_method(ss, cc, doublings=2, fix=FIX_LINEAR_PENULTIMATE) -> Method:
    m = Method()
    for i, v in enumerate(ss):
        m.ss[i] = float(np.float32(v))
    for i, v in enumerate(cc):
        m.cc[i] = float(np.float32(v))
    m.n_ss, m.n_cc, m.doublings, m.fix = len(ss), len(cc), doublings, fix
    return m


def paper_method(variant: int) -> Method:
    """The paper's method (variant N or A) as a general Method."""
    o = opts(variant)
    k = o.coeffs
    return make_method([k.ss1, k.ss2, k.ss3, k.ss4], [k.cc1, k.cc2, k.cc3], o.doublings, o.fix)


_lib = None
_P = ctypes.c_void_p


def _load():
    global _lib
    if _lib is not None:
        return _lib
    with _load_lock:
        return _load_locked()


def _load_locked():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        sig = {
            "oracle_variant_opts": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(Opts)]),
            "oracle_reduce_turns": (ctypes.c_float, [ctypes.c_float]),
            "oracle_poly_quarter": (None, [ctypes.c_float, ctypes.POINTER(Coeffs),
                                           ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
            "oracle_double_angle": (None, [ctypes.c_float, ctypes.c_float, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
            "oracle_pair_from_q": (None, [ctypes.c_float, ctypes.POINTER(Opts),
                                          ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
            "sincos_oracle": (ctypes.c_int, [_P, _P, _P, ctypes.c_size_t, ctypes.c_int]),
            "sincos_oracle_opts": (ctypes.c_int, [_P, _P, _P, ctypes.c_size_t, ctypes.POINTER(Opts)]),
            "oracle_error_stats": (None, [_P, _P, _P, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(Stats)]),
            "oracle_error_stats_interleaved": (None, [_P, _P, ctypes.c_size_t, ctypes.c_int,
                                                      ctypes.POINTER(Stats)]),
            "oracle_grid_stats": (None, [ctypes.POINTER(Opts), ctypes.c_uint64, ctypes.c_int,
                                         ctypes.POINTER(Stats)]),
            "oracle_sweep_bits": (None, [ctypes.POINTER(Opts), ctypes.c_int, ctypes.c_uint32,
                                         ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(Stats)]),
            "oracle_hash_bits": (None, [ctypes.POINTER(Opts), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.POINTER(ctypes.c_uint64)]),
            "oracle_hash_outputs": (ctypes.c_uint64, [_P, _P, _P, ctypes.c_size_t, ctypes.c_uint32]),
            "oracle_phase_points": (ctypes.c_int, [_P, _P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, _P, _P]),
            "oracle_phase_grid": (ctypes.c_int, [_P, ctypes.c_size_t, _P, ctypes.c_size_t, ctypes.c_int,
                                                 ctypes.c_int, _P, _P]),
            "oracle_nudft": (ctypes.c_int, [_P, ctypes.c_size_t, _P, _P, ctypes.c_size_t, ctypes.c_int,
                                            ctypes.c_int, _P]),
            "oracle_method_pair_from_q": (ctypes.c_int, [ctypes.c_float, ctypes.POINTER(Method),
                                                         ctypes.POINTER(ctypes.c_float),
                                                         ctypes.POINTER(ctypes.c_float)]),
            "oracle_method_sincos": (ctypes.c_int, [_P, _P, _P, ctypes.c_size_t, ctypes.POINTER(Method)]),
            "oracle_method_sweep_q": (None, [ctypes.POINTER(Method), ctypes.c_uint32, ctypes.c_uint32,
                                             ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(Stats)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def opts(variant: int) -> Opts:
    o = Opts()
    if _load().oracle_variant_opts(variant, ctypes.byref(o)) != 0:
        raise ValueError(f"unknown oracle variant {variant}")
    return o


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def reduce_turns(theta: float) -> float:
    """A1 turn reduction of one angle (Fig. 1)."""
    return float(_load().oracle_reduce_turns(theta))


def poly_quarter(q: float, variant_or_opts=VARIANT_N):
    """A2 quarter-angle series at reduced turn q (Fig. 1) -> (s, c)."""
    o = variant_or_opts if isinstance(variant_or_opts, Opts) else opts(variant_or_opts)
    s, c = ctypes.c_float(), ctypes.c_float()
    _load().oracle_poly_quarter(q, ctypes.byref(o.coeffs), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def double_angle(s: float, c: float, form: int = DOUBLING_EQ1):
    """A3 one doubling, Eq. (1) P:77-79 (or the rejected Eq. (2)) -> (s', c')."""
    so, co = ctypes.c_float(), ctypes.c_float()
    _load().oracle_double_angle(s, c, form, ctypes.byref(so), ctypes.byref(co))
    return so.value, co.value


def pair_from_q(q: float, variant_or_opts=VARIANT_N):
    o = variant_or_opts if isinstance(variant_or_opts, Opts) else opts(variant_or_opts)
    s, c = ctypes.c_float(), ctypes.c_float()
    _load().oracle_pair_from_q(q, ctypes.byref(o), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def sincos(theta, variant_or_opts=VARIANT_N):
    """Full pipeline over an array -> (sin, cos) float32 arrays (plain scalar loop)."""
    theta = _f32(theta)
    s = np.empty_like(theta)
    c = np.empty_like(theta)
    lib = _load()
    if isinstance(variant_or_opts, Opts):
        lib.sincos_oracle_opts(theta.ctypes.data, s.ctypes.data, c.ctypes.data, theta.size,
                               ctypes.byref(variant_or_opts))
    else:
        if lib.sincos_oracle(theta.ctypes.data, s.ctypes.data, c.ctypes.data, theta.size,
                             int(variant_or_opts)) != 0:
            raise ValueError(f"unknown oracle variant {variant_or_opts}")
    return s, c


def sincos_into(theta: np.ndarray, s: np.ndarray, c: np.ndarray, variant: int) -> None:
    """Like sincos() but into caller buffers (used by the threaded cpu_baseline)."""
    if _load().sincos_oracle(theta.ctypes.data, s.ctypes.data, c.ctypes.data, theta.size, variant) != 0:
        raise ValueError(f"unknown oracle variant {variant}")


UNITS_RADIANS, UNITS_TURNS = 0, 1


def phase_points(f, t, units: int, variant: int):
    """NEXT(1): pairs of the phases RN(f[k] * t[k]) (radians or turns) -> (sin, cos)."""
    f, t = _f32(f), _f32(t)
    assert f.size == t.size
    s = np.empty_like(f)
    c = np.empty_like(f)
    if _load().oracle_phase_points(f.ctypes.data, t.ctypes.data, f.size, units, variant, s.ctypes.data,
                                   c.ctypes.data) != 0:
        raise ValueError("bad variant or units")
    return s, c


def phase_grid(f, t, units: int, variant: int):
    """NEXT(1): row-major grid (i, j) -> pair of RN(f[i] * t[j]); returns (sin, cos) of shape (nf, nt)."""
    f, t = _f32(f), _f32(t)
    s = np.empty((f.size, t.size), dtype=np.float32)
    c = np.empty_like(s)
    if _load().oracle_phase_grid(f.ctypes.data, f.size, t.ctypes.data, t.size, units, variant, s.ctypes.data,
                                 c.ctypes.data) != 0:
        raise ValueError("bad variant or units")
    return s, c


def nudft(f, t, a, units: int, variant: int) -> np.ndarray:
    """NEXT(2): F_k = sum_j a_j e^{i p_kj}, p_kj = RN(f_k t_j), pairs by the method, products and
    sums in double.  a: complex64 array (or interleaved float32); returns complex128 (nf,)."""
    f, t = _f32(f), _f32(t)
    a = np.ascontiguousarray(a)
    a = a.view(np.float32) if np.iscomplexobj(a) else _f32(a)
    a = np.ascontiguousarray(a.astype(np.float32, copy=False))
    assert a.size == 2 * t.size
    out = np.empty(2 * f.size, dtype=np.float64)
    if _load().oracle_nudft(f.ctypes.data, f.size, t.ctypes.data, a.ctypes.data, t.size, units, variant,
                            out.ctypes.data) != 0:
        raise ValueError("bad variant or units")
    return out.view(np.complex128)


def method_pair_from_q(q: float, m: Method):
    s, c = ctypes.c_float(), ctypes.c_float()
    if _load().oracle_method_pair_from_q(q, ctypes.byref(m), ctypes.byref(s), ctypes.byref(c)) != 0:
        raise ValueError("invalid method")
    return s.value, c.value


def method_sincos(theta, m: Method):
    """NEXT(3): the general method over an array -> (sin, cos)."""
    theta = _f32(theta)
    s = np.empty_like(theta)
    c = np.empty_like(theta)
    if _load().oracle_method_sincos(theta.ctypes.data, s.ctypes.data, c.ctypes.data, theta.size,
                                    ctypes.byref(m)) != 0:
        raise ValueError("invalid method")
    return s, c


def method_sweep_q(m: Method, lo_bits: int = 0, hi_bits: int = 0x3F000000, stride: int = 1,
                   nthreads: int = 0) -> Stats:
    """Kernel-only error stats of a method over fp32 q in [0, 1/2] (every `stride`-th pattern)."""
    st = Stats()
    _load().oracle_method_sweep_q(ctypes.byref(m), lo_bits, hi_bits, stride, nthreads, ctypes.byref(st))
    return st


def error_stats(theta, s, c, ref: int = REF_DOUBLE) -> Stats:
    """P:135-139 metrics of outputs (s, c) against libm double (or long double)."""
    theta, s, c = _f32(theta), _f32(s), _f32(c)
    st = Stats()
    _load().oracle_error_stats(theta.ctypes.data, s.ctypes.data, c.ctypes.data, theta.size, ref,
                               ctypes.byref(st))
    return st


def error_stats_interleaved(theta, cs, ref: int = REF_DOUBLE) -> Stats:
    theta, cs = _f32(theta), _f32(cs)
    st = Stats()
    _load().oracle_error_stats_interleaved(theta.ctypes.data, cs.ctypes.data, theta.size, ref,
                                           ctypes.byref(st))
    return st


def grid_stats(variant_or_opts, m: int = 1 << 24, ref: int = REF_DOUBLE) -> Stats:
    o = variant_or_opts if isinstance(variant_or_opts, Opts) else opts(variant_or_opts)
    st = Stats()
    _load().oracle_grid_stats(ctypes.byref(o), m, ref, ctypes.byref(st))
    return st


def sweep_bits(variant_or_opts, mode: int, lo_bits: int, hi_bits: int, nthreads: int = 0) -> Stats:
    """Exhaustive stats over fp32 patterns [lo_bits, hi_bits]; mode 0 = theta, 1 = q (kernel-only)."""
    o = variant_or_opts if isinstance(variant_or_opts, Opts) else opts(variant_or_opts)
    st = Stats()
    _load().oracle_sweep_bits(ctypes.byref(o), mode, lo_bits, hi_bits, nthreads, ctypes.byref(st))
    return st


def hash_bits(variant_or_opts, lo_bits: int, hi_bits: int, nthreads: int = 0):
    """(hash, nan_pairs, exact_(0,1)_pairs) over theta = bits(u), u in [lo_bits, hi_bits]."""
    o = variant_or_opts if isinstance(variant_or_opts, Opts) else opts(variant_or_opts)
    h, nn, ex = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_hash_bits(ctypes.byref(o), lo_bits, hi_bits, nthreads, ctypes.byref(h),
                             ctypes.byref(nn), ctypes.byref(ex))
    return h.value, nn.value, ex.value


def hash_outputs(s=None, c=None, cs=None, first_bits: int = 0) -> int:
    """The same hash over given outputs (split s/c, or interleaved cs), u = first_bits + i."""
    lib = _load()
    if cs is not None:
        cs = _f32(cs)
        return int(lib.oracle_hash_outputs(None, None, cs.ctypes.data, cs.size // 2, first_bits))
    s, c = _f32(s), _f32(c)
    return int(lib.oracle_hash_outputs(s.ctypes.data, c.ctypes.data, None, s.size, first_bits))
