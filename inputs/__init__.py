"""Seeded synthetic inputs for the BASELINE.json configs.

Shared by the oracle side and the product side, so it holds none of the
method's arithmetic -- only the counter-based generator in ``gen.c`` and the
configs' value distributions.  Element ``i`` of config ``c`` is a pure function
of ``(c, i)``: ranges and index samples can be generated independently.

Config ids: 1..5 are BASELINE.json ``configs[0..4]`` (C1..C5); 0 is "raw fp32
bit patterns" (theta_i = bits(i)) for whole-input-space sweeps.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsincos_inputs.so")

CONFIG_NAMES = {
    0: "all-fp32-bit-patterns",
    1: "C1: 2^20 U[-pi,pi) seed 0",
    2: "C2: 2^28 U[-1e4,1e4] seed 1",
    3: "C3: 2^24 edge/stress set seed 2",
    4: "C4: 2^30 NUFFT phases 2pi f_i t_j seed 3",
    5: "C5: 2^32 N(0,100^2) seed 4",
}


_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile gen.c into libsincos_inputs.so (gcc, OpenMP): to a temporary file renamed into
    place, under a lock, so concurrent first uses never load a half-written library."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = f"{_LIB}.{os.getpid()}.{threading.get_ident()}.tmp"
            subprocess.check_call([
                "gcc", "-O2", "-std=c99", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
                "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


_lib = None
_load_lock = threading.Lock()


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
        lib.sincos_gen_size.restype = ctypes.c_uint64
        lib.sincos_gen_size.argtypes = [ctypes.c_int]
        lib.sincos_gen_range.restype = ctypes.c_int
        lib.sincos_gen_range.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_void_p, ctypes.c_int]
        lib.sincos_gen_at.restype = ctypes.c_int
        lib.sincos_gen_at.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        lib.sincos_gen_urand.restype = ctypes.c_double
        lib.sincos_gen_urand.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib = lib
    return _lib


def size(config: int) -> int:
    """Element count of a config (C1 2^20, C2 2^28, C3 2^24, C4 2^30, C5 2^32)."""
    return int(_load().sincos_gen_size(config))


def generate(config: int, start: int = 0, count: int | None = None, out: np.ndarray | None = None,
             nthreads: int = 0) -> np.ndarray:
    """Elements [start, start+count) of ``config`` as float32 (into ``out`` if given;
    ``out`` may be any C-contiguous float32 buffer, e.g. a pinned torch tensor's numpy view)."""
    if count is None:
        count = size(config) - start
    if out is None:
        out = np.empty(count, dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.size >= count
    rc = _load().sincos_gen_range(config, start, count, out.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError(f"unknown config {config}")
    return out


def generate_at(config: int, idx: np.ndarray) -> np.ndarray:
    """Elements ``idx`` (uint64 indices) of ``config``."""
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(idx.size, dtype=np.float32)
    rc = _load().sincos_gen_at(config, idx.ctypes.data, idx.size, out.ctypes.data)
    if rc != 0:
        raise ValueError(f"unknown config {config}")
    return out


def urand(seed: int, stream: int, i: int) -> float:
    """The raw counter-based uniform u(seed, stream, i) in [0, 1)."""
    return float(_load().sincos_gen_urand(seed, stream, i))
