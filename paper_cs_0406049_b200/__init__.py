"""paper_cs_0406049_b200 -- thin Python binding of libsincos_pairs.so.

The hot path of Mendenhall, "A Fast, Vectorizable Algorithm for Producing
Single-Precision Sine-Cosine Pairs" (arXiv cs/0406049) as one hand-written
sm_100a kernel behind a C ABI (include/sincos_pairs.h).  This module only
marshals arguments (torch tensors -> device pointers, the current CUDA
stream); every step of the path runs in the library's kernels.  There is no
CPU fallback: if the library cannot be loaded, or a tensor is not a CUDA
tensor, the call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

__all__ = [
    # the hot path
    "NORMALIZED", "RENORMALIZED", "SincosError", "lib", "library_path", "sincos", "cis", "sincos_pairs",
    "sincos_pairs_host", "host_workspace_min_bytes",
    # multi-GPU / statistics (8(e))
    "shard_range", "sincos_pairs_sharded", "sincos_pairs_sharded_stats", "nccl_available", "error_stats",
    # NEXT rows (8(f))
    "RADIANS", "TURNS", "phase_grid", "sincos_turns", "nudft", "nudft_chunk", "Method", "make_method",
    "PAPER_METHODS", "FIX_LINEAR", "FIX_RECIPROCAL", "FIX_NONE", "sincos_pairs_method", "sincos_pairs_dtype",
    "interleave", "deinterleave",
    # the fixed kernel configuration, context and test hooks
    "LAUNCH", "null_4in8out", "compare_cuda", "debug_reciprocal", "debug_packed_check", "launch_count",
]

NORMALIZED = 0      # method 1, P:124-150 (Fig. 1 FASTER_SINCOS)
RENORMALIZED = 1    # method 2, P:152-172 (exact reciprocal renormalisation)
_VARIANTS = {"normalized": NORMALIZED, "n": NORMALIZED, "renormalized": RENORMALIZED, "a": RENORMALIZED,
             "angle_accurate": RENORMALIZED}

_STATUS = {0: "ok", 1: "invalid argument", 2: "overlap", 3: "cuda error", 4: "nccl error"}

_PKG = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_PKG, "libsincos_pairs.so")


class SincosError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = f"{what}: {_STATUS.get(status, status)}"
        if status == 3 and _lib is not None:
            msg += f" (cudaError {_lib.sincos_last_cuda_error()})"
        if status == 4 and _lib is not None:
            msg += f" (ncclResult {_lib.sincos_last_nccl_error()})"
        super().__init__(msg)


class Stats(ctypes.Structure):
    """sincos_stats_t (64 bytes)."""
    _fields_ = [("n", ctypes.c_uint64), ("nan_count", ctypes.c_uint64), ("max_comb", ctypes.c_double),
                ("sum_sq", ctypes.c_double), ("max_amp", ctypes.c_double), ("kernel_ms", ctypes.c_double),
                ("worst_theta", ctypes.c_float), ("device", ctypes.c_uint32), ("reserved", ctypes.c_uint64)]


class Shard(ctypes.Structure):
    """sincos_shard_t."""
    _fields_ = [("device", ctypes.c_int), ("theta_dev", ctypes.c_void_p), ("sin_dev", ctypes.c_void_p),
                ("cos_dev", ctypes.c_void_p), ("inter_dev", ctypes.c_void_p), ("n", ctypes.c_size_t),
                ("stream", ctypes.c_void_p)]


class Method(ctypes.Structure):
    """sincos_method_t (NEXT(3))."""
    _fields_ = [("ss", ctypes.c_float * 8), ("n_ss", ctypes.c_int), ("cc", ctypes.c_float * 8),
                ("n_cc", ctypes.c_int), ("doublings", ctypes.c_int), ("fix", ctypes.c_int)]


FIX_LINEAR, FIX_RECIPROCAL, FIX_NONE = 0, 1, 3

# The paper's two methods as explicit tables (PAPER.md P:140-148 / Fig. 1).
PAPER_METHODS = {
    NORMALIZED: ([1.5707963235, -0.645963615, 0.0796819754, -0.0046075748],
                 [-1.2336977925, 0.2536086171, -0.0204391631], 2, FIX_LINEAR),
    RENORMALIZED: ([1.5707963268, -0.6466386396, 0.0679105987, -0.0011573807],
                   [-1.2341299769, 0.2465220241, -0.0123926179], 2, FIX_RECIPROCAL),
}


def make_method(ss, cc, doublings=2, fix=FIX_LINEAR) -> Method:
    """A sincos_method_t from coefficient lists (rounded to fp32 as Fig. 1 does)."""
    import numpy as np
    m = Method()
    for i, v in enumerate(ss):
        m.ss[i] = float(np.float32(v))
    for i, v in enumerate(cc):
        m.cc[i] = float(np.float32(v))
    m.n_ss, m.n_cc, m.doublings, m.fix = len(ss), len(cc), int(doublings), int(fix)
    return m


_lib = None
_P, _S, _I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
_SIGS = {
    "sincos_pairs": (_I, [_P, _P, _P, _P, _S, _I, _P]),
    "sincos_pairs_host": (_I, [_P, _P, _P, _P, _S, _I, _P, _S, _P]),
    "sincos_host_workspace_min_bytes": (_S, []),
    "sincos_shard_range": (_I, [_S, _I, _I, ctypes.POINTER(_S), ctypes.POINTER(_S)]),
    "sincos_pairs_sharded": (_I, [ctypes.POINTER(Shard), _I, _I]),
    "sincos_stats_workspace_bytes": (_S, []),
    "sincos_error_stats": (_I, [_P, _P, _P, _P, _S, _P, _P, _P]),
    "sincos_debug_packed_check": (_I, [_I, _P, _P, _P]),
    "sincos_null_4in8out": (_I, [_P, _P, _P, _P, _S, _P]),
    "sincos_compare_cuda": (_I, [_P, _P, _P, _P, _S, _I, _P]),
    "sincos_debug_reciprocal": (_I, [_P, _P, _S, _P]),
    "sincos_status_string": (ctypes.c_char_p, [_I]),
    "sincos_last_cuda_error": (_I, []),
    "sincos_version": (ctypes.c_char_p, []),
    "sincos_launch_count": (ctypes.c_uint64, []),
    "sincos_phase_grid": (_I, [_P, _S, _P, _S, _P, _P, _P, _I, _I, _P]),
    "sincos_pairs_method": (_I, [_P, _P, _P, _P, _S, ctypes.POINTER(Method), _P]),
    "sincos_pairs_dtype": (_I, [_P, _P, _P, _P, _S, _I, _I, _P]),
    "sincos_pairs_sharded_stats": (_I, [ctypes.POINTER(Shard), _I, _I, _P]),
    "sincos_nccl_available": (_I, []),
    "sincos_last_nccl_error": (_I, []),
    "sincos_interleave": (_I, [_P, _P, _P, _S, _P]),
    "sincos_deinterleave": (_I, [_P, _P, _P, _S, _P]),
    "sincos_nudft_method": (_I, [_P, _S, _P, _P, _S, _P, _I, ctypes.POINTER(Method), _P, _S, _P]),
    "sincos_nudft_chunk": (_S, [_S]),
    "sincos_nudft_workspace_bytes": (_S, [_S, _S]),
    "sincos_nudft": (_I, [_P, _S, _P, _P, _S, _P, _I, _I, _P, _S, _P]),
}

CMP_LIBM_SINCOSF = 3      # comparison only: CUDA libm sincosf / sincospif in the fused sum
CMP_INTRINSIC_SINCOSF = 4  # comparison only: __sincosf

RADIANS, TURNS = 0, 1
EXPORTS = tuple(_SIGS)


def _load(path: str, sigs: dict):
    if not os.path.exists(path):
        raise ImportError(f"{os.path.basename(path)} not found at {path}")
    L = ctypes.CDLL(path)
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


_lib_lock = threading.Lock()


def lib():
    """Load libsincos_pairs.so (building it in-tree with nvcc if it is missing or stale; once, even
    when several threads ask at the same time)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                from . import _build
                _lib = _load(_build.build(), _SIGS)
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise SincosError(status, what)


def _variant(v) -> int:
    if isinstance(v, str):
        return _VARIANTS[v.lower()]
    return int(v)


def _ptr(t, name: str, n=None, dtype="float32", host: bool = False, device=None):
    """Check one buffer argument and return its data pointer (None passes through as NULL).

    Every tensor must be contiguous, of `dtype` (a torch dtype name, or None for any), on the
    right side of the bus -- a CUDA tensor (on `device` when given) for the device entry points,
    a CPU tensor for the host path -- and, when `n` is given, hold exactly n elements.  The
    library trusts these sizes: a short output would be written past its end."""
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if dtype is not None and t.dtype != getattr(torch, dtype):
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if host:
        if t.device.type != "cpu":
            raise ValueError(f"{name} must be a host (CPU) tensor for the host-buffer path")
    else:
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
        if device is not None and t.device != device:
            raise ValueError(f"{name} is on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} must hold {n} elements, got {t.numel()}")
    return t.data_ptr()


def _flat(t, name: str):
    """A 1-D view of a contiguous tensor (never a copy: a non-contiguous `out` is refused
    instead of silently receiving nothing)."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.view(-1)


def _stream(stream, device) -> int:
    """The cudaStream_t handle: `stream` (a torch CUDA stream, or a raw handle), else the current
    stream of `device`.  A torch stream of another device is refused (its work would run on the
    wrong GPU's queue while the kernel reads this one's memory)."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    if hasattr(stream, "cuda_stream"):
        sd = getattr(stream, "device", None)
        if sd is not None and device is not None and torch.device(device).type == "cuda" and \
                torch.device(sd).index != torch.device(device).index:
            raise ValueError(f"stream is on {sd}, the tensors on {device}")
        return stream.cuda_stream
    return int(stream)


def _record(stream, device, *tensors):
    """Temporaries allocated here on the current stream but used by a launch on another
    `stream`: tell the caching allocator, so their blocks are not handed to new work while
    that launch may still read or write them."""
    import torch
    if stream is None:
        return
    s = stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(int(stream), device=device)
    if s.cuda_stream == torch.cuda.current_stream(device).cuda_stream:
        return
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(s)


def _on_tensor_device(fn):
    """Run a device entry point with the CUDA device of its tensors current (the C ABI works on
    the current device's buffers and stream); tensors on two different devices are refused."""
    import functools

    import torch
    Tensor = torch.Tensor

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        dev = None
        for a in list(args) + list(kwargs.values()):
            if isinstance(a, Tensor) and a.is_cuda:
                if dev is None:
                    dev = a.get_device()
                elif a.get_device() != dev:
                    raise ValueError(f"{fn.__name__}: tensors on different devices")
        if dev is None or dev == torch.cuda.current_device():
            return fn(*args, **kwargs)              # the common case: no device switch
        with torch.cuda.device(dev):
            return fn(*args, **kwargs)
    return wrapped


@_on_tensor_device
def sincos_pairs(theta, sin_out=None, cos_out=None, interleaved_out=None, variant=NORMALIZED, stream=None):
    """C-ABI sincos_pairs on CUDA tensors (asynchronous on `stream`, default: current stream).

    Split form: sin_out[i], cos_out[i]; interleaved form: interleaved_out (float32, 2n) holds
    {cos, sin} per element (view as complex64 for e^{i theta})."""
    n = theta.numel()
    d = theta.device
    st = lib().sincos_pairs(_ptr(theta, "theta", device=d), _ptr(sin_out, "sin_out", n, device=d),
                            _ptr(cos_out, "cos_out", n, device=d),
                            _ptr(interleaved_out, "interleaved_out", 2 * n, device=d), n, _variant(variant),
                            _stream(stream, d))
    _check(st, "sincos_pairs")


def sincos(theta, variant="normalized", interleaved=False, out=None, stream=None):
    """Allocate outputs (or take `out`, contiguous: a strided `out` is refused, never silently
    left unwritten) and run the hot path.  Returns (sin, cos) or, if interleaved, a (..., 2)
    float32 tensor of {cos, sin} rows."""
    import torch
    th = theta.contiguous().view(-1)     # an input may be strided: a contiguous copy is read
    if interleaved:
        o = out if out is not None else torch.empty(theta.shape + (2,), dtype=torch.float32, device=theta.device)
        sincos_pairs(th, interleaved_out=_flat(o, "out"), variant=variant, stream=stream)
        _record(stream, theta.device, th, *(() if out is not None else (o,)))
        return o
    s, c = out if out is not None else (torch.empty(theta.shape, dtype=torch.float32, device=theta.device),
                                             torch.empty(theta.shape, dtype=torch.float32, device=theta.device))
    sincos_pairs(th, _flat(s, "out[0]"), _flat(c, "out[1]"), variant=variant, stream=stream)
    _record(stream, theta.device, th, *(() if out is not None else (s, c)))
    return s, c


@_on_tensor_device
def phase_grid(f, t, sin_out=None, cos_out=None, interleaved_out=None, units=RADIANS, variant=NORMALIZED,
               stream=None):
    """NEXT(1) C-ABI sincos_phase_grid: pairs of p_ij = RN(f[i] * t[j]) (radians, or turns with
    units=TURNS) for the row-major nf x nt grid, into split or interleaved outputs."""
    nf, nt = f.numel(), t.numel()
    n = nf * nt
    d = f.device
    st = lib().sincos_phase_grid(_ptr(f, "f", device=d), nf, _ptr(t, "t", device=d), nt,
                                 _ptr(sin_out, "sin_out", n, device=d), _ptr(cos_out, "cos_out", n, device=d),
                                 _ptr(interleaved_out, "interleaved_out", 2 * n, device=d), int(units),
                                 _variant(variant), _stream(stream, d))
    _check(st, "sincos_phase_grid")


def cis(theta, variant="normalized", stream=None):
    """e^{i theta} as a complex64 tensor of theta's shape: the interleaved {cos, sin} output of
    the hot path viewed as complex (reading G13: struct phase {c, s} = re, im)."""
    import torch
    o = sincos(theta, variant=variant, interleaved=True, stream=stream)
    return torch.view_as_complex(o)


def sincos_turns(x, variant="normalized", interleaved=False, out=None, stream=None):
    """Pairs of angles given in TURNS (x = theta / 2 pi): the method from the reduction on
    (P:53-54), without the 1/2 pi scaling and its rounding.  Served by the C-ABI
    sincos_phase_grid with f = [1] (p = RN(1 * x) = x exactly): one row of nt = n pairs.
    Returns (sin 2 pi x, cos 2 pi x) or, if interleaved, a (..., 2) tensor of {cos, sin} rows."""
    import torch
    one = torch.ones(1, dtype=torch.float32, device=x.device)
    xf = x.contiguous().view(-1)
    if interleaved:
        o = out if out is not None else torch.empty(x.shape + (2,), dtype=torch.float32, device=x.device)
        phase_grid(one, xf, interleaved_out=_flat(o, "out"), units=TURNS, variant=variant, stream=stream)
        _record(stream, x.device, one, xf, *(() if out is not None else (o,)))
        return o
    s, c = out if out is not None else (torch.empty(x.shape, dtype=torch.float32, device=x.device),
                                             torch.empty(x.shape, dtype=torch.float32, device=x.device))
    phase_grid(one, xf, _flat(s, "out[0]"), _flat(c, "out[1]"), units=TURNS, variant=variant, stream=stream)
    _record(stream, x.device, one, xf, *(() if out is not None else (s, c)))
    return s, c


@_on_tensor_device
def sincos_pairs_method(theta, method: Method, sin_out=None, cos_out=None, interleaved_out=None, stream=None):
    """NEXT(3) C-ABI sincos_pairs_method: the method with the given series / doublings / fix."""
    n = theta.numel()
    d = theta.device
    st = lib().sincos_pairs_method(_ptr(theta, "theta", device=d), _ptr(sin_out, "sin_out", n, device=d),
                                   _ptr(cos_out, "cos_out", n, device=d),
                                   _ptr(interleaved_out, "interleaved_out", 2 * n, device=d), n,
                                   ctypes.byref(method), _stream(stream, d))
    _check(st, "sincos_pairs_method")


_DTYPES = {"float32": 0, "float16": 1, "bfloat16": 2}


@_on_tensor_device
def sincos_pairs_dtype(theta, sin_out=None, cos_out=None, interleaved_out=None, variant=NORMALIZED, stream=None):
    """NEXT(4) C-ABI sincos_pairs_dtype: outputs in the dtype of the given tensors (float32,
    float16 or bfloat16); 16-bit values are the method's fp32 pair rounded to nearest even."""
    outs = [o for o in (sin_out, cos_out, interleaved_out) if o is not None]
    if not outs:
        raise ValueError("sincos_pairs_dtype: no output given")
    dt = str(outs[0].dtype).replace("torch.", "")
    if dt not in _DTYPES or any(o.dtype != outs[0].dtype for o in outs):
        raise TypeError("outputs must share one dtype of float32, float16, bfloat16")
    n = theta.numel()
    d = theta.device
    st = lib().sincos_pairs_dtype(_ptr(theta, "theta", device=d), _ptr(sin_out, "sin_out", n, dt, device=d),
                                  _ptr(cos_out, "cos_out", n, dt, device=d),
                                  _ptr(interleaved_out, "interleaved_out", 2 * n, dt, device=d), n,
                                  _variant(variant), _DTYPES[dt], _stream(stream, d))
    _check(st, "sincos_pairs_dtype")


@_on_tensor_device
def interleave(sin_in, cos_in, interleaved_out, stream=None):
    """NEXT(4): split fp32 (sin[], cos[]) -> interleaved {cos, sin}."""
    n = sin_in.numel()
    d = sin_in.device
    st = lib().sincos_interleave(_ptr(sin_in, "sin", device=d), _ptr(cos_in, "cos", n, device=d),
                                 _ptr(interleaved_out, "inter", 2 * n, device=d), n, _stream(stream, d))
    _check(st, "sincos_interleave")


@_on_tensor_device
def deinterleave(interleaved_in, sin_out, cos_out, stream=None):
    """NEXT(4): interleaved {cos, sin} fp32 -> split (sin[], cos[])."""
    n = sin_out.numel()
    d = sin_out.device
    st = lib().sincos_deinterleave(_ptr(interleaved_in, "inter", 2 * n, device=d), _ptr(sin_out, "sin", device=d),
                                   _ptr(cos_out, "cos", n, device=d), n, _stream(stream, d))
    _check(st, "sincos_deinterleave")


def nudft_chunk(nt: int) -> int:
    return int(lib().sincos_nudft_chunk(nt))


@_on_tensor_device
def nudft(f, t, a, out=None, units=RADIANS, variant=NORMALIZED, workspace=None, stream=None, method=None):
    """NEXT(2) C-ABI sincos_nudft: out[k] = sum_j a[j] e^{i RN(f[k] t[j])} (complex64 a, out;
    float32 f, t; CUDA tensors).  With `method` (a Method), sincos_nudft_method: the pairs of
    that general method (NEXT(3)).  Returns out."""
    import torch
    nf, nt = f.numel(), t.numel()
    d = f.device
    if a.dtype == torch.complex64:
        a = torch.view_as_real(a)
    ac = a.contiguous()
    if out is None:
        out = torch.empty(nf, dtype=torch.complex64, device=d)
    o = torch.view_as_real(out) if out.dtype == torch.complex64 else out
    need = int(lib().sincos_nudft_workspace_bytes(nf, nt))
    if workspace is None:
        workspace = torch.empty(max(need, 8), dtype=torch.uint8, device=d)
    ws_bytes = workspace.numel() * workspace.element_size()
    ptrs = (_ptr(f, "f", device=d), nf, _ptr(t, "t", device=d), _ptr(ac, "a", 2 * nt, device=d), nt,
            _ptr(o, "out", 2 * nf, device=d), int(units))
    wsp = _ptr(workspace, "workspace", dtype=None, device=d)
    if method is not None:
        st = lib().sincos_nudft_method(*ptrs, ctypes.byref(method), wsp, ws_bytes, _stream(stream, d))
    else:
        st = lib().sincos_nudft(*ptrs, _variant(variant), wsp, ws_bytes, _stream(stream, d))
    _record(stream, d, ac, workspace, out)
    _check(st, "sincos_nudft_method" if method is not None else "sincos_nudft")
    return out


def host_workspace_min_bytes() -> int:
    return int(lib().sincos_host_workspace_min_bytes())


def sincos_pairs_host(theta, sin_out=None, cos_out=None, interleaved_out=None, variant=NORMALIZED,
                      workspace=None, stream=None):
    """C-ABI sincos_pairs_host on HOST (CPU) tensors, pinned for overlap; `workspace` is a CUDA
    tensor whose device runs the pipeline.  Synchronous."""
    import torch
    if workspace is None or not isinstance(workspace, torch.Tensor) or not workspace.is_cuda:
        raise ValueError("workspace must be a CUDA tensor")
    n = theta.numel()
    dev = workspace.device
    with torch.cuda.device(dev):
        st = lib().sincos_pairs_host(_ptr(theta, "theta", host=True), _ptr(sin_out, "sin_out", n, host=True),
                                     _ptr(cos_out, "cos_out", n, host=True),
                                     _ptr(interleaved_out, "interleaved_out", 2 * n, host=True), n,
                                     _variant(variant), _ptr(workspace, "workspace", dtype=None, device=dev),
                                     workspace.numel() * workspace.element_size(), _stream(stream, dev))
    _check(st, "sincos_pairs_host")


def shard_range(n: int, nshards: int, g: int):
    """[lo, hi) of shard g (host logic only, no CUDA)."""
    lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
    if lib().sincos_shard_range(n, nshards, g, ctypes.byref(lo), ctypes.byref(hi)) != 0:
        raise ValueError(f"bad shard {g} of {nshards}")
    return lo.value, hi.value


def _shard_array(shards):
    """sincos_shard_t records; every buffer of a shard on the shard's device, sizes checked.
    A shard may name its device explicitly ("device"), else theta's."""
    arr = (Shard * len(shards))()
    for i, sh in enumerate(shards):
        th = sh["theta"]
        d = th.device
        n = th.numel()
        arr[i].device = int(sh.get("device", d.index))
        arr[i].theta_dev = _ptr(th, "theta", device=d)
        arr[i].sin_dev = _ptr(sh.get("sin"), "sin", n, device=d)
        arr[i].cos_dev = _ptr(sh.get("cos"), "cos", n, device=d)
        arr[i].inter_dev = _ptr(sh.get("inter"), "inter", 2 * n, device=d)
        arr[i].n = n
        arr[i].stream = _stream(sh.get("stream"), d)
    return arr


def sincos_pairs_sharded(shards, variant=NORMALIZED):
    """Single-process multi-device launch (one host thread per device).  shards: list of dicts
    with theta, sin/cos or inter tensors, optional stream (and optional device override)."""
    _check(lib().sincos_pairs_sharded(_shard_array(shards), len(shards), _variant(variant)), "sincos_pairs_sharded")


def sincos_pairs_sharded_stats(shards, variant=NORMALIZED) -> list:
    """C-ABI sincos_pairs_sharded_stats: one shard per device, launched, its stats and kernel
    time reduced on its device, the 64-B records all-gathered over NCCL.  Returns the records."""
    arr = _shard_array(shards)
    out = (Stats * len(shards))()
    _check(lib().sincos_pairs_sharded_stats(arr, len(shards), _variant(variant), out), "sincos_pairs_sharded_stats")
    res = []
    for s in out:
        d = {k: getattr(s, k) for k, _ in Stats._fields_}
        d["rms"] = (s.sum_sq / s.n) ** 0.5 if s.n else 0.0
        res.append(d)
    return res


def nccl_available() -> bool:
    return bool(lib().sincos_nccl_available())


@_on_tensor_device
def error_stats(theta, sin_out=None, cos_out=None, interleaved_out=None, stream=None) -> dict:
    """KB5 fp64 error statistics of outputs on the device (P:135-139 metrics).  Synchronous."""
    import torch
    d = theta.device
    n = theta.numel()
    ws = torch.empty(lib().sincos_stats_workspace_bytes(), dtype=torch.uint8, device=d)
    rec = torch.zeros(ctypes.sizeof(Stats), dtype=torch.uint8, device=d)
    st = lib().sincos_error_stats(_ptr(theta, "theta", device=d), _ptr(sin_out, "sin_out", n, device=d),
                                  _ptr(cos_out, "cos_out", n, device=d),
                                  _ptr(interleaved_out, "interleaved_out", 2 * n, device=d), n, rec.data_ptr(),
                                  ws.data_ptr(), _stream(stream, d))
    _record(stream, d, ws, rec)
    _check(st, "sincos_error_stats")
    if stream is not None:
        torch.cuda.ExternalStream(_stream(stream, d), device=d).synchronize()
    raw = bytes(rec.cpu().numpy().tobytes())
    s = Stats.from_buffer_copy(raw)
    out = {k: getattr(s, k) for k, _ in Stats._fields_}
    out["rms"] = (s.sum_sq / s.n) ** 0.5 if s.n else 0.0
    out["raw"] = raw
    return out


# The one kernel configuration of the product library (sincos_launch.h Tuning): 128-thread
# blocks, the full grid (one 256-bit trip per thread), 8 floats per access, no unroll.  The
# alternatives exist only in the A/B build (paper_cs_0406049_b200.ab; tests and tools).
LAUNCH = {"threads": 128, "grid": "full (one trip per thread)", "vec": 8, "unroll": 1, "pdl": True}


@_on_tensor_device
def compare_cuda(theta, sin_out=None, cos_out=None, interleaved_out=None, which=3, stream=None):
    """Context (bench): the hot path's kernel shape with CUDA sincosf (which=3) or __sincosf (4)."""
    n = theta.numel()
    d = theta.device
    _check(lib().sincos_compare_cuda(_ptr(theta, "theta", device=d), _ptr(sin_out, "sin_out", n, device=d),
                                     _ptr(cos_out, "cos_out", n, device=d),
                                     _ptr(interleaved_out, "interleaved_out", 2 * n, device=d), n, int(which),
                                     _stream(stream, d)), "sincos_compare_cuda")


@_on_tensor_device
def null_4in8out(theta, sin_out=None, cos_out=None, interleaved_out=None, stream=None):
    n = theta.numel()
    d = theta.device
    _check(lib().sincos_null_4in8out(_ptr(theta, "theta", device=d), _ptr(sin_out, "sin_out", n, device=d),
                                     _ptr(cos_out, "cos_out", n, device=d),
                                     _ptr(interleaved_out, "interleaved_out", 2 * n, device=d), n,
                                     _stream(stream, d)), "sincos_null_4in8out")


@_on_tensor_device
def debug_reciprocal(d, out, stream=None):
    _check(lib().sincos_debug_reciprocal(_ptr(d, "d", device=d.device), _ptr(out, "out", d.numel(), device=d.device),
                                         d.numel(), _stream(stream, d.device)), "sincos_debug_reciprocal")


def debug_packed_check(variant=NORMALIZED, method=None, stream=None) -> int:
    """Test hook: mismatching output components of the packed-fp32 method against the scalar
    method over all 2^32 fp32 inputs (radians and turns).  Synchronous; 0 expected."""
    import torch
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    _check(lib().sincos_debug_packed_check(-1 if variant == -1 else _variant(variant),
                                           ctypes.byref(method) if method is not None else None,
                                           cnt.data_ptr(), _stream(stream, cnt.device)),
           "sincos_debug_packed_check")
    return int(cnt.item())


def launch_count() -> int:
    return int(lib().sincos_launch_count())
