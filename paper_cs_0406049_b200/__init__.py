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

__all__ = [
    # the hot path
    "NORMALIZED", "RENORMALIZED", "SincosError", "lib", "library_path", "sincos", "cis", "sincos_pairs",
    "sincos_pairs_host", "host_workspace_min_bytes", "Item", "BatchTable", "sincos_pairs_batched", "sincos_batched",
    # multi-GPU / statistics (8(e))
    "shard_range", "sincos_pairs_sharded", "sincos_pairs_sharded_stats", "nccl_available", "error_stats",
    # NEXT rows (8(f))
    "RADIANS", "TURNS", "phase_grid", "sincos_turns", "nudft", "nudft_chunk", "Method", "make_method",
    "PAPER_METHODS", "FIX_LINEAR", "FIX_RECIPROCAL", "FIX_NONE", "sincos_pairs_method", "sincos_pairs_dtype",
    "interleave", "deinterleave",
    # tuning, context and test hooks
    "set_launch_config", "get_launch_config", "set_realign", "set_pdl", "set_nudft_packed", "null_4in8out",
    "compare_cuda", "debug_reciprocal", "debug_packed_check", "launch_count",
]

NORMALIZED = 0      # method 1, P:124-150 (Fig. 1 FASTER_SINCOS)
RENORMALIZED = 1    # method 2, P:152-172 (exact reciprocal renormalisation)
_VARIANTS = {"normalized": NORMALIZED, "n": NORMALIZED, "renormalized": RENORMALIZED, "a": RENORMALIZED,
             "angle_accurate": RENORMALIZED}

_STATUS = {0: "ok", 1: "invalid argument", 2: "overlap", 3: "cuda error"}

_PKG = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_PKG, "libsincos_pairs.so")


class SincosError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        msg = f"{what}: {_STATUS.get(status, status)}"
        if status == 3 and _lib is not None:
            msg += f" (cudaError {_lib.sincos_last_cuda_error()})"
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
    "sincos_set_launch_config": (_I, [_I, _I, _I, _I, _I]),
    "sincos_set_nudft_packed": (_I, [_I]),
    "sincos_set_realign": (_I, [_I]),
    "sincos_set_pdl": (_I, [_I]),
    "sincos_pairs_batched": (_I, [ctypes.c_void_p, _I, _I, _P]),
    "sincos_debug_packed_check": (_I, [_I, _P, _P, _P]),
    "sincos_get_launch_config": (None, [ctypes.POINTER(_I)] * 5),
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


def lib():
    """Load libsincos_pairs.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    if _lib is None:
        from . import _build
        path = _build.build()
        if not os.path.exists(path):
            raise ImportError(f"libsincos_pairs.so not found at {path}")
        L = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise SincosError(status, what)


def _variant(v) -> int:
    if isinstance(v, str):
        return _VARIANTS[v.lower()]
    return int(v)


def _ptr(t, name: str, device_required: bool = True) -> int:
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32, got {t.dtype}")
    if device_required and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _stream(stream, device) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _on_tensor_device(fn):
    """Run a device entry point with the CUDA device of its tensors current (the C ABI works on
    the current device's buffers and stream); tensors on two different devices are refused."""
    import functools

    import torch
    Tensor = torch.Tensor

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        dev = None
        for a in args:
            if isinstance(a, Tensor) and a.is_cuda:
                if dev is None:
                    dev = a.get_device()
                elif a.get_device() != dev:
                    raise ValueError(f"{fn.__name__}: tensors on different devices")
        for a in kwargs.values():
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
    if interleaved_out is not None and interleaved_out.numel() != 2 * n:
        raise ValueError("interleaved_out must hold 2*n floats")
    for o in (sin_out, cos_out):
        if o is not None and o.numel() != n:
            raise ValueError("outputs must hold n floats")
    st = lib().sincos_pairs(_ptr(theta, "theta"), _ptr(sin_out, "sin_out"), _ptr(cos_out, "cos_out"),
                            _ptr(interleaved_out, "interleaved_out"), n, _variant(variant),
                            _stream(stream, theta.device))
    _check(st, "sincos_pairs")


def sincos(theta, variant="normalized", interleaved=False, out=None, stream=None):
    """Allocate outputs and run the hot path.  Returns (sin, cos) or, if interleaved, a (n, 2)
    float32 tensor of {cos, sin} rows."""
    import torch
    if interleaved:
        o = out if out is not None else torch.empty(theta.shape + (2,), dtype=torch.float32, device=theta.device)
        sincos_pairs(theta.reshape(-1), interleaved_out=o.reshape(-1), variant=variant, stream=stream)
        return o
    s, c = out if out is not None else (torch.empty_like(theta), torch.empty_like(theta))
    sincos_pairs(theta.reshape(-1), s.reshape(-1), c.reshape(-1), variant=variant, stream=stream)
    return s, c


@_on_tensor_device
def phase_grid(f, t, sin_out=None, cos_out=None, interleaved_out=None, units=RADIANS, variant=NORMALIZED,
               stream=None):
    """NEXT(1) C-ABI sincos_phase_grid: pairs of p_ij = RN(f[i] * t[j]) (radians, or turns with
    units=TURNS) for the row-major nf x nt grid, into split or interleaved outputs."""
    nf, nt = f.numel(), t.numel()
    n = nf * nt
    if interleaved_out is not None and interleaved_out.numel() != 2 * n:
        raise ValueError("interleaved_out must hold 2*nf*nt floats")
    for o in (sin_out, cos_out):
        if o is not None and o.numel() != n:
            raise ValueError("outputs must hold nf*nt floats")
    st = lib().sincos_phase_grid(_ptr(f, "f"), nf, _ptr(t, "t"), nt, _ptr(sin_out, "sin_out"),
                                 _ptr(cos_out, "cos_out"), _ptr(interleaved_out, "interleaved_out"), int(units),
                                 _variant(variant), _stream(stream, f.device))
    _check(st, "sincos_phase_grid")


class Item(ctypes.Structure):
    """sincos_item_t: one array of a batched call."""
    _fields_ = [("theta", ctypes.c_void_p), ("sin", ctypes.c_void_p), ("cos", ctypes.c_void_p),
                ("inter", ctypes.c_void_p), ("n", ctypes.c_uint64)]


class BatchTable:
    """A validated, reusable item table for sincos_pairs_batched (the sincos_item_t layout as one
    uint64 array): build it once for a fixed set of buffers, then run() costs one C call --
    the per-item Python work (~1 us each) is paid once, not per call.  Keeps the tensors alive."""

    def __init__(self, thetas, sin_outs=None, cos_outs=None, interleaved_outs=None):
        self.tab = _batch_table(thetas, sin_outs, cos_outs, interleaved_outs)
        self.tensors = (list(thetas), sin_outs, cos_outs, interleaved_outs)
        self.count = len(thetas)

    def run(self, variant=NORMALIZED, stream=None):
        import torch
        if self.count:
            st = lib().sincos_pairs_batched(self.tab.ctypes.data, self.count, _variant(variant),
                                            _stream(stream, torch.device("cuda", torch.cuda.current_device())))
            _check(st, "sincos_pairs_batched")


def _batch_table(thetas, sin_outs, cos_outs, interleaved_outs):
    import numpy as np
    import torch
    k = len(thetas)
    tab = np.zeros((k, 5), dtype=np.uint64)
    if k == 0:
        return tab
    dev = torch.cuda.current_device()

    def ok(t, name):
        if t.dtype != torch.float32 or not t.is_cuda or t.get_device() != dev or not t.is_contiguous():
            raise ValueError(f"{name}: every tensor must be a contiguous float32 CUDA tensor on the current device")
        return t.data_ptr()

    tab[:, 0] = [ok(t, "theta") for t in thetas]
    n = np.array([t.numel() for t in thetas], dtype=np.uint64)
    tab[:, 4] = n
    if interleaved_outs is not None:
        if len(interleaved_outs) != k or any(o.numel() != 2 * int(m) for o, m in zip(interleaved_outs, n)):
            raise ValueError("interleaved_outs must hold 2*n floats each")
        tab[:, 3] = [ok(o, "interleaved_out") for o in interleaved_outs]
    else:
        if len(sin_outs) != k or len(cos_outs) != k or any(
                so.numel() != int(m) or co.numel() != int(m) for so, co, m in zip(sin_outs, cos_outs, n)):
            raise ValueError("outputs must hold n floats each")
        tab[:, 1] = [ok(o, "sin_out") for o in sin_outs]
        tab[:, 2] = [ok(o, "cos_out") for o in cos_outs]
    return tab


def sincos_pairs_batched(thetas, sin_outs=None, cos_outs=None, interleaved_outs=None, variant=NORMALIZED,
                         stream=None):
    """C-ABI sincos_pairs_batched: many arrays in one launch (per 480 arrays).  thetas: list of
    CUDA float32 contiguous tensors on the current device; outputs: lists of the same length
    (split) or interleaved_outs.  The item table is built as one uint64 array (the
    sincos_item_t layout: 4 pointers + n), so marshalling costs ~1 us per item."""
    BatchTable(thetas, sin_outs, cos_outs, interleaved_outs).run(variant, stream)


def sincos_batched(thetas, variant="normalized", interleaved=False, stream=None):
    """Allocate outputs and run many arrays in one launch; returns a list of (sin, cos) or of
    (n, 2) {cos, sin} tensors."""
    import torch
    if interleaved:
        outs = [torch.empty(t.shape + (2,), dtype=torch.float32, device=t.device) for t in thetas]
        sincos_pairs_batched([t.reshape(-1) for t in thetas], interleaved_outs=[o.reshape(-1) for o in outs],
                             variant=variant, stream=stream)
        return outs
    ss = [torch.empty_like(t) for t in thetas]
    cs = [torch.empty_like(t) for t in thetas]
    sincos_pairs_batched([t.reshape(-1) for t in thetas], [x.reshape(-1) for x in ss], [x.reshape(-1) for x in cs],
                         variant=variant, stream=stream)
    return list(zip(ss, cs))


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
    Returns (sin 2 pi x, cos 2 pi x) or, if interleaved, a (n, 2) tensor of {cos, sin} rows."""
    import torch
    one = torch.ones(1, dtype=torch.float32, device=x.device)
    xf = x.reshape(-1)
    if interleaved:
        o = out if out is not None else torch.empty(x.shape + (2,), dtype=torch.float32, device=x.device)
        phase_grid(one, xf, interleaved_out=o.reshape(-1), units=TURNS, variant=variant, stream=stream)
        return o
    s, c = out if out is not None else (torch.empty_like(x), torch.empty_like(x))
    phase_grid(one, xf, s.reshape(-1), c.reshape(-1), units=TURNS, variant=variant, stream=stream)
    return s, c


@_on_tensor_device
def sincos_pairs_method(theta, method: Method, sin_out=None, cos_out=None, interleaved_out=None, stream=None):
    """NEXT(3) C-ABI sincos_pairs_method: the method with the given series / doublings / fix."""
    n = theta.numel()
    st = lib().sincos_pairs_method(_ptr(theta, "theta"), _ptr(sin_out, "sin_out"), _ptr(cos_out, "cos_out"),
                                   _ptr(interleaved_out, "interleaved_out"), n, ctypes.byref(method),
                                   _stream(stream, theta.device))
    _check(st, "sincos_pairs_method")


def _ptr_any(t, name: str):
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA tensor (no CPU fallback)")
    return t.data_ptr()


@_on_tensor_device
def sincos_pairs_dtype(theta, sin_out=None, cos_out=None, interleaved_out=None, variant=NORMALIZED, stream=None):
    """NEXT(4) C-ABI sincos_pairs_dtype: outputs in the dtype of the given tensors (float32,
    float16 or bfloat16); 16-bit values are the method's fp32 pair rounded to nearest even."""
    import torch
    outs = [o for o in (sin_out, cos_out, interleaved_out) if o is not None]
    dt = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}[outs[0].dtype]
    if any(o.dtype != outs[0].dtype for o in outs):
        raise TypeError("outputs must share one dtype")
    n = theta.numel()
    st = lib().sincos_pairs_dtype(_ptr(theta, "theta"), _ptr_any(sin_out, "sin_out"), _ptr_any(cos_out, "cos_out"),
                                  _ptr_any(interleaved_out, "interleaved_out"), n, _variant(variant), dt,
                                  _stream(stream, theta.device))
    _check(st, "sincos_pairs_dtype")


@_on_tensor_device
def interleave(sin_in, cos_in, interleaved_out, stream=None):
    """NEXT(4): split fp32 (sin[], cos[]) -> interleaved {cos, sin}."""
    st = lib().sincos_interleave(_ptr(sin_in, "sin"), _ptr(cos_in, "cos"), _ptr(interleaved_out, "inter"),
                                 sin_in.numel(), _stream(stream, sin_in.device))
    _check(st, "sincos_interleave")


@_on_tensor_device
def deinterleave(interleaved_in, sin_out, cos_out, stream=None):
    """NEXT(4): interleaved {cos, sin} fp32 -> split (sin[], cos[])."""
    st = lib().sincos_deinterleave(_ptr(interleaved_in, "inter"), _ptr(sin_out, "sin"), _ptr(cos_out, "cos"),
                                   sin_out.numel(), _stream(stream, sin_out.device))
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
    if a.dtype == torch.complex64:
        a = torch.view_as_real(a)
    if a.numel() != 2 * nt:
        raise ValueError("a must hold nt complex values")
    if out is None:
        out = torch.empty(nf, dtype=torch.complex64, device=f.device)
    o = torch.view_as_real(out) if out.dtype == torch.complex64 else out
    need = int(lib().sincos_nudft_workspace_bytes(nf, nt))
    if workspace is None:
        workspace = torch.empty(max(need, 8), dtype=torch.uint8, device=f.device)
    ws_bytes = workspace.numel() * workspace.element_size()
    if method is not None:
        st = lib().sincos_nudft_method(_ptr(f, "f"), nf, _ptr(t, "t"), _ptr(a.contiguous(), "a"), nt,
                                       _ptr(o, "out"), int(units), ctypes.byref(method), workspace.data_ptr(),
                                       ws_bytes, _stream(stream, f.device))
        _check(st, "sincos_nudft_method")
        return out
    st = lib().sincos_nudft(_ptr(f, "f"), nf, _ptr(t, "t"), _ptr(a.contiguous(), "a"), nt, _ptr(o, "out"),
                            int(units), _variant(variant), workspace.data_ptr(), ws_bytes,
                            _stream(stream, f.device))
    _check(st, "sincos_nudft")
    return out


def host_workspace_min_bytes() -> int:
    return int(lib().sincos_host_workspace_min_bytes())


def sincos_pairs_host(theta, sin_out=None, cos_out=None, interleaved_out=None, variant=NORMALIZED,
                      workspace=None, stream=None):
    """C-ABI sincos_pairs_host on HOST tensors (pinned for overlap); `workspace` is a CUDA uint8/float
    tensor on the current device.  Synchronous."""
    import torch
    n = theta.numel()
    ws_bytes = workspace.numel() * workspace.element_size()
    dev = workspace.device
    st = lib().sincos_pairs_host(_ptr(theta, "theta", False), _ptr(sin_out, "sin_out", False),
                                 _ptr(cos_out, "cos_out", False), _ptr(interleaved_out, "interleaved_out", False),
                                 n, _variant(variant), workspace.data_ptr(), ws_bytes, _stream(stream, dev))
    _check(st, "sincos_pairs_host")


def shard_range(n: int, nshards: int, g: int):
    """[lo, hi) of shard g (host logic only, no CUDA)."""
    lo, hi = ctypes.c_size_t(), ctypes.c_size_t()
    if lib().sincos_shard_range(n, nshards, g, ctypes.byref(lo), ctypes.byref(hi)) != 0:
        raise ValueError(f"bad shard {g} of {nshards}")
    return lo.value, hi.value


def sincos_pairs_sharded(shards, variant=NORMALIZED):
    """Single-process multi-device launch.  shards: list of dicts with device, theta,
    sin/cos or inter tensors, optional stream."""
    arr = (Shard * len(shards))()
    for i, sh in enumerate(shards):
        th = sh["theta"]
        arr[i].device = th.device.index
        arr[i].theta_dev = _ptr(th, "theta")
        arr[i].sin_dev = _ptr(sh.get("sin"), "sin")
        arr[i].cos_dev = _ptr(sh.get("cos"), "cos")
        arr[i].inter_dev = _ptr(sh.get("inter"), "inter")
        arr[i].n = th.numel()
        arr[i].stream = _stream(sh.get("stream"), th.device)
    _check(lib().sincos_pairs_sharded(arr, len(shards), _variant(variant)), "sincos_pairs_sharded")


def _shard_array(shards):
    arr = (Shard * len(shards))()
    for i, sh in enumerate(shards):
        th = sh["theta"]
        arr[i].device = th.device.index
        arr[i].theta_dev = _ptr(th, "theta")
        arr[i].sin_dev = _ptr(sh.get("sin"), "sin")
        arr[i].cos_dev = _ptr(sh.get("cos"), "cos")
        arr[i].inter_dev = _ptr(sh.get("inter"), "inter")
        arr[i].n = th.numel()
        arr[i].stream = _stream(sh.get("stream"), th.device)
    return arr


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
    """KB5 fp64 error statistics of outputs on the device (P:135-139 metrics)."""
    import torch
    dev = theta.device
    ws = torch.empty(lib().sincos_stats_workspace_bytes(), dtype=torch.uint8, device=dev)
    rec = torch.zeros(ctypes.sizeof(Stats), dtype=torch.uint8, device=dev)
    st = lib().sincos_error_stats(_ptr(theta, "theta"), _ptr(sin_out, "sin_out"), _ptr(cos_out, "cos_out"),
                                  _ptr(interleaved_out, "interleaved_out"), theta.numel(), rec.data_ptr(),
                                  ws.data_ptr(), _stream(stream, dev))
    _check(st, "sincos_error_stats")
    raw = bytes(rec.cpu().numpy().tobytes())
    s = Stats.from_buffer_copy(raw)
    d = {k: getattr(s, k) for k, _ in Stats._fields_}
    d["rms"] = (s.sum_sq / s.n) ** 0.5 if s.n else 0.0
    d["raw"] = raw
    return d


DEFAULT_LAUNCH = dict(threads=128, blocks_per_sm=0, vec=8, unroll=1, prefetch=0)


def set_launch_config(threads=None, blocks_per_sm=None, vec=None, unroll=None, prefetch=None):
    """Set the process-global launch configuration; omitted fields take the library defaults."""
    cfg = dict(DEFAULT_LAUNCH)
    for k, v in (("threads", threads), ("blocks_per_sm", blocks_per_sm), ("vec", vec), ("unroll", unroll),
                 ("prefetch", prefetch)):
        if v is not None:
            cfg[k] = int(v)
    if lib().sincos_set_launch_config(cfg["threads"], cfg["blocks_per_sm"], cfg["vec"], cfg["unroll"],
                                      cfg["prefetch"]) != 0:
        raise ValueError(f"unsupported launch config {cfg}")


def set_realign(on) -> int:
    """Unshared-alignment path: register re-alignment (True / 1, default), one element per thread
    (False / 0), re-alignment in its 128-bit form only (2, A/B), or 1 with the phase grid's
    ragged rows through its flat kernel instead of the row kernel (3, A/B).  Returns the
    previous value."""
    v = on if on in (2, 3) else (1 if on else 0)
    prev = lib().sincos_set_realign(v)
    if prev < 0:
        raise ValueError(on)
    return prev


def set_pdl(on: bool) -> bool:
    """Programmatic dependent launch of the hot kernel (True, default) or plain launches."""
    prev = lib().sincos_set_pdl(1 if on else 0)
    if prev < 0:
        raise ValueError(on)
    return bool(prev)


def set_nudft_packed(on: bool) -> bool:
    """Select the packed-fp32 (FFMA2) or scalar kernels of the fused sum; returns the previous setting."""
    prev = lib().sincos_set_nudft_packed(1 if on else 0)
    if prev < 0:
        raise ValueError(on)
    return bool(prev)


def get_launch_config() -> dict:
    v = [ctypes.c_int() for _ in range(5)]
    lib().sincos_get_launch_config(*[ctypes.byref(x) for x in v])
    return dict(zip(("threads", "blocks_per_sm", "vec", "unroll", "prefetch"), (x.value for x in v)))


@_on_tensor_device
def compare_cuda(theta, sin_out=None, cos_out=None, interleaved_out=None, which=3, stream=None):
    """Context (bench): the hot path's kernel shape with CUDA sincosf (which=3) or __sincosf (4)."""
    _check(lib().sincos_compare_cuda(_ptr(theta, "theta"), _ptr(sin_out, "sin_out"), _ptr(cos_out, "cos_out"),
                                     _ptr(interleaved_out, "interleaved_out"), theta.numel(), int(which),
                                     _stream(stream, theta.device)), "sincos_compare_cuda")


@_on_tensor_device
def null_4in8out(theta, sin_out=None, cos_out=None, interleaved_out=None, stream=None):
    _check(lib().sincos_null_4in8out(_ptr(theta, "theta"), _ptr(sin_out, "sin_out"), _ptr(cos_out, "cos_out"),
                                     _ptr(interleaved_out, "interleaved_out"), theta.numel(),
                                     _stream(stream, theta.device)), "sincos_null_4in8out")


@_on_tensor_device
def debug_reciprocal(d, out, stream=None):
    _check(lib().sincos_debug_reciprocal(_ptr(d, "d"), _ptr(out, "out"), d.numel(), _stream(stream, d.device)),
           "sincos_debug_reciprocal")


def debug_packed_check(variant=NORMALIZED, method=None, stream=None) -> int:
    """Test hook: mismatching output components of the packed-fp32 method against the scalar
    method over all 2^32 fp32 inputs (radians and turns).  Synchronous; 0 expected."""
    import torch
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    _check(lib().sincos_debug_packed_check(-1 if variant == -1 else _variant(variant), ctypes.byref(method) if method is not None else None,
                                           cnt.data_ptr(), _stream(stream, cnt.device)),
           "sincos_debug_packed_check")
    return int(cnt.item())


def launch_count() -> int:
    return int(lib().sincos_launch_count())
