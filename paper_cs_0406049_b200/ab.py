"""The A/B build of the library -- for tests and tools only, never the product path.

libsincos_pairs_ab.so is built from the same sources with -DSINCOS_AB (paper_cs_0406049_b200
/_build.py): the same entry points, plus the settable kernel forms and launch shapes that the
product fixes (csrc/sincos_ab.h, sincos_ab_set) and sincos_pairs_batched.  They exist to
measure the alternatives DESIGN.md section 5 compares, and to keep those kernels parity-tested.

    with ab.knobs(realign=0):          # every binding call inside runs on the A/B build
        sp.sincos_pairs(theta, s, c)   # ... through its one-element-per-thread kernel

`knobs` swaps the binding's library for the A/B build and sets the knobs for the duration of
the block, then restores the defaults and the product library (single-threaded use).
"""
from __future__ import annotations

import contextlib
import ctypes
import threading

from . import _build

KNOBS = {"threads": 0, "blocks_per_sm": 1, "vec": 2, "unroll": 3, "prefetch": 4, "realign": 5, "pdl": 6,
         "nudft_packed": 7}
DEFAULTS = {"threads": 128, "blocks_per_sm": 0, "vec": 8, "unroll": 1, "prefetch": 0, "realign": 1, "pdl": 1,
            "nudft_packed": 1}

_ab = None


class Item(ctypes.Structure):
    """sincos_item_t: one array of a batched call."""
    _fields_ = [("theta", ctypes.c_void_p), ("sin", ctypes.c_void_p), ("cos", ctypes.c_void_p),
                ("inter", ctypes.c_void_p), ("n", ctypes.c_uint64)]


_ab_lock = threading.Lock()


def lib():
    """Load libsincos_pairs_ab.so (building it in-tree if missing or stale)."""
    global _ab
    if _ab is None:
        with _ab_lock:
            if _ab is None:
                import paper_cs_0406049_b200 as sp
                P, I = ctypes.c_void_p, ctypes.c_int
                sigs = dict(sp._SIGS)
                sigs.update({"sincos_ab_set": (I, [I, I]), "sincos_ab_get": (I, [I]),
                             "sincos_pairs_batched": (I, [P, I, I, P])})
                _ab = sp._load(_build.build_ab(), sigs)
    return _ab


def set_knob(name: str, value) -> int:
    """Set one knob of the A/B build (process-global there); returns the previous value."""
    prev = lib().sincos_ab_set(KNOBS[name], int(value))
    if prev < 0:
        raise ValueError(f"unsupported {name}={value}")
    return prev


def reset():
    for k, v in DEFAULTS.items():
        set_knob(k, v)


@contextlib.contextmanager
def knobs(**kw):
    """Run the binding on the A/B build with the given knobs (others at their defaults)."""
    import paper_cs_0406049_b200 as sp
    L = lib()
    prev_lib = sp._lib
    reset()
    try:
        for k, v in kw.items():
            if k == "launch":                 # (threads, blocks_per_sm, vec, unroll, prefetch)
                for name, x in zip(("threads", "blocks_per_sm", "vec", "unroll", "prefetch"), v):
                    set_knob(name, x)
            else:
                set_knob(k, v)
        sp._lib = L
        yield L
    finally:
        sp._lib = prev_lib
        reset()


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


class BatchTable:
    """A validated, reusable item table for sincos_pairs_batched (the sincos_item_t layout as one
    uint64 array): build it once for a fixed set of buffers, then run() costs one C call.
    Keeps the tensors alive."""

    def __init__(self, thetas, sin_outs=None, cos_outs=None, interleaved_outs=None):
        self.tab = _batch_table(thetas, sin_outs, cos_outs, interleaved_outs)
        self.tensors = (list(thetas), sin_outs, cos_outs, interleaved_outs)
        self.count = len(thetas)

    def run(self, variant=0, stream=None):
        import torch

        import paper_cs_0406049_b200 as sp
        if self.count:
            st = lib().sincos_pairs_batched(self.tab.ctypes.data, self.count, sp._variant(variant),
                                            sp._stream(stream, torch.device("cuda", torch.cuda.current_device())))
            sp._check(st, "sincos_pairs_batched")


def sincos_pairs_batched(thetas, sin_outs=None, cos_outs=None, interleaved_outs=None, variant=0, stream=None):
    """sincos_pairs_batched of the A/B build: many arrays in one launch (per 480 arrays)."""
    BatchTable(thetas, sin_outs, cos_outs, interleaved_outs).run(variant, stream)


# ---- persistent switches for tools/ (a probe process that measures one alternative) ----------
def use(on: bool = True):
    """Route the binding to the A/B build (on) or back to the product library (off)."""
    import paper_cs_0406049_b200 as sp
    sp._lib = lib() if on else None


def set_launch_config(threads=128, blocks_per_sm=0, vec=8, unroll=1, prefetch=0):
    use()
    for name, x in zip(("threads", "blocks_per_sm", "vec", "unroll", "prefetch"),
                       (threads, blocks_per_sm, vec, unroll, prefetch)):
        set_knob(name, x)


def set_realign(v) -> int:
    use()
    return set_knob("realign", v if v in (2, 3) else int(bool(v)))


def set_pdl(on) -> bool:
    use()
    return bool(set_knob("pdl", int(bool(on))))


def set_nudft_packed(on) -> bool:
    use()
    return bool(set_knob("nudft_packed", int(bool(on))))
