"""Build libsincos_pairs.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Flags: -fmad=false (no contraction beyond the explicit __fmaf_rn of Fig. 1),
-ftz=false / -prec-div=true / -prec-sqrt=true (IEEE fp32; never --use_fast_math),
-lineinfo (ncu source view), cudart linked statically (the library runs inside a
torch cu128 process with its own cudart; streams/contexts are shared through
the driver).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsincos_pairs.so")
# the A/B build: the same sources with -DSINCOS_AB (settable kernel forms, csrc/sincos_ab.h);
# loaded by tests/ and tools/ only, never by the product binding
AB_LIB = os.path.join(PKG, "libsincos_pairs_ab.so")
AB_FLAGS = ("-DSINCOS_AB",)
HEADER = os.path.join(ROOT, "include", "sincos_pairs.h")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-shared", "-cudart", "static",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in deps)


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, extra_flags=(), out: str | None = None,
          link_flags=()) -> str:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file), then link the shared
    library (cudart static).  extra_flags: e.g. -D switches for A/B builds; out: another path;
    link_flags: extra flags for the link step (e.g. sanitizer runtimes)."""
    out = out or LIB
    if out in (LIB, AB_LIB) and not force and not _stale(out):
        return out
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static")]
    with tempfile.TemporaryDirectory() as tmp:
        objs = []

        def one(src):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [nvcc(), *compile_flags, *extra_flags, "-c", "-o", obj, src]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            subprocess.check_call(cmd, cwd=PKG)
            return obj

        with ThreadPoolExecutor(max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
            objs = list(ex.map(one, sources()))
        tmp_out = f"{out}.{os.getpid()}.{threading.get_ident()}.tmp"      # renamed into place: atomic
        subprocess.check_call([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                               "-Xcompiler", "-fPIC", *link_flags, "-o", tmp_out, *objs], cwd=PKG)
    os.replace(tmp_out, out)
    return out


def build_ab(force: bool = False) -> str:
    """libsincos_pairs_ab.so (tests and tools only)."""
    return build(force=force, extra_flags=AB_FLAGS, out=AB_LIB)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
    if "--ab" in sys.argv:
        print(build_ab(force="--force" in sys.argv))
