"""The host C code -- the oracle (oracle/*.c) and the input generators (inputs/gen.c) -- under
AddressSanitizer and UndefinedBehaviorSanitizer (SURVEY 4 sanitizer row; CPU only).
tests/c/oracle_sanitize.c calls every entry point on exactly-sized buffers, degenerate shapes
and special values; any sanitizer report aborts it (-fno-sanitize-recover=all)."""
import glob
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_oracle_and_generators_clean_under_asan_ubsan(tmp_path):
    exe = str(tmp_path / "oracle_sanitize")
    srcs = [os.path.join(ROOT, "tests", "c", "oracle_sanitize.c")] + sorted(
        glob.glob(os.path.join(ROOT, "oracle", "*.c"))) + [os.path.join(ROOT, "inputs", "gen.c")]
    cmd = ["gcc", "-std=c99", "-D_GNU_SOURCE", "-O1", "-g", "-fno-omit-frame-pointer", "-ffp-contract=off",
           "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-fopenmp", "-o", exe, *srcs, "-lm"]
    subprocess.check_call(cmd)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1",
               OMP_NUM_THREADS="2")
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "oracle_sanitize: ok" in r.stdout


@pytest.mark.skipif(shutil.which("gcc") is None or shutil.which("nvcc") is None and
                    not os.path.exists("/usr/local/cuda/bin/nvcc"), reason="needs gcc and nvcc")
def test_library_host_logic_clean_under_asan_ubsan(tmp_path):
    """The library's host code (argument validation before any CUDA call, the sharder's
    range arithmetic up to n = 2^64 - 1, workspace sizing) built with
    -fsanitize=address,undefined and driven without a GPU (tests/c/abi_sanitize.py)."""
    import sys
    sys.path.insert(0, ROOT)
    from paper_cs_0406049_b200 import _build
    lib = str(tmp_path / "libsincos_san.so")
    _build.build(extra_flags=["-Xcompiler", "-fsanitize=address,-fsanitize=undefined,-fno-omit-frame-pointer"],
                 out=lib, link_flags=["-Xlinker", "-lasan", "-Xlinker", "-lubsan"])
    pre = " ".join(subprocess.check_output(["gcc", f"-print-file-name={x}"], text=True).strip()
                   for x in ("libasan.so", "libubsan.so"))
    env = dict(os.environ, LD_PRELOAD=pre, ASAN_OPTIONS="detect_leaks=0", UBSAN_OPTIONS="halt_on_error=1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "c", "abi_sanitize.py"), lib],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "san_abi ok" in r.stdout, r.stdout + r.stderr[-3000:]
