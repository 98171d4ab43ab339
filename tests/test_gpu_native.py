"""The C ABI from a plain C program (tests/c/abi_native.c), linked against libsincos_pairs.so
and the C oracle: compiled here with gcc (no GPU needed to build), run with ``-m gpu``."""
import os
import subprocess

import pytest

import oracle
import paper_cs_0406049_b200 as sp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_driver():
    out = os.path.join(ROOT, "tests", "c", "abi_native")
    lib_dir = os.path.dirname(sp.lib()._name)
    odir = os.path.dirname(oracle.build())
    subprocess.check_call([
        "gcc", "-O2", "-std=c99", "-D_GNU_SOURCE", "-o", out, os.path.join(ROOT, "tests", "c", "abi_native.c"),
        f"-I{CUDA}/include", f"-L{lib_dir}", f"-L{odir}", f"-L{CUDA}/lib64",
        "-lsincos_pairs", "-loracle", "-lcudart", "-lm",
        f"-Wl,-rpath,{lib_dir}:{odir}:{CUDA}/lib64"])
    return out


def test_driver_builds():
    assert os.path.exists(build_driver())


@pytest.mark.gpu
def test_driver_runs_on_the_gpu():
    exe = build_driver()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_native: ok, 0 mismatches" in r.stdout
