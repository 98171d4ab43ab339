"""The C-ABI library without a GPU: it builds for sm_100a, loads, exports every symbol
include/*.h declares, validates arguments before any CUDA call, and its SASS keeps the
value path branch-free (tiers T1 and T5)."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

import paper_cs_0406049_b200 as sp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OK, INVALID, OVERLAP = 0, 1, 2


@pytest.fixture(scope="module")
def L():
    return sp.lib()


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        names |= set(re.findall(r"SINCOS_API\s+[\w\s\*]*?\b(sincos_\w+)\s*\(", src))
    return names


def test_every_declared_symbol_is_exported(L):
    names = declared_symbols()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", sp.library_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sincos_\w+)", out))
    assert names <= exported, names - exported
    assert set(sp.EXPORTS) <= names
    for n in names:
        getattr(L, n)


def test_only_the_abi_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", sp.library_path], capture_output=True, text=True).stdout
    ours = [s for s in re.findall(r"\bT (\w+)", out) if not s.startswith("_")]
    assert set(ours) == declared_symbols(), set(ours) ^ declared_symbols()


def test_version_and_status_strings(L):
    assert b"sm_100a" in L.sincos_version()
    for s in range(5):
        assert L.sincos_status_string(s)
    assert b"NCCL" in L.sincos_status_string(4)


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", sp.library_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


A = 0x10000  # fake, 256-aligned "device" addresses: validation never dereferences them


def test_validation_before_cuda(L):
    # n == 0 is a no-op, pointers may be NULL
    assert L.sincos_pairs(None, None, None, None, 0, 0, None) == OK
    # NULL theta, neither / both output forms, unknown variant
    assert L.sincos_pairs(None, A, 2 * A, None, 16, 0, None) == INVALID
    assert L.sincos_pairs(A, None, None, None, 16, 0, None) == INVALID
    assert L.sincos_pairs(A, 2 * A, 3 * A, 4 * A, 16, 0, None) == INVALID
    assert L.sincos_pairs(A, 2 * A, None, None, 16, 0, None) == INVALID
    assert L.sincos_pairs(A, 2 * A, 3 * A, None, 16, 7, None) == INVALID
    assert L.sincos_pairs(A, 2 * A, 3 * A, None, 16, -1, None) == INVALID
    # not 4-byte aligned
    assert L.sincos_pairs(A + 2, 2 * A, 3 * A, None, 16, 0, None) == INVALID
    assert L.sincos_pairs(A, 2 * A + 1, 3 * A, None, 16, 0, None) == INVALID


def test_overlap_rules(L):
    n = 1024
    # sin and cos overlap
    assert L.sincos_pairs(A, 2 * A, 2 * A + 4 * (n - 1), None, n, 0, None) == OVERLAP
    # partial theta / sin overlap
    assert L.sincos_pairs(A, A + 4, 3 * A, None, n, 0, None) == OVERLAP
    # theta inside the interleaved output
    assert L.sincos_pairs(A + 8, None, None, A, n, 0, None) == OVERLAP
    # exact in-place theta == sin is allowed: passes validation, then needs CUDA
    st = L.sincos_pairs(A, A, 3 * A, None, n, 0, None)
    assert st in (OK, 3)  # 3 = SINCOS_ERR_CUDA here (no GPU)


def test_phase_grid_validation(L):
    """NEXT(1) sincos_phase_grid: same conventions, checked before any CUDA call."""
    f, t = A, 2 * A
    assert L.sincos_phase_grid(None, 0, None, 5, None, None, None, 0, 0, None) == OK       # empty grid
    assert L.sincos_phase_grid(f, 4, t, 8, 3 * A, 4 * A, None, 2, 0, None) == INVALID       # bad units
    assert L.sincos_phase_grid(f, 4, t, 8, 3 * A, 4 * A, None, 0, 5, None) == INVALID       # bad variant
    assert L.sincos_phase_grid(None, 4, t, 8, 3 * A, 4 * A, None, 0, 0, None) == INVALID    # no f
    assert L.sincos_phase_grid(f, 4, t, 8, 3 * A, None, None, 0, 0, None) == INVALID        # half a split form
    assert L.sincos_phase_grid(f, 4, t, 8, 3 * A, 4 * A, 5 * A, 1, 0, None) == INVALID      # both forms
    assert L.sincos_phase_grid(f, 1 << 40, t, 1 << 40, 3 * A, 4 * A, None, 0, 0, None) == INVALID  # overflow
    assert L.sincos_phase_grid(f, 4, t, 8, f + 4, 4 * A, None, 0, 0, None) == OVERLAP       # output over f
    assert L.sincos_phase_grid(f, 4, t, 8, None, None, t - 16, 1, 0, None) == OVERLAP       # output over t
    assert L.sincos_phase_grid(f, 4, t, 8, 3 * A, 3 * A + 64, None, 0, 0, None) == OVERLAP  # sin over cos
    assert L.sincos_phase_grid(f, 4, t, 8, 3 * A, 4 * A, None, 0, 0, None) in (OK, 3)       # valid: needs CUDA


def test_sharded_stats_validation(L):
    """The single-process NCCL stats path refuses bad shard lists before any CUDA call, and binds
    NCCL at run time (libnccl.so.2 is present in this image)."""
    assert sp.nccl_available()
    arr = (sp.Shard * 2)()
    arr[0].device = arr[1].device = 0                       # two shards on one device
    out = (sp.Stats * 2)()
    assert L.sincos_pairs_sharded_stats(arr, 2, 0, out) == INVALID
    assert L.sincos_pairs_sharded_stats(arr, 0, 0, out) == INVALID
    assert L.sincos_pairs_sharded_stats(None, 1, 0, out) == INVALID


def test_host_path_validation(L):
    assert L.sincos_pairs_host(None, None, None, None, 0, 0, None, 0, None) == OK
    buf = (ctypes.c_float * 64)()
    p = ctypes.addressof(buf)
    assert L.sincos_pairs_host(p, p + 64, p + 128, None, 16, 0, None, 1 << 30, None) == INVALID  # no workspace
    assert L.sincos_pairs_host(p, p + 64, p + 128, None, 16, 0, A, 100, None) == INVALID          # too small
    assert L.sincos_pairs_host(p, p + 4, p + 128, None, 16, 0, A, 1 << 30, None) == OVERLAP


def test_no_tuning_state_in_the_product():
    """The product library has one fixed kernel configuration: no setter of launch shape,
    re-alignment, PDL or kernel form is exported (those live in the A/B build only)."""
    out = subprocess.run(["nm", "-D", "--defined-only", sp.library_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sincos_\w+)", out))
    assert not {s for s in exported if "_set_" in s or s.startswith("sincos_ab_") or "batched" in s}, exported
    from paper_cs_0406049_b200 import _build
    ab_out = subprocess.run(["nm", "-D", "--defined-only", _build.build_ab()], capture_output=True, text=True).stdout
    ab_exported = set(re.findall(r"\bT (sincos_\w+)", ab_out))
    assert ab_exported == exported | {"sincos_ab_set", "sincos_ab_get", "sincos_pairs_batched"}, ab_exported ^ exported


def test_ab_knob_validation():
    from paper_cs_0406049_b200 import ab
    L = ab.lib()
    for knob, bad in ((0, 100), (1, -1), (2, 3), (3, 3), (4, 2), (5, 4), (6, 2), (7, 2), (8, 0), (-1, 0)):
        assert L.sincos_ab_set(knob, bad) == -1, (knob, bad)
    assert L.sincos_ab_set(0, 512) == 128 and L.sincos_ab_get(0) == 512
    ab.reset()
    assert [L.sincos_ab_get(k) for k in range(8)] == list(ab.DEFAULTS.values())


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 1000, 1 << 20, (1 << 32) + 5, (1 << 30) + 3])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_shard_range_partitions(n, G):
    """contiguous, 8-element aligned starts, cover [0, n) exactly, balanced."""
    ranges = [sp.shard_range(n, G, g) for g in range(G)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (lo, hi), (lo2, _) in zip(ranges, ranges[1:]):
        assert hi == lo2
    for lo, hi in ranges:
        assert lo % 8 == 0 and lo <= hi
        assert hi - lo <= -(-n // G) + 8
    with pytest.raises(ValueError):
        sp.shard_range(n, G, G)


def test_stats_record_is_64_bytes(L):
    assert ctypes.sizeof(sp.Stats) == 64
    assert L.sincos_stats_workspace_bytes() > 0


def _sass():
    return subprocess.run(["cuobjdump", "-sass", sp.library_path], capture_output=True, text=True).stdout


def test_sass_value_path_branch_free():
    """no CALL/FCHK/BSSY slow paths (as __frcp_rn / __fdiv_rn would bring); the
    variant-A reciprocal is MUFU.RCP + FFMA Newton, variant N has no MUFU at all; no fp64;
    the branch count does not grow with the elements per thread (value path branch-free)."""
    sass = _sass()
    funcs = re.split(r"\n\s*Function : ", sass)
    loop_bra = {f.split("\n", 1)[0]: len(re.findall(r"\bBRA\b", f)) for f in funcs
                if "nudft_partial" in f.split("\n", 1)[0] and "ILi4E" in f.split("\n", 1)[0]}
    seen = 0
    for f in funcs:
        name = f.split("\n", 1)[0]
        if ("sincos_vec_kernel" not in name and "phase_grid_vec" not in name and "nudft_partial" not in name
                and "sincos_shift8_kernel" not in name):
            continue
        body = f
        m = re.search(r"ILi(\d+)E", name)
        tid = int(m.group(1)) if m else -1
        nbra = len(re.findall(r"\bBRA\b", body))
        if tid == 3:
            # the comparison kernel with CUDA's sincosf (radians) carries its large-argument
            # (Payne-Hanek) slow path; sincospif (turns) needs none
            if "ILi3ELb0" in name:
                assert nbra > 16 or " CALL" in body, name
            continue
        if tid == 4:
            continue                     # __sincosf comparison kernel
        seen += 1
        assert " CALL" not in body and "FCHK" not in body, name
        if tid < 16 and "nudft_partial" in name:
            # the fused sum's loops (tiles, chunks, the term loop unrolled by 8 with its
            # remainder) carry more branches: no more than its __sincosf comparison twin, whose
            # per-term path has no value-dependent branch at all
            twin = re.sub(r"ILi\d+E", "ILi4E", name, count=1)
            twin = re.sub(r"(ILi4ELb[01]E)Lb1E", r"\1Lb0E", twin)
            assert nbra <= loop_bra.get(twin, 16), (name, nbra, loop_bra.get(twin))
        elif tid < 16:                   # NEXT(3) kernels also branch on the warp-uniform doubling count
            assert nbra <= 16, (name, nbra)
        if tid == 1 or (tid >= 16 and (tid - 16) % 4 == 1):
            assert re.search(r"MUFU\.RCP\b", body) and "DFMA" not in body and "MUFU.RCP64H" not in body, name
        if tid == 0 or (tid >= 16 and (tid - 16) % 4 != 1):
            assert "MUFU" not in body and "DFMA" not in body, name
        if "sincos_vec_kernel" in name:
            # the loads/stores are the wide streaming forms
            assert re.search(r"LDG\.E\.[A-Z0-9.]*(128|256)", body), name
            assert re.search(r"STG\.E\.[A-Z0-9.]*(128|256)", body), name
    assert seen >= 24 + 42 + 8 + 24       # vector, theta re-aligning (256-bit), phase-grid, fused-sum instances


def test_sass_other_kernel_forms_have_no_slow_paths():
    """The re-aligning (KB3b, KB3c and its hybrid) and phase-grid (row, short-row, staged, tiny)
    forms evaluate the same method: no FCHK (fp32 division slow path), no fp64, and the method's
    reciprocal only in variant A -- each variant-A instance has more MUFU.RCP than its variant-N
    twin (whose MUFU.RCP, where present, belong to integer divisions of an index by a run-time
    row length)."""
    sass = _sass()
    funcs = re.split(r"\n\s*Function : ", sass)
    rcp = {}
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        form = next((k for k in ("sincos_outshift_kernel", "sincos_outshift_hyb_kernel", "phase_grid_staged", "phase_grid_tiny",
                                 "phase_grid_short", "phase_grid_rows") if k in name), None)
        if form is None:
            continue
        m = re.search(r"ILi(\d+)E", name)
        if not m or int(m.group(1)) not in (0, 1):
            continue                     # the no-math ceiling instances
        # (a CALL may appear: the 64-bit integer division of a pair index by the row length)
        assert "FCHK" not in f and "DFMA" not in f and "MUFU.RCP64H" not in f, name
        rcp[name] = len(re.findall(r"MUFU\.RCP\b", f))
    pairs = 0
    for name, k in rcp.items():
        if re.search(r"ILi0E", name):
            twin = name.replace("ILi0E", "ILi1E", 1)
            assert twin in rcp, twin
            assert rcp[twin] > k, (name, k, rcp[twin])
            pairs += 1
    assert pairs >= 64 + 4 + 2 * 2 * 13 + 8, pairs   # outshift split + interleaved, staged, tiny/short/rows


def test_product_never_touches_the_oracle():
    """The oracle is test infrastructure: nothing under the package imports, links or includes it."""
    pkg = os.path.join(ROOT, "paper_cs_0406049_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if not os.path.isfile(path) or path.endswith(".so") or "__pycache__" in path:
            continue
        src = open(path, errors="ignore").read()
        assert not re.search(r"\bimport\s+oracle|from\s+oracle|sincos_oracle|liboracle", src), path


def _nudft_forms(lib_path):
    sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    packed = scalar = 0
    for f in re.split(r"\n\s*Function : ", sass):
        name = f.split("\n", 1)[0]
        if "nudft_partial" not in name:
            continue
        m = re.search(r"nudft_partialILi(\d+)ELb([01])ELb([01])E", name)
        assert m, name
        n2 = len(re.findall(r"\bFFMA2\b", f)) + len(re.findall(r"\bFMUL2\b", f))
        if m.group(3) == "1":
            packed += 1
            assert n2 >= 20 and re.search(r"\bFADD2\b", f), (name, n2)
        else:
            scalar += 1
            assert n2 == 0, (name, n2)
    return packed, scalar


def test_sass_packed_fused_sum_uses_ffma2():
    """The fused sum's kernels (PACK = true, last template flag) run the method and the complex
    MAC on sm_100a's two-lane fp32 instructions.  The product has only those, plus the scalar
    comparison kernels with CUDA's own functions (radians / turns x sincosf / __sincosf); the
    A/B build adds a scalar twin (no FFMA2) of every packed kernel."""
    from paper_cs_0406049_b200 import _build
    packed, scalar = _nudft_forms(sp.library_path)
    assert packed >= 24 and scalar == 4, (packed, scalar)
    packed_ab, scalar_ab = _nudft_forms(_build.build_ab())
    assert packed_ab == packed and scalar_ab == scalar + packed, (packed_ab, scalar_ab)


def test_nudft_chunk_rule():
    """The fused sum's fp32 run length (it enters the error bound): 256 for short sums, else
    1024, whatever nt (longer sums use more segments, not longer fp32 runs)."""
    L = sp.lib()
    assert L.sincos_nudft_chunk(1000) == 256 and L.sincos_nudft_chunk(4095) == 256
    for nt in (4096, 1 << 15, 1 << 26, 65535 * 1024 + 1, 10 ** 9, 1 << 36):
        assert L.sincos_nudft_chunk(nt) == 1024


def test_nudft_workspace_sizes_host_only():
    """Pure host functions: no crash or division by zero on degenerate shapes; 16 B per
    frequency per segment, at most 65535 segments."""
    L = sp.lib()
    for nf, nt in ((0, 0), (0, 5), (5, 0), (1, 1), (1 << 15, 1 << 15), (10, 10 ** 9), (10 ** 6, 100)):
        ws = L.sincos_nudft_workspace_bytes(nf, nt)
        assert ws % 16 == 0 and ws <= 16 * max(nf, 1) * 65535


def test_alignment_checks_of_the_other_entry_points(L):
    """Every entry point refuses pointers its kernels could not access aligned -- before any
    CUDA call (fake addresses are never dereferenced)."""
    P, S, I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    L.sincos_error_stats.argtypes = [P, P, P, P, S, P, P, P]
    L.sincos_error_stats.restype = I
    assert L.sincos_error_stats(A, 2 * A, 3 * A, None, 16, 4 * A + 4, 5 * A, None) == INVALID   # record 4-B
    assert L.sincos_error_stats(A, 2 * A, 3 * A, None, 16, 4 * A, 5 * A + 4, None) == INVALID   # workspace
    assert L.sincos_error_stats(A + 2, 2 * A, 3 * A, None, 16, 4 * A, 5 * A, None) == INVALID   # theta 2-B
    L.sincos_nudft.argtypes = [P, S, P, P, S, P, I, I, P, S, P]
    L.sincos_nudft.restype = I
    ws = L.sincos_nudft_workspace_bytes(100, 5000)
    assert L.sincos_nudft(A, 100, 2 * A, 3 * A, 5000, 4 * A, 0, 0, 5 * A + 8, ws, None) == INVALID  # ws 8-B
    assert L.sincos_nudft(A, 100, 2 * A, 3 * A, 5000, 4 * A, 0, 0, 5 * A, ws - 1, None) == INVALID  # ws short
    assert L.sincos_nudft(A, 100, 2 * A, 3 * A + 4, 5000, 4 * A, 0, 0, 5 * A, ws, None) == INVALID  # a 4-B
    assert L.sincos_nudft(A, 100, 2 * A, 3 * A, 5000, 4 * A + 4, 0, 0, 5 * A, ws, None) == INVALID  # out 4-B
    L.sincos_debug_reciprocal.argtypes = [P, P, S, P]
    L.sincos_debug_reciprocal.restype = I
    assert L.sincos_debug_reciprocal(A + 1, 2 * A, 8, None) == INVALID
    L.sincos_compare_cuda.argtypes = [P, P, P, P, S, I, P]
    L.sincos_compare_cuda.restype = I
    assert L.sincos_compare_cuda(A + 4, 2 * A, 3 * A, None, 64, 3, None) == INVALID          # needs 32-B
    assert L.sincos_compare_cuda(A, 2 * A, 3 * A, None, 64, 5, None) == INVALID              # which
    L.sincos_debug_packed_check.argtypes = [I, P, P, P]
    L.sincos_debug_packed_check.restype = I
    assert L.sincos_debug_packed_check(0, None, A + 4, None) == INVALID
    assert L.sincos_debug_packed_check(7, None, A, None) == INVALID


def test_batched_validation_before_cuda():
    """sincos_pairs_batched (A/B build) validates every item before launching anything (fake
    addresses)."""
    from paper_cs_0406049_b200 import ab
    L = ab.lib()
    Item = ab.Item
    assert L.sincos_pairs_batched(None, 0, 0, None) == OK                 # empty batch
    assert L.sincos_pairs_batched(None, -1, 0, None) == INVALID
    good = Item(A, 2 * A, 3 * A, None, 64)
    bad_forms = Item(A, 2 * A, None, None, 64)                            # half a split form
    bad_align = Item(A + 2, 2 * A, 3 * A, None, 64)
    overlap = Item(A, 2 * A, 2 * A + 8, None, 64)
    for bad, want in ((bad_forms, INVALID), (bad_align, INVALID), (overlap, OVERLAP)):
        arr = (Item * 3)(good, good, bad)
        assert L.sincos_pairs_batched(ctypes.addressof(arr), 3, 0, None) == want
    arr = (Item * 1)(good)
    assert L.sincos_pairs_batched(ctypes.addressof(arr), 1, 9, None) == INVALID  # variant


def test_host_path_binding_refuses_a_host_workspace():
    """The host-buffer path's workspace is device memory: a CPU tensor is refused in Python,
    before the library is called."""
    import torch
    with pytest.raises(ValueError, match="workspace"):
        sp.sincos_pairs_host(torch.zeros(16), torch.zeros(16), torch.zeros(16), workspace=torch.zeros(1 << 20))


def test_binding_refuses_a_stream_of_another_device():
    """A torch stream object of another GPU is refused before the library is called (its queue
    would order the launch against the wrong device's work); a raw handle passes through."""
    import torch

    class FakeStream:                    # the two attributes the binding reads of a torch stream
        def __init__(self, idx):
            self.cuda_stream, self.device = 0x1234, torch.device("cuda", idx)

    assert sp._stream(FakeStream(0), torch.device("cuda", 0)) == 0x1234
    assert sp._stream(0x5678, torch.device("cuda", 0)) == 0x5678
    with pytest.raises(ValueError, match="stream is on cuda:1"):
        sp._stream(FakeStream(1), torch.device("cuda", 0))
