"""bench.py -- sincos pairs/s and HBM GB/s of the hot path on N B200 (one process per GPU).

Workload: BASELINE.json configs[1] ("C2"): 2^28 fp32 angles
U[-1e4, 1e4] (seed 1) per GPU, split sin/cos outputs, BOTH coefficient variants.
One step = one pass of the whole hot path over the batch for each variant (two
kernel launches, 2 x 2^28 pairs).  At N GPUs every rank owns a contiguous 2^28-
element shard of the same counter-based stream (weak scaling; no collective on
the data path).  Inputs (1 GiB) exceed L2 (126 MB), so no flush between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle on the host
cores instead (the tier's reference arm; rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402

CONFIG_ID = 2                       # BASELINE.json configs[1]
N_PER_RANK = 1 << 28
BYTES_PER_PAIR = 12                 # 4 B theta in + 8 B (sin, cos) out -- SURVEY 8(d)
METRIC = "sincos pairs/sec and achieved HBM GB/s vs peak at 1/2/4/8 B200; max error"
WORKLOAD = "C2: 2^28 fp32 angles U[-1e4,1e4] seed 1 per GPU, split sin/cos, both variants (N then A) per step"
L2_FLUSH_BYTES = 512 << 20         # > 4x the 126 MB L2: written before every step of the small configs
FALLBACK_HBM_GBS = 6650.0           # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="BASELINE config (default c2 = configs[1], weak scaling; c1/c3/c4/c5 strong, sharded)")
    # (not "--n": torch.distributed.run would take it for an abbreviation of its own options)
    ap.add_argument("--n-per-rank", dest="n", type=int, default=N_PER_RANK,
                    help="elements per rank for c2 (default 2^28)")
    ap.add_argument("--e2e-max", type=int, default=1 << 28, help="elements per rank in the e2e leg")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded oracle sample for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the NEXT-row side measurements")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for the stats gather / time max (gloo: flow testing only)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (flow testing of the N>1 host path on a 1-GPU box; gloo only)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, burst)"
        except (ValueError, KeyError, TypeError) as e:
            return FALLBACK_HBM_GBS, f"fallback (B200_PROFILING.md; MEASURED_PEAKS.json unreadable: {e!r})"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(n, interleaved=False):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu captures
    (the full-set capture of the bench kernel, else the per-config DRAM capture for this n and
    layout: profiles/ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        k = d.get("dominant", {})
        if int(k.get("n", -1)) == n and not interleaved:
            return float(k["dram_bytes_read"]) + float(k["dram_bytes_write"])
        for c in d.get("by_config", {}).values():
            if int(c["n"]) == n and bool(c["interleaved"]) == bool(interleaved):
                return float(c["dram_bytes_read"]) + float(c["dram_bytes_write"])
    except Exception:
        pass
    return None


# ---- clocks during the timed region (NVML, polled) ------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, local_rank):
        self.samples, self.mem, self.reasons, self.ok = [], [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [x for x in vis.split(",") if x.strip()]
            index = int(ids[local_rank]) if local_rank < len(ids) and ids[local_rank].strip().isdigit() else local_rank
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report null clocks
            self.err = repr(e)
        self._stop = threading.Event()

    def _run(self):
        # SM clock and event reasons as fast as NVML answers (the C2 timed region is ~20 ms);
        # the memory clock every 8th sample
        k = 0
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                if k % 8 == 0:
                    self.mem.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_MEM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            k += 1
            time.sleep(0.0002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "mem_mhz": statistics.median(self.mem) if self.mem else None,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ---- the oracle as a CPU baseline ---------------------------------------------------------
def cpu_oracle_rate(theta: np.ndarray, seconds: float, workload: str = "C2"):
    """Time the oracle as it stands on all host cores (chunked threads; ctypes releases the
    GIL) on a bounded prefix of the workload, both variants alternately, until `seconds`."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    cores = os.cpu_count() or 1
    chunk = 1 << 18
    m = min(theta.size, chunk * cores * 4)
    th = np.ascontiguousarray(theta[:m])
    s = np.empty_like(th)
    c = np.empty_like(th)
    spans = [(i, min(i + chunk, m)) for i in range(0, m, chunk)]
    pairs, t0 = 0, time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        v = 0
        while True:
            list(ex.map(lambda ab: oracle.sincos_into(th[ab[0]:ab[1]], s[ab[0]:ab[1]], c[ab[0]:ab[1]], v), spans))
            pairs += m
            v ^= 1
            if time.perf_counter() - t0 >= seconds and v == 0:
                break
    dt = time.perf_counter() - t0
    # one thread as well, on a 2^22-element prefix, both variants
    m1 = min(m, 1 << 22)
    t1 = time.perf_counter()
    for v in (0, 1):
        oracle.sincos_into(th[:m1], s[:m1], c[:m1], v)
    one = 2 * m1 / (time.perf_counter() - t1)
    cpu_model = ""
    try:
        cpu_model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        pass
    libm = libm_sincosf_rate(th, s, c, cores, min(seconds, 3.0))
    return {"value": pairs / dt, "unit": "pairs/s", "cores": cores, "kind": "oracle",
            "sample": f"first {m} elements of the {workload} workload, variants N and A alternately, "
                      f"{pairs} pairs in {dt:.1f} s on {cores} threads (plain scalar C oracle)",
            "seconds": dt, "ns_per_pair": 1e9 * dt / pairs, "GBps": 12 * pairs / dt / 1e9,
            "single_thread_pairs_per_s": one, "single_thread_ns_per_pair": 1e9 / one,
            "single_thread_sample": f"first {m1} elements, both variants", "cpu_model": cpu_model,
            "context_glibc_sincosf": libm}


def libm_sincosf_rate(th, s, c, cores, seconds):
    """Context only (SURVEY 8(d) optional row): glibc sincosf over the same sample on all host
    cores (tools/libm_baseline.c, compiled here with gcc); None if no compiler."""
    import ctypes
    import subprocess
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    try:
        so = os.path.join(tempfile.gettempdir(), f"libm_baseline_{os.getpid()}.so")
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", so,
                               os.path.join(ROOT, "tools", "libm_baseline.c"), "-lm"])
        L = ctypes.CDLL(so)
        L.libm_sincosf_array.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
    except Exception as e:
        return {"error": repr(e)}
    chunk = 1 << 18
    m = th.size
    spans = [(i, min(i + chunk, m)) for i in range(0, m, chunk)]
    pairs, t0 = 0, time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        while time.perf_counter() - t0 < seconds:
            list(ex.map(lambda ab: L.libm_sincosf_array(th[ab[0]:ab[1]].ctypes.data, s[ab[0]:ab[1]].ctypes.data,
                                                        c[ab[0]:ab[1]].ctypes.data, ab[1] - ab[0]), spans))
            pairs += m
    dt = time.perf_counter() - t0
    try:
        os.remove(so)
    except OSError:
        pass
    return {"value": pairs / dt, "unit": "pairs/s", "cores": cores, "what": "glibc sincosf, not the method"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    per_step = min(args.n, 1 << 22)
    th = inputs.generate(CONFIG_ID, 0, per_step)
    # warm-up and timed steps: each step = the oracle over a bounded sample, both variants
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    cores = os.cpu_count() or 1
    chunk = 1 << 18
    sample = np.ascontiguousarray(th[:per_step])
    s = np.empty_like(sample)
    c = np.empty_like(sample)
    spans = [(i, min(i + chunk, per_step)) for i in range(0, per_step, chunk)]

    def step(ex):
        for v in (0, 1):
            list(ex.map(lambda ab: oracle.sincos_into(sample[ab[0]:ab[1]], s[ab[0]:ab[1]], c[ab[0]:ab[1]], v),
                        spans))

    with ThreadPoolExecutor(cores) as ex:
        for _ in range(args.warmup):
            step(ex)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step(ex)
        dt = time.perf_counter() - t0
    pairs = 2 * per_step * args.steps
    val = pairs / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD + f"; reference arm: CPU oracle on a {per_step}-element prefix per "
                                          "variant per step", "n_per_rank": args.n},
        "cpu_baseline": {"value": val, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {per_step} elements of C2 per variant per step, {args.steps} steps"},
        "e2e": {"value": val, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm -------------------------------------------------------------------------------
def host_input(W, lo, hi, pinned=True):
    """This rank's inputs [lo, hi) of the workload's counter stream, generated on the host."""
    import torch
    t = torch.empty(hi - lo, dtype=torch.float32)
    if pinned:
        t = t.pin_memory()
    # this rank's share of the host cores (a launcher sets OMP_NUM_THREADS=1 per rank)
    local = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    inputs.generate(W.config, lo, hi - lo, out=t.numpy(), nthreads=max(1, (os.cpu_count() or 1) // local))
    return t


def c4_axes(turns):
    """BASELINE configs[3] axes (2^15 frequencies x 2^15 jittered times); radians: fl32(2 pi f)."""
    nf = nt = 1 << 15
    f = np.array([512.0 * inputs.urand(3, 0, i) for i in range(nf)])
    t = np.array([(j + inputs.urand(3, 1, j)) * 2.0 ** -15 for j in range(nt)])
    if not turns:
        f = 2 * np.pi * f
    return f.astype(np.float32), t.astype(np.float32)


def measure_phase_grid(dev, stream, peak, reps=10):
    """NEXT(1) side measurement (outside the timed region of the main metric): the C4 phase
    grid formed in the kernel (sincos_phase_grid, interleaved, 8 B written per pair, nothing
    read), against the materialised path (theta array in HBM: 12 B per pair)."""
    import torch

    import paper_cs_0406049_b200 as sp
    out = {"workload": "C4 shape: 2^15 f x 2^15 t = 2^30 pairs, interleaved {cos, sin}, phases formed in-kernel",
           "bytes_per_pair": 8, "peak": peak, "unit": "GB/s"}
    o = torch.empty(2 << 30, dtype=torch.float32, device=dev)
    for units, uname in ((sp.RADIANS, "radians"), (sp.TURNS, "turns")):
        f, t = c4_axes(units == sp.TURNS)
        fd, td = torch.from_numpy(f).to(dev), torch.from_numpy(t).to(dev)
        for v, vname in ((sp.NORMALIZED, "N"), (sp.RENORMALIZED, "A")):
            for _ in range(2):
                sp.phase_grid(fd, td, interleaved_out=o, units=units, variant=v, stream=stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                sp.phase_grid(fd, td, interleaved_out=o, units=units, variant=v, stream=stream)
            b.record(stream)
            torch.cuda.synchronize(dev)
            ms = a.elapsed_time(b) / reps
            gbs = 8 * (1 << 30) / (ms / 1e3) / 1e9
            out[f"{uname}_{vname}"] = {"ms": ms, "pairs_per_s": (1 << 30) / (ms / 1e3), "GBps": gbs,
                                       "frac": gbs / peak}
    # ragged rows (not whole 256-bit vectors): the row kernel (nt = 2^15 - 1), the short-row
    # kernel (nt = 1001) and the staged short-row kernel (nt = 5), turns, variant N, ~2^30 pairs each
    for nt in ((1 << 15) - 1, 1001, 5):
        nf = (1 << 30) // nt
        fd = torch.rand(nf, device=dev, generator=torch.Generator(device=dev).manual_seed(5)) * 512
        td = torch.rand(nt, device=dev, generator=torch.Generator(device=dev).manual_seed(6))
        oo = o[: 2 * nf * nt]
        for _ in range(2):
            sp.phase_grid(fd, td, interleaved_out=oo, units=sp.TURNS, variant=sp.NORMALIZED, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            sp.phase_grid(fd, td, interleaved_out=oo, units=sp.TURNS, variant=sp.NORMALIZED, stream=stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        gbs = 8 * nf * nt / (ms / 1e3) / 1e9
        out[f"ragged_nt{nt}_turns_N"] = {"nf": nf, "nt": nt, "ms": ms, "pairs_per_s": nf * nt / (ms / 1e3),
                                         "GBps": gbs, "frac": gbs / peak,
                                         "GBps_with_f_reads": (8 + 4 / nt) * nf * nt / (ms / 1e3) / 1e9,
                                         "kernel": "row" if nt >= 1024 else "short-row" if nt > 7 else "staged"}
    del o
    torch.cuda.empty_cache()
    return out


def fit_method(doublings, n_ss, n_cc):
    """NEXT(3): a regenerated angle-accurate method (coeff_fit, exact reciprocal fix)."""
    import paper_cs_0406049_b200 as sp
    from paper_cs_0406049_b200 import coeff_fit
    ss, cc = coeff_fit.fit_angle(doublings, n_ss, n_cc).fp32()
    return sp.make_method(list(ss), list(cc), doublings, sp.FIX_RECIPROCAL)


def measure_methods(dev, stream, th, outs, peak, reps=10):
    """NEXT(3) side measurement: sincos_pairs_method on the C2 batch (HBM-bound like the hot
    path) for the paper's tables and a regenerated 1-doubling method."""
    import torch

    import paper_cs_0406049_b200 as sp
    n = th.numel()
    res = {"workload": "C2 batch, split outputs", "bytes_per_pair": BYTES_PER_PAIR, "peak": peak}
    for name, m in (("paper_N_table", sp.make_method(*sp.PAPER_METHODS[sp.NORMALIZED])),
                    ("paper_A_table", sp.make_method(*sp.PAPER_METHODS[sp.RENORMALIZED])),
                    ("angle_fit_1dbl_deg3_2", fit_method(1, 3, 2))):
        s, c = outs
        for _ in range(2):
            sp.sincos_pairs_method(th, m, s, c, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            sp.sincos_pairs_method(th, m, s, c, stream=stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        gbs = BYTES_PER_PAIR * n / (ms / 1e3) / 1e9
        res[name] = {"ms": ms, "GBps": gbs, "frac": gbs / peak}
    return res


def measure_cuda_functions(dev, stream, th, outs, peak, reps=10):
    """Context (SURVEY 8(d) optional rows): the hot path's kernel shape with CUDA's sincosf and
    __sincosf instead of the paper's method, same 12 B/pair traffic on the C2 batch -- an
    HBM-bound kernel sits at the same roofline whatever the per-element math."""
    import torch

    import paper_cs_0406049_b200 as sp
    n = th.numel()
    res = {"workload": "C2 batch, split outputs", "bytes_per_pair": BYTES_PER_PAIR, "peak": peak,
           "note": "not the paper's method; context only"}
    s, c = outs
    for which, name in ((3, "cuda_sincosf"), (4, "cuda___sincosf")):
        for _ in range(2):
            sp.compare_cuda(th, s, c, which=which, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            sp.compare_cuda(th, s, c, which=which, stream=stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        gbs = BYTES_PER_PAIR * n / (ms / 1e3) / 1e9
        res[name] = {"ms": ms, "GBps": gbs, "frac": gbs / peak}
    return res


def measure_dtypes(dev, stream, th, peak, reps=10):
    """NEXT(4) side measurement: sincos_pairs_dtype with 16-bit split outputs on the C2 batch
    (8 algorithmic bytes per pair: 4 in, 2 x 2 out)."""
    import torch

    import paper_cs_0406049_b200 as sp
    n = th.numel()
    res = {"workload": "C2 batch, split 16-bit outputs", "bytes_per_pair": 8, "peak": peak}
    for dt, name in ((torch.float16, "fp16"), (torch.bfloat16, "bf16")):
        s = torch.empty(n, dtype=dt, device=dev)
        c = torch.empty(n, dtype=dt, device=dev)
        for v, vname in ((sp.NORMALIZED, "N"), (sp.RENORMALIZED, "A")):
            for _ in range(2):
                sp.sincos_pairs_dtype(th, s, c, variant=v, stream=stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                sp.sincos_pairs_dtype(th, s, c, variant=v, stream=stream)
            b.record(stream)
            torch.cuda.synchronize(dev)
            ms = a.elapsed_time(b) / reps
            gbs = 8 * n / (ms / 1e3) / 1e9
            res[f"{name}_{vname}"] = {"ms": ms, "pairs_per_s": n / (ms / 1e3), "GBps": gbs, "frac": gbs / peak}
        del s, c
    return res


ALU_PEAK_OPS = 148 * 128 * 1.965e9   # FP32-pipe lane-ops/s at the max SM clock (FMA = 1 op)
# algorithmic FP32-pipe ops per term of the fused sum, variant N: the phase product (1), the
# method (11 FMUL + 10 FFMA + 1 FADD + 1 FRND = 23; turns skips the 1/2pi FMUL), the complex MAC (4)
NUDFT_OPS = {"radians": 28, "turns": 27}
# variant A: the fix f = RN(1/d) instead of N's two FFMA -- d = fma(s2, s2, RN(c2 c2)) (FMUL + FFMA)
# and the Newton step on the MUFU.RCP seed (2 FFMA; the MUFU itself issues on the XU pipe): +2
NUDFT_OPS_A = {"radians": 30, "turns": 29}


def measure_nudft(dev, stream, reps=5):
    """NEXT(2) side measurement: the fused Huygens / non-uniform Fourier sum at the C4 shape
    (2^15 frequencies x 2^15 jittered times = 2^30 terms, random complex amplitudes).  FP32-ALU
    bound: achieved = algorithmic FP32-pipe ops/s vs 148 SMs x 128 lanes x 1.965 GHz.  The same
    fused kernel with CUDA's sincosf (sincospif in turns) and __sincosf is timed as context."""
    import torch

    import paper_cs_0406049_b200 as sp
    nf = nt = 1 << 15
    rng = np.random.default_rng(7)
    a = torch.from_numpy((rng.normal(size=nt) + 1j * rng.normal(size=nt)).astype(np.complex64)).to(dev)
    out = torch.empty(nf, dtype=torch.complex64, device=dev)
    ws = torch.empty(sp.lib().sincos_nudft_workspace_bytes(nf, nt), dtype=torch.uint8, device=dev)
    res = {"workload": "C4 shape: 2^15 f x 2^15 t = 2^30 terms, complex64 amplitudes", "bound": "alu",
           "peak_ops_per_s": ALU_PEAK_OPS, "ops_per_term": NUDFT_OPS, "ops_per_term_A": NUDFT_OPS_A,
           "kernel": "packed fp32 (FFMA2/FMUL2/FADD2, two frequencies per instruction)"}
    ks = torch.arange(0, nf, nf // 16, device=dev)
    asum = float(a.abs().sum())
    for units, uname in ((sp.RADIANS, "radians"), (sp.TURNS, "turns")):
        f, t = c4_axes(units == sp.TURNS)
        fd, td = torch.from_numpy(f).to(dev), torch.from_numpy(t).to(dev)
        # fp64 reference of 16 sampled outputs (torch, complex128): sum_j a_j exp(i p_kj) with the
        # same rounded phases p_kj = RN(f_k t_j) -- measures each variant's pair error
        p = (fd[ks, None] * td[None, :]).double()
        ang = p if units == sp.RADIANS else 2 * np.pi * (p - torch.round(p))
        ref = (a.to(torch.complex128)[None, :] * torch.exp(1j * ang)).sum(dim=1)
        for v, vname in ((sp.NORMALIZED, "N"), (sp.RENORMALIZED, "A"), (sp.CMP_LIBM_SINCOSF, "cuda_sincosf"),
                         (sp.CMP_INTRINSIC_SINCOSF, "cuda___sincosf"), ("m132", "method_1dbl_deg3_2_angle")):
            kw = {"method": fit_method(1, 3, 2)} if v == "m132" else {"variant": v}
            sp.nudft(fd, td, a, out=out, units=units, workspace=ws, stream=stream, **kw)
            err = float((out[ks].to(torch.complex128) - ref).abs().max()) / asum
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                sp.nudft(fd, td, a, out=out, units=units, workspace=ws, stream=stream, **kw)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / reps
            terms = (nf * nt) / (ms / 1e3)
            r = {"ms": ms, "terms_per_s": terms, "max_err_over_sum_abs_a": err}
            if vname in ("N", "A"):
                r["alu_frac"] = terms * (NUDFT_OPS if vname == "N" else NUDFT_OPS_A)[uname] / ALU_PEAK_OPS
            res[f"{uname}_{vname}"] = r
    return res


def pcie_roofline(th_h, n, nvar, dev, outs_h):
    """The e2e leg's ceiling: one step's bytes (nvar x 4n B H2D, nvar x 8n B D2H) through plain
    pinned cudaMemcpyAsync copies between the pipeline's OWN host buffers (theta in, the output
    arrays out) and the device -- each direction alone, and both directions concurrently on two
    streams, which is how the pipeline runs them.  step_floor_ms = the concurrent time (the
    binding one when the link is not fully duplex), never less than either direction alone.
    (The same buffers: on these VMs the pinned pages of one allocation can sit behind a slower
    host path than another's -- a whole e2e run once read 0.89 of a roofline measured on a
    separate buffer.)"""
    import torch
    dbuf = torch.empty(2 * n, dtype=torch.float32, device=dev)
    outs = [o.view(-1) for o in outs_h]          # sin, cos (n each) or interleaved (2n)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(h2d, d2h):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize(dev)
        if h2d:
            ev[0].record(s_in)
            with torch.cuda.stream(s_in):
                for _ in range(nvar):
                    dbuf[:n].copy_(th_h, non_blocking=True)
            ev[1].record(s_in)
        if d2h:
            ev[2].record(s_out)
            with torch.cuda.stream(s_out):
                for _ in range(nvar):
                    off = 0
                    for o in outs:
                        o.copy_(dbuf[off:off + o.numel()], non_blocking=True)
                        off += o.numel()
            ev[3].record(s_out)
        torch.cuda.synchronize(dev)
        ms_in = ev[0].elapsed_time(ev[1]) if h2d else 0.0
        ms_out = ev[2].elapsed_time(ev[3]) if d2h else 0.0
        return ms_in, ms_out

    for _ in range(2):
        timed(True, True)
    ms_h2d = min(timed(True, False)[0] for _ in range(3))
    ms_d2h = min(timed(False, True)[1] for _ in range(3))
    both = min((max(r[0], r[1]) for r in (timed(True, True) for _ in range(3))))
    floor = max(both, ms_h2d, ms_d2h)
    del dbuf
    return {"h2d_GBps": nvar * 4 * n / (ms_h2d / 1e3) / 1e9, "d2h_GBps": nvar * 8 * n / (ms_d2h / 1e3) / 1e9,
            "h2d_ms": ms_h2d, "d2h_ms": ms_d2h, "concurrent_ms": both, "step_floor_ms": floor,
            "how": "pinned copies of one step's bytes between the pipeline's own host buffers and the device; "
                   "concurrent = H2D and D2H on two streams at once (max of the two event spans); best of 3"}


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_cs_0406049_b200 as sp
    from paper_cs_0406049_b200.sharding import WORKLOADS, gather_records, max_over_ranks, summarize

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cdev = dev if args.backend == "nccl" else None      # where the collectives' tensors live
    W = WORKLOADS[args.workload]
    if args.n and args.workload == "c2":
        W = type(W)(**{**W.__dict__, "n": args.n})
    lo, hi = W.rank_range(world, rank)
    n = hi - lo
    variants = (sp.NORMALIZED, sp.RENORMALIZED)
    stream = torch.cuda.current_stream(dev)

    # inputs resident in HBM before timing (H2D excluded here; the e2e leg includes it)
    e2e_n = min(n, args.e2e_max)
    th_h = host_input(W, lo, lo + e2e_n, pinned=True)
    th = torch.empty(n, dtype=torch.float32, device=dev)
    th[:e2e_n].copy_(th_h)
    chunk = 1 << 28
    for off in range(e2e_n, n, chunk):
        m = min(chunk, n - off)
        th[off:off + m].copy_(host_input(W, lo + off, lo + off + m, pinned=False))

    def alloc_out():
        if W.interleaved:
            return {"interleaved_out": torch.empty(2 * n, dtype=torch.float32, device=dev)}
        return {"sin_out": torch.empty(n, dtype=torch.float32, device=dev),
                "cos_out": torch.empty(n, dtype=torch.float32, device=dev)}

    outs = {v: alloc_out() for v in variants}

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 3)):
        for v in variants:
            sp.sincos_pairs(th, variant=v, stream=stream, **outs[v])
    # Launch-bound (L2-resident) workloads replay the step from a CUDA graph: the whole step (one
    # launch per variant) captured once on a side stream and replayed once per step, so host launch
    # latency does not set the time.  The per-kernel durations then come from graphs of GRAPH_REPS
    # back-to-back launches of one variant (untimed for the metric), i.e. the kernel's own time.
    use_graph = 12 * n < (256 << 20)
    GRAPH_REPS = 20
    if use_graph:
        cap = torch.cuda.Stream(dev)
        side = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        step_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(step_graph, stream=cap):
            # the two variants are independent (same theta, separate outputs): two graph branches,
            # so the latency-bound small launches overlap instead of running back to back
            side.wait_stream(cap)
            sp.sincos_pairs(th, variant=variants[0], stream=cap, **outs[variants[0]])
            sp.sincos_pairs(th, variant=variants[1], stream=side, **outs[variants[1]])
            cap.wait_stream(side)
        rep_graphs = {}
        for v in variants:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                for _ in range(GRAPH_REPS):
                    sp.sincos_pairs(th, variant=v, stream=cap, **outs[v])
            rep_graphs[v] = g
        stream.wait_stream(cap)
        torch.cuda.synchronize(dev)
        for _ in range(3):
            step_graph.replay()

    # CUDA events on the launching stream bracket the timed region.  No event between the launches:
    # a recorded event breaks the programmatic-dependent-launch overlap of back-to-back kernels
    # (~1.5% of a step), so the kernels' average launch duration is the region's
    # time over its launches (both launches are the one streaming kernel, variant N and variant A),
    # and the per-variant split is timed after the region, each variant back to back.
    # Working sets below 2x the 126 MB L2 (C1, C3): L2 is flushed before every step (a 512 MiB
    # write, outside the timed spans) and each step is timed by its own pair of events; the
    # device time is the sum of the step spans.
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev) if use_graph else None
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    spans = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)] if use_graph else []
    barrier()
    launches0 = sp.launch_count()
    with ClockSampler(local_rank) as clk:
        wall0 = time.perf_counter()          # host wall clock: from the barrier to the final sync
        t_start.record(stream)
        for k in range(args.steps):
            if use_graph:
                flush.fill_(float(k))
                spans[k][0].record(stream)
                step_graph.replay()
                spans[k][1].record(stream)
                continue
            for v in variants:
                sp.sincos_pairs(th, variant=v, stream=stream, **outs[v])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        wall_ms = 1e3 * (time.perf_counter() - wall0)
    barrier()
    launches = sp.launch_count() - launches0 if not use_graph else len(variants) * args.steps
    region_ms = sum(a_.elapsed_time(b_) for a_, b_ in spans) if use_graph else t_start.elapsed_time(t_end)
    ms_max = max_over_ranks(region_ms, world, cdev)
    wall_ms_max = max_over_ranks(wall_ms, world, cdev)
    if use_graph:
        per_kernel = {v: [] for v in variants}
        for _ in range(5):
            for v in variants:
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                flush.fill_(0.0)
                a_.record(stream)
                rep_graphs[v].replay()
                b_.record(stream)
                torch.cuda.synchronize(dev)
                per_kernel[v].append(a_.elapsed_time(b_) / GRAPH_REPS)
    else:
        # per variant, untimed: R launches of one variant back to back between two events
        per_kernel = {v: [] for v in variants}
        for _ in range(3):
            for v in variants:
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                for _ in range(5):
                    sp.sincos_pairs(th, variant=v, stream=stream, **outs[v])
                b_.record(stream)
                torch.cuda.synchronize(dev)
                per_kernel[v].append(a_.elapsed_time(b_) / 5)
    units_all = W.n * world if W.weak else W.n
    pairs_total = len(variants) * units_all * args.steps
    value = pairs_total / (ms_max / 1e3)

    # roofline of the dominant kernel on this rank: the streaming kernel's average launch duration
    # over the timed region (graph-replayed sizes: the per-variant graphs of back-to-back launches)
    avg = {v: statistics.mean(per_kernel[v]) for v in variants}
    dom = max(variants, key=lambda v: avg[v])
    peak, peak_src = peaks()
    launch_ms = avg[dom] if use_graph else t_start.elapsed_time(t_end) / (len(variants) * args.steps)
    achieved = BYTES_PER_PAIR * n / (launch_ms / 1e3) / 1e9
    vname = {0: "N", 1: "A"}
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(n, W.interleaved),
            "kernel": ("sincos_vec_kernel variant " + vname[dom]) if use_graph else
                      "sincos_vec_kernel (variants N and A alternating; average launch over the timed region)",
            "launch_ms": launch_ms, "bytes_per_launch": BYTES_PER_PAIR * n,
            "bytes_per_pair": BYTES_PER_PAIR, "peak_source": peak_src,
            "traffic_source": "profiles/ncu_summary.json (ncu --set full of this kernel; summary in "
                              "profiles/ncu_r02_summary.txt, launch list profiles/ncu_launches_r02.csv)",
            "frac_of_theoretical_8180": achieved / 8180.0,
            # B200_PROFILING.md: 7.7 TB/s is the HGX B200 HBM3e spec figure (8 TB/s DGX); 8180 is
            # the 3996 MHz memory clock x 2 x 8192 bits
            "frac_of_spec_7700": achieved / 7700.0,
            "per_variant_GBps": {vname[v]: BYTES_PER_PAIR * n / (avg[v] / 1e3) / 1e9 for v in variants},
            "per_variant_ms": {vname[v]: avg[v] for v in variants},
            "per_variant_how": "after the timed region: 3 x 5 launches of each variant back to back",
            "per_variant_ms_median_min": {vname[v]: [statistics.median(per_kernel[v]), min(per_kernel[v])]
                                          for v in variants}}

    # traffic ceiling: same access pattern and launch, no arithmetic (outside the timed region)
    o = outs[sp.NORMALIZED]
    for _ in range(3):
        sp.null_4in8out(th, stream=stream, **o)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    if use_graph:       # same launch mode as the kernels it bounds
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        null_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(null_graph, stream=cap):
            for _ in range(GRAPH_REPS):
                sp.null_4in8out(th, stream=cap, **o)
        stream.wait_stream(cap)
        null_graph.replay()
        reps = GRAPH_REPS
    e0.record(stream)
    if use_graph:
        null_graph.replay()
    else:
        for _ in range(reps):
            sp.null_4in8out(th, stream=stream, **o)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    null_ms = e0.elapsed_time(e1) / reps
    roof["ceiling_kernel_GBps"] = BYTES_PER_PAIR * n / (null_ms / 1e3) / 1e9
    roof["kernel_over_ceiling"] = null_ms / launch_ms

    # per-shard error statistics (fp64, on the device), gathered over NCCL -- not timed
    for v in variants:
        sp.sincos_pairs(th, variant=v, stream=stream, **outs[v])
    recs = []
    for v in variants:
        st = sp.error_stats(th, stream=stream, **outs[v])
        recs.append([float(st["n"]), float(st["nan_count"]), st["max_comb"], st["sum_sq"], st["max_amp"],
                     avg[v], float(rank), float(v)])
    summary = summarize(gather_records(recs, world, cdev))

    # end to end through the C ABI with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        if W.interleaved:
            oh = {"interleaved_out": torch.empty(2 * e2e_n, dtype=torch.float32).pin_memory()}
        else:
            oh = {"sin_out": torch.empty(e2e_n, dtype=torch.float32).pin_memory(),
                  "cos_out": torch.empty(e2e_n, dtype=torch.float32).pin_memory()}

        def e2e_step():
            for v in variants:
                sp.sincos_pairs_host(th_h, variant=v, workspace=ws, stream=stream, **oh)

        e2e_step()
        # the e2e roofline (below) is measured right before and right after the timed steps, the
        # better of the two kept: a slow phase of the host (these are VMs) then cannot fall on
        # the ceiling alone
        roof_before = pcie_roofline(th_h, e2e_n, len(variants), dev, list(oh.values()))
        barrier()
        k2 = max(1, min(args.e2e_steps, args.steps))
        # events on the caller's stream between the (synchronous) steps: each step's span
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(k2 + 1)]
        marks[0].record(stream)
        for k in range(k2):
            e2e_step()
            marks[k + 1].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        t2 = max_over_ranks(marks[0].elapsed_time(marks[-1]), world, cdev)
        step_ms = [marks[k].elapsed_time(marks[k + 1]) for k in range(k2)]
        e2e = {"value": world * len(variants) * e2e_n * k2 / (t2 / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": len(variants) * 4 * e2e_n, "d2h_bytes_per_step": len(variants) * 8 * e2e_n,
               "steps": k2, "elements_per_rank": e2e_n,
               "step_ms_min_median_max": [min(step_ms), statistics.median(step_ms), max(step_ms)],
               "path": "sincos_pairs_host: pinned host buffers, chunked H2D -> kernel -> D2H over 3 streams"}
        # the e2e roofline: one step's bytes through the PCIe copy engines with plain pinned copies,
        # H2D and D2H issued concurrently on two streams (as the pipeline runs them) and each alone
        roof_after = pcie_roofline(th_h, e2e_n, len(variants), dev, list(oh.values()))
        e2e["pcie"] = min((roof_before, roof_after), key=lambda r: r["step_floor_ms"])
        e2e["pcie"]["step_floor_ms_before_after"] = [roof_before["step_floor_ms"], roof_after["step_floor_ms"]]
        e2e["pcie"]["roofline_pairs_per_s"] = world * len(variants) * e2e_n / (e2e["pcie"]["step_floor_ms"] / 1e3)
        e2e["frac_of_pcie_roofline"] = e2e["value"] / e2e["pcie"]["roofline_pairs_per_s"]
        del ws, oh

    # every rank's clocks (the collectives end here; rank 0 alone continues)
    clocks = clk.result()
    clocks_all = [clocks]
    if world > 1:
        import torch.distributed as dist
        clocks_all = [None] * world
        dist.all_gather_object(clocks_all, clocks)
    nccl = None
    if world > 1:
        import torch.distributed as dist
        nccl = {"backend": dist.get_backend(), "comm_nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if args.backend == "nccl" else None,
                "same_device": bool(args.same_device),
                "nccl_init_log": nccl_init_lines() if rank == 0 and args.backend == "nccl" else None}
        # every collective is done: all ranks tear the process group down together, so rank 0's
        # remaining single-rank work (NEXT side measurements, the CPU baseline) never runs with a
        # communicator whose peers have exited
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return

    methods_res = None
    if not args.no_next and not W.interleaved:
        o = outs[sp.NORMALIZED]
        methods_res = measure_methods(dev, stream, th, (o["sin_out"], o["cos_out"]), peak)
        methods_res["dtypes"] = measure_dtypes(dev, stream, th, peak)
        methods_res["context_cuda_functions"] = measure_cuda_functions(dev, stream, th,
                                                                       (o["sin_out"], o["cos_out"]), peak)

    fused = nudft_res = None
    if not args.no_next:
        del outs
        torch.cuda.empty_cache()
        fused = measure_phase_grid(dev, stream, peak)
        nudft_res = measure_nudft(dev, stream)

    # the oracle on the host cores, after every other rank has finished its GPU work (so no
    # rank's host thread competes with it)
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_oracle_rate(th_h.numpy(), args.cpu_seconds, W.description.split(":")[0])

    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps,
        "wall_ms_per_step": wall_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak" if W.weak else "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": W.description, "n_per_rank": n, "pairs_per_step": len(variants) * units_all,
                   "global_batch": units_all, "parallelism": f"dp{world} (contiguous shards, no collective)" + (
                           "; SAME DEVICE: every rank on cuda:0 in its own context (time-sliced), a host-flow "
                           "test -- value is NOT a throughput measurement" if args.same_device else ""),
                   "l2": "inputs larger than L2 (4n B theta + 8n B outputs per launch vs 126 MB L2); no flush"
                         if not use_graph else
                         "L2 flushed (512 MiB write) before every step, outside the per-step event spans; "
                         "launch/latency-bound at this size (the per-kernel split: graphs of 20 launches "
                         "after a flush, so mostly L2-warm)",
                   "launch": sp.LAUNCH, "cuda_graph": use_graph},
        "hbm_GBps": BYTES_PER_PAIR * pairs_total / (ms_max / 1e3) / 1e9 / world,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "clocks_per_rank": clocks_all,
        "distributed": nccl,
        "max_error": summary["max_err"],
        "rms_error": summary["rms_err"],
        "error_reference": "fp64 sin/cos on the device (P:137-138 metric); large-|theta| reduction error "
                           "is the method's (BASELINE.md section 2), the kernel equals the oracle bit for bit",
        "shards": summary["shards"],
        "next_fused_phase": fused,
        "next_fused_nudft": nudft_res,
        "next_methods": methods_res,
        "paper_context": "PowerPC 7400 G4 500 MHz AltiVec: 140 ns per 4 pairs = 28.6 M pairs/s (P:177-180)",
    }
    print(json.dumps(line), flush=True)


def nccl_init_lines():
    """This process's NCCL communicator-init lines (NCCL_DEBUG=INFO, subsystem INIT, to
    NCCL_DEBUG_FILE), e.g. "... comm 0x... rank 0 nRanks 8 nNodes 1 localRanks 8 ..."; also
    echoed to stderr."""
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    if not path or "%" in path or not os.path.exists(path):
        return None
    keep = [l.strip() for l in open(path, errors="ignore") if "nRanks" in l or "Init COMPLETE" in l]
    for l in keep:
        print(l, file=sys.stderr, flush=True)
    return keep[:8]


def die(msg: str, code: int = 2):
    print(f"bench.py: {msg}", file=sys.stderr, flush=True)
    sys.exit(code)


def visible_gpus() -> int:
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def self_launch(args) -> int:
    """`python bench.py --gpus N` (N > 1) without a launcher: re-run this command under
    torch.distributed.run with N ranks on this node (one process per GPU, rendezvous on
    127.0.0.1), so both invocation forms time N GPUs.  Returns the launcher's exit code."""
    import socket
    import subprocess
    if not args.same_device and visible_gpus() < args.gpus:
        die(f"--gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {visible_gpus()} "
            "(--same-device --backend gloo runs every rank on cuda:0: host-flow testing only)")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    launched = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus < 1:
        die("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if not launched and args.gpus > 1:
        sys.exit(self_launch(args))
    # from here on: one process per GPU, and the job is exactly --gpus ranks
    if world != args.gpus:
        die(f"--gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks")
    if args.same_device and args.backend != "gloo":
        die("--same-device needs --backend gloo (the ranks' kernels share one GPU: flow testing only)")
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    if not args.same_device and visible_gpus() < local_world:
        die(f"{local_world} ranks on this node but {visible_gpus()} visible CUDA devices")
    import torch
    import torch.distributed as dist
    gpu = 0 if args.same_device else local_rank
    if world > 1:
        torch.cuda.set_device(gpu)
        if args.backend == "nccl":
            # NCCL's INIT log (per process, to a file: on stdout it could follow the JSON line, and
            # several ranks writing one stderr file would clobber it); rank 0 copies its
            # communicator lines ("... nRanks N ...") to stderr and into the JSON line
            # (a launcher that set NCCL_DEBUG itself keeps NCCL's own log destination)
            if "NCCL_DEBUG" not in os.environ:
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/bench_nccl.{os.getpid()}.log")
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
            dist.barrier()
        else:
            dist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, gpu)
    finally:
        if world > 1 and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
