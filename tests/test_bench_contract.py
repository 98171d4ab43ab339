"""bench.py's output contract (the driver parses one JSON line): the reference arm on the CPU
here (it times the oracle; under torchrun only rank 0 prints), and our arm on a GPU (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = json.load(open(os.path.join(ROOT, "BASELINE.json")))


def run(args, timeout=600, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def check_common(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["metric"] == BASE["metric"]
    assert d["unit"] == "pairs/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["vs_baseline"] is None and d["data"] == "synthetic" and d["dtype"] == "f32"
    assert "workload" in d["config"] and d["warmup"] >= 3
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    assert d["cpu_baseline"]["kind"] == "oracle"


def test_reference_arm_contract():
    d = run(["--impl", "reference", "--steps", "2", "--warmup", "3"])
    check_common(d)
    assert d["impl"] == "reference" and d["steps"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_under_torchrun_prints_once():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"


@pytest.mark.gpu
def test_our_arm_contract_on_gpu():
    d = run(["--steps", "3", "--warmup", "3", "--no-next", "--e2e-max", str(1 << 24), "--cpu-seconds", "1"])
    check_common(d)
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["steps"] == 3
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] == 2 * 3
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 4 * (1 << 24) and d["e2e"]["d2h_bytes_per_step"] == 2 * 8 * (1 << 24)
    assert d["max_error"] < 1e-3                     # C2's reduction error, [X12] 7.9e-4


def run_rc(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    return r.returncode, r.stdout, r.stderr


def test_gpus_n_without_enough_devices_fails_loudly():
    """`bench.py --gpus 2` never silently times one GPU: without a launcher it re-runs itself under
    torch.distributed.run with 2 ranks, and refuses (non-zero exit, no JSON line) when fewer than
    2 CUDA devices are visible -- here, on the CPU-only container, none are."""
    import torch
    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        pytest.skip("this box has >= 2 GPUs")
    rc, out, err = run_rc(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert rc != 0
    assert not [l for l in out.splitlines() if l.startswith("{")]
    assert "--gpus 2 needs 2 visible CUDA devices" in err


def test_world_size_must_equal_gpus():
    """Under a launcher the rank count must be exactly --gpus (2 ranks started, --gpus 3 asked)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29573", os.path.join(ROOT, "bench.py"),
           "--gpus", "3", "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode != 0
    assert "--gpus 3 but the launcher started WORLD_SIZE=2 ranks" in r.stderr
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_same_device_needs_gloo():
    rc, out, err = run_rc(["--gpus", "1", "--same-device", "--steps", "1", "--warmup", "3"])
    assert rc != 0 and "--same-device needs --backend gloo" in err


@pytest.mark.gpu
def test_gpus_2_self_launch_same_device():
    """The driver's plain form with N = 2 (no torchrun): bench.py launches 2 ranks itself; on a
    1-GPU box --same-device --backend gloo puts both on cuda:0 (flow only).  Rank 0 prints one
    line for 2 ranks: both ranks' shards and clocks, the oracle baseline, the e2e leg."""
    d = run(["--gpus", "2", "--backend", "gloo", "--same-device", "--steps", "3", "--warmup", "3", "--no-next",
             "--n-per-rank", str(1 << 24), "--e2e-max", str(1 << 22), "--cpu-seconds", "1"])
    check_common(d)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert sorted({s["rank"] for s in d["shards"]}) == [0, 1] and len(d["shards"]) == 4
    assert d["cpu_baseline"] is not None and d["cpu_baseline"]["cores"] >= 1
    assert d["distributed"]["comm_nranks"] == 2 and d["distributed"]["same_device"] is True
    assert len(d["clocks_per_rank"]) == 2
    assert d["config"]["global_batch"] == 2 * (1 << 24)
    assert d["e2e"]["frac_of_pcie_roofline"] > 0


def test_every_bench_option_survives_torchrun_parsing():
    """bench.py re-runs itself under torch.distributed.run; that launcher's argparse takes any
    prefix of its own options (e.g. "--n" for --nnodes/--nproc-per-node) and rejects ambiguous
    ones before the script's arguments -- so no bench option may be such a prefix."""
    import re

    from torch.distributed.run import get_args_parser
    src = open(os.path.join(ROOT, "bench.py")).read()
    opts = sorted(set(re.findall(r'add_argument\(\s*"(--[\w-]+)"', src)))
    assert "--gpus" in opts and "--n-per-rank" in opts
    argv = ["--nnodes=1", "--nproc-per-node=2", "bench.py"]
    for o in opts:
        argv += [o, "1"]
    ns = get_args_parser().parse_args(argv)
    assert ns.training_script == "bench.py" and len(ns.training_script_args) == 2 * len(opts)


@pytest.mark.gpu
def test_gpus_2_on_a_one_gpu_box_fails_loudly():
    """On the one-GPU box: `--gpus 2` without --same-device refuses (non-zero exit, no JSON line)
    instead of timing one GPU."""
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this box has >= 2 GPUs")
    rc, out, err = run_rc(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert rc != 0 and not [l for l in out.splitlines() if l.startswith("{")]
    assert "--gpus 2 needs 2 visible CUDA devices, found 1" in err
