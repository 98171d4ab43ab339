"""Multi-GPU (SURVEY 4 tier T3): only runs on a box with >= 2 GPUs (skipped on this 1-GPU pool).

bench.py under torchrun, one process per GPU over NCCL: every rank's shard stats arrive through
the NCCL all-gather, the time is the max over ranks, and the line is the whole job's; the
strong-scaling workload's concatenated shards are the one-GPU array (checked through the
gathered per-shard element counts)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("workload", ["c2", "c4"])
def test_torchrun_nccl_bench(workload):
    G = ngpus()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(ROOT, "bench.py"),
           "--gpus", str(G), "--workload", workload, "--steps", "3", "--warmup", "3",
           "--no-next", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == G and line["value"] > 0
    assert line["scaling"] == ("weak" if workload == "c2" else "strong")
    shards = line["shards"]
    assert len(shards) == 2 * G and {s["rank"] for s in shards} == set(range(G))
    if workload == "c4":
        import inputs
        per_variant = [s["n"] + s["nan"] for s in shards if s["variant"] == "N"]
        assert sum(per_variant) == inputs.size(4)


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
def test_plain_invocation_self_launches_every_gpu():
    """`python bench.py --gpus G` without a launcher: G ranks over NCCL, one per GPU; the line
    carries every rank's shards and clocks and the communicator's rank count."""
    G = ngpus()
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(G), "--steps", "3", "--warmup", "3",
           "--no-next", "--e2e-max", str(1 << 22), "--cpu-seconds", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == G and line["distributed"]["comm_nranks"] == G
    assert len(line["clocks_per_rank"]) == G and {s["rank"] for s in line["shards"]} == set(range(G))
    assert line["cpu_baseline"] is not None and line["roofline"]["traffic"] is not None
