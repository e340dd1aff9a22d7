"""bench.py keeps the driver's contract: one JSON line with the required keys, for the default
run, for the reference arm, and (GPU) for a 2-rank torchrun launch sharing one GPU over gloo."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config"]


def _last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_reference_arm_cpu():
    """--impl reference runs the restated CPU path (no GPU needed) and prints one JSON line."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    d = _last_json(out.stdout)
    for key in REQUIRED + ["cpu_baseline", "e2e", "impl"]:
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"


def test_warmup_floor():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "2"],
                         cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert out.returncode != 0


@pytest.mark.gpu
def test_default_bench_line():
    out = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "3", "--e2e-steps", "1",
                          "--cpu-elems", "1000000"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr
    d = _last_json(out.stdout)
    for key in REQUIRED + ["roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"]:
        assert key in d, key
    assert d["gpu_launches"] == 40  # prep_dyn + the stream kernel per step (large call: B staged by prep)
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0.5 < r["frac"] < 1.3
    assert d["e2e"]["h2d_bytes_per_step"] > 7e9


@pytest.mark.gpu
def test_two_rank_torchrun_shared_gpu():
    env = dict(os.environ, TSM2X_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3",
           "--e2e-steps", "0", "--workload", "tsm2r_fp64_n2"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _last_json(out.stdout)
    assert d["n_gpus"] == 2 and d["config"]["m_total"] == 2 * d["config"]["m_per_gpu"]
    assert d["scaling"] == "weak" and d["value"] > 0
