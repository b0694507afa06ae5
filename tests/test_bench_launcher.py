"""CPU: bench.py's self-launch path (`--gpus N` without a launcher starts the N
ranks itself; gloo rendezvous on 127.0.0.1) and the reference arm's isolation
from the product library."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints, once
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,config,parallelism", [(2, "c2", "row-strips-x2"), (3, "c5", "images-x3")])
def test_self_launch_strong_scaling(gpus, config, parallelism):
    line = _run(["--gpus", str(gpus), "--config", config, "--dry-run"])
    assert line["n_gpus"] == gpus and line["scaling"] == "strong"
    assert line["config"]["parallelism"] == parallelism
    c = {"c2": 2048 * 2048, "c5": 256 * 1024 * 1024}[config]
    assert line["pixels"] == c  # the ranks' outputs cover the workload exactly once


def test_weak_scaling_is_one_workload_per_rank():
    line = _run(["--gpus", "2", "--config", "c1", "--dry-run", "--scaling", "weak"])
    assert line["scaling"] == "weak" and line["pixels"] == 2 * 512 * 512


def test_reference_arm_never_loads_the_product():
    line = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"])
    assert line["impl"] == "reference" and line["value"] > 0
    assert not any("libfourierbf_b200" in p for p in line["native_libs"])
    assert "oracle/_ref/libfbf_ref.so" in line["native_libs"]
