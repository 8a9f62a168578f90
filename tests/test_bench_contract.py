"""bench.py's JSON-line contract, checked on CPU through the reference arm
(the GPU arm's line is produced on the B200; tests/test_gpu_* cover it)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT, env=dict(os.environ, RANK="0", WORLD_SIZE="1"))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["steps"] == 1 and line["warmup"] == 3
    assert line["metric"] == "spin-flip attempts/sec" and line["unit"] == "attempts/s"
    assert line["higher_is_better"] is True and line["value"] > 0
    assert line["config"]["workload"].startswith("2D Ising 32x32")
    cb = line["cpu_baseline"]
    assert cb["value"] == line["value"] and cb["kind"] == "port" and cb["cores"] >= 1 and cb["sample"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_gpus_flag_refuses_missing_gpus():
    """--gpus N without torchrun self-launches N ranks, after checking that N
    GPUs are visible: this CPU container has none, so it must refuse loudly."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0
    assert "--gpus 2 needs 2 visible GPUs" in out.stderr
    assert not out.stdout.strip()


def test_gpus_flag_must_match_launched_world():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0"))
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr
