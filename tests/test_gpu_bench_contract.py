"""bench.py's JSON line for our arm on the GPU (small config): every key of
the contract, with the roofline / cpu_baseline / e2e / clocks objects."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,extra", [("c3", []), ("c1", []), ("c5", []),
                                          # the --gpus launcher: re-run under torchrun (one rank here)
                                          ("c3", ["--gpus", "1", "--spawn"]),
                                          # the multi-GPU code paths at one rank: NCCL all-gather per
                                          # interval (C3), peer-memory resident rounds (C5)
                                          ("c3", ["--sharded"]), ("c5", ["--sharded"])])
def test_our_arm_line(config, extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", "4",
                          "--warmup", "3", "--no-exact"] + extra, capture_output=True, text=True, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 4 and line["warmup"] == 3 and line["value"] > 0
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    if "--spawn" not in extra:
        assert line["roofline"]["kernel"] is not None
    cb = line["cpu_baseline"]
    if "--sharded" in extra:  # the coordinator path (N > 1 under torchrun) leaves the CPU baseline to the N = 1 run
        assert cb is None
    else:
        assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] > 0
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] >= line["steps"]
    assert line["clocks"]["sm_mhz"] is not None
    assert "l2" in line["config"] and line["config"]["workload"].startswith("2D Ising")


def test_gpus_beyond_visible_refused():
    import torch
    n = torch.cuda.device_count() + 1
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0 and f"--gpus {n} needs {n} visible GPUs" in out.stderr
