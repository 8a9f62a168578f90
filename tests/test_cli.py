"""The B200 CLI keeps the reference CLI's contract (ref:cli.py): flags,
precedence, presets, seeds, output schemas and exit codes.  CPU tests use a
stand-in for run(); the GPU tests compare observables.csv byte for byte with
the reference CLI's own output (tests/golden/cli.json)."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2512_03825_b200 import cli
from paper_2512_03825_b200.executor import RunRecord

GOLD = json.load(open(os.path.join(GOLDEN, "cli.json")))


def test_derive_seed_matches_reference():
    for key, want in GOLD["seeds"].items():
        m, p, r = key.split("|")
        assert cli.derive_seed(int(m), p, int(r)) == want


def test_precedence_flags_over_file_over_preset(tmp_path):
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"size": 12, "replicas": 6, "preset": "paper-small", "reps": 3}))
    spec = cli.parse_config(["--config", str(f), "--replicas", "9"])
    assert spec.base.side == 12 and spec.base.replicas == 9     # file, flag
    assert spec.base.iterations == 100_000 and spec.reps == 3    # preset, file
    assert spec.kind == "single" and spec.record_mode == "observables"
    spec = cli.parse_config(["--sweep", "swap_sweep"])
    assert spec.axis == (0, 100, 1000, 10000) and spec.record_mode == "none"
    spec = cli.parse_config(["--sweep-mode", "checkerboard", "--size", "8", "--iters", "640",
                             "--swap-interval", "64", "--record-every", "2"])
    assert spec.base.sweep_mode == "checkerboard" and spec.base.record_every == 2


@pytest.mark.parametrize("argv", [
    ["--bogus"], ["--size", "1"], ["--sweep", "size_sweep", "--axis", "8,1"],
    ["--sweep", "replica_scaling", "--axis", "a,b"], ["--reps", "0"], ["--config", "/nope.json"],
    ["--sweep", "swap_sweep", "--axis", ""], ["--sweep-mode", "checkerboard", "--size", "7"],
    ["--devices", "a,b"], ["--devices", "0,0", "--sweep-mode", "checkerboard", "--iters", "1024",
                           "--swap-interval", "64"],
])
def test_usage_errors_exit_1(argv, capsys):
    assert cli.main(argv) == 1
    assert "error" in capsys.readouterr().err


def test_devices_flag_and_file_key(tmp_path):
    spec = cli.parse_config(["--devices", "0,1", "--sweep-mode", "checkerboard", "--iters", "1024",
                             "--swap-interval", "64", "--size", "8"])
    assert spec.base.devices == (0, 1)
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"size": 8, "iters": 1024, "swap_interval": 64, "sweep_mode": "checkerboard",
                             "devices": [2, 3, 4]}))
    assert cli.parse_config(["--config", str(f)]).base.devices == (2, 3, 4)


def test_devices_without_torchrun_is_a_usage_error(tmp_path, monkeypatch, capsys):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    argv = ["--devices", "0,1", "--sweep-mode", "checkerboard", "--iters", "1024", "--swap-interval", "64",
            "--size", "8", "--out", str(tmp_path)]
    assert cli.main(argv) == 1
    assert "torchrun --nproc-per-node 2" in capsys.readouterr().err


def test_unknown_config_key(tmp_path):
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"size": 8, "colour": "blue"}))
    with pytest.raises(cli.UsageError):
        cli.parse_config(["--config", str(f)])


def _fake_run(cfg):
    R, N = cfg.replicas, cfg.iterations
    e = np.arange(R * N, dtype=np.float64).reshape(R, N)
    return RunRecord(config=cfg, temperatures=np.linspace(1, 2, R), energies=e,
                     magnetizations=e / 10, states=None, swap_rounds=1, swaps_attempted=4,
                     swaps_accepted=cfg.seed % 3, rng_positions=np.zeros(R, np.int64),
                     round_entry_iterations=None, init_seconds=0.1, exec_seconds=0.2,
                     total_seconds=0.3 + 0.1 * cfg.workers)


def test_sweep_outputs_and_failure_rows(tmp_path, monkeypatch):
    monkeypatch.setattr(cli, "run", _fake_run)
    monkeypatch.setattr("paper_2512_03825_b200.kernels.warm_kernels", lambda: None)
    out = tmp_path / "w"
    assert cli.main(["--sweep", "worker_scaling", "--axis", "1,2", "--reps", "2", "--iters", "5",
                     "--replicas", "2", "--out", str(out), "--record", "observables"]) == 0
    rows = [cli.TimingRow.from_csv(x) for x in (out / "timings.csv").read_text().splitlines()[1:]]
    assert [r.sweep_point for r in rows] == ["W=1", "W=1", "W=2", "W=2"]
    assert rows[0].seed == rows[2].seed != rows[1].seed    # W points share seeds
    summary = json.loads((out / "summary.json").read_text())
    assert summary["baseline"] == "W=1"
    assert abs(summary["points"][1]["speedup"] - 0.4 / 0.5) < 1e-12
    assert (out / "observables-W=2-rep1.csv").exists()

    def boom(cfg):
        raise RuntimeError("injected, failure")
    monkeypatch.setattr(cli, "run", boom)
    out2 = tmp_path / "f"
    assert cli.main(["--iters", "5", "--replicas", "2", "--out", str(out2)]) == 2
    row = cli.TimingRow.from_csv((out2 / "timings.csv").read_text().splitlines()[1])
    assert row.status == "error: injected; failure"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["single", "replica_sweep", "worker_sweep"])
def test_cli_outputs_match_reference_cli(tmp_path, name):
    case = GOLD["cases"][name]
    assert cli.main(case["argv"] + ["--out", str(tmp_path)]) == case["rc"]
    assert sorted(os.listdir(tmp_path)) == case["files"]
    for f, digest in case["digests"].items():
        assert hashlib.sha256((tmp_path / f).read_bytes()).hexdigest() == digest, f
    rows = (tmp_path / "timings.csv").read_text().splitlines()
    hdr = rows[0].split(",")
    keep = [i for i, c in enumerate(hdr) if c not in ("init_s", "exec_s", "total_s")]
    assert [",".join(r.split(",")[i] for i in keep) for r in rows] == case["timings_stable"]


@pytest.mark.gpu
def test_cli_devices_world1_equals_single_device(tmp_path):
    argv = ["--size", "64", "--replicas", "6", "--iters", str(20 * 4096), "--swap-interval", "8192",
            "--sweep-mode", "checkerboard", "--seed", "5"]
    assert cli.main(argv + ["--out", str(tmp_path / "a")]) == 0
    assert cli.main(argv + ["--devices", "0", "--out", str(tmp_path / "b")]) == 0
    assert (tmp_path / "a" / "observables.csv").read_bytes() == (tmp_path / "b" / "observables.csv").read_bytes()


@pytest.mark.gpu
def test_cli_checkerboard_run_is_reproducible(tmp_path):
    argv = ["--size", "64", "--replicas", "8", "--iters", str(50 * 4096), "--swap-interval",
            "4096", "--sweep-mode", "checkerboard", "--seed", "3"]
    assert cli.main(argv + ["--out", str(tmp_path / "a")]) == 0
    assert cli.main(argv + ["--out", str(tmp_path / "b")]) == 0
    a = (tmp_path / "a" / "observables.csv").read_bytes()
    assert a == (tmp_path / "b" / "observables.csv").read_bytes()
    lines = a.decode().splitlines()
    assert lines[0] == "replica,temperature,iteration,energy,magnetization"
    assert len(lines) == 1 + 8 * 50 and lines[1].split(",")[2] == str(4096 - 1)
