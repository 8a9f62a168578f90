"""Benchmark harness on the B200 engine: the reference CLI's contract.

    python -m paper_2512_03825_b200.cli [--size L --replicas R --iters N
        --swap-interval I --workers W --seed S --J J --B B --init-up F
        --preset desk|paper-small|paper-full --sweep KIND --axis a,b,c
        --reps K --out DIR --record none|observables|full --config FILE.json
        --sweep-mode exact|checkerboard --record-every K --device D | --devices 0,1,...]

Same flags, precedence (flags > JSON config > preset), presets, sweep kinds,
seed derivation, output files and exit codes as `isingpt` (ref:cli.py:1-411):
timings.csv, observables.csv / observables-<point>-rep<k>.csv, states*.npz
and summary.json, exit 0 / 1 (usage) / 2 (a failed row).  The three flags
after --config are extensions: the chain (the reference's, default, or the
checkerboard sweep), the checkerboard sampling stride and the GPU; --devices
runs every point on several GPUs, one process per GPU (launch the CLI under
torchrun --nproc-per-node len(devices); rank 0 writes the output files).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np

from .executor import SWEEP_MODES, ConfigurationError, RunRecord, SimulationConfig, run
from .lattice import IsingParams

SWEEP_KINDS = ("single", "worker_scaling", "replica_scaling", "swap_sweep", "size_sweep")
RECORD_CHOICES = {"none": "none", "observables": "observables", "full": "full_states"}

# ref:cli.py:39-52 (values are the reference's)
PRESETS = {
    "desk": {"size": 32, "replicas": 16, "iters": 50_000, "swap_interval": 100, "workers": 4,
             "seed": 42, "J": 1.0, "B": 0.0, "init_up": 0.5},
    "paper-small": {"size": 100, "replicas": 128, "iters": 100_000, "swap_interval": 100,
                    "workers": 4, "seed": 42, "J": 1.0, "B": 0.0, "init_up": 0.5},
    "paper-full": {"size": 300, "replicas": 1500, "iters": 300_000, "swap_interval": 0,
                   "workers": 16, "seed": 42, "J": 1.0, "B": 0.0, "init_up": 0.5},
}
DEFAULT_AXES = {"single": (), "worker_scaling": (1, 2, 4, 8),
                "replica_scaling": (16, 32, 64, 128), "swap_sweep": (0, 100, 1000, 10000),
                "size_sweep": (8, 12, 16, 24, 32)}
SETTINGS = ("size", "replicas", "iters", "swap_interval", "workers", "seed", "J", "B", "init_up")
EXTENSIONS = ("sweep_mode", "record_every", "device", "devices")
FILE_KEYS = SETTINGS + ("preset", "sweep", "axis", "reps", "out", "record") + EXTENSIONS
TIMINGS_COLUMNS = ("sweep_point", "rep", "workers", "replicas", "L", "iters", "swap_interval",
                   "seed", "init_s", "exec_s", "total_s", "swaps_attempted", "swaps_accepted",
                   "status")
OBSERVABLES_COLUMNS = ("replica", "temperature", "iteration", "energy", "magnetization")
_AXIS_RULES = {"worker_scaling": ("workers", 1), "replica_scaling": ("replicas", 1),
               "swap_sweep": ("swap_interval", 0), "size_sweep": ("size", 2)}
_POINT_FIELD = {"worker_scaling": ("W", "workers"), "replica_scaling": ("R", "replicas"),
                "swap_sweep": ("I", "swap_interval"), "size_sweep": ("L", "side")}


class UsageError(Exception):
    """Bad flags or config file (exit code 1)."""


@dataclass(frozen=True)
class SweepSpec:
    kind: str
    base: SimulationConfig
    axis: tuple[int, ...]
    reps: int
    out_dir: Path
    record_mode: str


@dataclass
class TimingRow:
    sweep_point: str
    rep: int
    workers: int
    replicas: int
    L: int
    iters: int
    swap_interval: int
    seed: int
    init_s: float
    exec_s: float
    total_s: float
    swaps_attempted: int
    swaps_accepted: int
    status: str

    def to_csv(self) -> str:
        return ",".join(str(getattr(self, name)) for name in TIMINGS_COLUMNS)

    @classmethod
    def from_csv(cls, line: str) -> "TimingRow":
        fields = line.rstrip("\n").split(",")
        if len(fields) != len(TIMINGS_COLUMNS):
            raise ValueError(f"expected {len(TIMINGS_COLUMNS)} columns, got {len(fields)}")
        casts = (str,) + (int,) * 7 + (float,) * 3 + (int, int, str)
        return cls(*(cast(v) for cast, v in zip(casts, fields)))


class _ArgParser(argparse.ArgumentParser):
    def error(self, message):  # usage problems exit with 1, not argparse's 2
        raise UsageError(message)


def _parser() -> _ArgParser:
    p = _ArgParser(prog="paper_2512_03825_b200.cli",
                   description="PT Metropolis benchmark sweeps on the B200 engine")
    for flag, typ, dest in [("--size", int, "size"), ("--replicas", int, "replicas"),
                            ("--iters", int, "iters"), ("--swap-interval", int, "swap_interval"),
                            ("--workers", int, "workers"), ("--seed", int, "seed"),
                            ("--J", float, "J"), ("--B", float, "B"),
                            ("--init-up", float, "init_up"), ("--reps", int, "reps"),
                            ("--record-every", int, "record_every"), ("--device", int, "device")]:
        p.add_argument(flag, type=typ, dest=dest)
    p.add_argument("--preset", choices=sorted(PRESETS))
    p.add_argument("--sweep", choices=SWEEP_KINDS)
    p.add_argument("--axis")
    p.add_argument("--out")
    p.add_argument("--record", choices=sorted(RECORD_CHOICES))
    p.add_argument("--config")
    p.add_argument("--sweep-mode", choices=SWEEP_MODES, dest="sweep_mode")
    p.add_argument("--devices")
    return p


def _devices(v) -> tuple | None:
    """--devices 0,1,2 (or a JSON list) -> (0, 1, 2)."""
    if v is None:
        return None
    try:
        items = v.split(",") if isinstance(v, str) else list(v)
        return tuple(int(x) for x in items if str(x).strip() != "")
    except (TypeError, ValueError) as exc:
        raise UsageError(f"devices must be comma-separated GPU indices, got {v!r}") from exc


def derive_seed(master_seed: int, point_id: str, rep: int) -> int:
    """sha256 of "master|point|rep", first 8 bytes big-endian, 63 bits
    (ref:cli.py:157-161): stable across Python runs and repetitions."""
    h = hashlib.sha256(f"{master_seed}|{point_id}|{rep}".encode()).digest()
    return int.from_bytes(h[:8], "big") & 0x7FFFFFFFFFFFFFFF


def _load_file(path_str: str | None) -> dict:
    if path_str is None:
        return {}
    path = Path(path_str)
    if not path.is_file():
        raise UsageError(f"config file not found: {path}")
    try:
        cfg = json.loads(path.read_text())
    except json.JSONDecodeError as exc:
        raise UsageError(f"config file is not valid JSON: {exc}") from exc
    extra = sorted(set(cfg) - set(FILE_KEYS))
    if extra:
        raise UsageError(f"unknown config file key(s): {', '.join(extra)}")
    return cfg


def _pick(ns, cfg: dict, key: str, default=None):
    """flag > config file > default"""
    v = getattr(ns, key, None)
    if v is not None:
        return v
    return cfg.get(key, default)


def parse_config(argv: list[str] | None = None) -> SweepSpec:
    ns = _parser().parse_args(argv)
    cfg = _load_file(ns.config)
    preset = ns.preset or cfg.get("preset") or "desk"
    if preset not in PRESETS:
        raise UsageError(f"unknown preset: {preset}")
    setting = {k: _pick(ns, cfg, k, PRESETS[preset][k]) for k in SETTINGS}
    kind = _pick(ns, cfg, "sweep", "single")
    if kind not in SWEEP_KINDS:
        raise UsageError(f"sweep must be one of {SWEEP_KINDS}, got {kind!r}")
    if ns.axis is not None:
        try:
            axis = tuple(int(t) for t in ns.axis.split(",") if t.strip())
        except ValueError as exc:
            raise UsageError(f"axis values must be integers: {ns.axis!r}") from exc
    else:
        axis = tuple(int(t) for t in cfg["axis"]) if "axis" in cfg else DEFAULT_AXES[kind]
    if kind != "single" and not axis:
        raise UsageError(f"axis must be non-empty for sweep kind {kind}")
    if kind in _AXIS_RULES:
        name, lo = _AXIS_RULES[kind]
        bad = [v for v in axis if v < lo]
        if bad:
            raise UsageError(f"axis: {name} must be >= {lo}, got {bad[0]}")
    reps = _pick(ns, cfg, "reps", 1)
    if reps < 1:
        raise UsageError(f"reps must be >= 1, got {reps}")
    record = _pick(ns, cfg, "record") or ("observables" if kind == "single" else "none")
    if record not in RECORD_CHOICES:
        raise UsageError(f"record must be one of {sorted(RECORD_CHOICES)}, got {record!r}")
    try:
        base = SimulationConfig(
            side=int(setting["size"]), replicas=int(setting["replicas"]),
            iterations=int(setting["iters"]), swap_interval=int(setting["swap_interval"]),
            workers=int(setting["workers"]), seed=int(setting["seed"]),
            params=IsingParams(J=float(setting["J"]), B=float(setting["B"])),
            init_up_fraction=float(setting["init_up"]), record_mode=RECORD_CHOICES[record],
            sweep_mode=_pick(ns, cfg, "sweep_mode", "exact"),
            record_every=int(_pick(ns, cfg, "record_every", 1)),
            device=_pick(ns, cfg, "device"), devices=_devices(_pick(ns, cfg, "devices")))
        base.validate()
    except (ConfigurationError, ValueError) as exc:
        raise UsageError(str(exc)) from exc
    return SweepSpec(kind, base, axis, int(reps), Path(_pick(ns, cfg, "out", "results")),
                     RECORD_CHOICES[record])


def _points(spec: SweepSpec) -> list[tuple[str, SimulationConfig]]:
    if spec.kind == "single":
        return [("single", spec.base)]
    tag, field = _POINT_FIELD[spec.kind]
    return [(f"{tag}={v}", replace(spec.base, **{field: v})) for v in spec.axis]


def _observable_iterations(record: RunRecord) -> np.ndarray:
    """Column -> iteration index: per attempt for the reference chain; the
    last attempt of each recorded sweep for the checkerboard chain."""
    n = record.energies.shape[1]
    if record.sweep_mode == "checkerboard":
        per = record.config.record_every * record.config.side ** 2
        return (np.arange(n, dtype=np.int64) + 1) * per - 1
    return np.arange(n, dtype=np.int64)


def write_observables(path: Path, record: RunRecord) -> None:
    """replica,temperature,iteration,energy,magnetization (ref:cli.py:276-287)."""
    its = _observable_iterations(record).tolist()
    out = [",".join(OBSERVABLES_COLUMNS)]
    for r, (t, er, mr) in enumerate(zip(record.temperatures, record.energies,
                                        record.magnetizations)):
        ts = repr(float(t))
        out += [f"{r},{ts},{i},{e!r},{m!r}" for i, e, m in zip(its, er.tolist(), mr.tolist())]
    path.write_text("\n".join(out) + "\n")


def emit_speedup_table(rows: list[TimingRow], baseline: str) -> list[tuple[str, float, float]]:
    """(point, baseline mean total / point mean total, std of per-rep ratios)
    over status-ok rows (ref:cli.py:290-311)."""
    good = [r for r in rows if r.status == "ok"]
    ref_totals = [r.total_s for r in good if r.sweep_point == baseline]
    if not ref_totals:
        raise ValueError(f"baseline point {baseline!r} has no successful rows")
    ref_mean = float(np.mean(ref_totals))
    out = []
    for point in dict.fromkeys(r.sweep_point for r in rows):
        tot = [r.total_s for r in good if r.sweep_point == point]
        if tot:
            out.append((point, ref_mean / float(np.mean(tot)),
                        float(np.std([ref_mean / t for t in tot]))))
    return out


def _summary(spec: SweepSpec, rows: list[TimingRow]) -> dict:
    baseline = "W=1" if spec.kind == "worker_scaling" else None
    speed = {}
    if baseline:
        try:
            speed = {p: v for p, v, _ in emit_speedup_table(rows, baseline)}
        except ValueError:
            baseline = None
    pts = []
    for point in dict.fromkeys(r.sweep_point for r in rows):
        good = [r for r in rows if r.sweep_point == point and r.status == "ok"]
        att = sum(r.swaps_attempted for r in good)
        pts.append({"point": point,
                    "mean_total_s": float(np.mean([r.total_s for r in good])) if good else None,
                    "std_total_s": float(np.std([r.total_s for r in good])) if good else None,
                    "swap_accept_rate": sum(r.swaps_accepted for r in good) / att if att else 0.0,
                    "speedup": speed.get(point)})
    return {"sweep": spec.kind, "baseline": baseline, "points": pts}


def _join_devices(spec: SweepSpec) -> int:
    """--devices with several GPUs: this process is one rank of a torchrun
    launch (RANK / LOCAL_RANK / WORLD_SIZE from the environment); joins the
    NCCL process group every run() of the sweep shards over.  Returns the
    rank (0 without --devices or with one device)."""
    devs = spec.base.devices
    if devs is None or len(devs) == 1:
        return 0
    import os

    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world != len(devs):
            raise UsageError(f"--devices names {len(devs)} GPUs: launch with torchrun --nproc-per-node "
                             f"{len(devs)} (WORLD_SIZE is {world})")
        rank = int(os.environ["RANK"])
        torch.cuda.set_device(devs[rank])
        dist.init_process_group("nccl", device_id=torch.device("cuda", devs[rank]))
    torch.cuda.set_device(devs[dist.get_rank()])
    return dist.get_rank()


def run_sweep(spec: SweepSpec) -> int:
    """Every point x repetition, sequentially; failures become rows and the
    sweep goes on; exit 2 if any row failed (ref:cli.py:314-368).  With
    several --devices every rank runs every point; rank 0 writes the files."""
    rank = _join_devices(spec)
    writer = rank == 0
    if writer:
        spec.out_dir.mkdir(parents=True, exist_ok=True)
    from .kernels import warm_kernels

    warm_kernels()  # CUDA context + module load outside the timed runs
    one_file = spec.kind == "single" and spec.reps == 1
    rows = []
    for point_id, cfg in _points(spec):
        for rep in range(spec.reps):
            # worker count is not part of the workload: W points share seeds
            seed = derive_seed(spec.base.seed, "" if spec.kind == "worker_scaling" else point_id,
                               rep)
            rc = replace(cfg, seed=seed, record_mode=spec.record_mode)
            rec = None
            try:
                rec = run(rc)
                status = "ok" if rec.valid else f"error: {rec.error}"
            except Exception as exc:  # noqa: BLE001 - a failed point is a row
                status = f"error: {exc}"
            status = status.replace(",", ";").replace("\n", " ")
            rows.append(TimingRow(point_id, rep, rc.workers, rc.replicas, rc.side, rc.iterations,
                                  rc.swap_interval, seed,
                                  rec.init_seconds if rec else 0.0,
                                  rec.exec_seconds if rec else 0.0,
                                  rec.total_seconds if rec else 0.0,
                                  rec.swaps_attempted if rec else 0,
                                  rec.swaps_accepted if rec else 0, status))
            if writer:
                print(f"[b200] {point_id} rep {rep}: {status}"
                      + (f" total {rec.total_seconds:.3f}s" if rec else ""), file=sys.stderr)
            if writer and rec is not None and rec.valid and spec.record_mode != "none":
                suffix = "" if one_file else f"-{point_id}-rep{rep}"
                write_observables(spec.out_dir / f"observables{suffix}.csv", rec)
                if rec.states is not None:
                    np.savez_compressed(spec.out_dir / f"states{suffix}.npz", states=rec.states,
                                        temperatures=rec.temperatures)
    if not writer:
        return 0 if all(r.status == "ok" for r in rows) else 2
    (spec.out_dir / "timings.csv").write_text(
        ",".join(TIMINGS_COLUMNS) + "\n" + "".join(r.to_csv() + "\n" for r in rows))
    (spec.out_dir / "summary.json").write_text(json.dumps(_summary(spec, rows), indent=2) + "\n")
    return 0 if all(r.status == "ok" for r in rows) else 2


def main(argv: list[str] | None = None) -> int:
    try:
        spec = parse_config(argv)
    except UsageError as exc:
        print(f"paper_2512_03825_b200: error: {exc}", file=sys.stderr)
        return 1
    t0 = time.perf_counter()
    try:
        code = run_sweep(spec)
    except UsageError as exc:
        print(f"paper_2512_03825_b200: error: {exc}", file=sys.stderr)
        return 1
    print(f"[b200] sweep finished in {time.perf_counter() - t0:.1f}s, outputs in {spec.out_dir}",
          file=sys.stderr)
    return code


if __name__ == "__main__":
    sys.exit(main())
