"""run(SimulationConfig) -> RunRecord: the drop-in for isingpt.executor.run.

Same dataclasses, validation, interval plan, swap schedule and record fields
as the reference (executor.py:28-300).  The state lives on the GPU for the
whole run (engine.py); the host only walks the interval plan and launches.

Extensions (all defaulted so reference configs run unchanged):

* ``sweep_mode``: "exact" (default) runs the reference's random-site chain,
  bit-exact with isingpt; "checkerboard" runs Mode F,
  where ``iterations`` and ``swap_interval`` must be whole sweeps (multiples
  of side**2) and observables are recorded per sweep (every
  ``record_every`` sweeps), shape (R, sweeps // record_every).
* ``record_every`` (exact chain, record_mode="observables"): keep every
  k-th column of the reference's per-attempt series -- column c is the
  reference's column (c+1)k - 1, shape (R, iterations // k).
* ``temperatures``: explicit ladder (e.g. tempering.geometric_ladder);
  default is the reference's build_ladder.
* ``device``: CUDA device index.  ``workers`` is validated and recorded
  but the GPU replaces the thread pool.
* ``devices``: the GPUs of a multi-GPU checkerboard run, one process per
  device (torchrun).  Rank r of the default process
  group runs on ``devices[r]`` and owns the lattice rows
  ``assign_replicas(replicas, len(devices))[r]``; exchanges all-gather the
  per-lattice (S, Bond) pairs (NCCL) or, on the resident path, go through
  NVLink peer memory.  Every rank returns the same RunRecord.  With one
  device and no process group, run() opens a world-1 NCCL group itself.
* ``return_final_state``: also return the final lattices (by row) and
  slot_to_row, for parity checks.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .lattice import IsingParams
from .tempering import build_ladder

RECORD_MODES = ("none", "observables", "full_states")
SWEEP_MODES = ("exact", "checkerboard")
KERNELS = ("auto", "sweep", "resident")
MASK64 = (1 << 64) - 1


class ConfigurationError(ValueError):
    """Invalid simulation configuration; raised before any work starts."""


@dataclass(frozen=True)
class SimulationConfig:
    """All parameters of a single run (executor.py:35-67, plus extensions)."""

    side: int = 32
    replicas: int = 16
    iterations: int = 50_000
    swap_interval: int = 100  # 0 disables swaps
    workers: int = 4
    seed: int = 42
    params: IsingParams = field(default_factory=IsingParams)
    init_up_fraction: float = 0.5
    record_mode: str = "observables"
    # --- extensions
    sweep_mode: str = "exact"
    temperatures: tuple | None = None
    record_every: int = 1
    device: int | None = None
    devices: tuple | None = None
    return_final_state: bool = False
    # checkerboard: "sweep" (launches per interval), "resident" (1 launch/run);
    # exact: "sweep" (launches per interval), "auto"/"resident": rounds inside
    # the commit launches when every slot fits one CTA (R <= 32)
    kernel: str = "auto"

    def validate(self) -> None:
        if self.side < 2:
            raise ConfigurationError(f"side must be >= 2, got {self.side}")
        if self.replicas < 1:
            raise ConfigurationError(f"replicas must be >= 1, got {self.replicas}")
        if self.iterations < 1:
            raise ConfigurationError(f"iterations must be >= 1, got {self.iterations}")
        if self.swap_interval < 0:
            raise ConfigurationError(f"swap_interval must be >= 0, got {self.swap_interval}")
        if self.workers < 1:
            raise ConfigurationError(f"workers must be >= 1, got {self.workers}")
        if not 0.0 <= self.init_up_fraction <= 1.0:
            raise ConfigurationError(
                f"init_up_fraction must be in [0, 1], got {self.init_up_fraction}")
        if self.record_mode not in RECORD_MODES:
            raise ConfigurationError(
                f"record_mode must be one of {RECORD_MODES}, got {self.record_mode!r}")
        if self.sweep_mode not in SWEEP_MODES:
            raise ConfigurationError(
                f"sweep_mode must be one of {SWEEP_MODES}, got {self.sweep_mode!r}")
        if self.temperatures is not None:
            t = np.asarray(self.temperatures, dtype=np.float64)
            if t.shape != (self.replicas,) or not np.all(t > 0) or not np.all(np.isfinite(t)):
                raise ConfigurationError(
                    "temperatures must be `replicas` positive finite values")
        if self.kernel not in KERNELS:
            raise ConfigurationError(f"kernel must be one of {KERNELS}, got {self.kernel!r}")
        if self.record_every < 1:
            raise ConfigurationError(f"record_every must be >= 1, got {self.record_every}")
        if self.devices is not None:
            devs = list(self.devices)
            if (not devs or any(not isinstance(d, (int, np.integer)) or isinstance(d, bool) or d < 0
                                for d in devs) or len(set(devs)) != len(devs)):
                raise ConfigurationError(
                    f"devices must be distinct non-negative device indices, got {self.devices!r}")
            if self.device is not None:
                raise ConfigurationError("set either device or devices, not both")
            if len(devs) > 1 and self.sweep_mode != "checkerboard":
                raise ConfigurationError(
                    "the exact chain runs on one device; multi-GPU runs need sweep_mode='checkerboard'")
            if len(devs) > 8:
                raise ConfigurationError("at most 8 devices (one NVLink node)")
            if self.record_mode == "full_states" and len(devs) > 1:
                raise ConfigurationError("full_states recording is single-device")
        if self.sweep_mode == "exact" and self.record_every > 1:
            if self.record_mode != "observables":
                raise ConfigurationError("record_every > 1 subsamples record_mode='observables' only")
            if self.record_every > self.iterations:
                raise ConfigurationError("record_every exceeds the number of iterations")
        if self.sweep_mode == "checkerboard":
            n = self.side * self.side
            if self.side % 2:
                raise ConfigurationError(
                    f"side must be even for the checkerboard sweep, got {self.side}")
            if self.iterations % n or self.swap_interval % n:
                raise ConfigurationError(
                    "iterations and swap_interval must be whole sweeps (multiples of side**2) "
                    "in checkerboard mode")
            if (self.iterations // n) // self.record_every < 1 and self.record_mode != "none":
                raise ConfigurationError("record_every exceeds the number of sweeps")

    def ladder(self) -> np.ndarray:
        if self.temperatures is not None:
            return np.asarray(self.temperatures, dtype=np.float64)
        return build_ladder(self.replicas)


@dataclass
class RunRecord:
    """Everything one run produced (executor.py:70-88, plus extensions).

    Checkerboard records (``sweep_mode="checkerboard"``): ``rng_positions``
    is the init phase's stream consumption (L^2 - 1 per slot; Mode F draws
    are addressed by slot, sweep, colour and site, so no position advances
    after init), and ``round_entry_iterations[k]`` is the iteration count
    (sweeps x L^2) every slot had completed when round k was decided -- the
    reference's barrier audit (executor.py:228-229,253-256).  On the
    resident path the rounds run inside one launch behind a grid barrier and
    the row is the schedule's value; the barrier itself is what every
    resident parity test checks.
    """

    config: SimulationConfig
    temperatures: np.ndarray
    energies: np.ndarray | None
    magnetizations: np.ndarray | None
    states: np.ndarray | None
    swap_rounds: int
    swaps_attempted: int
    swaps_accepted: int
    rng_positions: np.ndarray
    round_entry_iterations: np.ndarray | None
    init_seconds: float
    exec_seconds: float
    total_seconds: float
    valid: bool = True
    error: str | None = None
    # --- extensions
    sweep_mode: str = "exact"
    swap_near_ties: int = 0
    final_spins: np.ndarray | None = None
    slot_to_row: np.ndarray | None = None


def assign_replicas(replica_count: int, workers: int) -> list[tuple[int, int]]:
    """Contiguous ranges, sizes differing by at most one (executor.py:91-102);
    also the row sharding across GPUs (distributed.py)."""
    if workers < 1:
        raise ConfigurationError(f"workers must be >= 1, got {workers}")
    base, extra = divmod(replica_count, workers)
    bounds, lo = [], 0
    for w in range(workers):
        hi = lo + base + (1 if w < extra else 0)
        bounds.append((lo, hi))
        lo = hi
    return bounds


def _interval_plan(iterations: int, interval: int) -> list[tuple[int, int | None]]:
    """(target count, swap round or None) per interval (executor.py:111-125)."""
    plan: list[tuple[int, int | None]] = []
    if interval > 0:
        k = 1
        while k * interval < iterations:
            plan.append((k * interval, k - 1))
            k += 1
    plan.append((iterations, None))
    return plan


def _resident_wins(L: int, swap_every_sweeps: int) -> bool:
    """The resident run (sweeps and rounds in one launch) below L = 1024,
    where the one-launch-per-interval sweep kernel does not apply and the
    per-launch sweeps are launch-latency bound, and for per-sweep exchanges.
    Measured (one B200, attempts/s, resident vs sweep path): 512^2 x 64 every
    10 sweeps 1.57e12 vs 9.1e11; 384^2 x 64 every 5: 1.13e12 vs 4.2e11;
    512^2 x 256 every 10: 2.25e12 vs 2.0e12; 1024^2 x 64 every sweep: 1.73e12
    vs 1.68e12; 1024^2 x 16 every 10: 1.06e12 vs 1.61e12."""
    return L < 1024 or swap_every_sweeps == 1


class _StateStream:
    """full_states recording for the checkerboard chain: each sample is
    unpacked on the device in slot order into one of two staging buffers and
    copied asynchronously into its own contiguous block of a pinned host array
    (n_samples, R, L, L), so the copy of sample c overlaps the sweeps towards
    sample c+1; result() returns the reference's (R, n_samples, L, L) layout."""

    def __init__(self, R: int, n: int, L: int, dev):
        self.host = torch.empty((n, R, L, L), dtype=torch.int8, pin_memory=True)
        self.stage = [torch.empty((R, L, L), dtype=torch.int8, device=dev) for _ in range(2)]
        self.done = [torch.cuda.Event(), torch.cuda.Event()]
        self.copy = torch.cuda.Stream(dev)
        self.k = 0

    def push(self, eng, col: int) -> None:
        b = self.k & 1
        self.done[b].synchronize()  # the copy that last used this buffer finished
        eng.snapshot_by_slot(self.stage[b])
        self.copy.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.copy):
            self.host[col].copy_(self.stage[b], non_blocking=True)
            self.done[b].record(self.copy)
        self.k += 1

    def result(self) -> np.ndarray:
        self.copy.synchronize()
        return np.ascontiguousarray(self.host.numpy().transpose(1, 0, 2, 3))


def _sync(dev):
    torch.cuda.synchronize(dev)


def run(config: SimulationConfig) -> RunRecord:
    """Execute one simulation on the GPU: init phase, then synchronized
    intervals.  Mid-run failures return a record flagged invalid
    (executor.py:283-299); invalid configurations raise first."""
    config.validate()
    if config.sweep_mode == "checkerboard":
        return _run_checkerboard(config)
    return _run_exact(config)


def _run_exact(config: SimulationConfig) -> RunRecord:
    from .engine import ExactEngine, require_cuda

    t_start = time.perf_counter()
    R, L, N, I = config.replicas, config.side, config.iterations, config.swap_interval
    rec_flag = RECORD_MODES.index(config.record_mode)
    dev = require_cuda(config.devices[0] if config.devices is not None else config.device)
    temps = config.ladder()
    eng = None
    errors: list[BaseException] = []
    obs_e = obs_m = states = None
    rounds = attempted = 0
    snaps = None
    init_seconds = exec_seconds = 0.0
    with torch.cuda.device(dev):
        t0 = time.perf_counter()
        eng = ExactEngine(L, R, temps, config.seed, config.params.J, config.params.B,
                          config.init_up_fraction, dev)
        eng.init_state()
        k = config.record_every
        sub = rec_flag == 1 and k > 1  # subsampled observables: column c = state after (c+1)k iterations
        if rec_flag >= 1:
            ncol = N // k if sub else N
            obs_e = torch.empty((R, ncol), dtype=torch.float64, device=dev)
            obs_m = torch.empty((R, ncol), dtype=torch.float64, device=dev)
        if rec_flag == 2:
            states = torch.empty((R, N, L, L), dtype=torch.int8, device=dev)
        if sub:
            eng.advance(0, 1)  # iteration 0 (executor.py:218-220)
        else:
            eng.advance(0, 1, obs_e, obs_m, rec_flag, states)

        def sample(done: int) -> None:
            # the reference's column done-1 (kernels.py:103-105): E and sum(s)/L^2 by slot
            if done % k == 0:
                obs_e[:, done // k - 1].copy_(eng.energies)
                obs_m[:, done // k - 1].copy_(eng.spin_sums.to(torch.float64) / float(L * L))
        _sync(dev)
        init_seconds = time.perf_counter() - t0

        t1 = time.perf_counter()
        plan = _interval_plan(N, I)
        n_rounds = sum(1 for _, ri in plan if ri is not None)
        snaps = np.zeros((n_rounds, R), dtype=np.int64) if rec_flag >= 1 and n_rounds else None
        completed = 1
        try:
            if sub:
                for target, ri in plan:
                    while completed < target:
                        nxt = min(target, (completed // k + 1) * k)
                        eng.advance(completed, nxt - completed)
                        completed = nxt
                        sample(completed)
                    if ri is None:
                        continue
                    if snaps is not None:
                        snaps[ri, :] = completed
                    rounds += 1
                    attempted += eng.exchange(ri)
            elif config.kernel != "sweep" and eng.resident_ok(rec_flag):
                # few small lattices (the reference's C1): the whole run with its
                # rounds in chunked launches (csrc/exact.cu, exact_resident_kernel)
                eng.run_resident(1, N - 1, I, N, obs_e, obs_m)
                for target, ri in plan:
                    if ri is None:
                        continue
                    if snaps is not None:
                        snaps[ri, :] = target
                    rounds += 1
                    attempted += max(0, (R - ri % 2) // 2)
            else:
                for target, ri in plan:
                    if target > completed:
                        eng.advance(completed, target - completed, obs_e, obs_m, rec_flag, states)
                    completed = target
                    if ri is None:
                        continue
                    if snaps is not None:
                        snaps[ri, :] = completed  # == iters_done of every slot
                    rounds += 1
                    attempted += eng.exchange(ri)
            _sync(dev)
        except BaseException as exc:  # noqa: BLE001 - any failure invalidates the run
            errors.append(exc)
        exec_seconds = time.perf_counter() - t1

    valid = not errors
    accepted, near = eng.swap_counts() if valid else (0, 0)
    return RunRecord(
        config=config, temperatures=temps,
        energies=obs_e.cpu().numpy() if (valid and obs_e is not None) else None,
        magnetizations=obs_m.cpu().numpy() if (valid and obs_m is not None) else None,
        states=states.cpu().numpy() if (valid and states is not None) else None,
        swap_rounds=rounds, swaps_attempted=attempted, swaps_accepted=accepted,
        rng_positions=eng.positions.cpu().numpy() if valid else np.zeros(R, np.int64),
        round_entry_iterations=snaps, init_seconds=init_seconds, exec_seconds=exec_seconds,
        total_seconds=time.perf_counter() - t_start, valid=valid,
        error=None if valid else repr(errors[0]), sweep_mode="exact", swap_near_ties=near,
        final_spins=eng.final_spins() if (valid and config.return_final_state) else None,
        slot_to_row=eng.slot_to_row.cpu().numpy() if (valid and config.return_final_state) else None)


def _process_group(config: SimulationConfig) -> bool:
    """The process group a ``devices`` run shards over; opens a world-1 NCCL
    group when there is none and one device is named (returns True then, so
    the caller closes it).  Raises ConfigurationError before any work when
    the launch does not match ``devices``."""
    import os
    import socket

    import torch.distributed as dist

    n = len(config.devices)
    if dist.is_available() and dist.is_initialized():
        if dist.get_world_size() != n:
            raise ConfigurationError(
                f"devices names {n} GPU(s) but the process group has {dist.get_world_size()} rank(s)")
        return False
    if n != 1:
        raise ConfigurationError(
            f"devices={tuple(config.devices)!r}: a multi-GPU run is one process per device; launch it "
            f"with torchrun --nproc-per-node {n} (or init the process group) and call run() on every rank")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", int(config.devices[0])))
    return True


def _run_checkerboard(config: SimulationConfig) -> RunRecord:
    from .engine import require_cuda

    sharded = config.devices is not None
    own_group = _process_group(config) if sharded else False
    try:
        if sharded:
            import torch.distributed as dist
            dev = require_cuda(config.devices[dist.get_rank()])
        else:
            dev = require_cuda(config.device)
        return _checkerboard_on(config, dev, sharded)
    finally:
        if own_group:
            import torch.distributed as dist
            dist.destroy_process_group()


def _checkerboard_on(config: SimulationConfig, dev, sharded: bool) -> RunRecord:
    from .engine import CheckerboardEngine

    t_start = time.perf_counter()
    R, L = config.replicas, config.side
    n_sites = L * L
    sweeps, every_sw = config.iterations // n_sites, config.swap_interval // n_sites
    record = config.record_mode != "none"
    temps = config.ladder()
    errors: list[BaseException] = []
    drv = peers = None
    with torch.cuda.device(dev):
        t0 = time.perf_counter()
        if sharded:
            from .distributed import ShardedCheckerboard
            drv = ShardedCheckerboard(L, R, temps, config.seed, config.params.J, config.params.B,
                                      config.init_up_fraction, device=dev)
            eng = drv.eng
            drv.init_state()
        else:
            eng = CheckerboardEngine(L, R, temps, config.seed, config.params.J, config.params.B,
                                     config.init_up_fraction, dev)
            eng.init_state()
        n_samples = sweeps // config.record_every if record else 0
        obs_e = torch.zeros((R, n_samples), dtype=torch.float64, device=dev) if record else None
        obs_m = torch.zeros((R, n_samples), dtype=torch.float64, device=dev) if record else None
        full = config.record_mode == "full_states"
        states = _StateStream(R, n_samples, L, dev) if full else None
        _sync(dev)
        init_seconds = time.perf_counter() - t0

        t1 = time.perf_counter()
        plan = _interval_plan(sweeps, every_sw)
        n_rounds = sum(1 for _, ri in plan if ri is not None)
        snaps = np.zeros((n_rounds, R), dtype=np.int64) if record and n_rounds else None
        done = rounds = attempted = 0
        use_resident = not full and (config.kernel == "resident" or
                                     (config.kernel == "auto" and _resident_wins(L, every_sw)))
        try:
            if use_resident:
                # the whole run in one persistent launch (per rank; across
                # ranks the rounds go through peer memory); the schedule is
                # replayed on the host only for the bookkeeping fields
                rec_every = config.record_every if record else 0
                if sharded:
                    from .distributed import PeerBuffers, resident_sharded
                    peers = PeerBuffers(R, dev)
                    resident_sharded(drv, peers, 0, sweeps, sweeps, every_sw, rec_every, obs_e, obs_m)
                else:
                    eng.run_resident(0, sweeps, sweeps, every_sw, rec_every, obs_e, obs_m)
                for target, ri in plan:
                    if ri is None:
                        continue
                    if snaps is not None:
                        snaps[ri, :] = target * n_sites
                    rounds += 1
                    attempted += max(0, (R - ri % 2) // 2)
                plan = []
            gathered = -1  # sweep count at which every lattice's (S, Bond) was last all-gathered
            for target, ri in plan:
                while done < target:
                    if record:
                        nxt = min(target, (done // config.record_every + 1) * config.record_every)
                    else:
                        nxt = target
                    eng.sweeps(done, nxt - done)
                    done = nxt
                    if record and done % config.record_every == 0:
                        if sharded and gathered != done:
                            drv.gather_stats()
                            gathered = done
                        eng.observe(obs_e, obs_m, done // config.record_every - 1)
                        if full:
                            states.push(eng, done // config.record_every - 1)
                if ri is None:
                    continue
                if snaps is not None:
                    snaps[ri, :] = done * n_sites
                rounds += 1
                if sharded and gathered != done:
                    drv.gather_stats()
                    gathered = done
                attempted += eng.exchange(ri)
            _sync(dev)
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)
        finally:
            if peers is not None:
                peers.close()
        exec_seconds = time.perf_counter() - t1

    valid = not errors
    accepted, near = eng.swap_counts() if valid else (0, 0)
    final = None
    if valid and config.return_final_state:
        final = _gather_lattices(drv) if sharded else eng.final_spins()
    return RunRecord(
        config=config, temperatures=temps,
        energies=obs_e.cpu().numpy() if (valid and record) else None,
        magnetizations=obs_m.cpu().numpy() if (valid and record) else None,
        states=states.result() if (valid and full) else None, swap_rounds=rounds,
        swaps_attempted=attempted, swaps_accepted=accepted,
        # Mode F draws are addressed by (slot, sweep, colour, site) and never
        # advance a stream position; the init phase's Fisher-Yates is the only
        # positional consumer (L^2 - 1 draws of stream r, kernels.py:26-45)
        rng_positions=np.full(R, n_sites - 1, dtype=np.int64),
        round_entry_iterations=snaps, init_seconds=init_seconds, exec_seconds=exec_seconds,
        total_seconds=time.perf_counter() - t_start, valid=valid,
        error=None if valid else repr(errors[0]), sweep_mode="checkerboard", swap_near_ties=near,
        final_spins=final,
        slot_to_row=eng.slot_to_row.cpu().numpy() if (valid and config.return_final_state) else None)


def _gather_lattices(drv) -> np.ndarray:
    """Every rank's int8 lattices, in row order, on every rank."""
    from .distributed import all_gather_into

    eng = drv.eng
    loc = eng.spins_int8()
    pad = torch.zeros((drv.maxc, eng.L, eng.L), dtype=torch.int8, device=loc.device)
    pad[: loc.shape[0]].copy_(loc)
    out = torch.empty((drv.world * drv.maxc, eng.L, eng.L), dtype=torch.int8, device=loc.device)
    all_gather_into(out, pad, drv.group)
    parts = [out[g * drv.maxc: g * drv.maxc + (h - l)] for g, (l, h) in enumerate(drv.bounds)]
    return torch.cat(parts).cpu().numpy()
