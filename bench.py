"""Benchmark: spin-flip attempts/s of the PT Metropolis sampling loop.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c1|c2|c4|c5]

--gpus N without a torchrun environment re-launches this script under
``python -m torch.distributed.run --nproc-per-node N`` (one rank per GPU,
127.0.0.1 rendezvous) after checking that N GPUs are visible; under torchrun
WORLD_SIZE must equal N.  Either mismatch exits non-zero with a message.

Workload (default, BASELINE.json configs[2], the config the metric's target is
quoted on): 2D Ising 1024^2, 256 replicas, linear ladder 1+3i/R, J=1, B=0,
exchange every 10 sweeps.  A step = one exchange interval = 10 checkerboard
sweeps of every replica + one swap round (energies from the fused reduction,
reference swap rule).  Attempts per step = R * L^2 * 10.

* value: device-resident, CUDA events around each step, L2 flushed between
  steps (256 MiB write), max over ranks.
* e2e: the host-buffer plugin call (kernels.cb_interval -> C ABI
  ptmh_host_cb_interval) on pinned int8 lattices, host<->device copies of the
  lattices inside the timed region, pipelined against the sweeps.  For the
  resident configurations (C1, C2, C5: 100 one-sweep intervals per step in
  one launch) the e2e step is the same 100 intervals: int8 lattices and the
  permutation in from pinned host memory, load_spins -> run_resident ->
  spins_int8, lattices, permutation and (S, Bond) back.
* roofline: the half-sweep kernel, algorithmic bytes = 0.25 B per attempt
  (1-bit spin read + written) x R*L^2/2 attempts per launch,
  over its CUDA-event duration inside the timed steps.
* cpu_baseline / --impl reference: the reference's own algorithm (random-site
  chain, kernels.py:62-113) restated in C (oracle/, "port") on all host cores
  over a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (L, R, sweeps per exchange interval, description)
    "c1": (32, 8, 1, "2D Ising 32x32, 8 replicas, geometric T-ladder, exchange every sweep"),
    "c2": (256, 64, 1, "2D Ising 256x256, 64 replicas, exchange every sweep"),
    "c3": (1024, 256, 10, "2D Ising 1024x1024, 256 replicas, exchange every 10 sweeps"),
    "c4": (4096, 512, 10, "2D Ising 4096x4096, 512 replicas, exchange every 10 sweeps"),
    "c5": (64, 4096, 1, "2D Ising 64x64, 4096 replicas, exchange every sweep"),
}
# exchange intervals per timed step: one for the big lattices, 100 (one
# persistent launch of 100 sweeps + 100 rounds) where an interval is 1 sweep
INTERVALS_PER_STEP = {"c1": 100, "c2": 100, "c3": 1, "c4": 1, "c5": 100}
SEED = 42
ALG_BYTES_PER_ATTEMPT = 0.25  # 1-bit multispin coding: read + write one bit


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def _issue(cfg_name):
    """IPC / ALU-pipe share of the hot kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")) as f:
            return json.load(f)[cfg_name].get("issue")
    except Exception:  # noqa: BLE001
        return None


def _traffic(cfg_name):
    """dram bytes per half-sweep launch from the committed ncu --set full
    capture summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        ent = d.get(cfg_name)
        return None if ent is None else float(ent["dram_bytes_per_launch"])
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        # NVML is initialised here, before the timed region (nvmlInit can take
        # longer than a whole C3 run); each query then costs ~1 ms
        self._nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._bits = (nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                          nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap)
            self._smax = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._nv = nv
        except Exception:  # noqa: BLE001
            self._nv = None

    def _run(self):
        nv, h, bits = self._nv, getattr(self, "_h", None), getattr(self, "_bits", ())
        smax = getattr(self, "_smax", None)
        while not self._stop.is_set():
            try:
                if nv is not None:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.samples.append([str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), str(smax)]
                                        + ["Active" if r & b else "Not Active" for b in bits])
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------ CPU reference --
def cpu_reference_rate(L, R, attempts_per_slot, threads, reps=1):
    """Reference random-site chain (oracle C port of kernels.py:62-113,
    executor.py:227-245 worker pool) on `threads` host cores; returns
    (attempts/s, attempts, seconds)."""
    import oracle

    rs = np.random.default_rng(SEED)
    spins = (rs.integers(0, 2, size=(R, L, L)) * 2 - 1).astype(np.int8)
    betas = 1.0 / oracle.build_ladder(R)
    energies = np.array([oracle.lattice_energy(spins[r], 1.0, 0.0) for r in range(R)])
    sums = spins.reshape(R, -1).sum(axis=1).astype(np.int64)
    s2r = np.arange(R, dtype=np.int64)
    pos = np.full(R, L * L - 1, dtype=np.uint64)
    iters = np.zeros(R, dtype=np.int64)
    oracle.advance_block_mt(spins, s2r, betas, 1.0, 0.0, energies, sums, pos, iters, SEED, 1,
                            max(1, attempts_per_slot // 100), threads)  # warm
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.advance_block_mt(spins, s2r, betas, 1.0, 0.0, energies, sums, pos, iters, SEED,
                                1, attempts_per_slot, threads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    n = R * attempts_per_slot
    return n / best, n, best


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# ----------------------------------------------------------------- launcher --
def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _visible_gpus() -> int:
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _launch_ranks(args) -> int:
    """Re-run this script as args.gpus ranks under torchrun (one per GPU);
    returns the exit code.  Refuses (exit 2) when fewer GPUs are visible."""
    if args.impl == "ours":
        have = _visible_gpus()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, this host has {have}",
                  file=sys.stderr, flush=True)
            return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the init log shows the rank count
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
    cmd += [a for a in sys.argv[1:] if a != "--spawn"]
    return subprocess.run(cmd, env=env).returncode


# --------------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the exact-chain side measurement")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU coordinator (NCCL all_gather) even at one rank")
    ap.add_argument("--spawn", action="store_true",
                    help="launch the ranks under torchrun even for --gpus 1 (tests the launcher)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus < 1:
        print("bench.py: --gpus must be >= 1", file=sys.stderr)
        sys.exit(2)
    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.spawn):
        sys.exit(_launch_ranks(args))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']} ranks were launched",
              file=sys.stderr, flush=True)
        sys.exit(2)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    L, R, every, desc = CONFIGS[args.config]
    ips = INTERVALS_PER_STEP[args.config]
    attempts_per_step = R * L * L * every * ips
    config = {"workload": desc, "side": L, "replicas": R, "sweeps_per_step": every * ips,
              "exchange_rounds_per_step": ips,
              "attempts_per_step": attempts_per_step, "J": 1.0, "B": 0.0,
              "ladder": "geometric 4^(i/(R-1))" if args.config == "c1" else "linear 1+3i/R",
              "sweep": "checkerboard, 1-bit multispin", "l2": "flushed between steps (256 MiB write)",
              "chain": "checkerboard Metropolis (Mode F, DESIGN.md 3): a different Markov chain from the "
                       "reference's random-site chain, statistically equal to it; the like-for-like, "
                       "bit-exact reference chain is the exact_chain entry",
              "parallelism": f"rows sharded over {world} GPU(s), energies all-gathered"}
    metric = "spin-flip attempts/sec"

    if args.impl == "reference":
        if rank != 0:
            return
        world = max(world, args.gpus)
        config = dict(config, sweep="reference random-site chain (kernels.py:62-113), int8 spins",
                      chain="the reference's random-site Metropolis chain (its C restatement, oracle/)",
                      parallelism=f"{host_cores()} host threads over replica blocks "
                                  "(executor.py:227-245)", l2="n/a (CPU)")
        threads = host_cores()
        per_slot = max(1000, int(2.5e7 // R))  # ~1 s of 8-core work per step
        # each step: every slot of the timed shape advances per_slot attempts
        # of the reference chain (a bounded sample of the config's step)
        config = dict(config, attempts_per_step=R * per_slot,
                      config_attempts_per_step=attempts_per_step)
        for _ in range(args.warmup):  # warm-up on the timed shape
            cpu_reference_rate(L, R, max(100, per_slot // 10), threads)
        times = []
        for _ in range(args.steps):
            rate, n, dt = cpu_reference_rate(L, R, per_slot, threads)
            times.append(dt)
        tot = sum(times)
        val = args.steps * R * per_slot / tot
        line = {"metric": metric, "value": val, "unit": "attempts/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
                "scaling": "none", "vs_baseline": None, "dtype": "int8/f64", "data": "synthetic",
                "impl": "reference", "config": config,
                "note": "the reference runs on the host CPU (rank 0 only); n_gpus is the job's GPU count",
                "cpu_baseline": {"value": val, "unit": "attempts/s", "cores": threads, "kind": "port",
                                 "sample": f"{R} slots x {per_slot} random-site attempts per step "
                                           f"(reference chain kernels.py:62-113, C port, "
                                           f"{threads} threads)"},
                "e2e": {"value": val, "unit": "attempts/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    from paper_2512_03825_b200 import geometric_ladder, build_ladder, kernels
    from paper_2512_03825_b200.distributed import ShardedCheckerboard
    from paper_2512_03825_b200.engine import CheckerboardEngine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    clk = ClockSampler(local_rank)
    sharded = world > 1 or args.sharded
    if sharded:
        if "RANK" not in os.environ:  # --sharded without torchrun: a world of one
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))
        dist.init_process_group("nccl", device_id=dev)
    temps = geometric_ladder(R) if args.config == "c1" else build_ladder(R)
    if sharded:
        drv = ShardedCheckerboard(L, R, temps, SEED, device=local_rank)
        eng = drv.eng
        drv.init_state()
    else:
        drv = None
        eng = CheckerboardEngine(L, R, temps, SEED, 1.0, 0.0, 0.5, local_rank)
        eng.init_state()
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    state = {"sweep": 0, "round": 0}
    from paper_2512_03825_b200.executor import _resident_wins
    # small lattices, exchange every sweep: one persistent launch per step;
    # across GPUs the rounds go through peer memory (distributed.PeerBuffers)
    resident = _resident_wins(L, every)
    peers = None
    if sharded and resident:
        from paper_2512_03825_b200.distributed import PeerBuffers, resident_sharded
        peers = PeerBuffers(R, dev)
        config["parallelism"] = (f"rows sharded over {world} GPU(s), exchange rounds through peer "
                                 f"memory (CUDA IPC, no collective)")
    # the engine's sweeps() takes the one-launch persistent path here
    # (csrc/checkerboard.cu: cb_sweeps_persistent, J > 0, B = 0, L % 512 == 0)
    persistent = not resident and eng.persistent and L >= 1024 and L % 512 == 0
    big = 1 << 30  # run length for the resident kernel: every interval ends in a round

    def step(sweep_events=None):
        t0 = state["sweep"]
        if resident:  # one persistent launch = `ips` intervals, sweeps + exchange rounds
            if sweep_events is not None:
                sweep_events[0][0].record(stream)
            if peers is not None:
                resident_sharded(drv, peers, t0, every * ips, big, every)
            else:
                eng.run_resident(t0, every * ips, big, every)
            if sweep_events is not None:
                sweep_events[0][1].record(stream)
            state["sweep"] += every * ips
            state["round"] += ips
            return
        if ips != 1:
            raise ValueError("multi-interval steps are only defined for the resident path")
        if sweep_events is not None:
            sweep_events[0][0].record(stream)
        eng.sweeps(t0, every)
        if sweep_events is not None:
            sweep_events[0][1].record(stream)
        if drv is not None:
            drv.gather_stats()
        eng.exchange(state["round"])
        state["sweep"] += every
        state["round"] += 1

    step_ms, sweep_ms = [], []
    with clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        for it in range(args.steps):
            # per-launch events in every 4th timed step (they cost ~1-2 us each)
            probe = it % 4 == 0
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))] \
                if probe else None
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if sharded:
                dist.barrier()
            torch.cuda.synchronize()
            # L2 flush, then the step: its launches are queued while the GPU
            # runs the flush, so the timed region (s0 .. s1) holds the step's
            # GPU work and not the host's launch latency
            flush.zero_()
            s0.record(stream)
            step(ev)
            s1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            if probe:
                sweep_ms.extend(a.elapsed_time(b) for a, b in ev)
    from paper_2512_03825_b200 import _lib
    launched = _lib.cb_last_launch()  # this thread's last sweep launch (a timed step's)
    total_ms = sum(step_ms)
    if sharded:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = args.steps * attempts_per_step / (total_ms / 1e3)
    local_rows = eng.rows
    if resident:  # one launch per step: `every` sweeps of every lattice + the round
        sweep_ms = [m for m in sweep_ms if m > 0]
        launch_ms = statistics.mean(sweep_ms)
        bytes_per_launch = ALG_BYTES_PER_ATTEMPT * local_rows * L * L * every * ips
        kernel_name = launched["name"]
    elif persistent:  # one launch per interval: all 2*every half-sweeps
        launch_ms = statistics.mean(sweep_ms)
        bytes_per_launch = ALG_BYTES_PER_ATTEMPT * local_rows * L * L * every
        # the kernel the launcher picked for the timed steps (ptmh_cb_last_launch)
        kernel_name = launched["name"]
    else:
        launch_ms = statistics.mean(sweep_ms) / (2.0 * every)  # two colour launches per sweep
        bytes_per_launch = ALG_BYTES_PER_ATTEMPT * local_rows * L * L / 2
        kernel_name = launched["name"]
    achieved = bytes_per_launch / (launch_ms / 1e3) / 1e9
    peak, peak_kind = _peaks()
    traffic = _traffic(args.config) if not sharded and not resident else None

    # ---- end to end through the host-buffer plugin (rank 0, single device)
    e2e = None
    if not args.no_e2e and not sharded and resident:
        # the step's `ips` intervals in one resident launch, as the timed
        # step, with the lattices and the permutation in from pinned host
        # memory and the lattices, the permutation and every lattice's
        # (S, Bond) back, every step (the per-interval plugin call,
        # kernels.cb_interval, would time `ips` calls of a few us of work each)
        loc = eng.spins_int8()
        host = torch.empty(tuple(loc.shape), dtype=torch.int8).pin_memory()
        host.copy_(loc)
        dbuf = torch.empty_like(loc)
        s2r_h = eng.slot_to_row.cpu().pin_memory()
        r2s_h = eng.row_to_slot.cpu().pin_memory()
        stats_h = torch.empty(tuple(eng.stats.shape), dtype=torch.int64).pin_memory()
        sweep0 = state["sweep"]

        def e2e_step(t):
            dbuf.copy_(host, non_blocking=True)
            eng.slot_to_row.copy_(s2r_h, non_blocking=True)
            eng.row_to_slot.copy_(r2s_h, non_blocking=True)
            eng.load_spins(dbuf)
            eng.run_resident(t, every * ips, big, every)
            host.copy_(eng.spins_int8(), non_blocking=True)
            s2r_h.copy_(eng.slot_to_row, non_blocking=True)
            r2s_h.copy_(eng.row_to_slot, non_blocking=True)
            stats_h.copy_(eng.stats, non_blocking=True)

        for k in range(2):  # warm
            e2e_step(sweep0)
            sweep0 += every * ips
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for k in range(n_e2e):
            e2e_step(sweep0)
            sweep0 += every * ips
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        e2e = {"value": n_e2e * attempts_per_step / dt, "unit": "attempts/s",
               "h2d_bytes_per_step": int(R * L * L + 12 * R), "d2h_bytes_per_step": int(R * L * L + 28 * R),
               "path": "CheckerboardEngine.load_spins -> run_resident -> spins_int8 (the engine run() "
                       "drives): pinned int8 lattices + permutation in, lattices + permutation + "
                       f"(S, Bond) out, {ips} intervals per step in one resident launch; wall clock"}
    elif not args.no_e2e and not sharded:
        spins_h = eng.final_spins()
        pinned = torch.from_numpy(spins_h).pin_memory()
        sp = pinned.numpy()
        s2r = eng.slot_to_row.cpu().numpy().copy()
        betas = 1.0 / temps
        e = np.zeros(R)
        ss = np.zeros(R, dtype=np.int64)
        sweep0, rnd0 = state["sweep"], state["round"]
        for k in range(2):  # warm the workspace
            kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, SEED, sweep0, every, rnd0, e, ss)
            sweep0 += every
            rnd0 += 1
        n_e2e = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for k in range(n_e2e):
            kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, SEED, sweep0, every, rnd0, e, ss)
            sweep0 += every
            rnd0 += 1
        dt = time.perf_counter() - t0
        e2e = {"value": n_e2e * R * L * L * every / dt, "unit": "attempts/s",
               "h2d_bytes_per_step": int(R * L * L + R * 8 + R * 40 + R * 4 + R * 8),
               "d2h_bytes_per_step": int(R * L * L + R * 8 * 3 + 16),
               "path": "kernels.cb_interval -> ptmh_host_cb_interval (pinned int8 lattices)"}

    # ---- end to end across ranks (N > 1): the same interval through the
    # sharded driver, each rank's int8 lattices copied in from and out to
    # pinned host memory every step (the host plugin is single-device)
    if not args.no_e2e and sharded:
        loc = eng.spins_int8()
        host = torch.empty(tuple(loc.shape), dtype=torch.int8).pin_memory()
        host.copy_(loc)
        dbuf = torch.empty_like(loc)
        sweep0, rnd0 = state["sweep"], state["round"]

        def e2e_step(t, r):
            dbuf.copy_(host, non_blocking=True)
            eng.load_spins(dbuf)
            if resident:  # the step's intervals in one launch per rank, peer-memory rounds
                resident_sharded(drv, peers, t, every * ips, big, every)
            else:
                eng.sweeps(t, every)
                drv.gather_stats()
                eng.exchange(r)
            host.copy_(eng.spins_int8(), non_blocking=True)

        # (an e2e step is the timed step: one interval, or `ips` of them in one
        # resident launch)
        span = every * (ips if resident else 1)
        for k in range(2):  # warm
            e2e_step(sweep0, rnd0)
            sweep0 += span
            rnd0 += 1
        n_e2e = max(3, min(args.steps, 10))
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(n_e2e):
            e2e_step(sweep0, rnd0)
            sweep0 += span
            rnd0 += 1
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": n_e2e * R * L * L * span / float(dt.item()), "unit": "attempts/s",
               "h2d_bytes_per_step": int(R * L * L), "d2h_bytes_per_step": int(R * L * L),
               "path": "distributed.ShardedCheckerboard" + (" + resident_sharded" if resident else "")
                       + ", per-rank int8 lattices from / to pinned host memory each step (bytes summed "
                         "over ranks); wall clock, max over ranks"}

    # the bit-exact reference chain (sweep_mode="exact") on the same shape
    exact = None
    if rank == 0 and not sharded and not args.no_exact and L <= 4096:
        from paper_2512_03825_b200.engine import ExactEngine
        del eng
        torch.cuda.empty_cache()
        ex = ExactEngine(L, R, temps, SEED, 1.0, 0.0, 0.5, local_rank)
        ex.init_state()
        n_att = max(32, int(2e8 // R))
        done = 1
        # few slots (C1): the resident run WITH the config's swap rounds
        res = ex.resident_ok(0)
        I = every * L * L
        big = 1 << 60

        def adv(start, n):
            if res:
                ex.run_resident(start, n, I, big)
            else:
                ex.advance(start, n)

        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.3:  # warm, clocks up
            adv(done, n_att)
            done += n_att
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        adv(done, n_att)
        b.record(stream)
        torch.cuda.synchronize()
        exact = {"value": R * n_att / (a.elapsed_time(b) / 1e3), "unit": "attempts/s",
                 "chain": "reference random-site chain, bit-exact with isingpt ("
                          + ("resident run with a swap round every %d attempts" % I if res
                             else "two-phase kernels, no rounds") + ")",
                 "sample": f"{R} slots x {n_att} attempts, record none"}
        del ex

    cpu = None
    if rank == 0 and not sharded and not args.no_cpu:
        threads = host_cores()
        per_slot = max(1000, int(1.5e8 // R))
        rate, n, dt = cpu_reference_rate(L, R, per_slot, threads)
        cpu = {"value": rate, "unit": "attempts/s", "cores": threads, "kind": "port",
               "sample": f"{R} slots x {per_slot} random-site attempts on {L}^2 lattices "
                         f"({n:.3g} attempts, {dt:.1f} s; reference chain kernels.py:62-113 "
                         f"in C, {threads} threads)"}

    issue = _issue(args.config) if not resident and not sharded else None
    issue_frac = None
    if issue and issue.get("ipc_active"):  # ncu IPC of the same kernel / 4 issue slots per SM per cycle
        issue_frac = float(issue["ipc_active"][0]) / float(issue.get("ipc_peak", 4.0))
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "attempts/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u32 (1-bit spins), integer RNG", "data": "synthetic (seeded exact-count init)",
                "config": config,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "kernel": kernel_name, "launch_ms": launch_ms,
                             "alg_bytes_per_launch": bytes_per_launch, "peak_kind": peak_kind,
                             "note": "the bound is instruction issue (Philox + bit-sliced logic), not HBM: "
                                     "see issue_frac and DESIGN.md 5",
                             "issue_frac": issue_frac,
                             "issue_from_ncu": issue,
                             "traffic_note": "ncu dram read+write bytes per launch of the same kernel "
                                             "(profiles/ncu_sweep_summary.json); below the algorithmic "
                                             "bytes when the packed state stays in L2 across the "
                                             "launch's sweeps"},
                "cpu_baseline": cpu, "e2e": e2e, "exact_chain": exact,
                "gpu_launches": args.steps * (1 if resident else (1 if persistent else 2 * every) + 1),
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
