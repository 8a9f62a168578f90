"""Generate the golden fixtures in tests/golden/ by importing the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``isingpt`` read-only from /root/reference/pkg/src with numba's
cache redirected to /tmp and writes small .npz files that
pin the oracle (tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_exact.py).  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import isingpt  # noqa: E402
from isingpt import kernels, rng  # noqa: E402
from isingpt.executor import SimulationConfig, run  # noqa: E402
from isingpt.lattice import IsingParams  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
U = np.uint64


def philox_vectors():
    addrs = [(42, 0, 0), (42, 0, 1), (42, 1, 0), (42, 8, 3), (7, 3, 1023),
             (0, 0, 0), (2 ** 64 - 1, 3, 1), (2 ** 63 + 5, 2 ** 40, 12345),
             (123456789, 7, 99), (5, 2 ** 33 + 7, 2 ** 50 + 3)]
    rs = np.random.default_rng(2024)
    for _ in range(54):
        addrs.append((int(rs.integers(0, 2 ** 63)) * 2 + int(rs.integers(0, 2)),
                      int(rs.integers(0, 5000)), int(rs.integers(0, 2 ** 40))))
    a = np.array(addrs, dtype=np.uint64)
    w = np.array([int(rng._philox_word0(U(s), U(t), U(p))) for s, t, p in addrs],
                 dtype=np.uint64)
    u = np.array([float(rng.stream_uniform(U(s), U(t), U(p))) for s, t, p in addrs])
    np.savez_compressed(os.path.join(OUT, "philox4x64.npz"), addr=a, word0=w, uniform=u)


def kernel_vectors():
    out = {}
    # fill_lattice: several sides / up counts / streams
    cases = [(2, 2, 42, 0), (3, 4, 42, 1), (8, 32, 7, 3), (16, 100, 9, 5),
             (32, 512, 42, 0), (64, 2048, 42, 17), (5, 0, 1, 0), (5, 25, 1, 0)]
    for k, (L, up, seed, stream) in enumerate(cases):
        a = np.empty((L, L), dtype=np.int8)
        pos = kernels.fill_lattice(a, up, U(seed), U(stream), U(0))
        out[f"fill_{k}_args"] = np.array([L, up, seed, stream], dtype=np.int64)
        out[f"fill_{k}_out"] = a
        out[f"fill_{k}_pos"] = np.array([int(pos)], dtype=np.uint64)
        for J, B in [(1.0, 0.0), (1.0, 0.5), (-0.7, 0.3)]:
            out[f"fill_{k}_energy_{J}_{B}"] = np.array([kernels.lattice_energy(a, J, B)])
    # advance_block from a known state, with and without a field, recording
    for k, (L, R, J, B, nsteps) in enumerate([(8, 3, 1.0, 0.0, 500),
                                               (5, 2, 1.0, 0.25, 300),
                                               (16, 4, 0.8, -0.3, 2000)]):
        spins = np.empty((R, L, L), dtype=np.int8)
        positions = np.zeros(R, dtype=np.uint64)
        for r in range(R):
            positions[r] = kernels.fill_lattice(spins[r], (L * L) // 2, U(11), U(r), U(0))
        spins_in = spins.copy()
        energies = np.array([kernels.lattice_energy(spins[r], J, B) for r in range(R)])
        sums = spins.reshape(R, -1).sum(axis=1).astype(np.int64)
        slot_to_row = np.array(list(range(R))[::-1], dtype=np.int64)
        e_in, s_in = energies[slot_to_row].copy(), sums[slot_to_row].copy()
        energies, sums = e_in.copy(), s_in.copy()
        betas = 1.0 / isingpt.build_ladder(R)
        iters = np.zeros(R, dtype=np.int64)
        pos_in = positions.copy()
        obs_e = np.zeros((R, nsteps + 5)); obs_m = np.zeros((R, nsteps + 5))
        states = np.empty((1, 1, 1, 1), dtype=np.int8)
        kernels.advance_block(spins, slot_to_row, 0, R, betas, J, B, energies, sums,
                              positions, iters, U(11), 5, nsteps, obs_e, obs_m, 1, states)
        out[f"adv_{k}_args"] = np.array([L, R, nsteps], dtype=np.int64)
        out[f"adv_{k}_JB"] = np.array([J, B])
        out[f"adv_{k}_spins_in"] = spins_in
        out[f"adv_{k}_pos_in"] = pos_in
        out[f"adv_{k}_e_in"] = e_in
        out[f"adv_{k}_s_in"] = s_in
        out[f"adv_{k}_slot_to_row"] = slot_to_row
        out[f"adv_{k}_spins_out"] = spins
        out[f"adv_{k}_e_out"] = energies
        out[f"adv_{k}_s_out"] = sums
        out[f"adv_{k}_pos_out"] = positions
        out[f"adv_{k}_obs_e"] = obs_e[:, 5:]
        out[f"adv_{k}_obs_m"] = obs_m[:, 5:]
    # swap_chunk over many rounds with synthetic energies
    rs = np.random.default_rng(3)
    R = 33
    betas = 1.0 / isingpt.build_ladder(R)
    e0 = rs.integers(-2000, 0, R).astype(np.float64)
    s0 = rs.integers(-1024, 1024, R).astype(np.int64)
    str0 = np.arange(R, dtype=np.int64)
    e, s, st = e0.copy(), s0.copy(), str0.copy()
    accs = []
    for rnd in range(200):
        first = rnd % 2
        accs.append(kernels.swap_chunk(st, e, s, betas, U(99), R, rnd, first, 0,
                                       (R - first) // 2))
    out["swap_e0"], out["swap_s0"] = e0, s0
    out["swap_e"], out["swap_s"], out["swap_slot_to_row"] = e, s, st
    out["swap_acc"] = np.array(accs, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


RUNS = {
    # the executor test's small_config (tests/test_executor.py:15-19)
    "small": dict(side=8, replicas=5, iterations=3000, swap_interval=37, seed=7),
    "small_noswap": dict(side=8, replicas=5, iterations=3000, swap_interval=0, seed=7),
    "odd_L3": dict(side=3, replicas=2, iterations=20000, swap_interval=0, seed=42),
    "field": dict(side=6, replicas=4, iterations=4000, swap_interval=50, seed=5,
                  params=IsingParams(J=1.0, B=0.5)),
    "nonint": dict(side=7, replicas=3, iterations=2500, swap_interval=100, seed=13,
                   params=IsingParams(J=0.7, B=-0.2)),
    # C1 shape (32^2, 8 replicas, swap every sweep), 100 sweeps
    "c1_100sweeps": dict(side=32, replicas=8, iterations=102400, swap_interval=1024,
                         seed=42),
    "odd_replicas": dict(side=4, replicas=7, iterations=1500, swap_interval=10, seed=3),
}


def run_vectors():
    for name, kw in RUNS.items():
        cfg = SimulationConfig(workers=1, record_mode="observables", **kw)
        rec = run(cfg)
        params = kw.get("params", IsingParams())
        meta = np.array([cfg.side, cfg.replicas, cfg.iterations, cfg.swap_interval,
                         cfg.seed], dtype=np.int64)
        # keep fixtures small: full series for small runs, every 64th column +
        # the last one for the C1-shaped run (plus a digest of the full arrays)
        E, M = rec.energies, rec.magnetizations
        cols = np.arange(E.shape[1])
        if E.size > 200_000:
            cols = np.unique(np.concatenate([np.arange(0, E.shape[1], 64),
                                             [E.shape[1] - 1]]))
        import hashlib
        np.savez_compressed(
            os.path.join(OUT, f"run_{name}.npz"), meta=meta,
            JB=np.array([params.J, params.B]), temperatures=rec.temperatures,
            cols=cols, energies=E[:, cols], magnetizations=M[:, cols],
            sha_e=np.frombuffer(hashlib.sha256(E.tobytes()).digest(), np.uint8),
            sha_m=np.frombuffer(hashlib.sha256(M.tobytes()).digest(), np.uint8),
            swap=np.array([rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted],
                          dtype=np.int64),
            rng_positions=rec.rng_positions,
            round_entry=(rec.round_entry_iterations
                         if rec.round_entry_iterations is not None
                         else np.zeros((0, cfg.replicas), np.int64)))
    # full_states on a tiny run
    cfg = SimulationConfig(side=3, replicas=3, iterations=400, swap_interval=25,
                           workers=1, seed=21, record_mode="full_states")
    rec = run(cfg)
    np.savez_compressed(os.path.join(OUT, "run_full_states.npz"),
                        meta=np.array([3, 3, 400, 25, 21], dtype=np.int64),
                        states=rec.states, energies=rec.energies,
                        magnetizations=rec.magnetizations,
                        swap=np.array([rec.swap_rounds, rec.swaps_attempted,
                                       rec.swaps_accepted], dtype=np.int64))


def cli_vectors():
    """The reference CLI on small sweeps: observables.csv digests and the
    timings columns that do not depend on wall time."""
    import hashlib
    import tempfile
    from isingpt import cli
    out = {}
    cases = {
        "single": ["--size", "8", "--replicas", "4", "--iters", "2000", "--swap-interval", "50",
                   "--seed", "7", "--record", "observables"],
        "replica_sweep": ["--size", "6", "--iters", "1500", "--swap-interval", "30",
                          "--sweep", "replica_scaling", "--axis", "2,3", "--reps", "2",
                          "--record", "observables"],
        "worker_sweep": ["--size", "6", "--replicas", "3", "--iters", "800",
                         "--sweep", "worker_scaling", "--axis", "1,2", "--record", "none"],
    }
    for name, argv in cases.items():
        with tempfile.TemporaryDirectory() as d:
            rc = cli.main(argv + ["--out", d])
            files = sorted(os.listdir(d))
            digests = {f: hashlib.sha256(open(os.path.join(d, f), "rb").read()).hexdigest()
                       for f in files if f.startswith("observables")}
            rows = open(os.path.join(d, "timings.csv")).read().splitlines()
            hdr = rows[0].split(",")
            keep = [i for i, c in enumerate(hdr) if c not in ("init_s", "exec_s", "total_s")]
            stable = [",".join(r.split(",")[i] for i in keep) for r in rows]
            out[name] = {"argv": argv, "rc": rc, "files": files, "digests": digests,
                         "timings_stable": stable}
    seeds = {f"{m}|{p}|{r}": cli.derive_seed(m, p, r)
             for m in (0, 42, 2 ** 40) for p in ("", "single", "R=16", "L=8") for r in (0, 1, 5)}
    import json
    with open(os.path.join(OUT, "cli.json"), "w") as f:
        json.dump({"cases": out, "seeds": seeds}, f, indent=1)


def api_vectors():
    """isingpt.__all__ and the call signature of every public name, for the
    drop-in API test (tests/test_public_api.py)."""
    import inspect
    import json
    sigs = {}
    for name in isingpt.__all__:
        obj = getattr(isingpt, name)
        try:
            sig = inspect.signature(obj)
        except (TypeError, ValueError):
            sigs[name] = None
            continue
        sigs[name] = [[p.name, str(p.kind), None if p.default is inspect.Parameter.empty
                       else repr(p.default)] for p in sig.parameters.values()]
    with open(os.path.join(OUT, "api.json"), "w") as f:
        json.dump({"all": list(isingpt.__all__), "signatures": sigs}, f, indent=1)


def public_op_vectors():
    """The reference's per-replica public ops (rng.py, mh.py, tempering.py,
    analysis.py) on small cases, for the GPU-backed restatements."""
    from isingpt import analysis, mh, tempering
    from isingpt.rng import RngStream, SwapRng
    out = {}
    params = IsingParams(J=1.0, B=0.0)
    # RngStream / SwapRng
    st = RngStream(42, 3, 5)
    out["rng_uniforms"] = np.array([st.uniform() for _ in range(16)])
    out["rng_choose"] = np.array([st.choose(1000) for _ in range(16)], dtype=np.int64)
    out["rng_position"] = np.array([st.position], dtype=np.int64)
    sw = SwapRng(2 ** 63 + 11, 7)
    out["swap_uniforms"] = np.array([[sw.pair_uniform(r, p) for p in range(4)] for r in range(5)])
    # make_replica + mh_step loops (two couplings, one with a field)
    for tag, L, T, seed, idx, prm in (("a", 6, 2.0, 99, 0, params), ("b", 5, 1.5, 7, 3, IsingParams(J=1.0, B=0.5)),
                                      ("c", 8, 3.0, 2 ** 40 + 1, 11, IsingParams(J=-0.7, B=0.3))):
        rep = mh.make_replica(L, 0.5, T, seed, idx, prm)
        out[f"rep_{tag}_init"] = rep.lattice.spins.copy()
        out[f"rep_{tag}_init_pos"] = np.array([rep.rng.position], dtype=np.int64)
        out[f"rep_{tag}_init_e"] = np.array([rep.energy])
        acc, es = [], []
        for _ in range(300):
            acc.append(mh.mh_step(rep, prm))
            es.append(rep.energy)
        out[f"rep_{tag}_acc"] = np.array(acc, dtype=np.uint8)
        out[f"rep_{tag}_e"] = np.array(es)
        out[f"rep_{tag}_final"] = rep.lattice.spins.copy()
        out[f"rep_{tag}_pos"] = np.array([rep.rng.position], dtype=np.int64)
    # the PT composition of test_executor.py:80-104 (R=4, L=4, N=60, I=10)
    R, L, N, I = 5, 4, 120, 10
    temps = tempering.build_ladder(R)
    reps = [mh.make_replica(L, 0.5, float(temps[i]), 5, i, params) for i in range(R)]
    swap_rng = SwapRng(5, R)
    E = np.zeros((R, N))
    accs = []
    rnd = 0
    for it in range(N):
        for i, rep in enumerate(reps):
            mh.mh_step(rep, params)
            E[i, it] = rep.energy
        if (it + 1) % I == 0 and it + 1 < N:
            accs.append(tempering.execute_swap_round(reps, tempering.pairing(rnd, R), swap_rng))
            rnd += 1
    out["pt_E"] = E
    out["pt_acc"] = np.array(accs, dtype=np.int64)
    out["pt_final"] = np.stack([r.lattice.spins for r in reps])
    # analysis
    rs = np.random.default_rng(5)
    series = np.concatenate([np.linspace(0.0, 1.0, 400), 0.8 + 0.01 * rs.standard_normal(1600)])
    out["conv_series"] = series
    out["conv_result"] = np.array([
        -1 if (v := analysis.convergence_iteration(series, analysis.ConvergenceCriterion(window=w, tolerance=t)))
        is None else v for w, t in ((100, 0.02), (50, 0.005), (200, 0.05), (10, 1e-6))], dtype=np.int64)
    pts = np.array([[8, 120.0], [16, 530.0], [32, 2100.0], [64, 8800.0]])
    fit = analysis.fit_power_law(pts)
    out["fit_pts"] = pts
    out["fit"] = np.array([fit.exponent, fit.prefactor, fit.r_squared])
    states = (rs.integers(0, 2, size=(3, 5, 3, 3)) * 2 - 1).astype(np.int8)
    out["enc_states"] = states
    out["enc_codes"] = analysis.encode_configurations(states)
    for side, T, prm, tag in ((2, 2.0, params, "2"), (3, 2.5, IsingParams(J=1.0, B=0.5), "3"),
                              (4, 1.7, IsingParams(J=-0.5, B=0.2), "4")):
        out[f"boltz_{tag}"] = analysis.exact_boltzmann_distribution(side, T, prm)
    rec = run(SimulationConfig(side=6, replicas=3, iterations=4000, swap_interval=100, workers=1, seed=3))
    out["eq_mag_m"] = rec.magnetizations
    out["eq_mag_05"] = analysis.equilibrium_magnetization(rec)
    out["eq_mag_0"] = analysis.equilibrium_magnetization(rec, 0.0)
    out["eq_mag_09"] = analysis.equilibrium_magnetization(rec, 0.9)
    np.savez_compressed(os.path.join(OUT, "public_ops.npz"), **out)


if __name__ == "__main__":
    kernels.warm_kernels()
    if len(sys.argv) > 1:  # e.g. `make_golden.py api_vectors public_op_vectors`
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    cli_vectors()
    philox_vectors()
    kernel_vectors()
    run_vectors()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
