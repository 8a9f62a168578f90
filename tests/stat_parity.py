"""Statistical parity of the two chains, with seed-to-seed error bars.

Mode F (the checkerboard chain the throughput numbers run) and Mode E (the
reference's random-site chain, bit-exact with isingpt) must sample the same
Boltzmann distribution: per temperature slot, the post-burn-in averages of
E / L^2 and |m| from independent seeds agree within the combined standard
error, |mean_F - mean_E| < 4 sigma (the north star's "within stated error
bars"; the reference's own distributional tests: ref tests/test_sampling.py
:48-84).

Both chains run through run() with the reference ladder (1 + 3i/R), J = 1,
B = 0, an exchange every sweep, observables every sweep (the exact chain's
record_every = L^2 keeps every L^2-th column of the reference's series).
The runs start from the ordered state (init_up_fraction = 1): from a random
start the low-temperature slots coarsen for ~L^2 sweeps at L = 256, so the
averages would measure two different relaxations instead of equilibrium.

    python tests/stat_parity.py [--out profiles/r2_stat_parity.json]

runs the table on the GPU; tests/test_gpu_stat_parity.py runs it as a test.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# (L, R, sweeps, burn-in sweeps, seeds per chain)
CASES = ((64, 8, 4000, 1000, 8), (256, 8, 1500, 500, 8))
Z_MAX = 4.0


def chain_averages(L, R, sweeps, burn, seed, mode):
    from paper_2512_03825_b200 import SimulationConfig, run

    n = L * L
    kw = dict(side=L, replicas=R, iterations=sweeps * n, swap_interval=n, seed=seed,
              init_up_fraction=1.0, record_mode="observables", workers=1, device=0)
    if mode == "F":
        cfg = SimulationConfig(sweep_mode="checkerboard", record_every=1, **kw)
    else:
        cfg = SimulationConfig(sweep_mode="exact", record_every=n, **kw)
    rec = run(cfg)
    assert rec.valid, rec.error
    assert rec.energies.shape == (R, sweeps), rec.energies.shape
    assert rec.swap_near_ties == 0
    e = rec.energies[:, burn:] / n
    m = np.abs(rec.magnetizations[:, burn:])
    return e.mean(axis=1), m.mean(axis=1), rec.swaps_accepted / max(1, rec.swaps_attempted)


def parity_table(cases=CASES):
    from paper_2512_03825_b200 import build_ladder

    out = []
    for L, R, sweeps, burn, nseed in cases:
        per = {}
        t0 = time.perf_counter()
        for mode, base in (("E", 1000), ("F", 2000)):
            rows = [chain_averages(L, R, sweeps, burn, base + s, mode) for s in range(nseed)]
            per[mode] = (np.array([r[0] for r in rows]), np.array([r[1] for r in rows]),
                         float(np.mean([r[2] for r in rows])))
        temps = build_ladder(R)
        slots = []
        for k in range(R):
            ent = {"T": float(temps[k])}
            for name, idx in (("e_per_site", 0), ("abs_m", 1)):
                xe, xf = per["E"][idx][:, k], per["F"][idx][:, k]
                me, mf = float(xe.mean()), float(xf.mean())
                se = float(xe.std(ddof=1) / np.sqrt(xe.size))
                sf = float(xf.std(ddof=1) / np.sqrt(xf.size))
                sig = float(np.hypot(se, sf))
                z = (mf - me) / sig if sig > 0 else (0.0 if mf == me else float("inf"))
                ent[name] = {"exact": me, "exact_se": se, "checkerboard": mf, "checkerboard_se": sf,
                             "z": z}
            slots.append(ent)
        out.append({"L": L, "R": R, "sweeps": sweeps, "burn_in_sweeps": burn, "seeds_per_chain": nseed,
                    "swap_acceptance": {"exact": per["E"][2], "checkerboard": per["F"][2]},
                    "max_abs_z": max(abs(s[o]["z"]) for s in slots for o in ("e_per_site", "abs_m")),
                    "seconds": time.perf_counter() - t0, "slots": slots})
    return out


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    table = parity_table()
    doc = {"what": "Mode F (checkerboard) vs Mode E (reference random-site chain) per-slot averages, "
                   "independent seeds per chain, seed-to-seed standard errors; pass iff |z| < %g" % Z_MAX,
           "ladder": "1 + 3i/R", "J": 1.0, "B": 0.0, "exchange": "every sweep",
           "init": "ordered (init_up_fraction = 1)", "cases": table}
    txt = json.dumps(doc, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt + "\n")
    for c in table:
        print(f"L={c['L']} R={c['R']} sweeps={c['sweeps']} seeds={c['seeds_per_chain']} "
              f"max|z|={c['max_abs_z']:.2f} ({c['seconds']:.1f} s)")
        for s in c["slots"]:
            print(f"  T={s['T']:.3f}  e: {s['e_per_site']['exact']:+.5f}+-{s['e_per_site']['exact_se']:.5f} vs "
                  f"{s['e_per_site']['checkerboard']:+.5f}+-{s['e_per_site']['checkerboard_se']:.5f} "
                  f"(z {s['e_per_site']['z']:+.2f})   |m|: {s['abs_m']['exact']:.5f}+-{s['abs_m']['exact_se']:.5f} vs "
                  f"{s['abs_m']['checkerboard']:.5f}+-{s['abs_m']['checkerboard_se']:.5f} (z {s['abs_m']['z']:+.2f})")
    return 0 if all(c["max_abs_z"] < Z_MAX for c in table) else 1


if __name__ == "__main__":
    sys.exit(main())
