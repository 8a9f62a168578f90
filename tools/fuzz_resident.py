"""Randomised A/B of the resident run (every kernel the launcher picks:
registers, cluster shared memory, L2 clusters, warp- or CTA-owned lattices)
against the sweep path (bit-exact: the same chain) through run():
`python tools/fuzz_resident.py [n] [seed]`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2512_03825_b200 as p  # noqa: E402
from paper_2512_03825_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
kinds = {}
for case in range(n):
    L = int(rng.choice([2, 4, 8, 16, 32, 32, 48, 64, 64, 96, 128, 192, 256, 256, 320, 512]))
    R = int(rng.integers(1, 300 if L <= 64 else (80 if L <= 256 else 20)))
    sweeps = int(rng.integers(1, 12 if L <= 128 else 5))
    every = int(rng.integers(0, 4))
    J = float(rng.choice([1.0, 1.0, 0.5, -1.0]))
    B = float(rng.choice([0.0, 0.0, 0.0, 0.3]))
    rec_every = int(rng.integers(1, sweeps + 1))
    seed = int(rng.integers(1 << 40))
    recs = []
    for kernel in ("resident", "sweep"):
        cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=every * L * L,
                                 seed=seed, params=p.IsingParams(J=J, B=B), sweep_mode="checkerboard",
                                 record_every=rec_every, return_final_state=True, kernel=kernel)
        recs.append(p.run(cfg))
        if kernel == "resident":
            name = _lib.cb_last_launch()["name"]
    a, b = recs
    ok = a.valid and b.valid and np.array_equal(a.final_spins, b.final_spins) and \
        np.array_equal(a.energies, b.energies) and np.array_equal(a.slot_to_row, b.slot_to_row) and \
        (a.swaps_accepted == b.swaps_accepted)
    bad += not ok
    kinds[name] = kinds.get(name, 0) + 1
    if not ok:
        print(f"MISMATCH case {case}: L={L} R={R} sweeps={sweeps} every={every} J={J} B={B} rec={rec_every} "
              f"{name} {a.error} {b.error}", flush=True)
for k, v in sorted(kinds.items(), key=lambda kv: -kv[1]):
    print(f"{v:4d}  {k}")
print(f"{n - bad}/{n} equal")
sys.exit(1 if bad else 0)
