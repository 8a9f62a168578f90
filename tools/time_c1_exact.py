"""The reference's C1 run (32^2, 8 replicas, geometric ladder, 1e4 sweeps, a
round every sweep) through run(), exact chain: resident vs per-interval path."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2512_03825_b200 as p  # noqa: E402

L, R, sweeps = 32, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
temps = tuple(p.geometric_ladder(R))
for kernel in ("auto", "sweep"):
    for rec in ("none", "observables"):
        cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=L * L,
                                 temperatures=temps, record_mode=rec, kernel=kernel)
        p.run(p.SimulationConfig(side=L, replicas=R, iterations=20 * L * L, swap_interval=L * L,
                                 temperatures=temps, record_mode=rec, kernel=kernel))  # warm
        t0 = time.perf_counter()
        r = p.run(cfg)
        dt = time.perf_counter() - t0
        att = R * (sweeps * L * L - 1)
        print(f"C1 exact kernel={kernel} record={rec}: {dt:.3f} s total (exec {r.exec_seconds:.3f} s) "
              f"-> {att / r.exec_seconds:.3g} attempts/s, rounds {r.swap_rounds}", flush=True)
