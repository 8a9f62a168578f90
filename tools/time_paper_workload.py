"""The paper's own workload: a 300x300 lattice, J = 1,
B = 0, 300,000 single-spin attempts per replica, up to 1,500 replicas; the
paper reports its CUDA build finishing any replica count in < 1 s on an A100
(>= 4.5e8 attempts/s).  Both chains through run(), swaps every
sweep-equivalent (90,000 attempts) as in the reference CLI's default sweep."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_03825_b200 as p  # noqa: E402

L, N = 300, 300_000
for R in (100, 1500):
    for mode in ("checkerboard", "exact"):
        iters = N if mode == "exact" else (N // (L * L) + 1) * L * L  # whole sweeps for the checkerboard chain
        kw = dict(side=L, replicas=R, iterations=iters, swap_interval=L * L, seed=42, record_mode="none",
                  sweep_mode=mode)
        p.run(p.SimulationConfig(**dict(kw, iterations=2 * L * L)))  # warm
        t0 = time.perf_counter()
        r = p.run(p.SimulationConfig(**kw))
        wall = time.perf_counter() - t0
        print(f"R={R} {mode}: {R * iters:.3g} attempts, exec {r.exec_seconds * 1e3:.1f} ms, run() wall "
              f"{wall * 1e3:.1f} ms (init {r.init_seconds * 1e3:.1f} ms) -> {R * iters / r.exec_seconds:.3g} "
              f"attempts/s", flush=True)
