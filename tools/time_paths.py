"""Attempts/s of both checkerboard paths on each config, exchanges included.
    python tools/time_paths.py c1 c2 c3 c4 c5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2512_03825_b200 import build_ladder, geometric_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for name in (sys.argv[1:] or ["c1", "c2", "c3", "c5"]):
    L, R, every, _ = CONFIGS[name]
    temps = geometric_ladder(R) if name == "c1" else build_ladder(R)
    eng = CheckerboardEngine(L, R, temps, 42, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    n = max(every * 2, min(2000, int(2e10 // (R * L * L)) // every * every))
    total = 10 * n + 10

    def sweep_path(t0):
        def f():
            for s in range(t0, t0 + n, every):
                eng.sweeps(s, every)
                eng.exchange(s // every)
        return f

    sweep_path(0)()
    ms_s = timed(sweep_path(n))
    eng.run_resident(2 * n, n, total, every)
    ms_r = timed(lambda: eng.run_resident(3 * n, n, total, every))
    att = n * R * L * L
    print(f"{name}: L={L} R={R} every={every} sweeps={n}: sweep-path {att / ms_s / 1e9:.4g} T/s "
          f"({ms_s / n * 1e3:.1f} us/sweep) | resident {att / ms_r / 1e9:.4g} T/s "
          f"({ms_r / n * 1e3:.1f} us/sweep)", flush=True)
    del eng
    torch.cuda.empty_cache()
