"""Resident kernel: sweeps with vs without exchange rounds (grid syncs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

for name in sys.argv[1:] or ["c5", "c2"]:
    L, R, _, _ = CONFIGS[name]
    eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    n = 1000
    for every, label in ((0, "no rounds"), (1, "round every sweep"), (10, "round every 10")):
        eng.run_resident(0, 10, 1 << 30, every)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run_resident(100, n, 1 << 30, every)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(f"{name} {label}: {ms / n * 1e3:.2f} us/sweep -> {n * R * L * L / ms / 1e9:.3g} T/s",
              flush=True)
