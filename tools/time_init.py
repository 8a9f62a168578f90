"""Exact-count (Fisher-Yates) init time per config (outside every throughput timer)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

for name in sys.argv[1:] or ["c3", "c4"]:
    L, R, _, _ = CONFIGS[name]
    eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.init_state()
    torch.cuda.synchronize()
    print(f"{name}: init {time.perf_counter() - t0:.2f} s for {R} x {L}^2", flush=True)
    del eng
    torch.cuda.empty_cache()
