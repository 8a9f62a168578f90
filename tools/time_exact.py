"""Time the exact-chain advance (Mode E), CUDA events; warm-up of ~0.3 s of
GPU work, median of 5 repetitions.
    python tools/time_exact.py [L R nsteps] ..."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import ExactEngine  # noqa: E402

args = [int(x) for x in sys.argv[1:]] or [1024, 256, 200000, 32, 8, 200000, 64, 4096, 20000]
for L, R, n in zip(args[0::3], args[1::3], args[2::3]):
    eng = ExactEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    done = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:  # clocks up
        eng.advance(done, n)
        done += n
        torch.cuda.synchronize()
    rates = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.advance(done, n)
        b.record()
        torch.cuda.synchronize()
        done += n
        rates.append(R * n / a.elapsed_time(b) / 1e6)
    print(f"exact L={L} R={R}: {statistics.median(rates):.4g} G attempts/s "
          f"(min {min(rates):.4g}, max {max(rates):.4g})", flush=True)
    del eng
    torch.cuda.empty_cache()
