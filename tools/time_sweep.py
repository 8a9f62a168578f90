"""Time the checkerboard sweep kernels alone (CUDA events): ~0.3 s warm-up,
median of 5 repetitions.    python tools/time_sweep.py c3 c5 ..."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

persist = "--no-persist" not in sys.argv
for name in ([a for a in sys.argv[1:] if not a.startswith("--")] or ["c3"]):
    if name in CONFIGS:
        L, R, every, _ = CONFIGS[name]
    else:  # "L,R": e.g. 1024,32 = one rank's shard of C3 at 8 GPUs
        L, R = (int(x) for x in name.split(","))
    eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
    eng.persistent = persist
    eng.init_state()
    n = max(2, min(200, int(4e9 // (R * L * L))))
    t = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:
        eng.sweeps(t, n)
        t += n
        torch.cuda.synchronize()
    ms_all = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.sweeps(t, n)
        b.record()
        torch.cuda.synchronize()
        t += n
        ms_all.append(a.elapsed_time(b))
    ms = statistics.median(ms_all)
    print(f"{name}{'' if persist else ' (per-launch)'}: L={L} R={R} {n} sweeps {ms:.3f} ms -> {n * R * L * L / ms / 1e9:.4g} T attempts/s "
          f"({ms / n * 1e3:.1f} us/sweep; min {min(ms_all):.3f} max {max(ms_all):.3f} ms)", flush=True)
    del eng
    torch.cuda.empty_cache()
