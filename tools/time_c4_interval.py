"""C4 at the bench's interval (10 sweeps per persistent launch), CUDA events.
    python tools/time_c4_interval.py [sweeps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
L, R = 4096, 512
eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
eng.init_state()
t = 0
for _ in range(2):
    eng.sweeps(t, n)
    t += n
torch.cuda.synchronize()
ms = []
for _ in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.sweeps(t, n)
    b.record()
    torch.cuda.synchronize()
    t += n
    ms.append(a.elapsed_time(b))
m = statistics.median(ms)
print(f"c4 {n} sweeps per launch: {m:.3f} ms -> {n * R * L * L / m / 1e9:.4g} T attempts/s", flush=True)
