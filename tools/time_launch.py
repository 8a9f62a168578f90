"""Launch overhead: torch tiny kernels vs our sweep launches, eager vs CUDA graph."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

x = torch.zeros(1, device="cuda")


def wall(fn, n):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6


print("torch add_: issue %.2f us, total %.2f us per launch" % wall(lambda: x.add_(1), 2000))
for L, R in [(64, 1), (64, 4096), (32, 8), (256, 64)]:
    eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    st = {"t": 0}

    def sw():
        eng.sweeps(st["t"], 1)
        st["t"] += 1
    a, b = wall(sw, 500)
    print(f"sweep L={L} R={R}: issue {a:.2f} us, total {b:.2f} us per sweep (2 launches)")

    def ex():
        eng.exchange(st["t"])
        st["t"] += 1
    a, b = wall(ex, 500)
    print(f"exchange L={L} R={R}: issue {a:.2f} us, total {b:.2f} us per round (2 launches)")
    # graph of 10 sweeps + exchange (fixed indices: timing only)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        eng.sweeps(0, 10)
        eng.exchange(0)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        eng.sweeps(0, 10)
        eng.exchange(0)
    a, b = wall(g.replay, 200)
    print(f"graph(10 sweeps + exchange) L={L} R={R}: issue {a:.2f} us, total {b:.2f} us per replay "
          f"({b / 22:.2f} us per kernel)")
    del eng, g
