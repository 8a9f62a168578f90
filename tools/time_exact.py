"""Time the exact-chain advance kernel (Mode E), CUDA events.
    python tools/time_exact.py [L R nsteps] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import ExactEngine  # noqa: E402

args = [int(x) for x in sys.argv[1:]] or [1024, 256, 200000, 32, 8, 200000, 64, 4096, 20000]
for L, R, n in zip(args[0::3], args[1::3], args[2::3]):
    eng = ExactEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    eng.advance(0, 1000)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.advance(1000, n)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"exact L={L} R={R}: {R * n / ms / 1e6:.4g} G attempts/s ({ms:.1f} ms)", flush=True)
    del eng
    torch.cuda.empty_cache()
