"""Small driver for ncu: init a config, run a few sweeps + one exchange.

    python tools/prof_sweep.py [c3|c4|c5|c2|c1|L,R] [sweeps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if "," in name:  # "L,R": e.g. 1024,32 (a rank's C3 shard at 8 GPUs)
    L, R = map(int, name.split(","))
else:
    L, R, every, _ = CONFIGS[name]
eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
eng.init_state()
eng.sweeps(0, n)
eng.exchange(0)
torch.cuda.synchronize()
print("done", name, n)
