import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
every = int(sys.argv[2]) if len(sys.argv) > 2 else 0
L, R, _, _ = CONFIGS[name]
eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
eng.init_state()
eng.run_resident(0, 20, 1 << 30, every)
torch.cuda.synchronize()
