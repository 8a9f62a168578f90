"""C2 resident kernel, what the round costs: us per sweep with no rounds, with
the (S, Bond) recompute + observables every sweep but no exchange, and with a
round every sweep (tools/ only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    L, R, _, _ = CONFIGS[name]
    eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    n = 1000
    T = 1200  # sweeps in the run (the observables hold one column per sweep)
    obs_e = torch.zeros((R, T), dtype=torch.float64, device="cuda")
    obs_m = torch.zeros((R, T), dtype=torch.float64, device="cuda")
    for every, rec, label in ((0, 0, "no rounds"), (0, 1, "stats + record every sweep"), (1, 0, "round every sweep"),
                              (1, 1, "round + record every sweep")):
        kw = dict(record_every=rec, obs_e=obs_e, obs_m=obs_m) if rec else {}
        eng.run_resident(0, 10, T, every, **kw)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run_resident(100, n, T, every, **kw)
        b.record()
        torch.cuda.synchronize()
        print(f"{name} {label}: {a.elapsed_time(b) / n * 1e3:.2f} us/sweep", flush=True)
