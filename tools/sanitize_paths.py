"""compute-sanitizer driver (tools/ only): one small call of every kernel family -- persistent
sweeps, resident checkerboard (warp-owned lattices, clusters), exact windows, resident exact run.
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_paths.py"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2512_03825_b200 as p
from paper_2512_03825_b200.engine import CheckerboardEngine, ExactEngine
# persistent sweeps (small), resident checkerboard (warp-lat + cluster), exact windows + resident exact
e = CheckerboardEngine(1024, 2, np.array([1.5, 2.5]), 5, 1.0, 0.0, 0.5, 0); e.init_state(); e.sweeps(0, 2)
r = p.run(p.SimulationConfig(side=64, replicas=6, iterations=4 * 64 * 64, swap_interval=64 * 64, sweep_mode="checkerboard", seed=3))
r2 = p.run(p.SimulationConfig(side=256, replicas=2, iterations=3 * 256 * 256, swap_interval=256 * 256, sweep_mode="checkerboard", seed=4))
r3 = p.run(p.SimulationConfig(side=512, replicas=2, iterations=3000, swap_interval=0, record_mode="none", seed=5))
r4 = p.run(p.SimulationConfig(side=16, replicas=4, iterations=3000, swap_interval=100, seed=6))
torch.cuda.synchronize()
print("ok", r.valid, r2.valid, r3.valid, r4.valid)
