"""C3-shape host-plugin calls (cb_interval) on a warmed workspace: per-call time; PTMH_TRACE=1 adds the
chunk timeline (tools/ only)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_03825_b200 import build_ladder, kernels
from paper_2512_03825_b200.engine import CheckerboardEngine
L, R = 1024, 256
eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0); eng.init_state()
sp = torch.from_numpy(eng.final_spins()).pin_memory().numpy()
s2r = np.arange(R, dtype=np.int64); e = np.zeros(R); ss = np.zeros(R, dtype=np.int64)
betas = 1.0 / build_ladder(R)
for k in range(3):
    kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, 42, 10 * k, 10, k, e, ss)
t0 = time.perf_counter(); n = 5
for k in range(n):
    kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, 42, 30 + 10 * k, 10, 3 + k, e, ss)
print("per call %.2f ms" % ((time.perf_counter() - t0) / n * 1e3))
