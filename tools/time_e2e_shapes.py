"""Host-plugin call time (kernels.cb_interval, pinned int8 lattices) per
shape and chunk count: `python tools/time_e2e_shapes.py [L,R,sweeps ...]`."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_03825_b200 import build_ladder, kernels  # noqa: E402

shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or [
    (32, 8, 1), (256, 64, 1), (64, 4096, 1), (1024, 256, 10)]
for L, R, every in shapes:
    rng = np.random.default_rng(1)
    sp = torch.from_numpy((rng.integers(0, 2, (R, L, L)) * 2 - 1).astype(np.int8)).pin_memory().numpy()
    s2r = np.arange(R, dtype=np.int64)
    e, ss = np.zeros(R), np.zeros(R, dtype=np.int64)
    betas = 1.0 / build_ladder(R)
    for ch in ("default", "1", "2", "4", "8"):
        if ch == "default":
            os.environ.pop("PTMH_PLUGIN_CHUNKS", None)
        else:
            os.environ["PTMH_PLUGIN_CHUNKS"] = ch
        t = 0
        for _ in range(3):
            kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, 42, t, every, t, e, ss)
            t += every
        n = 20 if R * L * L < (1 << 26) else 5
        t0 = time.perf_counter()
        for _ in range(n):
            kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, 42, t, every, t, e, ss)
            t += every
        dt = (time.perf_counter() - t0) / n
        print("L=%d R=%d every=%d chunks=%s: %.1f us/call -> %.3g attempts/s"
              % (L, R, every, ch, dt * 1e6, R * L * L * every / dt))
    os.environ.pop("PTMH_PLUGIN_CHUNKS", None)
