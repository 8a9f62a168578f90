"""Where the end-to-end plugin call spends its time (C3 shape)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_03825_b200 import build_ladder, kernels  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

L, R = 1024, 256
nbytes = R * L * L
h = torch.empty(nbytes, dtype=torch.int8).pin_memory()
h2 = torch.empty(nbytes, dtype=torch.int8).pin_memory()
d = torch.empty(nbytes, dtype=torch.int8, device="cuda")
d2 = torch.empty(nbytes, dtype=torch.int8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("H2D 256MiB pinned: %.2f ms" % t(lambda: d.copy_(h, non_blocking=True)))
print("D2H 256MiB pinned: %.2f ms" % t(lambda: h.copy_(d, non_blocking=True)))


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print("H2D || D2H: %.2f ms" % t(both))
eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
eng.init_state()
sp = torch.from_numpy(eng.final_spins()).pin_memory().numpy()
s2r = np.arange(R, dtype=np.int64)
e, ss = np.zeros(R), np.zeros(R, dtype=np.int64)
betas = 1.0 / build_ladder(R)
state = {"t": 0}


def call(n_sweeps):
    def f():
        kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, 42, state["t"], n_sweeps, 0, e, ss)
        state["t"] += n_sweeps
    return f


print("cb_interval 0 sweeps: %.2f ms" % t(call(0), 3))
print("cb_interval 10 sweeps: %.2f ms" % t(call(10), 3))
from paper_2512_03825_b200 import _lib  # noqa: E402
st = torch.empty((R, 2), dtype=torch.int64, device="cuda")
dd = d.view(R, L, L)
strm = torch.cuda.current_stream().cuda_stream
print("row_stats int8: %.2f ms" % t(lambda: _lib.call("ptmh_row_stats", dd.data_ptr(), R, L, st.data_ptr(), strm)))
pk = eng.packed
print("pack: %.2f ms" % t(lambda: _lib.call("ptmh_cb_pack", dd.data_ptr(), R, L, pk.data_ptr(), strm)))
print("unpack: %.2f ms" % t(lambda: _lib.call("ptmh_cb_unpack", pk.data_ptr(), R, L, dd.data_ptr(), strm)))
print("cb_row_stats packed: %.2f ms" % t(lambda: _lib.call("ptmh_cb_row_stats", pk.data_ptr(), R, L, st.data_ptr(), strm)))
