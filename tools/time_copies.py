"""Bidirectional PCIe copy behaviour: whole vs chunked, same vs separate host buffer."""
import time

import torch

nb = 256 * 1024 * 1024
h = torch.empty(nb, dtype=torch.int8).pin_memory()
h2 = torch.empty(nb, dtype=torch.int8).pin_memory()
d = torch.empty(nb, dtype=torch.int8, device="cuda")
d2 = torch.empty(nb, dtype=torch.int8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def both(chunks, same):
    c = nb // chunks
    dst = h if same else h2

    def f():
        for k in range(chunks):
            with torch.cuda.stream(s1):
                d[k * c:(k + 1) * c].copy_(h[k * c:(k + 1) * c], non_blocking=True)
            with torch.cuda.stream(s2):
                j = (k + chunks // 2) % chunks
                dst[j * c:(j + 1) * c].copy_(d2[j * c:(j + 1) * c], non_blocking=True)
    return f


for chunks in (1, 8, 16):
    for same in (False, True):
        print(f"H2D||D2H chunks={chunks} same_host_buffer={same}: {t(both(chunks, same)):.2f} ms")

# copies while sweep kernels run on another stream
import os, sys  # noqa: E401,E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

eng = CheckerboardEngine(1024, 64, build_ladder(64), 42, 1.0, 0.0, 0.5, 0)
eng.init_state()
s3 = torch.cuda.Stream()


def with_compute(nsweeps):
    def f():
        with torch.cuda.stream(s3):
            eng.sweeps(0, nsweeps)
        both(16, True)()
    return f


for ns in (0, 20, 60):
    print(f"H2D||D2H + {ns} sweeps of 64 lattices on a third stream: {t(with_compute(ns), 3):.2f} ms")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s3):
    a.record()
    eng.sweeps(0, 60)
    b.record()
torch.cuda.synchronize()
print(f"60 sweeps alone: {a.elapsed_time(b):.2f} ms")
