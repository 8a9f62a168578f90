"""A/B of the resident kernels at C2-like shapes: us per sweep with a round
every sweep (and without rounds) for PTMH_RESIDENT_SMEM configurations
"cs,rows,threads" ("0" = resident.cu's cluster kernel)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2512_03825_b200 import build_ladder, _lib
from paper_2512_03825_b200.engine import CheckerboardEngine
L, R = int(sys.argv[2]), int(sys.argv[3])
eng = CheckerboardEngine(L, R, build_ladder(R), 42, 1.0, 0.0, 0.5, 0)
eng.init_state()
out = []
for every in (0, 1):
    n = 1000
    eng.run_resident(0, 10, 1 << 30, every)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.run_resident(100, n, 1 << 30, every)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    out.append(f"every={every}: {ms / n * 1e3:.2f} us/sweep {n * R * L * L / ms / 1e9:.3g} T/s")
print(_lib.cb_last_launch()["name"], "|", " | ".join(out), flush=True)
'''
shapes = [tuple(map(int, s.split("x"))) for s in (sys.argv[1:2] or ["256x64"])[0].split(",")]
cfgs = sys.argv[2:] or ["0", "1,2,256", "2,2,256", "2,1,512", "2,2,128", "4,2,128", "4,1,256", "2,4,128",
                        "4,2,256", "8,1,256"]
for L, R in shapes:
    for c in cfgs:
        env = dict(os.environ, PTMH_RESIDENT_SMEM=c)
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(L), str(R)], env=env, capture_output=True,
                           text=True, timeout=300)
        print(f"{L}^2 x {R} [{c}]", (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
