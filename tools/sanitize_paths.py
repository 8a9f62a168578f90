"""compute-sanitizer driver (tools/ only): one small call of every kernel family -- persistent
sweeps (2 lattices of 1024^2: the temporally blocked items), resident checkerboard (warp-owned
lattices; 256^2 lattices in cluster shared memory), exact windows, resident exact run,
the per-replica API (device draws, mh_steps, swap_pairs), the host interval plugin.
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
# the per-replica public API (uniforms_kernel, advance_kernel with a stream offset, swap_pairs_kernel)
reps = [p.make_replica(8, 0.5, 1.0 + i, 7, i, p.IsingParams()) for i in range(3)]
for _ in range(3):
    for rep in reps:
        p.mh_step(rep, p.IsingParams())
p.mh_steps(reps[0], p.IsingParams(), 100)
p.execute_swap_round(reps, p.pairing(0, 3), p.SwapRng(7, 3))
st = p.RngStream(1, 2); st.uniforms(1000)
# host interval plugin (pack, persistent / per-launch sweeps, unpack, exchange)
from paper_2512_03825_b200 import kernels
sp = np.empty((4, 64, 64), dtype=np.int8)
for k in range(4):
    kernels.fill_lattice(sp[k], 2048, 9, k, 0)
s2r = np.arange(4, dtype=np.int64); en = np.zeros(4); ss = np.zeros(4, dtype=np.int64)
kernels.cb_interval(sp, s2r, 1.0 / p.build_ladder(4), 1.0, 0.0, 9, 0, 2, 0, en, ss)
torch.cuda.synchronize()
print("ok", r.valid, r2.valid, r3.valid, r4.valid)
