"""Randomised A/B of the persistent sweep kernel against the per-launch
kernels (bit-exact lattices and stats), over shapes, row permutations, sweep
ranges and the PTMH_PERSIST_* knobs (temporally blocked items included):
`python tools/fuzz_persistent.py [n] [seed]`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_03825_b200 import build_ladder  # noqa: E402
from paper_2512_03825_b200.engine import CheckerboardEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
knobs = ("PTMH_PERSIST_ROWS", "PTMH_PERSIST_THREADS", "PTMH_PERSIST_BANDS", "PTMH_PERSIST_ITEMS_PER_SLOT",
         "PTMH_PERSIST_TB")
bad = 0
for case in range(n):
    L = int(rng.choice([1024, 1536, 2048]))
    R = int(rng.integers(1, 48 if L == 1024 else 12))
    first, ns = int(rng.integers(0, 50)), int(rng.integers(1, 7))
    env = {"PTMH_PERSIST_ROWS": str(rng.choice(["", "2", "4", "8", "16", "32"])),
           "PTMH_PERSIST_THREADS": str(rng.choice(["", "128", "256"])),
           "PTMH_PERSIST_BANDS": str(rng.choice(["", "0", "1"])),
           "PTMH_PERSIST_ITEMS_PER_SLOT": str(rng.choice(["", "0", "1"])),
           "PTMH_PERSIST_TB": str(rng.choice(["", "0", "1"]))}
    for k in knobs:
        if env[k]:
            os.environ[k] = env[k]
        else:
            os.environ.pop(k, None)
    perm = rng.permutation(R)
    r2s = np.empty(R, dtype=np.int64)
    r2s[perm] = np.arange(R)
    outs = []
    for persistent in (True, False):
        seed = 1234 + case
        eng = CheckerboardEngine(L, R, build_ladder(R), seed, 1.0, 0.0, 0.5, 0)
        eng.persistent = persistent
        eng.slot_to_row.copy_(torch.from_numpy(perm.astype(np.int64)))
        eng.row_to_slot.copy_(torch.from_numpy(r2s.astype(np.int32)))
        eng.init_state()
        eng.sweeps(first, ns)
        eng.sweeps(first + ns, 2)
        torch.cuda.synchronize()
        outs.append((eng.packed.clone(), eng.local_stats.clone(), int(eng._sync.abs().sum().item())))
        del eng
    ok = torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]) and outs[0][2] == 0
    bad += not ok
    print(f"case {case}: L={L} R={R} first={first} n={ns} {env} -> {'ok' if ok else 'MISMATCH'}", flush=True)
for k in knobs:
    os.environ.pop(k, None)
print(f"{n - bad}/{n} equal")
sys.exit(1 if bad else 0)
