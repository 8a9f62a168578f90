"""The reference itself (isingpt, numba) at the C3 shape beside its C port
(oracle.advance_block_mt, the bench's --impl reference arm), on this host's
cores: records the port / numba ratio (profiles/r2_reference_numba_vs_port.json).

Build container only (imports /root/reference read-only, numba cache in /tmp).

    python tools/time_numba_reference.py [--sweeps 1] [--out FILE]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_ref_cache")
sys.dont_write_bytecode = True
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(1, "/root/reference/pkg/src")

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=1024)
    ap.add_argument("--replicas", type=int, default=256)
    ap.add_argument("--sweeps", type=float, default=1.0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import isingpt
    from isingpt import kernels
    import oracle

    L, R = args.side, args.replicas
    W = len(os.sched_getaffinity(0))
    N = int(args.sweeps * L * L)
    kernels.warm_kernels()
    cfg = isingpt.SimulationConfig(side=L, replicas=R, iterations=N, swap_interval=10 * L * L, workers=W,
                                   seed=42, record_mode="none")
    rec = isingpt.run(cfg)
    numba_rate = R * (N - 1) / rec.exec_seconds
    # the port on the same shape and threads (bench.py cpu_reference_rate)
    from bench import cpu_reference_rate
    per_slot = max(1000, N // 4)
    port_rate, n, dt = cpu_reference_rate(L, R, per_slot, W)
    res = {"shape": f"{L}^2 x {R} slots", "host_threads": W,
           "numba": {"attempts_per_s": numba_rate, "attempts": R * (N - 1), "exec_seconds": rec.exec_seconds,
                     "init_seconds": rec.init_seconds, "api": "isingpt.executor.run(record_mode='none', "
                                                               f"workers={W})"},
           "port": {"attempts_per_s": port_rate, "attempts": n, "seconds": dt,
                    "api": "oracle.advance_block_mt (bench.py --impl reference)"},
           "port_over_numba": port_rate / numba_rate}
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
