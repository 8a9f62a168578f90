"""The multi-GPU coordinator over NCCL on the one GPU available (world 1):
the sharded path (all_gather of per-lattice stats, replicated exchange) must
give the oracle's chain.  World sizes 2-3 are covered over gloo on CPU
(tests/test_distributed_gloo.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_coordinator_over_nccl_world1():
    from paper_2512_03825_b200 import build_ladder
    from paper_2512_03825_b200.distributed import ShardedCheckerboard
    from paper_2512_03825_b200.executor import _interval_plan
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        L, R, sweeps, every, seed = 64, 7, 10, 2, 19
        drv = ShardedCheckerboard(L, R, build_ladder(R), seed, device=0)
        drv.init_state()
        done = 0
        for target, ri in _interval_plan(sweeps, every):
            drv.interval(done, target - done, ri)
            done = target
        ref = oracle.run_checkerboard(L, R, sweeps, every, seed, record=False)
        assert np.array_equal(drv.eng.final_spins(), ref.final_spins)
        assert np.array_equal(drv.eng.slot_to_row.cpu().numpy(), ref.slot_to_row)
        assert drv.eng.swap_counts()[0] == ref.swaps_accepted
    finally:
        dist.destroy_process_group()
