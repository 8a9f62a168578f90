"""World-size-2 run of the multi-GPU coordinator over gloo on CPU, with the
oracle-backed engine substituted for the CUDA one: sharded rows +
all-gathered (S, Bond) + replicated exchange must reproduce the
single-process checkerboard chain exactly, with identical permutations on
every rank."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, L, R, sweeps, every, seed, out_dir):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from cpu_engine import OracleCheckerboardEngine
    from paper_2512_03825_b200.distributed import ShardedCheckerboard
    from paper_2512_03825_b200.executor import _interval_plan
    temps = oracle.build_ladder(R)
    drv = ShardedCheckerboard(L, R, temps, seed, engine_cls=OracleCheckerboardEngine)
    drv.init_state()
    done = 0
    for target, ri in _interval_plan(sweeps, every):
        drv.interval(done, target - done, ri)
        done = target
    drv.gather_stats()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), spins=drv.eng.spins,
             s2r=drv.eng.slot_to_row, stats=drv.eng.stats.numpy(), acc=drv.eng.accepted,
             lo=drv.eng.row_lo, hi=drv.eng.row_hi)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,R", [(2, 5), (2, 8), (3, 7)])
def test_sharded_checkerboard_matches_single_process(tmp_path, world, R):
    L, sweeps, every, seed = 8, 12, 2, 17
    mp.spawn(_worker, args=(world, _free_port(), L, R, sweeps, every, seed, str(tmp_path)),
             nprocs=world, join=True)
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, record=False)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    spins = np.concatenate([o["spins"] for o in outs])
    assert np.array_equal(spins, ref.final_spins)
    for o in outs:
        assert np.array_equal(o["s2r"], ref.slot_to_row)
        assert int(o["acc"]) == ref.swaps_accepted
        assert np.array_equal(o["stats"], oracle.row_stats(ref.final_spins))
    sizes = [int(o["hi"]) - int(o["lo"]) for o in outs]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == R
