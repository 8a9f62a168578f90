"""run(SimulationConfig(devices=...)) as real separate processes: 2 and 3
ranks (one process each, sharing the one GPU of the test box, gloo moving
the CUDA tensors through host memory where NCCL would use NVLink) run the
sharded checkerboard chain through the public entry point and must all
return the single-process record, bit for bit.  The per-interval path is
used (kernel="sweep"): the resident path's in-kernel peer-flag rounds need
the ranks' kernels co-resident, which separate processes on one GPU do not
guarantee (tests/test_gpu_distributed.py co-runs them in one process)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
KW = dict(side=64, replicas=7, iterations=12 * 64 * 64, swap_interval=2 * 64 * 64, seed=29,
          sweep_mode="checkerboard", kernel="sweep", record_mode="observables", return_final_state=True)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2512_03825_b200.executor import SimulationConfig, _checkerboard_on
    cfg = SimulationConfig(devices=tuple(range(world)), **KW)
    cfg.validate()
    # every rank on the one physical GPU (run() would put rank r on devices[r])
    rec = _checkerboard_on(cfg, torch.device("cuda", 0), True)
    assert rec.valid, rec.error
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), e=rec.energies, m=rec.magnetizations,
             spins=rec.final_spins, s2r=rec.slot_to_row,
             swap=np.array([rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted]),
             entry=rec.round_entry_iterations)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_run_devices_separate_processes_equal_single_process(tmp_path, world):
    mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    from paper_2512_03825_b200 import SimulationConfig, run
    ref = run(SimulationConfig(device=0, **KW))
    for r in range(world):
        o = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(o["spins"], ref.final_spins)
        assert np.array_equal(o["s2r"], ref.slot_to_row)
        assert np.array_equal(o["e"].view(np.int64), ref.energies.view(np.int64))
        assert np.array_equal(o["m"].view(np.int64), ref.magnetizations.view(np.int64))
        assert o["swap"].tolist() == [ref.swap_rounds, ref.swaps_attempted, ref.swaps_accepted]
        assert np.array_equal(o["entry"], ref.round_entry_iterations)
