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


def _ipc_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)  # both ranks on the one GPU: CUDA IPC across processes
    from cuda.bindings import runtime as rt
    from paper_2512_03825_b200.distributed import PeerBuffers
    peers = PeerBuffers(5, torch.device("cuda", 0))
    # every rank writes (rank + 1) * 100 + g into flag slot [rank] of rank g's
    # buffer, and its rank into row `rank` of every peer's slot_stats[0]
    src = torch.empty(1, dtype=torch.int32, device="cuda")
    row = torch.full((2,), rank + 7, dtype=torch.int64, device="cuda")
    for g in range(world):
        src.fill_((rank + 1) * 100 + g)
        torch.cuda.synchronize()
        err, = rt.cudaMemcpy(peers.flag_peers[g] + 4 * rank, src.data_ptr(), 4,
                             rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
        assert err == rt.cudaError_t.cudaSuccess, err
        err, = rt.cudaMemcpy(peers.pub_peers[g] + 16 * rank, row.data_ptr(), 16,
                             rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
        assert err == rt.cudaError_t.cudaSuccess, err
    torch.cuda.synchronize()
    dist.barrier()
    flags = torch.empty(world, dtype=torch.int32, device="cuda")
    stats = torch.empty((world, 2), dtype=torch.int64, device="cuda")
    for dst, ptr, n in ((flags, peers.flags, 4 * world), (stats, peers.slot_stats, 16 * world)):
        err, = rt.cudaMemcpy(dst.data_ptr(), ptr, n, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
        assert err == rt.cudaError_t.cudaSuccess, err
    np.savez(os.path.join(out_dir, f"ipc{rank}.npz"), flags=flags.cpu().numpy(), stats=stats.cpu().numpy())
    dist.barrier()
    peers.close()
    dist.destroy_process_group()


def test_peer_buffers_ipc_two_processes(tmp_path):
    """PeerBuffers: CUDA IPC handles shared over the process group and opened
    as peer pointers (two processes on the one GPU): every rank's writes land
    in every other rank's round buffers."""
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_ipc_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for g in range(world):
        d = np.load(tmp_path / f"ipc{g}.npz")
        assert d["flags"].tolist() == [(r + 1) * 100 + g for r in range(world)]
        for r in range(world):
            assert d["stats"][r].tolist() == [r + 7, r + 7]


def test_resident_sharded_driver_world1():
    """distributed.resident_sharded (peer-buffer rounds, then the slots /
    counters / observables combination) over NCCL at world 1, in two
    segments with recording: equal to the engine's own resident run."""
    from paper_2512_03825_b200 import build_ladder
    from paper_2512_03825_b200.distributed import PeerBuffers, ShardedCheckerboard, resident_sharded
    from paper_2512_03825_b200.engine import CheckerboardEngine
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        L, R, total, every, rec, seed = 64, 12, 24, 1, 2, 23
        temps = build_ladder(R)
        ref = CheckerboardEngine(L, R, temps, seed, 1.0, 0.0, 0.5, 0)
        ref.init_state()
        roe = torch.zeros((R, total // rec), dtype=torch.float64, device="cuda")
        rom = torch.zeros_like(roe)
        ref.run_resident(0, 10, total, every, record_every=rec, obs_e=roe, obs_m=rom)
        ref.run_resident(10, total - 10, total, every, record_every=rec, obs_e=roe, obs_m=rom)
        drv = ShardedCheckerboard(L, R, temps, seed, device=0)
        drv.init_state()
        peers = PeerBuffers(R, torch.device("cuda", 0))
        oe = torch.zeros_like(roe)
        om = torch.zeros_like(rom)
        resident_sharded(drv, peers, 0, 10, total, every, record_every=rec, obs_e=oe, obs_m=om)
        resident_sharded(drv, peers, 10, total - 10, total, every, record_every=rec, obs_e=oe, obs_m=om)
        torch.cuda.synchronize()
        assert np.array_equal(drv.eng.final_spins(), ref.final_spins())
        assert torch.equal(drv.eng.slot_to_row, ref.slot_to_row)
        assert torch.equal(drv.eng.row_to_slot, ref.row_to_slot)
        assert drv.eng.swap_counts() == ref.swap_counts()
        assert torch.equal(oe, roe) and torch.equal(om, rom)
        peers.close()
    finally:
        dist.destroy_process_group()
