"""Parity at the benchmarked shapes, against the CPU oracle directly.

* C3 -- exactly bench.py's default step twice over: 256 lattices of 1024^2,
  seed 42, linear ladder 1+3i/R, J=1, B=0: parallel init, then for k = 0, 1
  ``sweeps(10k, 10)`` (ONE cb_sweeps_persistent<16,128> launch, asserted)
  and ``exchange(k)``.  Lattices, (S, Bond), slot_to_row and the accepted
  count must equal the oracle's chain (oracle.cb_sweep_mt restates
  or_cb_sweep over host threads; tests/test_oracle_mt.py pins the two).
* C4 -- the bench's C4 launch (512 lattices of 4096^2: the parallel init's
  multi-batch path, then cb_sweeps_persistent<32,128> with multi-block items
  and lattice-wide phases, asserted) on the GPU; a sample of the lattices is
  checked against the oracle's init and sweeps (the lattices are independent
  between exchange rounds, so each sampled lattice's chain is complete).
* A rank's C3 shard at 8 GPUs (32 lattices) -- the temporally blocked
  persistent launch (asserted), 10 and 7 sweeps, against the oracle.
"""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _by_row(slot_to_row):
    r2s = np.empty_like(slot_to_row)
    r2s[slot_to_row] = np.arange(slot_to_row.size)
    return r2s


def test_c3_bench_steps_equal_oracle():
    from paper_2512_03825_b200 import _lib, build_ladder
    from paper_2512_03825_b200.engine import CheckerboardEngine

    L, R, seed, every, J, B = 1024, 256, 42, 10, 1.0, 0.0
    temps = build_ladder(R)
    betas = 1.0 / temps
    torch.cuda.set_device(0)
    eng = CheckerboardEngine(L, R, temps, seed, J, B, 0.5, 0)
    eng.init_state()
    ref = np.empty((R, L, L), dtype=np.int8)
    oracle.fill_lattices_mt(ref, L * L // 2, seed)  # executor.py:203-205: row r from stream r
    assert np.array_equal(eng.final_spins(), ref)
    stats = oracle.row_stats_mt(ref)
    assert np.array_equal(eng.local_stats.cpu().numpy(), stats)
    thr, always = oracle.cb_tables(betas, J, B)
    s2r = np.arange(R, dtype=np.int64)
    accepted = 0
    for k in range(2):
        eng.sweeps(k * every, every)
        launch = _lib.cb_last_launch()
        assert launch["name"] == "cb_sweeps_persistent<16,128>", launch
        eng.exchange(k)
        r2s = _by_row(s2r)
        for t in range(k * every, (k + 1) * every):
            oracle.cb_sweep_mt(ref, r2s, thr, always, seed, t, stats)
        s = stats[s2r]
        energies = B * s[:, 0].astype(np.float64) - J * s[:, 1].astype(np.float64)
        sums = s[:, 0].copy()
        first = k % 2
        accepted += oracle.swap_chunk(s2r, energies, sums, betas, seed, R, k, first, 0, (R - first) // 2)
    torch.cuda.synchronize()
    assert np.array_equal(eng.final_spins(), ref)
    assert np.array_equal(eng.stats.cpu().numpy(), stats)
    assert np.array_equal(eng.slot_to_row.cpu().numpy(), s2r)
    assert eng.swap_counts() == (accepted, 0)
    # the by-slot energies the exchange used
    assert np.array_equal(eng.energies.cpu().numpy(), energies)


def test_c4_launch_on_sampled_lattices_equals_oracle():
    from paper_2512_03825_b200 import _lib, build_ladder
    from paper_2512_03825_b200.engine import CheckerboardEngine

    L, R, seed, n_sweeps, J, B = 4096, 512, 42, 4, 1.0, 0.0
    temps = build_ladder(R)
    torch.cuda.set_device(0)
    eng = CheckerboardEngine(L, R, temps, seed, J, B, 0.5, 0)
    eng.init_state()
    rows = np.array([0, 1, 255, 383, 511], dtype=np.int64)

    def sample():
        sel = eng.packed[torch.from_numpy(rows).to(eng.packed.device)].contiguous()
        out = torch.empty((rows.size, L, L), dtype=torch.int8, device=sel.device)
        _lib.call("ptmh_cb_unpack", sel.data_ptr(), rows.size, L, out.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        return out.cpu().numpy()

    ref = np.empty((rows.size, L, L), dtype=np.int8)
    for k, r in enumerate(rows):  # row r from stream r
        oracle.fill_lattices_mt(ref[k:k + 1], L * L // 2, seed, stream0=int(r))
    assert np.array_equal(sample(), ref)
    stats = oracle.row_stats_mt(ref)
    assert np.array_equal(eng.local_stats.cpu().numpy()[rows], stats)

    eng.sweeps(0, n_sweeps)
    launch = _lib.cb_last_launch()
    # the bench's C4 configuration (same shape, so the same launcher choice):
    # 32-row strips, multi-block items, lattice-wide phases
    assert launch["name"] == "cb_sweeps_persistent<32,128>" and launch["group"] >= 2 \
        and not launch["bands"], launch
    thr, always = oracle.cb_tables(1.0 / temps, J, B)
    r2s = rows.copy()  # no exchange yet: row r holds slot r
    for t in range(n_sweeps):
        oracle.cb_sweep_mt(ref, r2s, thr, always, seed, t, stats)
    torch.cuda.synchronize()
    assert np.array_equal(sample(), ref)
    assert np.array_equal(eng.local_stats.cpu().numpy()[rows], stats)


@pytest.mark.parametrize("n_sweeps", [10, 7])
def test_c3_rank_shard_temporally_blocked_equals_oracle(n_sweeps):
    """A rank's shard of C3 at 8 GPUs (32 lattices of 1024^2, the rows
    assign_replicas gives rank 3): the persistent launch runs temporally
    blocked there (asserted: one work item per (sweep, lattice, band), ping-
    pong buffers; an odd sweep count ends with the copy back), against the
    oracle's sweeps of the same rows."""
    from paper_2512_03825_b200 import _lib, build_ladder
    from paper_2512_03825_b200.engine import CheckerboardEngine

    L, R_total, G, rank, seed = 1024, 256, 8, 3, 42
    lo, hi = rank * R_total // G, (rank + 1) * R_total // G
    temps = build_ladder(R_total)
    torch.cuda.set_device(0)
    eng = CheckerboardEngine(L, R_total, temps, seed, 1.0, 0.0, 0.5, 0, row_range=(lo, hi))
    eng.init_state()
    ref = np.empty((hi - lo, L, L), dtype=np.int8)
    oracle.fill_lattices_mt(ref, L * L // 2, seed, stream0=lo)
    assert np.array_equal(eng.final_spins(), ref)
    stats = oracle.row_stats_mt(ref)
    eng.sweeps(0, n_sweeps)
    launch = _lib.cb_last_launch()
    assert launch["kind"] == 1 and launch["tb"], launch
    thr, always = oracle.cb_tables(1.0 / temps, 1.0, 0.0)
    r2s = np.arange(lo, hi, dtype=np.int64)  # no exchange yet: row r holds slot r
    for t in range(n_sweeps):
        oracle.cb_sweep_mt(ref, r2s, thr, always, seed, t, stats)
    torch.cuda.synchronize()
    assert np.array_equal(eng.final_spins(), ref)
    assert np.array_equal(eng.local_stats.cpu().numpy(), stats)
