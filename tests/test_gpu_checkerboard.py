"""Mode F (checkerboard, multispin-coded) on the GPU vs the CPU oracle:
bit-exact final lattices, per-lattice stats, observables, swap decisions."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import paper_2512_03825_b200 as p
    from paper_2512_03825_b200 import engine, kernels, tables
    return p, engine, kernels, tables


def _rand_spins(R, L, seed):
    rs = np.random.default_rng(seed)
    return (rs.integers(0, 2, size=(R, L, L)) * 2 - 1).astype(np.int8)


@pytest.mark.parametrize("L", [2, 4, 6, 10, 32, 64, 128, 192])
def test_pack_unpack_roundtrip_and_stats(mods, L):
    p, engine, _, _ = mods
    R = 3
    sp = _rand_spins(R, L, L)
    eng = engine.CheckerboardEngine(L, R, p.build_ladder(R), 1, 1.0, 0.0, 0.5, 0)
    eng.load_spins(torch.from_numpy(sp))
    assert np.array_equal(eng.final_spins(), sp)
    st = eng.local_stats.cpu().numpy()
    assert np.array_equal(st, oracle.row_stats(sp))
    assert np.array_equal(eng.audit_stats().cpu().numpy(), st)


@pytest.mark.parametrize("L,R,J,B,seed,nsweeps", [
    (64, 4, 1.0, 0.0, 42, 5),      # fast path
    (128, 3, 1.0, 0.0, 7, 4),
    (192, 2, 0.8, 0.0, 9, 3),
    (64, 3, 1.0, 0.5, 5, 4),       # field: 10-class path
    (128, 2, -1.0, 0.25, 6, 3),    # antiferromagnet with field
    (32, 5, 1.0, 0.0, 11, 6),      # generic path (L % 64 != 0)
    (10, 4, 1.0, 0.3, 12, 8),
    (2, 3, 1.0, 0.0, 13, 10),
    (6, 2, 0.5, -0.5, 14, 10),
])
def test_sweeps_match_oracle(mods, L, R, J, B, seed, nsweeps):
    p, engine, _, tables = mods
    temps = p.build_ladder(R)
    sp = _rand_spins(R, L, seed)
    eng = engine.CheckerboardEngine(L, R, temps, seed, J, B, 0.5, 0)
    perm = np.random.default_rng(seed).permutation(R)
    eng.slot_to_row.copy_(torch.from_numpy(perm.astype(np.int64)))
    r2s = np.empty(R, dtype=np.int64); r2s[perm] = np.arange(R)
    eng.row_to_slot.copy_(torch.from_numpy(r2s.astype(np.int32)))
    eng.load_spins(torch.from_numpy(sp))
    eng.sweeps(3, nsweeps)
    ref = sp.copy()
    stats = oracle.row_stats(ref)
    thr, always = oracle.cb_tables(1.0 / temps, J, B)
    t_thr, t_always = tables.cb_tables(1.0 / temps, J, B)
    assert np.array_equal(thr, t_thr) and always == (t_always & 0x3FF)
    for t in range(3, 3 + nsweeps):
        oracle.cb_sweep(ref, r2s, thr, always, seed, t, stats)
    got = eng.final_spins()
    assert np.array_equal(got, ref)
    assert np.array_equal(eng.local_stats.cpu().numpy(), stats)
    assert np.array_equal(eng.audit_stats().cpu().numpy(), stats)


@pytest.mark.parametrize("L,R,sweeps,every,seed,J,B,rec_every", [
    (64, 6, 20, 2, 42, 1.0, 0.0, 1),
    (32, 8, 30, 1, 3, 1.0, 0.0, 3),
    (128, 5, 12, 5, 4, 1.0, 0.1, 2),
    (4, 7, 50, 3, 5, 1.0, 0.0, 1),
])
def test_run_matches_oracle(mods, L, R, sweeps, every, seed, J, B, rec_every):
    p = mods[0]
    cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L,
                             swap_interval=every * L * L, seed=seed,
                             params=p.IsingParams(J=J, B=B), sweep_mode="checkerboard",
                             record_every=rec_every, return_final_state=True)
    rec = p.run(cfg)
    assert rec.valid, rec.error
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, J=J, B=B, record_every=rec_every)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.slot_to_row, ref.slot_to_row)
    assert np.array_equal(rec.energies, ref.energies)
    assert np.array_equal(rec.magnetizations, ref.magnetizations)
    assert (rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted) == \
        (ref.swap_rounds, ref.swaps_attempted, ref.swaps_accepted)
    assert rec.swap_near_ties == 0


@pytest.mark.parametrize("chunks,case", [(None, -1), ("3", -1)] + [(None, k) for k in range(8)])
def test_host_interval_plugin_matches_oracle(mods, monkeypatch, chunks, case):
    """One stream (small call, the default here) and 3 pipelined chunks; then
    randomised shapes, couplings, fields and chunk counts."""
    p, _, kernels, _ = mods
    L, R, seed, J, B, nsw = 64, 8, 21, 1.0, 0.0, 3
    if case >= 0:
        rng = np.random.default_rng(4000 + case)
        L = int(rng.choice([2, 4, 6, 10, 32, 64, 96, 128]))
        R = int(rng.integers(1, 12))
        seed = int(rng.integers(1 << 40))
        J = float(rng.choice([1.0, -1.0, 0.5]))
        B = float(rng.choice([0.0, 0.25, -0.5]))
        nsw = int(rng.integers(0, 4))
        chunks = str(rng.choice(["", "1", "2", "5"])) or None
    if chunks is not None:
        monkeypatch.setenv("PTMH_PLUGIN_CHUNKS", chunks)
    temps = p.build_ladder(R)
    betas = 1.0 / temps
    sp = np.empty((R, L, L), dtype=np.int8)
    for r in range(R):
        oracle.fill_lattice(sp[r], L * L // 2, seed, r, 0)
    ref = sp.copy()
    s2r = np.arange(R, dtype=np.int64)
    ref_s2r = s2r.copy()
    stats = oracle.row_stats(ref)
    thr, always = oracle.cb_tables(betas, J, B)
    done = 0
    for rnd in range(4):
        e = np.zeros(R); ss = np.zeros(R, dtype=np.int64)
        acc = kernels.cb_interval(sp, s2r, betas, J, B, seed, done, nsw, rnd, e, ss)
        r2s = np.empty(R, dtype=np.int64); r2s[ref_s2r] = np.arange(R)
        for t in range(done, done + nsw):
            oracle.cb_sweep(ref, r2s, thr, always, seed, t, stats)
        done += nsw
        s = stats[ref_s2r]
        re = B * s[:, 0] - J * s[:, 1].astype(np.float64)
        rs_ = s[:, 0].copy()
        racc = oracle.swap_chunk(ref_s2r, re, rs_, betas, seed, R, rnd, rnd % 2, 0,
                                 (R - rnd % 2) // 2)
        assert acc == racc
        assert np.array_equal(sp, ref)
        assert np.array_equal(s2r, ref_s2r)
        assert np.array_equal(e, re) and np.array_equal(ss, rs_)


def test_c3_scale_properties(mods):
    """BASELINE C3 shape (1024^2, 256 replicas): incremental stats equal the
    recomputed ones after an exchange interval, the run is deterministic, and
    the spin sums stay consistent with the packed state."""
    p, engine, _, _ = mods
    L, R = 1024, 256
    temps = p.build_ladder(R)
    outs = []
    for _ in range(2):
        eng = engine.CheckerboardEngine(L, R, temps, 42, 1.0, 0.0, 0.5, 0)
        eng.init_state()
        eng.sweeps(0, 10)
        eng.exchange(0)
        eng.sweeps(10, 2)
        st = eng.local_stats.clone()
        assert torch.equal(eng.audit_stats(), st)
        outs.append((st.cpu().numpy(), eng.slot_to_row.cpu().numpy(),
                     eng.packed.view(torch.int64).sum().item()))
        del eng
        torch.cuda.empty_cache()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


def test_one_lattice_matches_oracle_at_1024(mods):
    p, engine, _, _ = mods
    L, R = 1024, 2
    temps = np.array([1.5, 2.269])
    eng = engine.CheckerboardEngine(L, R, temps, 5, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    sp0 = eng.final_spins()
    eng.sweeps(0, 2)
    ref = sp0.copy()
    stats = oracle.row_stats(ref)
    thr, always = oracle.cb_tables(1.0 / temps, 1.0, 0.0)
    for t in range(2):
        oracle.cb_sweep(ref, np.arange(R, dtype=np.int64), thr, always, 5, t, stats)
    assert np.array_equal(eng.final_spins(), ref)
    assert np.array_equal(eng.local_stats.cpu().numpy(), stats)


@pytest.mark.parametrize("L,R,sweeps,every,seed,J,B,rec_every", [
    (64, 6, 20, 2, 42, 1.0, 0.0, 1),
    (64, 37, 15, 1, 8, 1.0, 0.0, 1),    # odd R, exchange every sweep
    (32, 8, 30, 1, 3, 1.0, 0.0, 3),     # segment gather (L = 32: two rows per word)
    (16, 5, 40, 1, 12, 1.0, 0.0, 1),    # segment gather, 4 rows per word
    (8, 9, 40, 2, 13, 1.0, 0.0, 2),     # segment gather, one word per colour
    (16, 6, 20, 1, 14, 1.0, 0.3, 1),    # segment gather, field: class plan
    (32, 4, 20, 1, 15, -1.0, 0.0, 1),   # segment gather, antiferromagnet
    (12, 5, 20, 1, 16, 1.0, 0.0, 1),    # generic gather (64 % L != 0)
    (64, 700, 6, 1, 17, 1.0, 0.0, 2),   # several lattices per CTA
    (16, 2000, 5, 1, 18, 1.0, 0.0, 1),  # many lattices per CTA, segment gather
    (128, 5, 12, 5, 4, 1.0, 0.1, 2),    # field: class plan
    (256, 3, 6, 2, 9, -1.0, 0.0, 1),    # antiferromagnet (cluster of 4 CTAs per lattice)
    (256, 5, 12, 1, 19, 1.0, 0.0, 2),   # ferro, cluster of 4 CTAs per lattice (the C2 choice)
    (512, 3, 6, 1, 20, 1.0, 0.0, 1),    # cluster of 8 CTAs per lattice
    (2, 7, 50, 3, 5, 1.0, 0.0, 1),
    (6, 4, 25, 0, 6, 0.5, -0.5, 5),     # no exchanges
    (8, 3, 9000, 1, 21, 1.0, 0.0, 50),  # > 4096 rounds: two segments of swap draws
    (64, 4096, 8, 1, 22, 1.0, 0.0, 2),  # C5's shape: point-to-point rounds, 28 warp-owned lattices per CTA
])
@pytest.mark.parametrize("p2p", [None, "0"])
def test_resident_run_matches_oracle(mods, monkeypatch, L, R, sweeps, every, seed, J, B, rec_every, p2p):
    """The resident run against the oracle; warp-owned lattices decide their
    rounds pairwise (point-to-point, default) or behind a grid barrier
    (PTMH_RESIDENT_P2P=0)."""
    if p2p is not None:
        monkeypatch.setenv("PTMH_RESIDENT_P2P", p2p)
    p = mods[0]
    cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L,
                             swap_interval=every * L * L, seed=seed,
                             params=p.IsingParams(J=J, B=B), sweep_mode="checkerboard",
                             record_every=rec_every, return_final_state=True, kernel="resident")
    rec = p.run(cfg)
    assert rec.valid, rec.error
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, J=J, B=B, record_every=rec_every)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.slot_to_row, ref.slot_to_row)
    assert np.array_equal(rec.energies, ref.energies)
    assert np.array_equal(rec.magnetizations, ref.magnetizations)
    assert (rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted) == \
        (ref.swap_rounds, ref.swaps_attempted, ref.swaps_accepted)
    if ref.round_entry_iterations is not None:
        assert np.array_equal(rec.round_entry_iterations[:, 0], ref.round_entry_iterations * L * L)


@pytest.mark.parametrize("case", range(32))
def test_resident_random_shapes_match_oracle(mods, case):
    """Randomised shapes, couplings and schedules through the resident kernel
    (every gather mode, clusters, warp-owned lattices) and the per-interval
    path, against the oracle."""
    p = mods[0]
    rng = np.random.default_rng(1000 + case)
    L = int(rng.choice([2, 4, 6, 8, 10, 16, 24, 32, 48, 64, 96, 128, 256]))
    R = int(rng.integers(1, 40 if L <= 64 else 6))
    sweeps = int(rng.integers(1, 12 if L <= 64 else 5))
    every = int(rng.integers(0, 4))
    J = float(rng.choice([1.0, -1.0, 0.5]))
    B = float(rng.choice([0.0, 0.0, 0.25, -0.5]))
    rec_every = int(rng.integers(1, min(3, sweeps) + 1))
    seed = int(rng.integers(1 << 40))
    kernel = str(rng.choice(["resident", "resident", "sweep", "auto"]))
    cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=every * L * L,
                             seed=seed, params=p.IsingParams(J=J, B=B), sweep_mode="checkerboard",
                             record_every=rec_every, return_final_state=True, kernel=kernel)
    rec = p.run(cfg)
    assert rec.valid, rec.error
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, J=J, B=B, record_every=rec_every)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.slot_to_row, ref.slot_to_row)
    assert np.array_equal(rec.energies, ref.energies)
    assert np.array_equal(rec.magnetizations, ref.magnetizations)
    assert (rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted) == \
        (ref.swap_rounds, ref.swaps_attempted, ref.swaps_accepted)


@pytest.mark.parametrize("cluster", ["1", "2", "8"])
def test_resident_cluster_sizes(mods, monkeypatch, cluster):
    """C2's lattice size (256^2) on other cluster sizes than the automatic 4."""
    monkeypatch.setenv("PTMH_RESIDENT_CLUSTER", cluster)
    p = mods[0]
    L, R, sweeps, every, seed = 256, 5, 8, 1, 23
    cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=every * L * L,
                             seed=seed, sweep_mode="checkerboard", record_every=2, return_final_state=True,
                             kernel="resident")
    rec = p.run(cfg)
    assert rec.valid, rec.error
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, record_every=2)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.energies, ref.energies)
    assert rec.swaps_accepted == ref.swaps_accepted


@pytest.mark.parametrize("L,R,sweeps,every,rec_every,cfg", [
    (256, 5, 8, 1, 2, None),         # automatic cluster size (C2's lattice)
    (256, 64, 6, 1, 3, None),        # C2's shape: 2-CTA clusters
    (256, 6, 7, 1, 1, "2,2,256"),
    (256, 3, 5, 2, 5, "1,2,256"),    # whole lattice in one CTA: halos wrap onto itself
    (256, 4, 6, 1, 2, "4,1,256"),
    (256, 4, 6, 3, 2, "2,4,128"),
    (256, 4, 4, 1, 1, "2,1,512"),
    (256, 4, 4, 1, 1, "8,2,128"),
    (128, 9, 9, 1, 3, "2,2,128"),
    (512, 3, 4, 1, 2, "8,2,128"),
    (512, 2, 3, 1, 3, "16,2,128"),   # non-portable cluster size
    (192, 4, 5, 1, 1, "1,1,256"),    # L/64 = 3 words per row
    (320, 3, 4, 2, 2, "5,2,256"),    # odd cluster size, 64-row bands
    (256, 7, 6, 0, 2, None),         # no exchanges
])
def test_cluster_smem_kernel_matches_oracle(mods, monkeypatch, L, R, sweeps, every, rec_every, cfg):
    """cb_cluster_smem_kernel (lattices in the shared memory of thread-block
    clusters, halos over DSMEM, point-to-point rounds) against the oracle,
    over cluster sizes, strip heights and CTA widths."""
    if cfg is not None:
        monkeypatch.setenv("PTMH_RESIDENT_SMEM", cfg)
    p = mods[0]
    from paper_2512_03825_b200 import _lib
    seed = 1000 + L + R
    cfg_run = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=every * L * L,
                                 seed=seed, sweep_mode="checkerboard", record_every=rec_every,
                                 return_final_state=True, kernel="resident")
    rec = p.run(cfg_run)
    assert rec.valid, rec.error
    assert _lib.cb_last_launch()["kind"] == 8
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, record_every=rec_every)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.slot_to_row, ref.slot_to_row)
    assert np.array_equal(rec.energies, ref.energies)
    assert np.array_equal(rec.magnetizations, ref.magnetizations)
    assert (rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted) == \
        (ref.swap_rounds, ref.swaps_attempted, ref.swaps_accepted)


@pytest.mark.parametrize("rows1,pre,expect", [("1", "1", (1, 512)), ("0", "1", (2, 256)), ("0", "0", (2, 256))])
def test_c2_shape_kernel_variants_match_oracle(mods, monkeypatch, rows1, pre, expect):
    """C2's shape (256^2 x 64, a round every sweep) on the launcher's choice
    (1-row strips on 512 threads, random planes drawn ahead of each pass and,
    across a round, for both slots the lattice may hold), on 2-row strips,
    and with the planes drawn inside the passes: all equal to the oracle."""
    monkeypatch.setenv("PTMH_SMEM_ROWS1", rows1)
    monkeypatch.setenv("PTMH_SMEM_PRE", pre)
    p = mods[0]
    from paper_2512_03825_b200 import _lib
    L, R, sweeps, seed = 256, 64, 5, 4242
    rec = p.run(p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=L * L, seed=seed,
                                   sweep_mode="checkerboard", record_every=1, return_final_state=True,
                                   kernel="resident"))
    assert rec.valid, rec.error
    launch = _lib.cb_last_launch()
    assert launch["kind"] == 8 and (launch["rows"], launch["threads"]) == expect and launch["group"] == 2
    ref = oracle.run_checkerboard(L, R, sweeps, 1, seed, record_every=1)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.slot_to_row, ref.slot_to_row)
    assert np.array_equal(rec.energies, ref.energies)
    assert rec.swaps_accepted == ref.swaps_accepted


@pytest.mark.parametrize("R,sweeps,every,rec_every,J", [
    (4096, 6, 1, 2, 1.0),   # C5's shape
    (333, 9, 1, 3, 1.0),    # ragged lattices per CTA
    (200, 7, 3, 7, 1.0),
    (97, 11, 0, 11, 1.0),   # no exchanges
    (130, 5, 1, 5, 0.5),    # another coupling (thresholds from J)
])
def test_reg64_kernel_matches_oracle(mods, R, sweeps, every, rec_every, J):
    """cb_resident_reg64_kernel (64^2 ferro lattices held in registers, a warp
    each: neighbour rows by shuffles, no memory traffic during the sweeps)
    against the oracle; the launch is asserted.  (Up to 64 lattices of 64^2
    the launcher puts every lattice in ONE CTA instead.)"""
    p = mods[0]
    from paper_2512_03825_b200 import _lib
    L, seed = 64, 600 + R
    cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=every * L * L,
                             seed=seed, params=p.IsingParams(J=J, B=0.0), sweep_mode="checkerboard",
                             record_every=rec_every, return_final_state=True, kernel="resident")
    rec = p.run(cfg)
    assert rec.valid, rec.error
    assert _lib.cb_last_launch()["kind"] == 9
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, J=J, record_every=rec_every)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.slot_to_row, ref.slot_to_row)
    assert np.array_equal(rec.energies, ref.energies)
    assert np.array_equal(rec.magnetizations, ref.magnetizations)
    assert (rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted) == \
        (ref.swap_rounds, ref.swaps_attempted, ref.swaps_accepted)


@pytest.mark.parametrize("J,B", [(1.0, 0.1), (-1.0, 0.0)])
def test_resident_large_lattices_non_ferro(mods, J, B):
    """The L2-resident kernel at 1024^2 x 32 with a round every sweep (a field
    or an antiferromagnet: no shared-memory kernel): its 4-CTA clusters of
    1024 threads cannot all be resident at once, so the launcher retries on
    smaller clusters (cudaErrorCooperativeLaunchTooLarge) -- and the next run
    on the same process is unaffected by that refused launch."""
    p = mods[0]
    L, R, sweeps = 1024, 32, 2
    for seed in (3, 4):
        cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=L * L, seed=seed,
                                 params=p.IsingParams(J=J, B=B), sweep_mode="checkerboard",
                                 return_final_state=True)
        rec = p.run(cfg)
        assert rec.valid, rec.error
        ref = oracle.run_checkerboard(L, R, sweeps, 1, seed, J=J, B=B)
        assert np.array_equal(rec.final_spins, ref.final_spins)
        assert np.array_equal(rec.energies, ref.energies)
        assert np.array_equal(rec.slot_to_row, ref.slot_to_row)


@pytest.mark.parametrize("R,sweeps,every,rec_every,J", [
    (8, 40, 1, 2, 1.0),     # C1's shape
    (3, 25, 1, 5, 1.0),
    (77, 9, 2, 3, 1.0),     # several lattices per CTA, ragged
    (5, 11, 0, 11, 1.0),    # no exchanges
    (6, 15, 1, 5, 0.5),
])
def test_reg32_kernel_matches_oracle(mods, R, sweeps, every, rec_every, J):
    """cb_resident_reg32_kernel (32^2 ferro lattices held in registers, a warp
    each: 16 lanes own a word of both colours, neighbour rows by shuffles and
    segment shifts) against the oracle; the launch is asserted."""
    p = mods[0]
    from paper_2512_03825_b200 import _lib
    L, seed = 32, 900 + R
    cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=every * L * L,
                             seed=seed, params=p.IsingParams(J=J, B=0.0), sweep_mode="checkerboard",
                             record_every=rec_every, return_final_state=True, kernel="resident")
    rec = p.run(cfg)
    assert rec.valid, rec.error
    assert _lib.cb_last_launch()["kind"] == 10
    ref = oracle.run_checkerboard(L, R, sweeps, every, seed, J=J, record_every=rec_every)
    assert np.array_equal(rec.final_spins, ref.final_spins)
    assert np.array_equal(rec.slot_to_row, ref.slot_to_row)
    assert np.array_equal(rec.energies, ref.energies)
    assert np.array_equal(rec.magnetizations, ref.magnetizations)
    assert (rec.swap_rounds, rec.swaps_attempted, rec.swaps_accepted) == \
        (ref.swap_rounds, ref.swaps_attempted, ref.swaps_accepted)


def test_resident_segments_compose(mods):
    """Two resident segments == one resident run == the sweep-kernel path."""
    p, engine, _, _ = mods
    L, R, total, every = 64, 9, 12, 3
    temps = p.build_ladder(R)
    outs = []
    for mode in ("one", "two", "sweep"):
        eng = engine.CheckerboardEngine(L, R, temps, 77, 1.0, 0.0, 0.5, 0)
        eng.init_state()
        if mode == "one":
            eng.run_resident(0, total, total, every)
        elif mode == "two":
            eng.run_resident(0, 5, total, every)
            eng.run_resident(5, total - 5, total, every)
        else:
            from paper_2512_03825_b200.executor import _interval_plan
            done = 0
            for target, ri in _interval_plan(total, every):
                eng.sweeps(done, target - done)
                done = target
                if ri is not None:
                    eng.exchange(ri)
        outs.append((eng.final_spins(), eng.slot_to_row.cpu().numpy(), eng.swap_counts()[0],
                     eng.local_stats.cpu().numpy()))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0])
        assert np.array_equal(o[1], outs[0][1])
        assert o[2] == outs[0][2]
        assert np.array_equal(o[3], outs[0][3])


@pytest.mark.parametrize("L,R,ladder", [(32, 8, "geometric"), (256, 64, "linear"), (64, 4096, "linear")])
def test_bench_e2e_round_trip_is_the_same_run(mods, L, R, ladder):
    """bench.py's e2e step for the resident configurations (C1, C2, C5):
    lattices and permutation to pinned host memory and back between
    resident segments (load_spins -> run_resident -> spins_int8) gives the
    run that never leaves the device."""
    p, engine, _, _ = mods
    temps = p.geometric_ladder(R) if ladder == "geometric" else p.build_ladder(R)
    big, every, seg, nseg = 1 << 30, 1, 20, 3
    ref = engine.CheckerboardEngine(L, R, temps, 42, 1.0, 0.0, 0.5, 0)
    ref.init_state()
    ref.run_resident(0, seg * nseg, big, every)
    eng = engine.CheckerboardEngine(L, R, temps, 42, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    host = torch.empty((R, L, L), dtype=torch.int8).pin_memory()
    host.copy_(eng.spins_int8())
    s2r_h = eng.slot_to_row.cpu().pin_memory()
    r2s_h = eng.row_to_slot.cpu().pin_memory()
    dbuf = torch.empty((R, L, L), dtype=torch.int8, device="cuda")
    for k in range(nseg):
        dbuf.copy_(host, non_blocking=True)
        eng.slot_to_row.copy_(s2r_h, non_blocking=True)
        eng.row_to_slot.copy_(r2s_h, non_blocking=True)
        eng.load_spins(dbuf)
        eng.run_resident(k * seg, seg, big, every)
        host.copy_(eng.spins_int8(), non_blocking=True)
        s2r_h.copy_(eng.slot_to_row, non_blocking=True)
        r2s_h.copy_(eng.row_to_slot, non_blocking=True)
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), ref.final_spins())
    assert np.array_equal(s2r_h.numpy(), ref.slot_to_row.cpu().numpy())
    assert np.array_equal(r2s_h.numpy(), ref.row_to_slot.cpu().numpy())
    assert np.array_equal(eng.stats.cpu().numpy(), ref.stats.cpu().numpy())
    assert eng.swap_counts() == ref.swap_counts()


def test_sweeps_match_oracle_at_2048(mods):
    """L >= 1024 takes the 16-rows-per-thread fast-path instantiation (also at 2048)."""
    p, engine, _, _ = mods
    L, R = 2048, 2
    temps = np.array([1.8, 2.6])
    eng = engine.CheckerboardEngine(L, R, temps, 21, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    sp0 = eng.final_spins()
    eng.sweeps(0, 1)
    ref = sp0.copy()
    stats = oracle.row_stats(ref)
    thr, always = oracle.cb_tables(1.0 / temps, 1.0, 0.0)
    oracle.cb_sweep(ref, np.arange(R, dtype=np.int64), thr, always, 21, 0, stats)
    assert np.array_equal(eng.final_spins(), ref)
    assert np.array_equal(eng.local_stats.cpu().numpy(), stats)


@pytest.mark.parametrize("L,R,sweeps,every,rec_every", [(4, 3, 40, 2, 1), (64, 4, 12, 3, 2),
                                                        (6, 5, 30, 1, 3)])
def test_full_states_match_oracle(mods, L, R, sweeps, every, rec_every):
    p = mods[0]
    rec = p.run(p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L,
                                   swap_interval=every * L * L, seed=31, sweep_mode="checkerboard",
                                   record_mode="full_states", record_every=rec_every))
    assert rec.valid, rec.error
    ref = oracle.run_checkerboard(L, R, sweeps, every, 31, record_every=rec_every, record_states=True)
    assert rec.states.shape == (R, sweeps // rec_every, L, L)
    assert np.array_equal(rec.states, ref.states)
    assert np.array_equal(rec.energies, ref.energies)
    # magnetisations are the recorded states' means (reference test_executor.py:172-181)
    assert np.array_equal(rec.magnetizations, rec.states.sum(axis=(2, 3)) / (L * L))


@pytest.mark.parametrize("L,R,first,nsweeps,per_slot,rows,threads", [
    (1024, 24, 3, 7, None, None, None), (1024, 256, 0, 10, None, None, None), (2048, 5, 1, 3, None, None, None),
    (2048, 5, 1, 3, "0", "16", None),    # 16 blocks per item: one item per lattice and phase
    (1024, 256, 0, 4, "0", "16", None),  # 4 blocks per item (auto: 128-thread items)
    (1024, 256, 0, 4, None, None, "256"),  # the full C3 shard on 256-thread items
    (1024, 32, 2, 5, None, "8", None),   # 8 rows per thread
    (1024, 32, 2, 5, None, "4", None),   # 4 rows per thread (a rank's C3 shard at 8 GPUs)
    (1024, 24, 3, 7, None, None, "128"),  # 128-thread items below their auto threshold
    (512, 9, 0, 6, "0", "4", None),      # L = 512, grouped 4-row items
    (512, 9, 0, 6, "0", "4", "128"),     # ... on 128-thread items
    (1024, 16, 1, 4, None, None, None),  # auto: 2 rows per thread (a rank's C3 shard at 16 GPUs)
    (1536, 3, 2, 3, None, "16", None),   # 9 blocks per lattice and phase (odd), WR = 24
    (1536, 3, 2, 3, None, "16", "128"),  # 18 blocks per lattice and phase
    (1536, 3, 2, 3, None, "32", "256"),  # 32 rows do not split 1536^2 into 256-thread blocks: 16 taken
    (2048, 4, 1, 3, None, "32", None),   # 32 rows per thread (the C4 choice), ties from L2
    (2048, 4, 1, 3, None, "32", "128"),  # ... on 128-thread items (the C4 launch)
    (1024, 8, 0, 2, "0", "32", None),    # 32 rows, grouped
])
@pytest.mark.parametrize("tb,bands", [(None, None), ("1", None), ("0", None), ("0", "0"), ("0", "1")])
def test_persistent_sweeps_equal_per_launch_path(mods, monkeypatch, L, R, first, nsweeps, per_slot, rows, threads,
                                                 tb, bands):
    """The one-launch dataflow path (cb_sweeps_persistent) and the per-launch
    half-sweep kernels give identical lattices and stats; the sync block is
    left zeroed for the next call.  tb = "1": temporally blocked items (a
    whole sweep of a band per item, ping-pong buffers; odd sweep counts end
    with the copy back) wherever items span whole lattice rows (the default
    for shards of <= 2^25 sites); tb = "0": per-colour items with band (or,
    bands "0", lattice-wide) dependencies."""
    p, engine, _, _ = mods
    from paper_2512_03825_b200 import _lib
    if tb is not None:
        monkeypatch.setenv("PTMH_PERSIST_TB", tb)
    if per_slot is not None:
        monkeypatch.setenv("PTMH_PERSIST_ITEMS_PER_SLOT", per_slot)
    if rows is not None:
        monkeypatch.setenv("PTMH_PERSIST_ROWS", rows)
    if threads is not None:
        monkeypatch.setenv("PTMH_PERSIST_THREADS", threads)
    if bands is not None:  # band dependencies forced on (where items span rows) / off
        monkeypatch.setenv("PTMH_PERSIST_BANDS", bands)
    temps = p.build_ladder(R)
    perm = np.random.default_rng(R).permutation(R)
    r2s = np.empty(R, dtype=np.int64); r2s[perm] = np.arange(R)
    outs = []
    for persistent in (True, False):
        eng = engine.CheckerboardEngine(L, R, temps, 99, 1.0, 0.0, 0.5, 0)
        eng.persistent = persistent
        eng.slot_to_row.copy_(torch.from_numpy(perm.astype(np.int64)))
        eng.row_to_slot.copy_(torch.from_numpy(r2s.astype(np.int32)))
        eng.init_state()
        eng.sweeps(first, nsweeps)
        if persistent and L >= 1024:  # (L = 512: the per-launch kernels either way)
            launch = _lib.cb_last_launch()
            assert launch["kind"] == 1
            # temporally blocked items: 128-thread items that span whole rows (L <= 8192)
            spans = launch["threads"] == 128 and 128 % (L // 64) == 0
            assert launch["tb"] == (spans and (tb == "1" or (tb is None and R * L * L <= 1 << 25)))
            # beyond 2^25 sites (16- / 32-row items) the blocked items stream through their band
            streamed = launch["tb"] and R * L * L > 1 << 25 and launch["rows"] in (16, 32)
            assert launch["streamed"] == streamed
        eng.sweeps(first + nsweeps, 1)  # a second call reuses the (re-zeroed) sync block
        torch.cuda.synchronize()
        if persistent:
            assert int(eng._sync.abs().sum().item()) == 0
        outs.append((eng.packed.clone(), eng.local_stats.clone(), eng.audit_stats()))
        del eng
        torch.cuda.empty_cache()
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(outs[0][1], outs[0][2])


@pytest.mark.parametrize("plugin_sync", ["0", "1"])
def test_host_interval_plugin_at_1024(mods, monkeypatch, plugin_sync):
    """The host plugin at L = 1024, with the chunks on the per-launch kernels
    (default) and on the persistent path: equal to the device engine (which
    matches the oracle, above)."""
    p, engine, kernels, _ = mods
    monkeypatch.setenv("PTMH_PLUGIN_SYNC", plugin_sync)
    L, R, seed = 1024, 6, 23
    temps = p.build_ladder(R)
    betas = 1.0 / temps
    eng = engine.CheckerboardEngine(L, R, temps, seed, 1.0, 0.0, 0.5, 0)
    eng.init_state()
    sp = eng.final_spins()
    s2r = np.arange(R, dtype=np.int64)
    prev = 0
    for rnd in range(2):
        e = np.zeros(R); ss = np.zeros(R, dtype=np.int64)
        acc = kernels.cb_interval(sp, s2r, betas, 1.0, 0.0, seed, 2 * rnd, 2, rnd, e, ss)
        eng.sweeps(2 * rnd, 2)
        eng.exchange(rnd)
        assert acc == eng.swap_counts()[0] - prev
        prev = eng.swap_counts()[0]
        assert np.array_equal(sp, eng.final_spins())
        assert np.array_equal(s2r, eng.slot_to_row.cpu().numpy())


def _random_sharded_cases(n):
    rng = np.random.default_rng(5000)
    out = []
    for _ in range(n):
        total = int(rng.integers(3, 25))
        out.append((int(rng.choice([8, 16, 32, 64, 128])), int(rng.integers(4, 60)), int(rng.integers(2, 5)),
                    total, int(rng.integers(1, 4)), int(rng.integers(1, min(5, total) + 1))))
    return out


@pytest.mark.parametrize("L,R,G,total,every,rec", [(64, 24, 2, 30, 1, 1), (64, 37, 3, 20, 2, 2),
                                                   (16, 40, 4, 25, 1, 5),
                                                   (256, 6, 2, 8, 1, 2),   # shared-memory clusters
                                                   (128, 9, 3, 7, 2, 1)] + _random_sharded_cases(6))
@pytest.mark.parametrize("p2p", [None, "0"])
def test_resident_sharded_virtual_ranks(mods, monkeypatch, L, R, G, total, every, rec, p2p):
    """The multi-GPU resident kernel (rounds exchanged through peer memory, no
    collective: pairwise round words where lattices are warp-owned, else
    flags + grid barriers; PTMH_RESIDENT_P2P=0 forces the latter) with G ranks
    co-running on ONE GPU, each on its own stream and a share of the SMs:
    after combining the ranks' parts it is the single-GPU resident run, bit
    for bit."""
    if p2p is not None:
        monkeypatch.setenv("PTMH_RESIDENT_P2P", p2p)
    p, engine, _, _ = mods
    from paper_2512_03825_b200.executor import assign_replicas
    temps, seed = p.build_ladder(R), 31
    ncols = total // rec
    ref = engine.CheckerboardEngine(L, R, temps, seed, 1.0, 0.0, 0.5, 0)
    ref.init_state()
    roe = torch.zeros((R, ncols), dtype=torch.float64, device="cuda")
    rom = torch.zeros_like(roe)
    ref.run_resident(0, total, total, every, record_every=rec, obs_e=roe, obs_m=rom)
    bounds = assign_replicas(R, G)
    engs = [engine.CheckerboardEngine(L, R, temps, seed, 1.0, 0.0, 0.5, 0, row_range=b) for b in bounds]
    for e in engs:
        e.init_state()
    pubs = [torch.zeros((2, R, 2), dtype=torch.int64, device="cuda") for _ in range(G)]
    flags = [torch.zeros(G, dtype=torch.int32, device="cuda") for _ in range(G)]
    oes = [torch.zeros((R, ncols), dtype=torch.float64, device="cuda") for _ in range(G)]
    oms = [torch.zeros_like(o) for o in oes]
    streams = [torch.cuda.Stream() for _ in range(G)]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    torch.cuda.synchronize()
    for g, e in enumerate(engs):
        with torch.cuda.stream(streams[g]):
            e.run_resident_sharded(0, total, total, every, g, G, [t.data_ptr() for t in pubs],
                                   [f.data_ptr() for f in flags], pubs[g], record_every=rec, obs_e=oes[g],
                                   obs_m=oms[g], max_ctas=sms // G - 2)
    torch.cuda.synchronize()
    r2s = np.concatenate([e.row_to_slot[e.row_lo:e.row_hi].cpu().numpy() for e in engs])
    assert np.array_equal(r2s, ref.row_to_slot.cpu().numpy())
    spins = np.concatenate([e.final_spins() for e in engs])
    assert np.array_equal(spins, ref.final_spins())
    stats = np.concatenate([e.local_stats.cpu().numpy() for e in engs])
    assert np.array_equal(stats, ref.local_stats.cpu().numpy())
    assert sum(e.swap_counts()[0] for e in engs) == ref.swap_counts()[0]
    assert torch.equal(sum(oes), roe) and torch.equal(sum(oms), rom)


@pytest.mark.parametrize("L,R,sweeps,every,J,B", [
    (96, 130, 3, 1, 1.0, 0.0), (192, 40, 3, 2, 1.0, 0.0), (320, 17, 2, 1, 1.0, 0.0),
    (512, 40, 3, 1, 1.0, 0.0), (512, 9, 4, 2, 0.5, 0.1), (640, 12, 2, 1, 1.0, 0.0),
    (1024, 20, 2, 1, 1.0, 0.0), (1024, 7, 2, 1, -1.0, 0.0), (1536, 5, 2, 1, 1.0, 0.0),
    (2048, 6, 2, 1, 1.0, 0.0), (2048, 3, 2, 1, 1.0, -0.2),
])
def test_resident_and_sweep_paths_agree(mods, L, R, sweeps, every, J, B):
    """Larger shapes than the oracle tests reach: the resident run (whichever
    kernel the launcher picks: shared-memory clusters, L2 clusters, CTA- or
    warp-owned lattices, with the cooperative-launch fallbacks) and the sweep
    path (persistent or per-launch kernels + exchange kernel) are the same
    chain, so their records must be identical."""
    p = mods[0]
    recs = []
    for kernel in ("resident", "sweep"):
        cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L, swap_interval=every * L * L,
                                 seed=L + R, params=p.IsingParams(J=J, B=B), sweep_mode="checkerboard",
                                 return_final_state=True, kernel=kernel)
        rec = p.run(cfg)
        assert rec.valid, (kernel, rec.error)
        recs.append(rec)
    a, b = recs
    assert np.array_equal(a.final_spins, b.final_spins)
    assert np.array_equal(a.energies, b.energies)
    assert np.array_equal(a.magnetizations, b.magnetizations)
    assert np.array_equal(a.slot_to_row, b.slot_to_row)
    assert (a.swaps_attempted, a.swaps_accepted) == (b.swaps_attempted, b.swaps_accepted)
