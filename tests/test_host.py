"""Host-side logic of the engine (CPU only): schedule, sharding, ladders,
pairing, swap rule, configuration validation and the acceptance tables.
Mirrors the reference's own unit tests (tests/test_executor.py,
tests/test_tempering.py) for the same functions."""

import math

import numpy as np
import pytest

import oracle
from paper_2512_03825_b200 import (ConfigurationError, IsingParams, SimulationConfig, SpinLattice,
                                   assign_replicas, build_ladder, flip_delta, geometric_ladder,
                                   magnetization_fraction, pairing, swap_probability, total_energy)
from paper_2512_03825_b200.executor import _interval_plan
from paper_2512_03825_b200.tables import cb_tables, class_delta, exact_tables


class TestAssignReplicas:  # reference tests/test_executor.py:22-47
    def test_paper_scale_partition(self):
        sizes = [hi - lo for lo, hi in assign_replicas(1500, 16)]
        assert sorted(set(sizes)) == [93, 94] and sum(sizes) == 1500

    def test_more_workers_than_replicas(self):
        assert [hi - lo for lo, hi in assign_replicas(4, 8)] == [1, 1, 1, 1, 0, 0, 0, 0]

    def test_ceiling_floor_rule(self):
        assert [hi - lo for lo, hi in assign_replicas(5, 2)] == [3, 2]

    def test_every_replica_exactly_once(self):
        for count, workers in [(7, 3), (16, 5), (2, 2), (9, 9), (256, 8), (4096, 8)]:
            covered = [i for lo, hi in assign_replicas(count, workers) for i in range(lo, hi)]
            assert covered == list(range(count))

    def test_invalid_workers(self):
        with pytest.raises(ConfigurationError):
            assign_replicas(4, 0)


class TestIntervalPlan:  # reference tests/test_executor.py:50-63
    def test_plans(self):
        assert _interval_plan(100, 0) == [(100, None)]
        assert _interval_plan(300, 100) == [(100, 0), (200, 1), (300, None)]
        assert _interval_plan(301, 100) == [(100, 0), (200, 1), (300, 2), (301, None)]
        assert _interval_plan(50, 100) == [(50, None)]
        assert _interval_plan(1, 1) == [(1, None)]

    @pytest.mark.parametrize("n,i", [(1000, 7), (10, 1), (64, 64), (65, 64), (3, 0)])
    def test_matches_oracle(self, n, i):
        assert _interval_plan(n, i) == oracle.interval_plan(n, i)


class TestLadderAndPairing:  # reference tests/test_tempering.py:15-77
    def test_ladder_exact_values(self):
        assert build_ladder(3).tolist() == [1.0, 2.0, 3.0]
        assert build_ladder(1).tolist() == [1.0]
        assert build_ladder(6).tolist() == [1.0, 1.5, 2.0, 2.5, 3.0, 3.5]
        assert np.array_equal(build_ladder(257), oracle.build_ladder(257))
        with pytest.raises(ValueError):
            build_ladder(0)

    def test_geometric_ladder(self):
        t = geometric_ladder(8)
        assert t[0] == 1.0 and math.isclose(t[-1], 4.0)
        assert np.allclose(t[1:] / t[:-1], 4.0 ** (1 / 7))

    def test_pairing(self):
        assert pairing(0, 4).pairs == ((0, 1), (2, 3))
        assert pairing(1, 4).pairs == ((1, 2),)
        assert pairing(7, 5).pairs == ((1, 2), (3, 4))
        assert pairing(0, 1).pairs == ()
        with pytest.raises(ValueError):
            pairing(-1, 4)

    def test_swap_probability_identities(self):
        rs = np.random.default_rng(0)
        for _ in range(200):
            bi, bj = rs.uniform(0.2, 1.0, 2)
            ei, ej = rs.uniform(-2000, 0, 2)
            p = swap_probability(bi, bj, ei, ej)
            q = swap_probability(bi, bj, ej, ei)  # x -> -x
            assert 0.0 <= p <= 1.0 and math.isclose(p + q, 1.0, rel_tol=0, abs_tol=1e-12)
        assert swap_probability(1.0, 0.5, -1e6, 0.0) == 0.0
        assert swap_probability(1.0, 0.5, 1e6, 0.0) == 1.0


class TestLatticeHelpers:  # reference tests/test_lattice.py:37-98
    def test_hand_energies(self):
        up = SpinLattice(np.ones((3, 3), dtype=np.int8))
        assert total_energy(up, IsingParams(1.0, 0.0)) == -18
        assert total_energy(up, IsingParams(-1.0, 0.0)) == 18
        chk = SpinLattice(np.array([[1, -1], [-1, 1]], dtype=np.int8))
        assert total_energy(chk, IsingParams(1.0, 0.0)) == 8
        assert flip_delta(up, (1, 1), IsingParams(1.0, 0.0)) == 8.0
        assert magnetization_fraction(up) == 1.0

    def test_flip_delta_equals_recompute(self):
        rs = np.random.default_rng(1)
        p = IsingParams(1.0, 0.5)
        for _ in range(50):
            L = int(rs.integers(2, 7))
            a = SpinLattice((rs.integers(0, 2, (L, L)) * 2 - 1).astype(np.int8))
            r, c = (int(x) for x in rs.integers(0, L, 2))
            b = a.copy()
            b.spins[r, c] *= -1
            assert flip_delta(a, (r, c), p) == total_energy(b, p) - total_energy(a, p)


class TestConfigValidation:  # reference tests/test_executor.py:217-224
    def test_rejected_before_any_work(self):
        base = dict(side=8, replicas=5, iterations=3000, swap_interval=37, workers=1, seed=7)
        for field, value in [("workers", 0), ("replicas", 0), ("iterations", 0), ("side", 1),
                             ("swap_interval", -1), ("init_up_fraction", 1.5),
                             ("record_mode", "bogus"), ("sweep_mode", "bogus")]:
            with pytest.raises(ConfigurationError) as err:
                SimulationConfig(**{**base, field: value}).validate()
            assert field.split("_")[0] in str(err.value)

    def test_checkerboard_constraints(self):
        ok = SimulationConfig(side=8, replicas=2, iterations=64 * 10, swap_interval=64,
                              sweep_mode="checkerboard")
        ok.validate()
        for kw in [dict(side=7, iterations=49, swap_interval=0),
                   dict(side=8, iterations=100, swap_interval=0),
                   dict(side=8, iterations=640, swap_interval=10)]:
            with pytest.raises(ConfigurationError):
                SimulationConfig(replicas=2, sweep_mode="checkerboard", **kw).validate()

    def test_temperatures_override(self):
        with pytest.raises(ConfigurationError):
            SimulationConfig(replicas=3, temperatures=(1.0, 2.0)).validate()
        with pytest.raises(ConfigurationError):
            SimulationConfig(replicas=2, temperatures=(1.0, -2.0)).validate()
        SimulationConfig(replicas=2, temperatures=(1.0, 2.0)).validate()


class TestTables:
    def test_class_delta_is_reference_expression(self):
        for J, B in [(1.0, 0.0), (0.7, -0.2), (-1.0, 0.5)]:
            for cls in range(10):
                s = 1 if cls >= 5 else -1
                nb = 2 * (cls % 5) - 4
                assert class_delta(cls, J, B) == 2.0 * s * (J * nb - B)  # kernels.py:94
                assert class_delta(cls, J, B) == oracle.class_delta(cls, J, B)

    def test_exact_tables_are_libm_exp(self):
        betas = 1.0 / build_ladder(16)
        tbl, dcls = exact_tables(betas, 1.0, 0.3)
        for k, b in enumerate(betas):
            for c in range(10):
                if dcls[c] > 0:
                    assert tbl[k, c] == math.exp(-b * dcls[c])  # kernels.py:98

    @pytest.mark.parametrize("J,B", [(1.0, 0.0), (1.0, 0.25), (-1.0, 0.0), (0.5, -1.0)])
    def test_cb_tables_match_oracle(self, J, B):
        betas = 1.0 / build_ladder(9)
        thr, always = cb_tables(betas, J, B)
        othr, oalways = oracle.cb_tables(betas, J, B)
        assert np.array_equal(thr, othr) and (always & 0x3FF) == oalways
        assert bool(always >> 16) == (B == 0.0)
        # threshold/2^32 approximates exp(-beta dE) from below within 2^-32
        for k, b in enumerate(betas):
            for c in range(10):
                if not (always >> c) & 1:
                    d = class_delta(c, J, B)
                    p = 0.5 if d == 0.0 else math.exp(-b * d)
                    assert 0 <= p - thr[k, c] / 2 ** 32 < 2 ** -32 + 1e-18

    def test_ferro_zero_field_always_mask(self):
        # the fast-path selector in csrc/checkerboard.cu expects classes 3..6 (k <= 1)
        _, always = cb_tables(1.0 / build_ladder(4), 1.0, 0.0)
        assert always == (1 << 16) | 0x078
