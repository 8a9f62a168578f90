"""Distributional checks on the GPU (reference tests/test_sampling.py,
tests/test_acceptance.py): both chains sample the Boltzmann distribution.

* exact chain: state marginal at L=3, T=2.5 vs full enumeration (TV < 0.02,
  test_acceptance.py:35-56);
* checkerboard chain: energy-level marginal of every slot vs enumeration at
  L=2 and L=4 under frequent exchanges (TV < 0.01 / 0.02,
  test_sampling.py:48-84 thresholds);
* checkerboard vs exact chain: <E> and <|m|> per temperature agree within
  5 combined standard errors (batch means) at L=16;
* phase transition at L=32 (test_acceptance.py:59-102 thresholds).
"""

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def exact_levels(L, T, J=1.0, B=0.0):
    """Energy levels and their Boltzmann weights by full enumeration
    (analysis.py:126-151 restated)."""
    n = L * L
    codes = np.arange(1 << n, dtype=np.int64)
    s = 2 * ((codes[:, None] >> np.arange(n)) & 1) - 1
    right = np.array([r * L + (c + 1) % L for r in range(L) for c in range(L)])
    down = np.array([((r + 1) % L) * L + c for r in range(L) for c in range(L)])
    bond = (s * s[:, right]).sum(1) + (s * s[:, down]).sum(1)
    E = B * s.sum(1) - J * bond
    w = np.exp(-(E - E.min()) / T)
    w /= w.sum()
    lv = np.unique(E)
    return lv, np.array([w[E == e].sum() for e in lv]), E, w


def tv(p, q):
    return 0.5 * float(np.abs(p - q).sum())


@pytest.fixture(scope="module")
def p():
    import paper_2512_03825_b200 as p
    return p


def test_exact_chain_state_distribution_L3(p):
    cfg = p.SimulationConfig(side=3, replicas=2, iterations=1_000_000, swap_interval=0, seed=42,
                             record_mode="full_states")
    rec = p.run(cfg)
    assert float(rec.temperatures[1]) == 2.5
    st = rec.states[1].reshape(-1, 9)
    codes = ((st > 0).astype(np.int64) << np.arange(9)).sum(1)
    emp = np.bincount(codes, minlength=512) / codes.size
    _, _, _, w = exact_levels(3, 2.5)
    assert tv(emp, w) < 0.02


@pytest.mark.parametrize("L,sweeps,every,tol", [(2, 400_000, 1, 0.01), (2, 400_000, 10, 0.01),
                                                (4, 200_000, 5, 0.02)])
def test_checkerboard_energy_marginals_under_swaps(p, L, sweeps, every, tol):
    R = 4
    cfg = p.SimulationConfig(side=L, replicas=R, iterations=sweeps * L * L,
                             swap_interval=every * L * L, seed=4, sweep_mode="checkerboard")
    rec = p.run(cfg)
    assert rec.swaps_accepted > 0
    burn = sweeps // 10
    for slot, T in enumerate(rec.temperatures):
        lv, pw, _, _ = exact_levels(L, float(T))
        e = rec.energies[slot, burn:]
        emp = np.array([(e == x).mean() for x in lv])
        assert abs(emp.sum() - 1.0) < 1e-12  # every sample is a valid level
        assert tv(emp, pw) < tol, (slot, T, tv(emp, pw))


def _batch_se(x, nb=50):
    b = x[: len(x) // nb * nb].reshape(nb, -1).mean(1)
    return b.mean(), b.std(ddof=1) / np.sqrt(nb)


def test_checkerboard_agrees_with_exact_chain(p):
    L, R = 16, 6
    n_sweeps = 20_000
    temps = (1.5, 2.0, 2.27, 2.5, 3.0, 3.5)
    cb = p.run(p.SimulationConfig(side=L, replicas=R, iterations=n_sweeps * L * L,
                                  swap_interval=L * L, seed=1, temperatures=temps,
                                  sweep_mode="checkerboard"))
    ex = p.run(p.SimulationConfig(side=L, replicas=R, iterations=n_sweeps * L * L // 4,
                                  swap_interval=L * L, seed=2, temperatures=temps))
    ex_e = ex.energies[:, L * L - 1::L * L]  # one sample per sweep
    ex_m = ex.magnetizations[:, L * L - 1::L * L]
    for k in range(R):
        for a, b in [(cb.energies[k, 2000:], ex_e[k, 500:]),
                     (np.abs(cb.magnetizations[k, 2000:]), np.abs(ex_m[k, 500:]))]:
            ma, sa = _batch_se(a)
            mb, sb = _batch_se(b)
            assert abs(ma - mb) < 5 * np.hypot(sa, sb) + 1e-9, (k, ma, mb, sa, sb)


def test_checkerboard_phase_transition(p):
    L, R = 32, 16
    rec = p.run(p.SimulationConfig(side=L, replicas=R, iterations=4000 * L * L,
                                   swap_interval=L * L, seed=3, sweep_mode="checkerboard"))
    temps = rec.temperatures
    mags = np.abs(rec.magnetizations[:, 2000:]).mean(1)
    assert np.all(mags[temps <= 1.5] > 0.9)
    assert np.all(mags[temps >= 3.5] < 0.3)
    k = int(np.argmax(mags[:-1] - mags[1:]))
    assert temps[k] >= 2.0 and temps[k + 1] <= 2.6


def test_checkerboard_state_marginal_L2(p):
    """reference tests/test_sampling.py:48-57 for the checkerboard chain: the
    full-state marginal of slot 1 (T = 2.5) vs exact enumeration."""
    sweeps = 200_000
    rec = p.run(p.SimulationConfig(side=2, replicas=2, iterations=sweeps * 4, swap_interval=0,
                                   seed=11, sweep_mode="checkerboard", record_mode="full_states"))
    st = rec.states[1].reshape(-1, 4)
    codes = ((st > 0).astype(np.int64) << np.arange(4)).sum(1)
    emp = np.bincount(codes, minlength=16) / codes.size
    _, _, _, w = exact_levels(2, 2.5)
    assert tv(emp, w) < 0.01
