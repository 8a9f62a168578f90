"""The drop-in API surface (CPU): every name of isingpt.__all__ exists with the
reference's call signature (fixture tests/golden/api.json, written by
tests/golden/make_golden.py from the reference itself), and the host-side
post-run analysis (analysis.py) reproduces the reference's results on the
fixture cases of tests/golden/public_ops.npz.  The GPU-backed per-replica
ops are checked in tests/test_gpu_public_api.py."""

import inspect
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2512_03825_b200 as pkg
from paper_2512_03825_b200 import analysis
from paper_2512_03825_b200.executor import ConfigurationError, SimulationConfig

API = json.load(open(os.path.join(GOLDEN, "api.json")))
OPS = np.load(os.path.join(GOLDEN, "public_ops.npz"))


def test_all_reference_names_exported():
    missing = sorted(set(API["all"]) - set(pkg.__all__))
    assert not missing, missing
    for name in API["all"]:
        assert hasattr(pkg, name), name


@pytest.mark.parametrize("name", sorted(API["signatures"]))
def test_signature_matches_reference(name):
    ref = API["signatures"][name]
    if ref is None:
        return
    ours = [[p.name, str(p.kind), None if p.default is inspect.Parameter.empty else repr(p.default)]
            for p in inspect.signature(getattr(pkg, name)).parameters.values()]
    # the reference's parameters, in order, with the same kinds and defaults;
    # extensions only after them and only with defaults
    assert ours[: len(ref)] == ref, (name, ours, ref)
    assert all(p[2] is not None for p in ours[len(ref):]), (name, ours[len(ref):])


def test_replica_validation_and_beta():
    from paper_2512_03825_b200 import IsingParams, Replica, RngStream, SpinLattice
    lat = SpinLattice(np.ones((2, 2), dtype=np.int8))
    r = Replica(lat, 2.0, -8.0, RngStream(1, 0), 0)
    assert r.beta == 0.5
    assert r.energy_drift(IsingParams()) == 0.0
    with pytest.raises(ValueError):
        Replica(lat, 0.0, 0.0, RngStream(1, 0), 0)
    with pytest.raises(ValueError):
        Replica(lat, 1.0, 0.0, RngStream(1, 0), -1)


def test_rng_stream_masks_like_reference():
    from paper_2512_03825_b200 import RngStream, SwapRng
    s = RngStream(-1, 2 ** 64 + 3, 7)
    assert (s.master_seed, s.stream_id, s.position) == (2 ** 64 - 1, 3, 7)
    assert repr(s) == "RngStream(master_seed=18446744073709551615, stream_id=3, position=7)"
    w = SwapRng(2 ** 65 + 2, 9)
    assert (w.master_seed, w.replica_count) == (2, 9)


def test_acceptance_probability_identities():
    from paper_2512_03825_b200 import acceptance_probability
    assert acceptance_probability(-4.0, 0.5) == 1.0
    assert acceptance_probability(0.0, 3.0) == 1.0
    assert acceptance_probability(8.0, 0.25) == np.exp(-2.0)


def test_convergence_iteration_matches_reference():
    series = OPS["conv_series"]
    got = []
    for w, t in ((100, 0.02), (50, 0.005), (200, 0.05), (10, 1e-6)):
        v = analysis.convergence_iteration(series, analysis.ConvergenceCriterion(window=w, tolerance=t))
        got.append(-1 if v is None else v)
    assert got == OPS["conv_result"].tolist()
    with pytest.raises(ValueError):
        analysis.convergence_iteration(series[:10], analysis.ConvergenceCriterion(window=10))
    with pytest.raises(ValueError):
        analysis.ConvergenceCriterion(window=0)
    with pytest.raises(ValueError):
        analysis.ConvergenceCriterion(tolerance=0.0)
    with pytest.raises(ValueError):
        analysis.ConvergenceCriterion(statistic="energy")


def test_fit_power_law_matches_reference():
    fit = analysis.fit_power_law(OPS["fit_pts"])
    np.testing.assert_allclose([fit.exponent, fit.prefactor, fit.r_squared], OPS["fit"], rtol=1e-12)
    exact = analysis.fit_power_law([[2, 8.0], [4, 32.0], [8, 128.0]])
    assert abs(exact.exponent - 2.0) < 1e-12 and exact.r_squared == 1.0
    for bad in ([[1, 2]], [[1, 2], [2, 3]], [[1, 2], [2, -3], [4, 5]], [1, 2, 3]):
        with pytest.raises(ValueError):
            analysis.fit_power_law(bad)


def test_encode_configurations_matches_reference():
    assert np.array_equal(analysis.encode_configurations(OPS["enc_states"]), OPS["enc_codes"])
    with pytest.raises(ValueError):
        analysis.encode_configurations(np.ones((5, 5), dtype=np.int8))


@pytest.mark.parametrize("side,T,J,B,tag", [(2, 2.0, 1.0, 0.0, "2"), (3, 2.5, 1.0, 0.5, "3"),
                                            (4, 1.7, -0.5, 0.2, "4")])
def test_exact_boltzmann_matches_reference(side, T, J, B, tag):
    p = analysis.exact_boltzmann_distribution(side, T, pkg.IsingParams(J=J, B=B))
    np.testing.assert_allclose(p, OPS[f"boltz_{tag}"], rtol=1e-12, atol=1e-300)
    assert abs(p.sum() - 1.0) < 1e-12
    with pytest.raises(ValueError):
        analysis.exact_boltzmann_distribution(5, 1.0, pkg.IsingParams())
    with pytest.raises(ValueError):
        analysis.exact_boltzmann_distribution(2, 0.0, pkg.IsingParams())


def test_equilibrium_magnetization_matches_reference():
    rec = SimpleNamespace(magnetizations=OPS["eq_mag_m"])
    for frac, key in ((0.5, "eq_mag_05"), (0.0, "eq_mag_0"), (0.9, "eq_mag_09")):
        np.testing.assert_allclose(analysis.equilibrium_magnetization(rec, frac), OPS[key], rtol=1e-14)
    with pytest.raises(ValueError):
        analysis.equilibrium_magnetization(SimpleNamespace(magnetizations=None))
    with pytest.raises(ValueError):
        analysis.equilibrium_magnetization(rec, 1.0)


def test_devices_validation():
    base = dict(side=8, replicas=4, iterations=640, swap_interval=64, sweep_mode="checkerboard")
    for bad in ((), (0, 0), (-1,), (0.5,), tuple(range(9))):
        with pytest.raises(ConfigurationError):
            SimulationConfig(devices=bad, **base).validate()
    with pytest.raises(ConfigurationError):
        SimulationConfig(devices=(0,), device=0, **base).validate()
    with pytest.raises(ConfigurationError):  # the exact chain is single-device
        SimulationConfig(side=8, replicas=4, devices=(0, 1)).validate()
    SimulationConfig(devices=(0, 1), **base).validate()
    SimulationConfig(side=8, replicas=4, devices=(3,)).validate()


def test_multi_device_run_needs_one_process_per_device():
    """devices=(0, 1) without a process group: ConfigurationError before any
    work (no GPU touched; this runs on CPU)."""
    from paper_2512_03825_b200 import run
    cfg = SimulationConfig(side=8, replicas=4, iterations=640, swap_interval=64,
                           sweep_mode="checkerboard", devices=(0, 1))
    with pytest.raises(ConfigurationError, match="torchrun"):
        run(cfg)
