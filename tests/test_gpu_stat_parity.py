"""Mode F vs Mode E with seed-to-seed error bars at the BASELINE lattice
sizes L = 64 (C5) and L = 256 (C2): |mean_F - mean_E| < 4 sigma for E/L^2 and
|m| in every temperature slot (tests/stat_parity.py; the committed table is
profiles/r2_stat_parity.json)."""

import numpy as np
import pytest

from stat_parity import CASES, Z_MAX, parity_table

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"L{c[0]}")
def test_checkerboard_and_exact_chain_agree_within_error_bars(case):
    (res,) = parity_table((case,))
    for s in res["slots"]:
        for obs in ("e_per_site", "abs_m"):
            d = s[obs]
            assert abs(d["z"]) < Z_MAX, (res["L"], s["T"], obs, d)
            assert np.isfinite(d["exact_se"]) and np.isfinite(d["checkerboard_se"])


def test_exact_record_every_keeps_reference_columns():
    """record_every = k on the exact chain keeps the reference's columns
    (c+1)k - 1 bit for bit (the statistical runs above rely on it)."""
    from paper_2512_03825_b200 import SimulationConfig, run
    base = dict(side=8, replicas=5, iterations=3000, swap_interval=37, workers=1, seed=7, device=0)
    full = run(SimulationConfig(**base))
    for k in (1, 37, 64, 100):
        sub = run(SimulationConfig(record_every=k, **base))
        assert np.array_equal(sub.energies, full.energies[:, k - 1::k][:, : 3000 // k])
        assert np.array_equal(sub.magnetizations, full.magnetizations[:, k - 1::k][:, : 3000 // k])
        assert (sub.swaps_accepted, sub.swap_rounds) == (full.swaps_accepted, full.swap_rounds)
        assert np.array_equal(sub.round_entry_iterations, full.round_entry_iterations)
