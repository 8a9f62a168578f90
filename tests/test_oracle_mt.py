"""The multi-threaded oracle drivers (oracle/ptmh_oracle.c or_*_mt) equal the
single-threaded restatements they batch: the headline-shape parity tests
(tests/test_gpu_headline.py) lean on them, so they are pinned here on CPU."""

import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("L,R,J,B,threads", [(6, 3, 1.0, 0.0, 2), (10, 4, 1.0, 0.5, 3),
                                             (34, 5, -0.7, 0.3, 4), (64, 6, 1.0, 0.0, 3),
                                             (128, 3, 1.0, 0.0, 8), (2, 4, 1.0, 0.0, 2)])
def test_cb_sweep_mt_equals_cb_sweep(L, R, J, B, threads):
    sp = np.empty((R, L, L), dtype=np.int8)
    oracle.fill_lattices_mt(sp, (L * L) // 2, 11, threads=threads)
    ref = np.empty_like(sp)
    for r in range(R):
        oracle.fill_lattice(ref[r], (L * L) // 2, 11, r, 0)
    assert np.array_equal(sp, ref)
    temps = 1.0 + 3.0 * np.arange(R) / R
    thr, always = oracle.cb_tables(1.0 / temps, J, B)
    a, b = sp.copy(), sp.copy()
    sa, sb = oracle.row_stats(a), oracle.row_stats_mt(b, threads)
    assert np.array_equal(sa, sb)
    r2s = np.random.default_rng(L).permutation(R).astype(np.int64)
    for t in range(6):
        oracle.cb_sweep(a, r2s, thr, always, 2 ** 40 + 9, t, sa)
        oracle.cb_sweep_mt(b, r2s, thr, always, 2 ** 40 + 9, t, sb, threads)
    assert np.array_equal(a, b)
    assert np.array_equal(sa, sb)
    assert np.array_equal(sb, oracle.row_stats(b))
