"""The Mode F chain definition itself (CPU): the synchronous checkerboard
kernel P0*P1 with the reference's Metropolis acceptance for dE != 0 and
probability 1/2 for dE == 0 has the Boltzmann distribution as its unique
stationary distribution (exact transition matrix at L=2), while acceptance 1
for dE == 0 (the reference's random-site value) makes it reducible -- the
reason for the 1/2.  Plus oracle runs vs enumeration."""

import itertools
import math

import numpy as np
import pytest

import oracle


def _kernel(L, T, neutral):
    n = L * L
    states = list(itertools.product([-1, 1], repeat=n))
    index = {s: i for i, s in enumerate(states)}

    def half(color):
        P = np.zeros((2 ** n, 2 ** n))
        for si, s in enumerate(states):
            a = np.array(s).reshape(L, L)
            cs = [(r, c) for r in range(L) for c in range(L) if (r + c) % 2 == color]
            probs = []
            for r, c in cs:
                nb = a[(r + 1) % L, c] + a[(r - 1) % L, c] + a[r, (c + 1) % L] + a[r, (c - 1) % L]
                d = 2.0 * a[r, c] * nb
                probs.append(1.0 if d < 0 else (neutral if d == 0 else math.exp(-d / T)))
            for flips in itertools.product([0, 1], repeat=len(cs)):
                b = a.copy()
                p = 1.0
                for f, (r, c), q in zip(flips, cs, probs):
                    p *= q if f else 1 - q
                    if f:
                        b[r, c] = -b[r, c]
                if p:
                    P[si, index[tuple(b.ravel())]] += p
        return P

    E = np.array([-sum(np.array(s).reshape(L, L)[r, c] * (np.array(s).reshape(L, L)[(r + 1) % L, c]
                                                         + np.array(s).reshape(L, L)[r, (c + 1) % L])
                       for r in range(L) for c in range(L)) for s in states], dtype=float)
    w = np.exp(-(E - E.min()) / T)
    return half(0) @ half(1), w / w.sum()


@pytest.mark.parametrize("T", [1.0, 2.5])
def test_neutral_half_gives_unique_boltzmann_stationary_state(T):
    P, pi = _kernel(2, T, 0.5)
    assert np.allclose(pi @ P, pi, atol=1e-14)           # invariance
    ev = np.sort(np.abs(np.linalg.eigvals(P)))[::-1]
    assert ev[1] < 1 - 1e-6                                # unique, aperiodic


@pytest.mark.parametrize("T", [1.0, 2.5])
def test_neutral_one_is_reducible(T):
    P, pi = _kernel(2, T, 1.0)
    assert np.allclose(pi @ P, pi, atol=1e-14)           # still invariant ...
    ev = np.sort(np.abs(np.linalg.eigvals(P)))[::-1]
    assert ev[2] > 1 - 1e-9                                # ... but not the only limit


@pytest.mark.parametrize("L,T,tol", [(2, 1.0, 0.005), (2, 2.5, 0.005), (4, 2.5, 0.01)])
def test_oracle_chain_energy_marginal(L, T, tol):
    sweeps = 200_000
    rec = oracle.run_checkerboard(L, 2, sweeps, 0, 11, temperatures=[T, T + 1.0], record=True)
    n = L * L
    codes = np.arange(1 << n, dtype=np.int64)
    s = 2 * ((codes[:, None] >> np.arange(n)) & 1) - 1
    right = [r * L + (c + 1) % L for r in range(L) for c in range(L)]
    down = [((r + 1) % L) * L + c for r in range(L) for c in range(L)]
    E = -((s * s[:, right]).sum(1) + (s * s[:, down]).sum(1))
    w = np.exp(-(E - E.min()) / T)
    w /= w.sum()
    e = rec.energies[0, sweeps // 10:]
    lv = np.unique(E)
    tv = 0.5 * sum(abs((e == x).mean() - w[E == x].sum()) for x in lv)
    assert tv < tol
