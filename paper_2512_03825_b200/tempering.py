"""Temperature ladder, pairing schedule and swap rule (isingpt tempering.py).

``build_ladder``, ``pairing`` and ``swap_probability`` are the reference's
host-side definitions.  The sampling loop's exchange is the device kernel
csrc/exact.cu swap_kernel; ``execute_swap_round`` (the per-replica API)
decides its pairs with the same device rule (swap_pairs_kernel).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np


def build_ladder(replica_count: int) -> np.ndarray:
    """T_i = 1 + 3 i / R (tempering.py:22-27)."""
    if replica_count < 1:
        raise ValueError(f"replica_count must be >= 1, got {replica_count}")
    i = np.arange(replica_count, dtype=np.float64)
    return 1.0 + i * 3.0 / replica_count


def geometric_ladder(replica_count: int, t_min: float = 1.0, t_max: float = 4.0) -> np.ndarray:
    """T_i = t_min * (t_max/t_min)^(i/(R-1)): the "geometric T-ladder" of
    BASELINE.json config C1 (an extension; the reference ladder is linear)."""
    if replica_count < 1:
        raise ValueError(f"replica_count must be >= 1, got {replica_count}")
    if replica_count == 1:
        return np.array([t_min], dtype=np.float64)
    i = np.arange(replica_count, dtype=np.float64)
    return t_min * (t_max / t_min) ** (i / (replica_count - 1))


@dataclass(frozen=True)
class SwapRound:
    """Pairs of one round (tempering.py:30-36)."""

    round_index: int
    parity: str
    pairs: tuple[tuple[int, int], ...]


def pairing(round_index: int, replica_count: int) -> SwapRound:
    """(0,1)(2,3).. on even rounds, (1,2)(3,4).. on odd ones (tempering.py:39-50)."""
    if round_index < 0:
        raise ValueError("round_index must be >= 0")
    first = round_index % 2
    pairs = tuple((i, i + 1) for i in range(first, replica_count - 1, 2))
    return SwapRound(round_index=round_index, parity="odd" if first else "even", pairs=pairs)


def swap_probability(beta_i: float, beta_j: float, energy_i: float, energy_j: float) -> float:
    """Saturating logistic of (b_i - b_j)(E_i - E_j) (tempering.py:53-65)."""
    x = (beta_i - beta_j) * (energy_i - energy_j)
    if x >= 0.0:
        return 1.0 / (1.0 + math.exp(-x))
    ex = math.exp(x)
    return ex / (1.0 + ex)


def execute_swap_round(replicas, swap_round: SwapRound, swap_rng) -> int:
    """Decide every pair of ``swap_round`` independently; returns the accepted
    count (tempering.py:68-86).

    Pair k draws ``swap_rng.pair_uniform(round_index, k)``; an accepted pair
    exchanges the two replicas' lattices and cached energies, while
    temperatures and streams stay with their slots.  The decisions are made
    on the device (``ptmh_host_swap_pairs``) by the exchange kernels' rule.
    """
    from . import _lib

    pairs = swap_round.pairs
    if not pairs:
        return 0
    pi = np.ascontiguousarray([i for i, _ in pairs], dtype=np.int64)
    pj = np.ascontiguousarray([j for _, j in pairs], dtype=np.int64)
    betas = np.ascontiguousarray([r.beta for r in replicas], dtype=np.float64)
    energies = np.ascontiguousarray([r.energy for r in replicas], dtype=np.float64)
    accept = np.zeros(len(pairs), dtype=np.uint8)
    ties = ctypes.c_int64(0)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.call("ptmh_host_swap_pairs", vp(pi), vp(pj), len(pairs), vp(betas), vp(energies),
              len(replicas), swap_rng.master_seed, swap_rng.replica_count,
              int(swap_round.round_index), vp(accept), ctypes.byref(ties))
    for (i, j), ok in zip(pairs, accept):
        if ok:
            a, b = replicas[i], replicas[j]
            a.lattice, b.lattice = b.lattice, a.lattice
            a.energy, b.energy = b.energy, a.energy
    return int(accept.sum())
