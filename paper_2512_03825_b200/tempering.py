"""Temperature ladder, pairing schedule and swap rule (isingpt tempering.py).

Host-side definitions.  The device exchange kernel (csrc/exact.cu
swap_kernel) evaluates the same rule for every pair of a round.
"""

from __future__ import annotations

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
