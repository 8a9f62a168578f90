"""Host-built acceptance tables (the only place exp() of dE is evaluated).

The reference evaluates ``math.exp(-beta * d)`` per attempt with the host
libm (kernels.py:98).  Both GPU chains look the value up instead:

* exact chain:  tbl[k, c] = math.exp(-beta_k * d_c), compared against the
  FP64 uniform exactly as the reference compares it;
* checkerboard: thr[k, c] = floor(math.exp(-beta_k * d_c) * 2^32), compared
  against a 32-bit uniform; dE < 0 always accepted, dE == 0 accepted with
  probability 1/2 (threshold 2^31) -- DESIGN.md section 3.2.

Python's math.exp is the host libm exp numba's math.exp lowers to, so the
tables reproduce the reference's acceptance decisions bit for bit.
"""

from __future__ import annotations

import math

import numpy as np

N_CLASSES = 10
SYMMETRIC_FLAG = 1 << 16


def class_delta(cls: int, J: float, B: float) -> float:
    """dE of class cls = 5*(s>0) + (nb+4)/2, spelled as kernels.py:94."""
    s = 1 if cls >= 5 else -1
    nb = 2 * (cls % 5) - 4
    return 2.0 * s * (J * nb - B)


def exact_tables(betas: np.ndarray, J: float, B: float) -> tuple[np.ndarray, np.ndarray]:
    dcls = np.array([class_delta(c, J, B) for c in range(N_CLASSES)], dtype=np.float64)
    tbl = np.ones((len(betas), N_CLASSES), dtype=np.float64)
    for k, beta in enumerate(np.asarray(betas, dtype=np.float64)):
        for c in range(N_CLASSES):
            if dcls[c] > 0.0:
                tbl[k, c] = math.exp(-float(beta) * float(dcls[c]))
    return tbl, dcls


def cb_tables(betas: np.ndarray, J: float, B: float) -> tuple[np.ndarray, int]:
    thr = np.full((len(betas), N_CLASSES), 0xFFFFFFFF, dtype=np.uint32)
    always = 0
    for c in range(N_CLASSES):
        d = class_delta(c, J, B)
        if d < 0.0:
            always |= 1 << c
            continue
        if d == 0.0:  # neutral: probability 1/2 keeps the checkerboard chain irreducible
            thr[:, c] = 0x80000000
            continue
        for k, beta in enumerate(np.asarray(betas, dtype=np.float64)):
            p = math.exp(-float(beta) * d)
            thr[k, c] = min(int(p * 4294967296.0), 0xFFFFFFFF)
    if B == 0.0:
        always |= SYMMETRIC_FLAG  # thresholds depend on the aligned count only
    return thr, always


def integer_energy_ok(J: float, B: float, energies) -> bool:
    """True when every energy increment is an integer, so FP64 sums are exact
    in any order (|values| far below 2^53)."""
    vals = [J, B] + [float(e) for e in np.asarray(energies).ravel()]
    return all(math.isfinite(v) and float(v).is_integer() and abs(v) < 1e15 for v in vals) \
        and abs(J) <= 1e6 and abs(B) <= 1e6
