"""The reference's kernel boundary, GPU-backed (isingpt/kernels.py).

Same names, signatures, dtypes and in-place semantics as the numba kernels
the reference executor calls as module attributes (executor.py:23,204-206,
218-220,241-245,258-260).  Each call goes through the host-buffer C ABI
(include/ptmh.h, ptmh_host_*): the caller's numpy arrays are copied to the
GPU, the CUDA kernel runs, results are copied back.  A user can therefore
install these functions as ``isingpt.kernels.<name>``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

MASK64 = (1 << 64) - 1


def _p(a: np.ndarray, dtype) -> ctypes.c_void_p:
    if a.dtype != np.dtype(dtype) or not a.flags.c_contiguous:
        raise TypeError(f"expected a C-contiguous {np.dtype(dtype)} array, got "
                        f"{a.dtype} (contiguous={a.flags.c_contiguous})")
    return a.ctypes.data_as(ctypes.c_void_p)


def fill_lattice(out: np.ndarray, up_count: int, seed, stream, position) -> np.uint64:
    """kernels.py:26-45; returns the new stream position."""
    newpos = ctypes.c_uint64(0)
    _lib.check(_lib.LIB.ptmh_host_fill_lattice(_p(out, np.int8), out.size, int(up_count),
                                               int(seed) & MASK64, int(stream) & MASK64,
                                               int(position) & MASK64, ctypes.byref(newpos)),
               "fill_lattice")
    return np.uint64(newpos.value)


def lattice_energy(spins: np.ndarray, J: float, B: float) -> float:
    """kernels.py:48-59."""
    if spins.ndim != 2 or spins.shape[0] != spins.shape[1]:
        raise ValueError("spins must be a square 2D array")
    e = ctypes.c_double(0.0)
    _lib.check(_lib.LIB.ptmh_host_lattice_energy(_p(spins, np.int8), spins.shape[0], float(J),
                                                 float(B), ctypes.byref(e)), "lattice_energy")
    return e.value


def advance_block(spins, slot_to_row, lo, hi, betas, J, B, energies, spin_sums, positions,
                  iters_done, seed, start_iter, nsteps, obs_e, obs_m, record, states) -> None:
    """kernels.py:62-113 (record 0/1/2; obs and states as the reference passes them)."""
    record = int(record)
    R = slot_to_row.shape[0]
    ncols = obs_e.shape[1] if record >= 1 else 0
    _lib.check(_lib.LIB.ptmh_host_advance_block(
        _p(spins, np.int8), spins.shape[0], spins.shape[1], _p(slot_to_row, np.int64), R,
        int(lo), int(hi), _p(betas, np.float64), float(J), float(B), _p(energies, np.float64),
        _p(spin_sums, np.int64), _p(positions, np.uint64), _p(iters_done, np.int64),
        int(seed) & MASK64, int(start_iter), int(nsteps),
        _p(obs_e, np.float64) if record >= 1 else None,
        _p(obs_m, np.float64) if record >= 1 else None, ncols, record,
        _p(states, np.int8) if record == 2 else None), "advance_block")


def swap_chunk(slot_to_row, energies, spin_sums, betas, seed, stream_base, round_index, first,
               pair_lo, pair_hi) -> int:
    """kernels.py:116-148; returns the accepted count."""
    acc = ctypes.c_int64(0)
    _lib.check(_lib.LIB.ptmh_host_swap_chunk(
        _p(slot_to_row, np.int64), _p(energies, np.float64), _p(spin_sums, np.int64),
        _p(betas, np.float64), slot_to_row.shape[0], int(seed) & MASK64, int(stream_base),
        int(round_index), int(first), int(pair_lo), int(pair_hi), ctypes.byref(acc)),
        "swap_chunk")
    return int(acc.value)


def cb_interval(spins, slot_to_row, betas, J, B, seed, first_sweep, n_sweeps, round_index,
                energies, spin_sums) -> int:
    """Mode F plugin call on host lattices: n_sweeps checkerboard sweeps then
    (round_index >= 0) one swap round; returns the accepted count.  spins
    (R, L, L) int8 and slot_to_row (R,) int64 are updated in place, energies /
    spin_sums (R,) receive the by-slot values after the round."""
    acc = ctypes.c_int64(0)
    R, L = spins.shape[0], spins.shape[1]
    _lib.check(_lib.LIB.ptmh_host_cb_interval(
        _p(spins, np.int8), R, L, _p(slot_to_row, np.int64), _p(betas, np.float64), float(J),
        float(B), int(seed) & MASK64, int(first_sweep), int(n_sweeps), int(round_index),
        _p(energies, np.float64), _p(spin_sums, np.int64), ctypes.byref(acc)), "cb_interval")
    return int(acc.value)


def warm_kernels() -> None:
    """kernels.py:151-168: one tiny call of every kernel (module load and
    CUDA context creation happen here, not in a timed run)."""
    spins = np.empty((1, 2, 2), dtype=np.int8)
    fill_lattice(spins[0], 2, 0, 0, 0)
    lattice_energy(spins[0], 1.0, 0.0)
    slot_to_row = np.arange(1, dtype=np.int64)
    betas = np.ones(1)
    energies = np.array([lattice_energy(spins[0], 1.0, 0.0)])
    sums = np.array([int(spins[0].sum())], dtype=np.int64)
    positions = np.zeros(1, dtype=np.uint64)
    iters = np.zeros(1, dtype=np.int64)
    obs = np.zeros((1, 2))
    states = np.empty((1, 2, 2, 2), dtype=np.int8)
    advance_block(spins, slot_to_row, 0, 1, betas, 1.0, 0.0, energies, sums, positions, iters,
                  0, 0, 2, obs, obs.copy(), 2, states)
    swap_chunk(slot_to_row, energies, sums, betas, 0, 1, 0, 0, 0, 0)
