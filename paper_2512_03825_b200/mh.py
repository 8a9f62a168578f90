"""Per-replica Metropolis-Hastings API of the reference (isingpt mh.py), GPU-backed.

``mh_step`` is the reference's spec-level definition of one attempt
(mh.py:73-88): draw a site, draw an acceptance uniform, flip with
probability min(1, exp(-beta dE)).  Here it runs as a one-slot
``advance_block`` on the device (csrc/exact.cu advance_kernel through
``ptmh_host_mh_steps``), with the replica's own stream id, so a loop of
``mh_step`` calls is bit-identical to the fused kernel the engine runs
(tests/test_gpu_public_api.py).  The replica object stays on the host, as
in the reference.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .lattice import IsingParams, SpinLattice, init_lattice, total_energy
from .rng import MASK64, RngStream


@dataclass
class Replica:
    """One chain: lattice, temperature, cached energy and private stream (mh.py:21-45).

    ``beta`` = 1/temperature is derived at construction; ``energy`` is kept
    current by :func:`mh_step`.
    """

    lattice: SpinLattice
    temperature: float
    energy: float
    rng: RngStream
    replica_index: int
    beta: float = field(init=False)

    def __post_init__(self):
        if not self.temperature > 0:
            raise ValueError(f"temperature must be positive, got {self.temperature}")
        if self.replica_index < 0:
            raise ValueError("replica_index must be >= 0")
        self.beta = 1.0 / self.temperature

    def energy_drift(self, params: IsingParams) -> float:
        """Cached energy minus a full recomputation (0 when consistent)."""
        return self.energy - total_energy(self.lattice, params)


def make_replica(side: int, up_fraction: float, temperature: float, master_seed: int,
                 replica_index: int, params: IsingParams) -> Replica:
    """Replica with stream id = replica_index, exact-count initial lattice
    (mh.py:48-56; the lattice is drawn on the device, lattice.init_lattice)."""
    stream = RngStream(master_seed, replica_index)
    lat = init_lattice(side, up_fraction, stream)
    return Replica(lattice=lat, temperature=temperature, energy=total_energy(lat, params),
                   rng=stream, replica_index=replica_index)


def propose(replica: Replica) -> tuple[int, int]:
    """Uniform trial site (row, col) from one draw (mh.py:59-63)."""
    side = replica.lattice.side
    k = replica.rng.choose(side * side)
    return divmod(k, side)


def acceptance_probability(delta_energy: float, beta: float) -> float:
    """min(1, exp(-beta dE)) (mh.py:66-70)."""
    return 1.0 if delta_energy <= 0.0 else math.exp(-beta * delta_energy)


def _advance(replica: Replica, params: IsingParams, nsteps: int) -> tuple[int, int]:
    spins = replica.lattice.spins
    if spins.dtype != np.int8 or not spins.flags.c_contiguous:
        raise TypeError("replica lattice must be a C-contiguous int8 array")
    before = int(spins.sum(dtype=np.int64))
    energy = ctypes.c_double(float(replica.energy))
    ssum = ctypes.c_int64(before)
    pos = ctypes.c_uint64(int(replica.rng.position) & MASK64)
    _lib.call("ptmh_host_mh_steps", spins.ctypes.data_as(ctypes.c_void_p), spins.shape[0],
              float(replica.beta), float(params.J), float(params.B), ctypes.byref(energy),
              ctypes.byref(ssum), replica.rng.master_seed, replica.rng.stream_id,
              ctypes.byref(pos), int(nsteps))
    replica.energy = energy.value
    replica.rng.position = int(pos.value)
    return before, int(ssum.value)


def mh_step(replica: Replica, params: IsingParams) -> bool:
    """One MH iteration (mh.py:73-88); True if the flip was accepted.

    Consumes exactly two draws (site, then acceptance uniform).  A flip
    always changes the spin sum by +-2, which is how acceptance is read back.
    """
    before, after = _advance(replica, params, 1)
    return after != before


def mh_steps(replica: Replica, params: IsingParams, nsteps: int) -> None:
    """Extension: ``nsteps`` consecutive mh_step calls in one device call."""
    if nsteps < 0:
        raise ValueError(f"nsteps must be >= 0, got {nsteps}")
    _advance(replica, params, nsteps)
