"""Counter-based random streams of the reference (isingpt rng.py), drawn on the GPU.

A draw is addressed by (master seed, stream id, position) and is word 0 of
Philox4x64-10 at counter (position, 0, stream, 0), key (seed, stream),
mapped to [0, 1) as (w >> 11) * 2^-53 (rng.py:40-67).  Stream ids 0..R-1
belong to the temperature slots, ids R, R+1, ... to the swap pairs
(rng.py:99-116).

The objects below keep the reference's host-side bookkeeping (the stream
position); every draw is computed by the device Philox (csrc/philox.cuh,
``ptmh_host_uniforms``), the same code the sampling kernels inline.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

MASK64 = 0xFFFFFFFFFFFFFFFF


def uniforms(seed: int, stream: int, position: int, n: int) -> np.ndarray:
    """The n consecutive uniforms of one stream from ``position`` on (float64)."""
    n = int(n)
    if n < 0:
        raise ValueError(f"n must be >= 0, got {n}")
    out = np.empty(n, dtype=np.float64)
    if n:
        _lib.call("ptmh_host_uniforms", int(seed) & MASK64, int(stream) & MASK64,
                  int(position) & MASK64, n, out.ctypes.data_as(ctypes.c_void_p))
    return out


def stream_uniform(seed, stream, position) -> float:
    """Uniform double in [0, 1) for the draw at (seed, stream, position) (rng.py:64-67)."""
    return float(uniforms(seed, stream, position, 1)[0])


class RngStream:
    """One random stream whose ``position`` counts the draws consumed (rng.py:70-96).

    Distinct (master_seed, stream_id) pairs are independent streams; the same
    pair replays the same sequence.
    """

    __slots__ = ("master_seed", "stream_id", "position")

    def __init__(self, master_seed: int, stream_id: int, position: int = 0):
        self.master_seed = int(master_seed) & MASK64
        self.stream_id = int(stream_id) & MASK64
        self.position = int(position)

    def uniform(self) -> float:
        """Next uniform in [0, 1); consumes one draw."""
        return float(self.uniforms(1)[0])

    def uniforms(self, n: int) -> np.ndarray:
        """Next n uniforms in one device call (extension); consumes n draws."""
        out = uniforms(self.master_seed, self.stream_id, self.position, n)
        self.position += int(n)
        return out

    def choose(self, n: int) -> int:
        """Uniform integer in [0, n); consumes one draw."""
        return int(self.uniform() * n)

    def __repr__(self) -> str:
        return (f"RngStream(master_seed={self.master_seed}, "
                f"stream_id={self.stream_id}, position={self.position})")


class SwapRng:
    """One uniform per (round index, pair index): stream replica_count + pair,
    position round index (rng.py:99-116), so swap draws never share a stream
    with a temperature slot."""

    __slots__ = ("master_seed", "replica_count")

    def __init__(self, master_seed: int, replica_count: int):
        self.master_seed = int(master_seed) & MASK64
        self.replica_count = int(replica_count)

    def pair_uniform(self, round_index: int, pair_index: int) -> float:
        return stream_uniform(self.master_seed, self.replica_count + int(pair_index),
                              int(round_index))
