"""Multi-GPU Parallel Tempering: lattices sharded by row, labels replicated.

One process per GPU (torchrun).  Rank g owns the contiguous block of lattice
rows ``assign_replicas(R, G)[g]`` (executor.py:91-102) -- initially a
temperature band -- and never moves a lattice.  Every rank keeps the full
slot_to_row / row_to_slot permutation, the threshold table and betas.

Per exchange round the only data that crosses GPUs is the per-lattice
(sum s, sum bonds) int64 pair: an all_gather of R x 16 bytes over NCCL
(NVLink).  Every rank then runs the identical exchange kernel (reference
swap rule and swap-RNG addresses, kernels.py:116-148) on identical inputs, so
the permutation stays identical everywhere without a second collective.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .executor import assign_replicas


class ShardedCheckerboard:
    """Checkerboard PT over the ranks of ``group``.

    ``engine_cls`` builds the per-rank state (default: the CUDA
    CheckerboardEngine); the CPU tests substitute an oracle-backed engine
    with the same interface to exercise this coordinator over gloo.
    """

    def __init__(self, side, replicas, temperatures, seed, J=1.0, B=0.0, up_fraction=0.5,
                 device=None, group=None, engine_cls=None):
        if engine_cls is None:
            from .engine import CheckerboardEngine as engine_cls
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.bounds = assign_replicas(replicas, self.world)
        lo, hi = self.bounds[self.rank]
        self.eng = engine_cls(side, replicas, temperatures, seed, J, B, up_fraction, device,
                              row_range=(lo, hi))
        self.maxc = max(h - l for l, h in self.bounds)
        dev = self.eng.stats.device
        self._send = torch.zeros((self.maxc, 2), dtype=torch.int64, device=dev)
        self._recv = torch.zeros((self.world * self.maxc, 2), dtype=torch.int64, device=dev)

    def init_state(self) -> None:
        self.eng.init_state()
        self.gather_stats()

    def gather_stats(self) -> None:
        """All lattices' (S, Bond) on every rank: one all_gather."""
        lo, hi = self.bounds[self.rank]
        self._send[: hi - lo].copy_(self.eng.local_stats)
        if all(h - l == self.maxc for l, h in self.bounds):
            # equal shards (C3: 256 over 1/2/4/8): gather straight into the stats
            dist.all_gather_into_tensor(self.eng.stats, self._send, group=self.group)
            return
        dist.all_gather_into_tensor(self._recv, self._send, group=self.group)
        for g, (l, h) in enumerate(self.bounds):
            if h > l:
                self.eng.stats[l:h].copy_(self._recv[g * self.maxc: g * self.maxc + (h - l)])

    def interval(self, first_sweep: int, n_sweeps: int, round_index: int | None) -> int:
        """n_sweeps local sweeps, then (round_index not None) the exchange."""
        self.eng.sweeps(first_sweep, n_sweeps)
        if round_index is None:
            return 0
        self.gather_stats()
        return self.eng.exchange(round_index)
