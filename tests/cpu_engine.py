"""Oracle-backed stand-in for engine.CheckerboardEngine (TEST ONLY): same
constructor and methods, CPU tensors, the C oracle doing the sweeps.  Lets
the multi-GPU coordinator (distributed.py) run over gloo on CPU."""

import numpy as np
import torch

import oracle


class OracleCheckerboardEngine:
    def __init__(self, side, replicas, temperatures, seed, J, B, up_fraction, device=None,
                 row_range=None):
        self.L, self.R = int(side), int(replicas)
        self.row_lo, self.row_hi = row_range if row_range is not None else (0, self.R)
        self.rows = self.row_hi - self.row_lo
        self.seed, self.J, self.B = int(seed), float(J), float(B)
        self.betas = 1.0 / np.asarray(temperatures, dtype=np.float64)
        self.thr, self.always = oracle.cb_tables(self.betas, self.J, self.B)
        self.up = round(up_fraction * self.L * self.L)
        self.spins = np.empty((self.rows, self.L, self.L), dtype=np.int8)
        self.stats = torch.zeros((self.R, 2), dtype=torch.int64)
        self.slot_to_row = np.arange(self.R, dtype=np.int64)
        self.accepted = 0

    @property
    def local_stats(self):
        return self.stats[self.row_lo:self.row_hi]

    def init_state(self):
        for r in range(self.row_lo, self.row_hi):
            oracle.fill_lattice(self.spins[r - self.row_lo], self.up, self.seed, r, 0)
        if self.rows:
            self.local_stats.copy_(torch.from_numpy(oracle.row_stats(self.spins)))

    def sweeps(self, first, n):
        if not self.rows:
            return
        r2s = np.empty(self.R, dtype=np.int64)
        r2s[self.slot_to_row] = np.arange(self.R)
        local_r2s = r2s[self.row_lo:self.row_hi].copy()
        st = self.local_stats.numpy()
        for t in range(first, first + n):
            oracle.cb_sweep(self.spins, local_r2s, self.thr, self.always, self.seed, t, st)

    def exchange(self, round_index):
        first = round_index % 2
        n_pairs = max(0, (self.R - first) // 2)
        s = self.stats.numpy()[self.slot_to_row]
        e = self.B * s[:, 0].astype(np.float64) - self.J * s[:, 1].astype(np.float64)
        sums = s[:, 0].copy()
        if n_pairs:
            self.accepted += oracle.swap_chunk(self.slot_to_row, e, sums, self.betas, self.seed,
                                               self.R, round_index, first, 0, n_pairs)
        return n_pairs
