"""Device-resident replica state and the calls that advance it.

Every tensor here lives in HBM for the whole run (allocated through torch's
caching allocator); each method is a handful of asynchronous launches of the
CUDA kernels in csrc/ through the C ABI (include/ptmh.h) on the current
torch stream.  Nothing is copied to the host until the run asks for results.

Two chains:

* ``ExactEngine`` -- the reference's random-site chain, bit-exact with
  ``isingpt.executor.run`` (csrc/exact.cu).
* ``CheckerboardEngine`` -- Mode F, the multispin-coded checkerboard sweep
  (csrc/checkerboard.cu), DESIGN.md section 3.

Lattice ("row") r of a run holds a configuration; slot k holds a temperature.
Exchanges permute slot_to_row / row_to_slot only -- lattices never move
(kernels.py:138-146 does the same with its row indirection).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .tables import cb_tables, exact_tables, integer_energy_ok

_P = lambda t: t.data_ptr() if t is not None else None  # noqa: E731


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


PARALLEL_FILL_MIN_SITES = 1 << 16  # below: the warp-sequential kernel (shared memory) wins
PARALLEL_FILL_WS_BYTES = 2 << 30


def fill_lattices(spins: torch.Tensor, L: int, up_count: int, seed: int, stream0: int,
                  stream: int) -> None:
    """Exact-count init of every lattice in `spins` (rows, L, L) int8 from
    stream stream0 + r, position 0 (executor.py:203-205, kernels.py:26-45)."""
    rows = spins.shape[0]
    if rows == 0:
        return
    if L * L < PARALLEL_FILL_MIN_SITES:
        _lib.call("ptmh_fill_lattices", _P(spins), rows, L, up_count, seed, stream0, 0, stream)
        return
    per_row = int(_lib.LIB.ptmh_fill_workspace_bytes(L, 1))
    k = max(1, min(rows, PARALLEL_FILL_WS_BYTES // per_row))
    ws = torch.empty(int(_lib.LIB.ptmh_fill_workspace_bytes(L, k)), dtype=torch.uint8,
                     device=spins.device)
    _lib.call("ptmh_fill_lattices_parallel", _P(spins), rows, L, up_count, seed, stream0, 0,
              _P(ws), ws.numel(), stream)
    del ws


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2512_03825_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    if isinstance(device, torch.device):
        return torch.device("cuda", device.index if device.index is not None
                            else torch.cuda.current_device())
    return torch.device("cuda", int(device))


class _Base:
    def __init__(self, side: int, replicas: int, temperatures: np.ndarray, seed: int,
                 J: float, B: float, up_fraction: float, device=None,
                 row_range: tuple[int, int] | None = None):
        self.dev = require_cuda(device)
        self.L, self.R = int(side), int(replicas)
        self.seed = int(seed) & ((1 << 64) - 1)
        self.J, self.B = float(J), float(B)
        self.temps = np.asarray(temperatures, dtype=np.float64)
        self.betas_np = 1.0 / self.temps  # executor.py:195
        self.up_count = round(up_fraction * self.L * self.L)  # executor.py:202
        lo, hi = row_range if row_range is not None else (0, self.R)
        self.row_lo, self.row_hi = int(lo), int(hi)
        self.rows = self.row_hi - self.row_lo
        d = self.dev
        self.betas = torch.from_numpy(self.betas_np.copy()).to(d)
        self.slot_to_row = torch.arange(self.R, dtype=torch.int64, device=d)
        self.counters = torch.zeros(2, dtype=torch.int64, device=d)  # accepted, near ties

    def _s(self) -> int:
        return _stream(self.dev)

    def swap_counts(self) -> tuple[int, int]:
        c = self.counters.cpu().tolist()
        return int(c[0]), int(c[1])


class ExactEngine(_Base):
    """The reference chain on device arrays (executor.py:196-220 state)."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        if self.rows != self.R:
            raise ValueError("the exact chain runs unsharded (one device)")
        d, R, L = self.dev, self.R, self.L
        # canonical state: 1 bit per spin (L2-resident commits); int8 only at
        # the boundaries (init, full_states recording, final_spins)
        self.spins = torch.empty((R, L, L), dtype=torch.int8, device=d)
        self.bits = torch.zeros((R, (L * L + 31) // 32), dtype=torch.int32, device=d)
        self.positions = torch.zeros(R, dtype=torch.int64, device=d)
        self.energies = torch.zeros(R, dtype=torch.float64, device=d)
        self.spin_sums = torch.zeros(R, dtype=torch.int64, device=d)
        self.iters_done = torch.zeros(R, dtype=torch.int64, device=d)
        tbl, dcls = exact_tables(self.betas_np, self.J, self.B)
        self.tbl = torch.from_numpy(tbl).to(d)
        self.dcls = torch.from_numpy(dcls).to(d)
        self.int_energy = 0

    def init_state(self) -> None:
        """executor.py:203-207: row r from stream r, position 0."""
        s = self._s()
        R, L = self.R, self.L
        fill_lattices(self.spins, L, self.up_count, self.seed, 0, s)
        stats = torch.empty((R, 2), dtype=torch.int64, device=self.dev)
        _lib.call("ptmh_row_stats", _P(self.spins), R, L, _P(stats), s)
        st = stats.cpu().numpy()
        # kernels.py:59 B*total - J*bond, evaluated with the same FP64 ops
        e = self.B * st[:, 0].astype(np.float64) - self.J * st[:, 1].astype(np.float64)
        self.energies.copy_(torch.from_numpy(e))
        self.spin_sums.copy_(torch.from_numpy(st[:, 0].copy()))
        self.positions.fill_(L * L - 1)  # fill_lattice consumes L^2-1 draws
        self.int_energy = int(integer_energy_ok(self.J, self.B, e))
        _lib.call("ptmh_bits_pack", _P(self.spins), R, L, _P(self.bits), s)

    def advance(self, start_iter: int, nsteps: int, obs_e=None, obs_m=None, record: int = 0,
                states=None, lo: int = 0, hi: int | None = None) -> None:
        """kernels.py:62-113 over slots [lo, hi)."""
        hi = self.R if hi is None else hi
        ncols = obs_e.shape[1] if obs_e is not None else 0
        if record <= 1 and nsteps > 0 and hi > lo and self.L <= 4096:
            # two-phase: parallel draws + dependency masks, then a light commit
            need = int(_lib.LIB.ptmh_advance_workspace_bytes(hi - lo, nsteps))
            if getattr(self, "_ws", None) is None or self._ws.numel() < need:
                self._ws = torch.empty(need, dtype=torch.uint8, device=self.dev)
            _lib.call("ptmh_advance_block_bits", _P(self.bits), self.L, _P(self.slot_to_row), lo,
                      hi, _P(self.tbl), _P(self.dcls), self.int_energy, _P(self.energies),
                      _P(self.spin_sums), _P(self.positions), _P(self.iters_done), self.seed,
                      start_iter, nsteps, _P(obs_e) if record else None,
                      _P(obs_m) if record else None, ncols, _P(self._ws), self._ws.numel(),
                      self._s())
            return
        # full_states: the per-attempt snapshot kernel works on int8 lattices
        _lib.call("ptmh_bits_unpack", _P(self.bits), self.R, self.L, _P(self.spins), self._s())
        _lib.call("ptmh_advance_block", _P(self.spins), self.L, _P(self.slot_to_row), lo, hi,
                  _P(self.tbl), _P(self.dcls), self.int_energy, _P(self.energies),
                  _P(self.spin_sums), _P(self.positions), _P(self.iters_done), self.seed,
                  start_iter, nsteps, _P(obs_e), _P(obs_m), ncols, record, _P(states), self._s())
        _lib.call("ptmh_bits_pack", _P(self.spins), self.R, self.L, _P(self.bits), self._s())

    def resident_ok(self, record: int) -> bool:
        """Whether run_resident applies: every slot in one CTA (R <= 32), bit
        lattices in shared memory, no per-attempt state snapshots."""
        return (self.R <= 32 and record <= 1 and self.L <= 4096
                and self.R * ((self.L * self.L + 31) // 32) * 4 <= 200 * 1024)

    def run_resident(self, start_iter: int, nsteps: int, swap_every: int, total_iters: int,
                     obs_e=None, obs_m=None) -> None:
        """Iterations start_iter .. start_iter+nsteps-1 WITH their swap rounds
        (executor.py:111-125, 227-262) in chunked launches: draws on the whole
        GPU, one CTA commits every slot in shared memory and runs the rounds
        (csrc/exact.cu, exact_resident_kernel)."""
        if nsteps <= 0:
            return
        need = int(_lib.LIB.ptmh_advance_workspace_bytes(self.R, nsteps))
        if getattr(self, "_ws", None) is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.dev)
        ncols = obs_e.shape[1] if obs_e is not None else 0
        _lib.call("ptmh_exact_run_resident", _P(self.bits), self.L, _P(self.slot_to_row), self.R,
                  _P(self.tbl), _P(self.dcls), self.int_energy, _P(self.energies), _P(self.spin_sums),
                  _P(self.positions), _P(self.iters_done), self.seed, start_iter, nsteps, swap_every,
                  total_iters, _P(self.betas), _P(self.counters), _P(obs_e), _P(obs_m), ncols,
                  _P(self._ws), self._ws.numel(), self._s())

    def exchange(self, round_index: int) -> int:
        """One swap round (executor.py:250-262, kernels.py:116-148); returns
        the number of pairs attempted."""
        first = round_index % 2
        n_pairs = max(0, (self.R - first) // 2)
        if n_pairs:
            _lib.call("ptmh_swap_chunk", _P(self.slot_to_row), _P(self.energies),
                      _P(self.spin_sums), _P(self.betas), self.R, self.seed, self.R,
                      round_index, first, 0, n_pairs, _P(self.counters),
                      self.counters.data_ptr() + 8, None, self._s())
        return n_pairs

    def final_spins(self) -> np.ndarray:
        _lib.call("ptmh_bits_unpack", _P(self.bits), self.R, self.L, _P(self.spins), self._s())
        return self.spins.cpu().numpy()


class CheckerboardEngine(_Base):
    """Mode F state: bit-packed lattices (rows, 2, W) uint32 + per-lattice
    (sum s, sum bonds) int64 kept current by the fused reduction."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        if self.L % 2:
            raise ValueError("the checkerboard sweep needs an even lattice side")
        d, R = self.dev, self.R
        self.W = int(_lib.LIB.ptmh_cb_words_per_color(self.L))
        self.packed = torch.zeros((self.rows, 2, self.W), dtype=torch.int32, device=d)
        self.stats = torch.zeros((R, 2), dtype=torch.int64, device=d)  # all lattices
        self.row_to_slot = torch.arange(R, dtype=torch.int32, device=d)
        thr, always = cb_tables(self.betas_np, self.J, self.B)
        self.thr = torch.from_numpy(thr.view(np.int32)).to(d)
        self.always = int(always)
        self.energies = torch.zeros(R, dtype=torch.float64, device=d)
        self.spin_sums = torch.zeros(R, dtype=torch.int64, device=d)
        # zeroed sync block of the persistent sweep path (left zeroed by every call)
        self.persistent = True
        self._sync = torch.zeros(int(_lib.LIB.ptmh_cb_sync_words(self.rows, self.L)), dtype=torch.int32, device=d)
        self._scratch = None  # the temporally blocked path's second state buffer (allocated on first use)

    @property
    def local_stats(self) -> torch.Tensor:
        return self.stats[self.row_lo:self.row_hi]

    def init_state(self) -> None:
        """Exact-count init identical to the reference (executor.py:203-207)
        for the local rows, then per-lattice stats and packing."""
        s = self._s()
        if self.rows == 0:
            return
        spins = torch.empty((self.rows, self.L, self.L), dtype=torch.int8, device=self.dev)
        fill_lattices(spins, self.L, self.up_count, self.seed, self.row_lo, s)
        _lib.call("ptmh_row_stats", _P(spins), self.rows, self.L, _P(self.local_stats), s)
        _lib.call("ptmh_cb_pack", _P(spins), self.rows, self.L, _P(self.packed), s)
        del spins

    def load_spins(self, spins: torch.Tensor) -> None:
        """Replace the local lattices with given int8 configurations."""
        s = self._s()
        spins = spins.to(self.dev, torch.int8).contiguous()
        _lib.call("ptmh_cb_pack", _P(spins), self.rows, self.L, _P(self.packed), s)
        # (S, Bond) from the packed words: the word-parallel kernel for L % 64 == 0
        _lib.call("ptmh_cb_row_stats", _P(self.packed), self.rows, self.L, _P(self.local_stats), s)

    def sweeps(self, first_sweep: int, n: int) -> None:
        if self.rows == 0 or n <= 0:
            return
        rts = self.row_to_slot[self.row_lo:self.row_hi]
        if self.persistent:
            # one persistent launch for all 2n half-sweeps where the kernel
            # supports it (csrc/checkerboard.cu, cb_sweeps_persistent); with a
            # scratch state buffer it runs temporally blocked (a whole sweep of
            # a band per work item, ping-pong between packed and scratch)
            if self._scratch is None and self.L >= 1024 and self.L % 512 == 0:
                self._scratch = torch.empty_like(self.packed)
            _lib.call("ptmh_cb_sweeps_ws", _P(self.packed), self.rows, self.L, _P(rts), _P(self.thr),
                      self.always, self.seed, first_sweep, n, _P(self.local_stats), _P(self._sync),
                      _P(self._scratch), self._s())
        else:
            _lib.call("ptmh_cb_sweeps", _P(self.packed), self.rows, self.L, _P(rts), _P(self.thr),
                      self.always, self.seed, first_sweep, n, _P(self.local_stats), self._s())

    def exchange(self, round_index: int) -> int:
        """Swap round on the energies of every lattice (self.stats must hold
        all lattices: the distributed driver all-gathers them first)."""
        first = round_index % 2
        _lib.call("ptmh_cb_exchange", _P(self.stats), _P(self.slot_to_row), _P(self.row_to_slot),
                  self.R, self.J, self.B, _P(self.betas), self.seed, round_index,
                  _P(self.energies), _P(self.spin_sums), _P(self.counters),
                  self.counters.data_ptr() + 8, self._s())
        return max(0, (self.R - first) // 2)

    def run_resident(self, first_sweep: int, n_sweeps: int, total_sweeps: int, swap_every: int,
                     record_every: int = 0, obs_e=None, obs_m=None) -> None:
        """Sweeps first..first+n-1 of a run of total_sweeps, with its swap
        rounds and observations, in ONE persistent launch (csrc/resident.cu).
        Single device only (every lattice local)."""
        if self.rows != self.R:
            raise ValueError("the resident kernel needs every lattice on one device")
        if getattr(self, "_s2r2", None) is None:
            self._s2r2 = torch.empty((2, self.R), dtype=torch.int64, device=self.dev)
            self._r2s2 = torch.empty((2, self.R), dtype=torch.int32, device=self.dev)
            self._slot_stats = torch.empty((2, self.R, 2), dtype=torch.int64, device=self.dev)
        self._s2r2[0].copy_(self.slot_to_row)
        self._r2s2[0].copy_(self.row_to_slot)
        out = ctypes.c_int(0)
        ncols = obs_e.shape[1] if obs_e is not None else 0
        # the segment's swap draws (point-to-point rounds where lattices are
        # warp-owned; csrc/resident.cu), in segments of <= 4096 rounds
        seg = n_sweeps
        if swap_every > 0:
            seg = max(swap_every, min(n_sweeps, 4096 * swap_every))
        done = 0
        while done < n_sweeps:
            n = min(seg, n_sweeps - done)
            t0 = first_sweep + done
            rounds = sum(1 for d in range(t0 + 1, t0 + n + 1)
                         if swap_every > 0 and d % swap_every == 0 and d < total_sweeps) if swap_every else 0
            ws = None
            if rounds:
                need = int(_lib.LIB.ptmh_cb_resident_ws_bytes(self.R, rounds))
                if getattr(self, "_res_ws", None) is None or self._res_ws.numel() < need:
                    self._res_ws = torch.empty(need, dtype=torch.uint8, device=self.dev)
                ws = self._res_ws
            _lib.call("ptmh_cb_run_resident_ws", _P(self.packed), self.R, self.L, _P(self._s2r2),
                      _P(self._r2s2), 0, _P(self.thr), self.always, self.seed, self.J, self.B,
                      _P(self.betas), _P(self.stats), _P(self._slot_stats), _P(self.counters), _P(obs_e),
                      _P(obs_m), ncols, t0, n, total_sweeps, swap_every, record_every,
                      ctypes.byref(out), _P(ws), ws.numel() if ws is not None else 0, self._s())
            if out.value != 0 and done + n < n_sweeps:
                self._s2r2[0].copy_(self._s2r2[out.value])
                self._r2s2[0].copy_(self._r2s2[out.value])
                out.value = 0
            done += n
        self.slot_to_row.copy_(self._s2r2[out.value])
        self.row_to_slot.copy_(self._r2s2[out.value])

    def run_resident_sharded(self, first_sweep: int, n_sweeps: int, total_sweeps: int, swap_every: int,
                             rank: int, world: int, pub_peers, flag_peers, slot_stats,
                             record_every: int = 0, obs_e=None, obs_m=None, max_ctas: int = 0) -> None:
        """One rank's part of a resident run over `world` GPUs (the local rows
        only); rounds exchange (S, Bond) through peer memory and flags
        (csrc/resident.cu).  pub_peers / flag_peers: device pointers (ints) of
        every rank's slot_stats (2, R, 2) int64 and flags (world,) uint32,
        [rank] = this rank's own.  Afterwards the local rows' slots are in
        row_to_slot[row_lo:row_hi]; counters, observables and slot_to_row hold
        this rank's part (ShardedCheckerboard combines them)."""
        if getattr(self, "_r2s2_loc", None) is None:
            self._s2r2_g = torch.empty((2, self.R), dtype=torch.int64, device=self.dev)
            self._r2s2_loc = torch.empty((2, max(1, self.rows)), dtype=torch.int32, device=self.dev)
        self._s2r2_g[0].copy_(self.slot_to_row)
        self._r2s2_loc[0, :self.rows].copy_(self.row_to_slot[self.row_lo:self.row_hi])
        out = ctypes.c_int(0)
        ncols = obs_e.shape[1] if obs_e is not None else 0
        pubs = (ctypes.c_void_p * world)(*[int(x) for x in pub_peers])
        flags = (ctypes.c_void_p * world)(*[int(x) for x in flag_peers])
        # (everything runs on the current stream: co-running ranks on one GPU
        # in the tests each use their own)
        # the point-to-point rounds' swap draws (csrc/resident.cu), when lattices are warp-owned
        rounds = sum(1 for d in range(first_sweep + 1, first_sweep + n_sweeps + 1)
                     if d % swap_every == 0 and d < total_sweeps) if swap_every > 0 else 0
        need = int(_lib.LIB.ptmh_cb_resident_ws_bytes(self.R, rounds)) if rounds else 0
        if need and (getattr(self, "_res_ws", None) is None or self._res_ws.numel() < need):
            self._res_ws = torch.empty(need, dtype=torch.uint8, device=self.dev)
        ws = self._res_ws if need else None
        _lib.call("ptmh_cb_run_resident_sharded_ws", _P(self.packed), self.rows, self.L, _P(self._s2r2_g),
                  _P(self._r2s2_loc), 0, _P(self.thr), self.always, self.seed, self.J, self.B,
                  _P(self.betas), _P(self.local_stats),
                  slot_stats if isinstance(slot_stats, int) else _P(slot_stats), _P(self.counters), _P(obs_e),
                  _P(obs_m), ncols, first_sweep, n_sweeps, total_sweeps, swap_every, record_every,
                  ctypes.byref(out), self.R, rank, world, self.row_lo, ctypes.cast(pubs, ctypes.c_void_p),
                  ctypes.cast(flags, ctypes.c_void_p), max_ctas, _P(ws), ws.numel() if ws is not None else 0,
                  self._s())
        self.row_to_slot[self.row_lo:self.row_hi].copy_(self._r2s2_loc[out.value, :self.rows])
        self.slot_to_row.copy_(self._s2r2_g[out.value])

    def observe(self, obs_e: torch.Tensor, obs_m: torch.Tensor, col: int) -> None:
        _lib.call("ptmh_cb_observe", _P(self.stats), _P(self.slot_to_row), self.R, self.L,
                  self.J, self.B, _P(obs_e), _P(obs_m), obs_e.shape[1], col, self._s())

    def snapshot_by_slot(self, out: torch.Tensor) -> None:
        """out (R, L, L) int8 <- every lattice, in slot order (full_states)."""
        _lib.call("ptmh_cb_unpack_slots", _P(self.packed), _P(self.slot_to_row), self.R, self.L,
                  _P(out), self._s())

    def audit_stats(self) -> torch.Tensor:
        """(S, Bond) recomputed from the packed lattices (local rows)."""
        out = torch.empty((self.rows, 2), dtype=torch.int64, device=self.dev)
        _lib.call("ptmh_cb_row_stats", _P(self.packed), self.rows, self.L, _P(out), self._s())
        return out

    def spins_int8(self) -> torch.Tensor:
        out = torch.empty((self.rows, self.L, self.L), dtype=torch.int8, device=self.dev)
        _lib.call("ptmh_cb_unpack", _P(self.packed), self.rows, self.L, _P(out), self._s())
        return out

    def final_spins(self) -> np.ndarray:
        return self.spins_int8().cpu().numpy()
