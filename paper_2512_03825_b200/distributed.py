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

import ctypes

import torch
import torch.distributed as dist

from .executor import assign_replicas


def _host_staged(group) -> bool:
    """gloo moves host tensors: CUDA tensors are staged through host memory
    (the CPU tests and multi-process tests on one GPU); NCCL moves them
    directly (NVLink)."""
    return dist.get_backend(group) == "gloo"


def all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None) -> None:
    """dist.all_gather_into_tensor for any backend."""
    if out.is_cuda and _host_staged(group):
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def all_reduce_sum(t: torch.Tensor, group=None) -> None:
    """dist.all_reduce (sum) for any backend."""
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


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
        if all(h - l == self.maxc for l, h in self.bounds):
            # equal shards (C3: 256 over 1/2/4/8): gather straight into the
            # stats, from a separate send buffer (no aliasing of input and
            # output, which only world-1 runs could test here)
            self._send.copy_(self.eng.local_stats)
            all_gather_into(self.eng.stats, self._send, self.group)
            return
        self._send[: hi - lo].copy_(self.eng.local_stats)
        all_gather_into(self._recv, self._send, self.group)
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


class PeerBuffers:
    """Every rank's round buffers, reachable from every other rank: each rank
    allocates its slot_stats (2, R, 2) int64 and flags (world,) uint32, shares
    CUDA IPC handles over the process group (one all_gather_object at setup)
    and opens the peers' buffers -- NVLink peer memory between the GPUs of a
    node.  Used by the multi-GPU resident kernel (csrc/resident.cu)."""

    def __init__(self, R: int, device, group=None):
        from . import _lib

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # own cudaMalloc allocations (an IPC handle names a whole allocation)
        self._own = []
        for nbytes in (2 * R * 2 * 8, 4 * self.world):
            p = ctypes.c_void_p()
            with torch.cuda.device(device):
                _lib.call("ptmh_peer_alloc", nbytes, ctypes.byref(p))
            self._own.append(p.value)
        self.slot_stats, self.flags = self._own  # device pointers
        nb = int(_lib.LIB.ptmh_ipc_handle_bytes())
        mine = []
        for ptr in self._own:
            h = (ctypes.c_char * nb)()
            _lib.call("ptmh_ipc_handle", ptr, h)
            mine.append(bytes(h))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        self.pub_peers, self.flag_peers = [], []
        for g in range(self.world):
            if g == self.rank:
                self.pub_peers.append(self.slot_stats)
                self.flag_peers.append(self.flags)
                continue
            ptrs = []
            for hb in allh[g]:
                p = ctypes.c_void_p()
                _lib.call("ptmh_ipc_open", ctypes.create_string_buffer(hb, nb), ctypes.byref(p))
                ptrs.append(p.value)
                self._opened.append(p.value)
            self.pub_peers.append(ptrs[0])
            self.flag_peers.append(ptrs[1])

    def close(self) -> None:
        from . import _lib

        for p in self._opened:
            _lib.call("ptmh_ipc_close", p)
        self._opened = []
        for p in self._own:
            _lib.call("ptmh_peer_free", p)
        self._own = []


def resident_sharded(drv: "ShardedCheckerboard", peers: PeerBuffers, first_sweep: int, n_sweeps: int,
                     total_sweeps: int, swap_every: int, record_every: int = 0, obs_e=None,
                     obs_m=None) -> None:
    """A resident run segment over the ranks of drv.group: one launch per
    rank, rounds through peer memory; then the ranks' parts are combined
    (all_gather of the local rows' slots, all_reduce of the swap counters and
    of the observables, which each rank wrote for the slots it held)."""
    eng = drv.eng
    lo, hi = drv.bounds[drv.rank]
    before = eng.counters.clone()
    cols = None
    if obs_e is not None and record_every > 0:
        # the columns recorded in this segment: each slot's entry is written
        # by the rank holding the slot at that sweep; zero them here so that
        # the other ranks contribute exact zeros to the combine below
        c0, c1 = first_sweep // record_every, (first_sweep + n_sweeps) // record_every
        if c1 > c0:
            cols = (c0, c1)
            obs_e[:, c0:c1].zero_()
            obs_m[:, c0:c1].zero_()
    eng.run_resident_sharded(first_sweep, n_sweeps, total_sweeps, swap_every, drv.rank, drv.world,
                             peers.pub_peers, peers.flag_peers, peers.slot_stats,
                             record_every=record_every, obs_e=obs_e, obs_m=obs_m)
    loc = torch.zeros(drv.maxc, dtype=torch.int32, device=eng.stats.device)
    loc[: hi - lo].copy_(eng.row_to_slot[lo:hi])
    allr = torch.empty(drv.world * drv.maxc, dtype=torch.int32, device=loc.device)
    all_gather_into(allr, loc, drv.group)
    for g, (l, h) in enumerate(drv.bounds):
        eng.row_to_slot[l:h].copy_(allr[g * drv.maxc: g * drv.maxc + (h - l)])
    eng.slot_to_row[eng.row_to_slot.long()] = torch.arange(eng.R, dtype=torch.int64, device=loc.device)
    delta = eng.counters - before  # this segment's counts on this rank
    all_reduce_sum(delta, drv.group)
    eng.counters.copy_(before + delta)
    if cols is not None:
        # one writer per entry, zeros elsewhere: an integer sum of the float64
        # bit patterns reproduces the writer's value exactly (signed zeros too)
        for o in (obs_e, obs_m):
            part = o[:, cols[0]:cols[1]].contiguous().view(torch.int64)
            all_reduce_sum(part, drv.group)
            o[:, cols[0]:cols[1]].copy_(part.view(torch.float64))
