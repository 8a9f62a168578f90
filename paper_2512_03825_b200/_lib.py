"""ctypes binding of libptmh.so (include/ptmh.h).

The CUDA library is the product: there is no CPU fallback.  Importing this
module raises if the library is missing, and every call raises
``PtmhError`` on a non-zero return code.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PTMH_LIB overrides the path (A/B builds of the same sources; tools/ only)
LIB_PATH = os.environ.get("PTMH_LIB") or os.path.join(_HERE, "libptmh.so")


class PtmhError(RuntimeError):
    """A libptmh call returned an error code."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i64, u64, f64, i32, u32 = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                               ctypes.c_int, ctypes.c_uint32)
    sigs = {
        "ptmh_abi_version": ([], i32),
        "ptmh_last_error": ([], ctypes.c_char_p),
        # host-buffer ABI (isingpt/kernels.py boundary)
        "ptmh_host_fill_lattice": ([P, i64, i64, u64, u64, u64, P], i32),
        "ptmh_host_lattice_energy": ([P, i64, f64, f64, P], i32),
        "ptmh_host_advance_block": ([P, i64, i64, P, i64, i64, i64, P, f64, f64, P, P, P, P,
                                     u64, i64, i64, P, P, i64, i32, P], i32),
        "ptmh_host_swap_chunk": ([P, P, P, P, i64, u64, i64, i64, i64, i64, i64, P], i32),
        "ptmh_host_cb_interval": ([P, i64, i64, P, P, f64, f64, u64, i64, i64, i64, P, P, P],
                                  i32),
        # the reference's per-replica public ops (rng.py, mh.py, tempering.py)
        "ptmh_host_uniforms": ([u64, u64, u64, i64, P], i32),
        "ptmh_host_swap_pairs": ([P, P, i64, P, P, i64, u64, i64, i64, P, P], i32),
        "ptmh_host_mh_steps": ([P, i64, f64, f64, f64, P, P, u64, u64, P, i64], i32),
        # device-resident ABI
        "ptmh_uniforms": ([u64, u64, u64, i64, P, P], i32),
        "ptmh_cb_last_launch": ([P], i32),
        "ptmh_fill_lattices": ([P, i64, i64, i64, u64, u64, u64, P], i32),
        "ptmh_row_stats": ([P, i64, i64, P, P], i32),
        "ptmh_fill_workspace_bytes": ([i64, i64], i64),
        "ptmh_fill_lattices_parallel": ([P, i64, i64, i64, u64, u64, u64, P, i64, P], i32),
        "ptmh_advance_block": ([P, i64, P, i64, i64, P, P, i32, P, P, P, P, u64, i64, i64,
                                P, P, i64, i32, P, P], i32),
        "ptmh_advance_workspace_bytes": ([i64, i64], i64),
        "ptmh_advance_block_ws": ([P, i64, P, i64, i64, P, P, i32, P, P, P, P, u64, i64, i64,
                                   P, P, i64, P, i64, P], i32),
        "ptmh_exact_run_resident": ([P, i64, P, i64, P, P, i32, P, P, P, P, u64, i64, i64, i64, i64, P, P,
                                     P, P, i64, P, i64, P], i32),
        "ptmh_bits_pack": ([P, i64, i64, P, P], i32),
        "ptmh_bits_unpack": ([P, i64, i64, P, P], i32),
        "ptmh_advance_block_bits": ([P, i64, P, i64, i64, P, P, i32, P, P, P, P, u64, i64, i64,
                                     P, P, i64, P, i64, P], i32),
        "ptmh_swap_chunk": ([P, P, P, P, i64, u64, i64, i64, i64, i64, i64, P, P, P, P], i32),
        "ptmh_cb_words_per_color": ([i64], i64),
        "ptmh_cb_exchange": ([P, P, P, i64, f64, f64, P, u64, i64, P, P, P, P, P], i32),
        "ptmh_cb_pack": ([P, i64, i64, P, P], i32),
        "ptmh_cb_unpack": ([P, i64, i64, P, P], i32),
        "ptmh_cb_sweeps": ([P, i64, i64, P, P, u32, u64, i64, i64, P, P], i32),
        "ptmh_cb_sync_words": ([i64, i64], i64),
        "ptmh_cb_sweeps_sync": ([P, i64, i64, P, P, u32, u64, i64, i64, P, P, P], i32),
        "ptmh_cb_sweeps_ws": ([P, i64, i64, P, P, u32, u64, i64, i64, P, P, P, P], i32),
        "ptmh_swap_decide": ([P, P, P, P, i64, P, P, P], i32),
        "ptmh_cb_row_stats": ([P, i64, i64, P, P], i32),
        "ptmh_cb_unpack_slots": ([P, P, i64, i64, P, P], i32),
        "ptmh_cb_run_resident": ([P, i64, i64, P, P, i32, P, u32, u64, f64, f64, P, P, P, P, P,
                                  P, i64, i64, i64, i64, i64, i64, P, P], i32),
        "ptmh_cb_resident_ws_bytes": ([i64, i64], i64),
        "ptmh_cb_run_resident_ws": ([P, i64, i64, P, P, i32, P, u32, u64, f64, f64, P, P, P, P, P,
                                     P, i64, i64, i64, i64, i64, i64, P, P, i64, P], i32),
        "ptmh_cb_run_resident_sharded_ws": ([P, i64, i64, P, P, i32, P, u32, u64, f64, f64, P, P, P, P, P,
                                             P, i64, i64, i64, i64, i64, i64, P, i64, i32, i32, i64, P, P,
                                             i32, P, i64, P], i32),
        "ptmh_cb_run_resident_sharded": ([P, i64, i64, P, P, i32, P, u32, u64, f64, f64, P, P, P, P, P,
                                          P, i64, i64, i64, i64, i64, i64, P, i64, i32, i32, i64, P, P,
                                          i32, P], i32),
        "ptmh_ipc_handle_bytes": ([], i64),
        "ptmh_ipc_handle": ([P, P], i32),
        "ptmh_ipc_open": ([P, P], i32),
        "ptmh_ipc_close": ([P], i32),
        "ptmh_peer_alloc": ([i64, P], i32),
        "ptmh_peer_free": ([P], i32),
        "ptmh_cb_slot_energies": ([P, P, i64, f64, f64, P, P, P], i32),
        "ptmh_cb_observe": ([P, P, i64, i64, f64, f64, P, P, i64, i64, P], i32),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib, sorted(sigs)


LIB, EXPORTED = _load()
ABI_VERSION = LIB.ptmh_abi_version()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = LIB.ptmh_last_error().decode(errors="replace")
        raise PtmhError(f"{what} failed (rc={rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(LIB, name)(*args), name)


def cb_last_launch() -> dict:
    """The sweep kernel this thread's last sweep call launched (ptmh_cb_last_launch)."""
    v = (ctypes.c_int32 * 6)()
    call("ptmh_cb_last_launch", v)
    kinds = {0: None, 1: "cb_sweeps_persistent<{r},{t}>{tb}", 2: "cb_half_sweep_ferro<{r},0|1>",
             3: "cb_half_sweep_fast<{r}>", 4: "cb_half_sweep_generic",
             5: "cb_resident_kernel (clusters of {r}, grid-barrier rounds)",
             6: "cb_resident_p2p_kernel (warp-owned lattices, point-to-point rounds)",
             7: "cb_resident_kernel (clusters of {r}, point-to-point rounds)",
             8: "cb_cluster_smem_kernel<{r},{t}> (lattices in the shared memory of {g}-CTA clusters, "
                "point-to-point rounds)",
             9: "cb_resident_reg64_kernel (64^2 lattices in registers, a warp each, point-to-point rounds)",
             10: "cb_resident_reg32_kernel (32^2 lattices in registers, a warp each, point-to-point rounds)"}
    k = kinds.get(v[0])
    return {"kind": v[0], "rows": v[1], "threads": v[2], "group": v[3], "bands": bool(v[4]), "tb": v[4] >= 2, "streamed": v[4] == 3,
            "grid": v[5], "name": k.format(r=v[1], t=v[2], g=v[3], tb=" (temporally blocked)" if v[4] == 2 else " (temporally blocked, streamed)" if v[4] == 3 else "")
            if k else None}
