"""The C-ABI library loads without a GPU and exports every entry point that
include/ptmh.h declares (no compute calls here)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "ptmh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ptmh_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_boundary():
    names = _declared()
    for n in ["ptmh_host_fill_lattice", "ptmh_host_lattice_energy", "ptmh_host_advance_block",
              "ptmh_host_swap_chunk", "ptmh_host_cb_interval", "ptmh_cb_sweeps",
              "ptmh_swap_chunk", "ptmh_advance_block", "ptmh_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2512_03825_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(_lib.EXPORTED)
    assert _lib.ABI_VERSION == 1


def test_library_is_sm100a():
    import subprocess
    from paper_2512_03825_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2512_03825_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt, f


def test_sync_block_size():
    """ptmh_cb_sync_words (host arithmetic only): ticket, CTAs out, one
    counter per lattice, and the persistent kernel's band counters (at most
    L^2 / 16384 per lattice where the persistent path applies)."""
    from paper_2512_03825_b200 import _lib
    f = _lib.LIB.ptmh_cb_sync_words
    assert f(256, 1024) == 2 + 256 + 256 * 64
    assert f(512, 4096) == 2 + 512 + 512 * 1024
    assert f(3, 1536) == 2 + 3 + 3 * (1536 * 1536 // 16384)
    assert f(8, 64) == 2 + 8  # no persistent path below L = 1024
    assert f(0, 1024) == 2
