"""Parallel exact-count init (csrc/init.cu) == the sequential Fisher-Yates
of the reference (kernels.py:26-45), bit for bit."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _parallel(L, rows, up, seed, stream0):
    from paper_2512_03825_b200 import _lib
    sp = torch.empty((rows, L, L), dtype=torch.int8, device="cuda")
    ws = torch.empty(int(_lib.LIB.ptmh_fill_workspace_bytes(L, 2)), dtype=torch.uint8, device="cuda")
    _lib.call("ptmh_fill_lattices_parallel", sp.data_ptr(), rows, L, up, seed, stream0, 0,
              ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    return sp.cpu().numpy()


def _sequential(L, rows, up, seed, stream0):
    from paper_2512_03825_b200 import _lib
    sp = torch.empty((rows, L, L), dtype=torch.int8, device="cuda")
    _lib.call("ptmh_fill_lattices", sp.data_ptr(), rows, L, up, seed, stream0, 0,
              torch.cuda.current_stream().cuda_stream)
    return sp.cpu().numpy()


@pytest.mark.parametrize("L,rows,upf,seed", [(2, 3, 0.5, 1), (3, 5, 0.3, 2), (8, 4, 0.5, 7),
                                            (33, 3, 0.9, 11), (64, 5, 0.5, 42), (256, 3, 0.5, 5),
                                            (512, 2, 0.0, 6), (512, 2, 1.0, 6)])
def test_parallel_equals_sequential_and_oracle(L, rows, upf, seed):
    up = round(upf * L * L)
    par = _parallel(L, rows, up, seed, 3)
    seq = _sequential(L, rows, up, seed, 3)
    assert np.array_equal(par, seq)
    for r in range(min(rows, 2)):
        ref = np.empty((L, L), dtype=np.int8)
        oracle.fill_lattice(ref, up, seed, 3 + r, 0)
        assert np.array_equal(par[r], ref)
    assert np.all((par == 1).sum(axis=(1, 2)) == up)


def test_parallel_init_at_1024():
    L, up = 1024, 1024 * 1024 // 2
    par = _parallel(L, 3, up, 42, 0)
    ref = np.empty((L, L), dtype=np.int8)
    oracle.fill_lattice(ref, up, 42, 2, 0)
    assert np.array_equal(par[2], ref)
