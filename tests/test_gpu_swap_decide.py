"""The resident kernels' exchange decision (csrc/rounds.cuh swap_decide: an
FP32 fast path, the exact FP64 evaluation within 1e-5 of the boundary)
against the reference rule evaluated on the host with Python's libm exp
(kernels.py:116-148, tempering.py:53-65), including u placed ulps away from
the FP64 probability on both sides: every decision not flagged as a near tie
(|u - p| <= 4 ulp, where the device exp may differ from glibc in the last
ulp) must equal the host's."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _host_prob(bd, ei, ej):
    x = bd * (ei - ej)
    if x >= 0.0:
        return 1.0 / (1.0 + math.exp(-x))
    ex = math.exp(x)
    return ex / (1.0 + ex)


def _cases(seed):
    rng = np.random.default_rng(seed)
    bd, ei, ej, u = [], [], [], []
    # realistic pairs: integer energies of an L = 256 lattice, ladder betas in [1/4, 1]
    for _ in range(4000):
        b1, b2 = sorted(rng.uniform(0.25, 1.0, 2))[::-1]
        e1, e2 = (float(v) for v in rng.integers(-2 * 65536, 2 * 65536, 2) // 4 * 4)
        bd.append(b1 - b2); ei.append(e1); ej.append(e2); u.append(float(rng.random()))
    # adversarial: u at, just below and just above p (ulps and small relative offsets)
    for _ in range(3000):
        b = float(rng.uniform(0.0, 0.2))
        d = float(rng.choice([-1.0, 1.0]) * rng.integers(0, 200) * 4)
        p = _host_prob(b, d, 0.0)
        if p <= 0.0:
            continue
        for k in (-1e-3, -1e-5, -2e-6, -1e-9, -3, -1, 0, 1, 3, 1e-9, 2e-6, 1e-5, 1e-3):
            uu = p + k * math.ulp(p) if isinstance(k, int) else p * (1.0 + k)
            if 0.0 <= uu < 1.0:
                bd.append(b); ei.append(d); ej.append(0.0); u.append(uu)
    return [np.array(a, dtype=np.float64) for a in (bd, ei, ej, u)]


@pytest.mark.parametrize("seed", [1, 2])
def test_swap_decide_equals_host_rule(seed):
    from paper_2512_03825_b200 import _lib
    bd, ei, ej, u = _cases(seed)
    n = bd.size
    dev = [torch.from_numpy(a).cuda() for a in (bd, ei, ej, u)]
    acc = torch.zeros(n, dtype=torch.uint8, device="cuda")
    near = torch.zeros(n, dtype=torch.uint8, device="cuda")
    _lib.call("ptmh_swap_decide", *[t.data_ptr() for t in dev], n, acc.data_ptr(), near.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    acc, near = acc.cpu().numpy().astype(bool), near.cpu().numpy().astype(bool)
    host = np.array([u[t] < _host_prob(bd[t], ei[t], ej[t]) for t in range(n)])
    assert np.array_equal(acc[~near], host[~near])
    # the near flag is raised only next to the boundary (and it is raised there)
    p = np.array([_host_prob(bd[t], ei[t], ej[t]) for t in range(n)])
    assert np.all(np.abs(u[near] - p[near]) <= 8 * np.spacing(p[near]) + 1e-300)
    assert near.sum() > 0 and not near[:4000].any()  # the realistic pairs are nowhere near
