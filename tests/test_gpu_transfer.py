"""Host transfers through pinned staging (capi.cu upload / download): arrays of
8 MB and more from pageable host memory are copied through two pinned 16 MB
buffers with a multi-threaded host memcpy. The staged path must move the
same bytes as the direct path (page-locked host buffers), including a
partial last chunk."""
import ctypes as C

import numpy as np
import pytest

from cases import problem, random_kappa
from paper_2103_11050_b200 import api

pytestmark = pytest.mark.gpu


def _pinned(n):
    import torch
    return torch.empty(n, dtype=torch.float64).pin_memory()


def _ptr(t):
    return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))


def test_staged_transfers_match_direct():
    nx = ny = 1024  # cells: 8 MiB per field (one staged chunk); faces: 16.8 MB (a full and a partial chunk)
    sim = api.Simulator(problem(nx, ny, 32, 32, random_kappa(nx, ny, 7)))
    try:
        rng = np.random.default_rng(11)
        s = rng.uniform(0.0, 1.0, sim.cells)
        u = rng.normal(0.0, 1e-3, sim.faces)
        # staged: numpy (pageable) in and out
        k_staged = sim.conductivity(s)
        s_staged = sim.upwind_step(s, 1.0, u, 1e-6)
        # direct: page-locked in and out
        import torch
        s_p, u_p = _pinned(sim.cells), _pinned(sim.faces)
        s_p.numpy()[:] = s
        u_p.numpy()[:] = u
        k_p, o_p = _pinned(sim.cells), _pinned(sim.cells)
        sim._check(sim.lib.conductivity(sim.h, _ptr(s_p), _ptr(k_p)))
        sim._check(sim.lib.upwind_step(sim.h, _ptr(s_p), 1.0, _ptr(u_p), 1e-6, _ptr(o_p)))
        torch.cuda.synchronize()
        assert np.array_equal(k_staged, k_p.numpy())
        assert np.array_equal(s_staged, o_p.numpy())
        # a face field round trip through divergence (16.8 MB upload, staged in two chunks)
        d_staged = sim.divergence(u)
        d_p = _pinned(sim.cells)
        sim._check(sim.lib.divergence(sim.h, _ptr(u_p), _ptr(d_p)))
        assert np.array_equal(d_staged, d_p.numpy())
    finally:
        sim.close()
