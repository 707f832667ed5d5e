"""BASELINE config builders: shapes, statistics and boundary data (host only)."""
import numpy as np
import pytest

from paper_2103_11050_b200 import api, configs


@pytest.mark.parametrize("name,nx,ny,nsx,nsy,M", [("C1", 64, 64, 4, 4, 5.0), ("C2", 256, 256, 16, 16, 5.0),
                                                  ("C3", 220, 60, 11, 3, 10.0), ("C4", 512, 512, 16, 16, 20.0)])
def test_shapes(name, nx, ny, nsx, nsy, M):
    c = configs.build(name)
    p = c.problem
    assert (p.nx, p.ny, p.nsx, p.nsy, p.viscosity_ratio) == (nx, ny, nsx, nsy, M)
    assert p.K.shape == (nx * ny,) and np.all(p.K > 0) and np.all(np.isfinite(p.K))
    assert p.bc.kind.shape == (2 * (nx + ny),)


def test_lognormal_statistics():
    K = configs.exp_covariance_lognormal(256, 256, 1.0, 1.0, 0.05, 4.0, seed=7)
    lnk = np.log(K)
    assert abs(lnk.mean()) < 0.5 and 2.0 < lnk.var() < 6.0
    K2 = configs.exp_covariance_lognormal(256, 256, 1.0, 1.0, 0.05, 4.0, seed=7)
    assert np.array_equal(K, K2)


def test_channel_field_contrast():
    c = configs.build("C3")
    lnk = np.log10(c.problem.K)
    chan = lnk > 0
    assert 0.3 < chan.mean() < 0.6
    assert np.median(lnk[chan]) - np.median(lnk[~chan]) > 4.0
    h = c.problem.ly / c.problem.ny
    inflow = -np.sum(c.problem.bc.value[c.problem.bc.kind == api.FLUX]) * h
    assert abs(inflow - 1.0) < 1e-12
    assert c.problem.bc.kind.tolist().count(api.PRESSURE) == 6


def test_white_noise():
    c = configs.build("C4")
    assert np.all(np.abs(c.problem.K - 1.0) <= 0.01)
