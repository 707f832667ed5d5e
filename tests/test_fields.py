"""Field generation on the device and the field files (include/mpm2p_fields.h,
SURVEY.md §8f-2), against the host restatement tests/field_ref.py."""
import os

import numpy as np
import pytest

from field_ref import channels as ref_channels, exp_lognormal as ref_exp, white_noise as ref_white
from paper_2103_11050_b200 import api, fields


@pytest.mark.parametrize("text", [False, True])
def test_field_files_roundtrip(tmp_path, text):
    """Binary and the reference's plain-matrix text (%.17g, fields_io.cpp:118-136)
    both round-trip bit for bit; load() detects the format by its magic."""
    rng = np.random.default_rng(1)
    K = np.exp(rng.standard_normal(37 * 23) * 3.0)
    p = tmp_path / ("k.txt" if text else "k.bin")
    (fields.save_text if text else fields.save)(p, 37, 23, K)
    assert np.array_equal(fields.load(p, 37, 23), K)
    with pytest.raises(api.ConfigError):
        fields.load(p, 23, 37)  # fields_io.cpp:100-104: shape mismatch
    with pytest.raises(api.ConfigError):
        fields.load(tmp_path / "missing.bin", 37, 23)


def test_text_loader_reads_reference_layout(tmp_path):
    """'nx ny' then ny rows of nx values, row j = cells j*nx .. j*nx+nx-1
    (fields_io.cpp:106-113); a short file is a parse failure."""
    p = tmp_path / "m.txt"
    p.write_text("3 2\n1 2 3\n4 5.5 6e-3\n")
    assert np.array_equal(fields.load(p, 3, 2), [1, 2, 3, 4, 5.5, 6e-3])
    p.write_text("3 2\n1 2 3\n4 5\n")
    with pytest.raises(api.ConfigError):
        fields.load(p, 3, 2)


def test_philox_reference_vector():
    """Philox4x32-10 known-answer vector (Random123 kat_vectors: counter 0, key 0)."""
    from field_ref import philox
    c = philox(np.array([0], np.uint64), 0, 0)
    assert [int(x[0]) for x in c] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,lx,ly,corr,var,seed", [(64, 64, 1.0, 1.0, 0.1, 1.0, 7), (96, 40, 2.0, 1.0, 0.05, 4.0, 8),
                                                        (33, 17, 1.0, 0.5, 0.2, 0.5, 9)])
def test_exp_lognormal_matches_host(nx, ny, lx, ly, corr, var, seed):
    kd = fields.exp_lognormal(nx, ny, lx, ly, corr, var, seed)
    kh = ref_exp(nx, ny, lx, ly, corr, var, seed)
    assert np.max(np.abs(np.log(kd) - np.log(kh))) < 1e-11


@pytest.mark.gpu
def test_white_noise_bitwise():
    assert np.array_equal(fields.white_noise(200, 130, 11, 0.01), ref_white(200, 130, 11, 0.01))


@pytest.mark.gpu
def test_channels_match_host():
    kd = fields.channels(220, 60, 11.0 / 3.0, 1.0, 103)
    kh, mask = ref_channels(220, 60, 11.0 / 3.0, 1.0, 103)
    same = np.abs(np.log(kd) - np.log(kh)) < 1e-12
    assert same.mean() > 0.9999
    assert 0.35 < mask.mean() < 0.6


@pytest.mark.gpu
def test_exp_lognormal_statistics_c5_size():
    """C5's field (4096^2, l = 0.02, variance 3) on the device: finite,
    positive, and ln K with mean ~0, variance ~3 and the exponential
    correlation at one correlation length."""
    n = 4096
    K = fields.exp_lognormal(n, n, 1.0, 1.0, 0.02, 3.0, 105)
    assert np.all(np.isfinite(K)) and np.all(K > 0)
    g = np.log(K).reshape(n, n)
    assert abs(g.mean()) < 0.3
    assert 2.4 < g.var() < 3.6
    lag = int(round(0.02 * n))  # one correlation length
    c = np.mean((g[:, :-lag] - g.mean()) * (g[:, lag:] - g.mean())) / g.var()
    assert abs(c - np.exp(-1.0)) < 0.1
