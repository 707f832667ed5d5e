"""Host restatement of the device field generators (csrc/fields.cu), test
infrastructure: Philox4x32-10 in numpy uint arithmetic, Box-Muller, and the
configs.py algorithms on top of them."""
from __future__ import annotations

import math

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox(idx, stream, seed):
    """Philox4x32-10 of counters (idx lo, idx hi, stream, 0) under key = seed."""
    idx = np.asarray(idx, np.uint64)
    c0 = (idx & MASK).astype(np.uint64)
    c1 = (idx >> np.uint64(32)).astype(np.uint64)
    c2 = np.full(idx.shape, stream, np.uint64)
    c3 = np.zeros(idx.shape, np.uint64)
    k0, k1 = np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF)
    for _ in range(10):
        p0, p1 = M0 * c0, M1 * c2
        h0, l0, h1, l1 = p0 >> np.uint64(32), p0 & MASK, p1 >> np.uint64(32), p1 & MASK
        n0 = h1 ^ c1 ^ np.uint64(k0)
        n2 = h0 ^ c3 ^ np.uint64(k1)
        c0, c1, c2, c3 = n0, l1, n2, l0
        k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
        k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
    return c0, c1, c2, c3


def uniform2(idx, stream, seed):
    c0, c1, c2, c3 = philox(idx, stream, seed)
    s53 = 1.0 / 9007199254740992.0
    u1 = (((c0 >> np.uint64(5)) << np.uint64(26)) | (c1 >> np.uint64(6))).astype(np.float64) + 1.0
    u2 = (((c2 >> np.uint64(5)) << np.uint64(26)) | (c3 >> np.uint64(6))).astype(np.float64) + 1.0
    return u1 * s53, u2 * s53


def normal2(idx, stream, seed):
    u1, u2 = uniform2(idx, stream, seed)
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2)


def exp_lognormal(nx, ny, lx, ly, corr_len, variance, seed):
    hx, hy = lx / nx, ly / ny
    mx, my = 2 * nx, 2 * ny
    ix = np.minimum(np.arange(mx), mx - np.arange(mx)) * hx
    iy = np.minimum(np.arange(my), my - np.arange(my)) * hy
    r = np.sqrt(iy[:, None] ** 2 + ix[None, :] ** 2)
    c = variance * np.exp(-r / corr_len)
    lam = np.clip(np.fft.fft2(c).real, 0.0, None)
    z1, z2 = normal2(np.arange(mx * my, dtype=np.uint64), 0, seed)
    xi = (z1 + 1j * z2).reshape(my, mx)
    z = np.fft.fft2(np.sqrt(lam / (mx * my)) * xi)
    return np.exp(z.real[:ny, :nx]).ravel()


def white_noise(nx, ny, seed, amp=0.01):
    u1, _ = uniform2(np.arange(nx * ny, dtype=np.uint64), 0, seed)
    return 1.0 + amp * (2.0 * u1 - 1.0)


def channels(nx, ny, lx, ly, seed, coverage=0.4, k_chan=1000.0, sd_chan=0.5, k_back=0.01, sd_back=1.0):
    hx, hy = lx / nx, ly / ny
    X = ((np.arange(nx) + 0.5) * hx)[None, :]
    Y = ((np.arange(ny) + 0.5) * hy)[:, None]
    mask = np.zeros((ny, nx), bool)
    for t in range(64):
        if mask.sum() >= coverage * nx * ny:
            break
        u = np.concatenate([np.array(uniform2(np.array([3 * t + k], np.uint64), 1, seed)).ravel() for k in range(3)])
        y0, amp, wav = u[0] * ly, (0.05 + 0.15 * u[1]) * ly, (0.3 + 0.5 * u[2]) * lx
        phi, half = 2.0 * math.pi * u[3], (0.03 + 0.04 * u[4]) * ly
        yc = y0 + amp * np.sin(2.0 * math.pi * X / wav + phi)
        mask |= np.abs(Y - yc) < half
    z1, _ = normal2(np.arange(nx * ny, dtype=np.uint64), 2, seed)
    z1 = z1.reshape(ny, nx)
    return np.where(mask, np.exp(math.log(k_chan) + sd_chan * z1), np.exp(math.log(k_back) + sd_back * z1)).ravel(), mask.ravel()
