"""The five BASELINE.json configurations (C1..C5) as seeded synthetic inputs.

BASELINE.json names no public dataset; every permeability field is generated
here from a per-config seed with the shapes and value distributions the
configs state, outside the hot path. Both the CUDA path
and the CPU oracle receive the same float64 array, so inputs are
bit-identical on both sides.

Porosity 0.2 is not modelled: with constant porosity the CFL step and the
saturation update scale together, so the discrete saturation sequence is
identical and only the physical-time label changes (
PVI divides by lx*ly as in proj/src/simulation.cpp:283).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import api


def exp_covariance_lognormal(nx, ny, lx, ly, corr_len, variance, seed):
    """ln K ~ Gaussian field with covariance variance*exp(-|x-y|/corr_len).

    Circulant embedding on the doubled periodic grid (FFT), negative
    embedding eigenvalues clipped to zero. Returns K row-major (j*nx + i).
    """
    hx, hy = lx / nx, ly / ny
    mx, my = 2 * nx, 2 * ny
    ix = np.minimum(np.arange(mx), mx - np.arange(mx)) * hx
    iy = np.minimum(np.arange(my), my - np.arange(my)) * hy
    r = np.sqrt(iy[:, None] ** 2 + ix[None, :] ** 2)
    c = variance * np.exp(-r / corr_len)
    lam = np.fft.fft2(c).real
    lam = np.clip(lam, 0.0, None)
    rng = np.random.default_rng(seed)
    xi = rng.standard_normal((my, mx)) + 1j * rng.standard_normal((my, mx))
    z = np.fft.fft2(np.sqrt(lam / (mx * my)) * xi)
    lnk = z.real[:ny, :nx]
    return np.exp(lnk).ravel().astype(np.float64)


def channel_field(nx, ny, lx, ly, seed, coverage=0.4, k_chan=1000.0, sd_chan=0.5, k_back=0.01, sd_back=1.0):
    """Sinuous high-k channels over a low-k background (config C3).

    Channels follow y = y0 + A sin(2 pi x / L + phi); they are added until
    about `coverage` of the cells are channel cells. ln K is Gaussian around
    ln k_chan (sd sd_chan) in channels and ln k_back (sd sd_back) elsewhere.
    """
    rng = np.random.default_rng(seed)
    x = (np.arange(nx) + 0.5) * (lx / nx)
    y = (np.arange(ny) + 0.5) * (ly / ny)
    X, Y = np.meshgrid(x, y)
    mask = np.zeros((ny, nx), bool)
    for _ in range(64):
        if mask.mean() >= coverage:
            break
        y0 = rng.uniform(0.0, ly)
        amp = rng.uniform(0.05, 0.2) * ly
        wav = rng.uniform(0.3, 0.8) * lx
        phi = rng.uniform(0.0, 2 * math.pi)
        half = rng.uniform(0.03, 0.07) * ly
        yc = y0 + amp * np.sin(2 * math.pi * X / wav + phi)
        mask |= np.abs(Y - yc) < half
    lnk = np.where(mask, rng.normal(math.log(k_chan), sd_chan, mask.shape),
                   rng.normal(math.log(k_back), sd_back, mask.shape))
    return np.exp(lnk).ravel().astype(np.float64)


def white_noise_field(nx, ny, seed, amp=0.01):
    """K = 1 + amp * U(-1, 1) (config C4)."""
    rng = np.random.default_rng(seed)
    return (1.0 + amp * rng.uniform(-1.0, 1.0, nx * ny)).astype(np.float64)


def quarter_five_spot(nx, ny, hy, k):
    """Injection through the first k west faces (total rate 1), production at
    the last k east faces (pressure 0), no flow elsewhere."""
    bc = api.BoundarySpec.uniform(nx, ny, (api.FLUX, 0.0), (api.FLUX, 0.0), (api.FLUX, 0.0), (api.FLUX, 0.0))
    bc.value[:k] = -1.0 / (k * hy)
    bc.kind[ny + ny - k: 2 * ny] = api.PRESSURE
    bc.value[ny + ny - k: 2 * ny] = 0.0
    return bc


@dataclasses.dataclass
class Config:
    name: str
    problem: api.Problem
    split: api.SplittingConfig
    inflow_sat: float = 1.0
    two_pass: bool = False  # "until breakthrough + 50%" (C3)
    description: str = ""

    @property
    def cells(self):
        return self.problem.nx * self.problem.ny

    def s0(self):
        return np.zeros(self.cells)


def build(name: str, te_override: int = 0) -> Config:
    """The BASELINE.json configs; `te_override` shortens the run (parity samples)."""
    n = name.upper()
    if n == "C1":
        nx = ny = 64
        K = exp_covariance_lognormal(nx, ny, 1.0, 1.0, 0.1, 1.0, seed=101)
        prob = api.Problem(nx, ny, 1.0, 1.0, 4, 4, K, api.unit_inflow(nx, ny), viscosity_ratio=5.0)
        sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, eta_mode=api.EPS_RELATIVE, cfl_safety=0.5, te=201)
        desc = "64x64 unit square, 4x4 subdomains of 16x16, exp-cov lognormal (l=0.1, var 1), M=5, unit inflow W / p=0 E, CFL 0.5, 200 saturation steps"
    elif n == "C2":
        nx = ny = 256
        K = exp_covariance_lognormal(nx, ny, 1.0, 1.0, 0.05, 4.0, seed=102)
        prob = api.Problem(nx, ny, 1.0, 1.0, 16, 16, K, api.pressure_drop(nx, ny), viscosity_ratio=5.0)
        sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, eta_mode=api.EPS_RELATIVE, cfl_safety=0.9, te=2001)
        desc = "256x256, 16x16 subdomains of 16x16, exp-cov lognormal (l=0.05, var 4), M=5, slab pressure drop, 2000 saturation steps"
    elif n == "C3":
        nx, ny = 220, 60
        lx, ly = 11.0 / 3.0, 1.0
        K = channel_field(nx, ny, lx, ly, seed=103)
        bc = quarter_five_spot(nx, ny, ly / ny, k=6)
        prob = api.Problem(nx, ny, lx, ly, 11, 3, K, bc, viscosity_ratio=10.0, space_kind=api.SPACE_LINEAR,
                           alpha=api.AlphaSpec(mode=api.ALPHA_ADAPTIVE))
        sp = api.SplittingConfig(method=api.MPM2P, eta=0.01, eta_mode=api.EPS_MOBILITY, cfl_safety=0.9,
                                 stop_on_breakthrough=True, max_steps_hard=20000)
        desc = "220x60 square cells, 11x3 subdomains of 20x20, channelized (~40% channels, ~5 decades), M=10, quarter-five-spot, linear spaces + adaptive alpha, to breakthrough + 50%"
        cfg = Config("C3", prob, sp, two_pass=True, description=desc)
        if te_override:
            cfg.split = dataclasses.replace(sp, stop_on_breakthrough=False, te=te_override)
            cfg.two_pass = False
        return cfg
    elif n == "C4":
        nx = ny = 512
        K = white_noise_field(nx, ny, seed=104)
        prob = api.Problem(nx, ny, 1.0, 1.0, 16, 16, K, api.pressure_drop(nx, ny), viscosity_ratio=20.0)
        sp = api.SplittingConfig(method=api.MPM2P, eta=0.05, eta_mode=api.EPS_MOBILITY, cfl_safety=0.9, te=5001)
        desc = "512x512, 16x16 subdomains of 32x32, K=1+0.01U(-1,1), M=20, slab pressure drop, mobility drift eta=0.05, 5000 saturation steps"
    elif n == "C5":
        nx = ny = 4096
        K = exp_covariance_lognormal(nx, ny, 1.0, 1.0, 0.02, 3.0, seed=105)
        prob = api.Problem(nx, ny, 1.0, 1.0, 128, 128, K, api.pressure_drop(nx, ny), viscosity_ratio=5.0)
        sp = api.SplittingConfig(method=api.MPM2P, eta=0.002, eta_mode=api.EPS_MOBILITY, cfl_safety=0.9, te=501)
        desc = "4096x4096, 128x128 subdomains of 32x32, exp-cov lognormal (l=0.02, var 3), M=5, slab pressure drop, 500 saturation steps"
    else:
        raise api.ConfigError(f"unknown config {name!r}; available: C1..C5")
    if te_override:
        sp = dataclasses.replace(sp, te=te_override)
    return Config(n, prob, sp, description=desc)


def breakthrough_plus_50(te_breakthrough_step: int) -> int:
    """te for the second C3 pass: ceil(1.5 b) + 1 elliptic solves."""
    return int(math.ceil(1.5 * te_breakthrough_step)) + 1
