"""Seeded permeability fields generated on the device, and the field files
(include/mpm2p_fields.h, csrc/fields.cu).

The reference's generate_gaussian (proj/src/fields_io.cpp:25-85) uses a dense
Cholesky and stops at 2^16 cells; these are the BASELINE configs' generators
(configs.py) at any size, with counter-based normals so a field depends only
on (shape, parameters, seed). load() reads the reference's plain-matrix text
(fields_io.cpp:91-116) or the binary format; save()/save_text() write them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import api

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmpm2p_fields.so")
_LIB = None
_dp = C.POINTER(C.c_double)


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"field library not built: {LIB_PATH} (run __graft_entry__.build())")
        d = C.CDLL(LIB_PATH)
        d.mpm2p_field_error.restype = C.c_char_p
        d.mpm2p_field_exp_lognormal.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                                C.c_double, C.c_uint64, _dp]
        d.mpm2p_field_white_noise.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_uint64, _dp]
        d.mpm2p_field_channels.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_double,
                                           C.c_double, C.c_double, C.c_double, C.c_double, _dp]
        for nm in ("mpm2p_field_save", "mpm2p_field_save_text", "mpm2p_field_load"):
            getattr(d, nm).argtypes = [C.c_char_p, C.c_int32, C.c_int32, _dp]
        _LIB = d
    return _LIB


_ERR = {2: api.ConfigError, 4: api.CapacityError, 5: api.CudaError, 6: api.InternalError}


def _check(rc):
    if rc != 0:
        raise _ERR.get(rc, RuntimeError)(_lib().mpm2p_field_error().decode())


def exp_lognormal(nx, ny, lx, ly, corr_len, variance, seed):
    K = np.empty(nx * ny)
    _check(_lib().mpm2p_field_exp_lognormal(nx, ny, lx, ly, corr_len, variance, seed, K.ctypes.data_as(_dp)))
    return K


def white_noise(nx, ny, seed, amp=0.01):
    K = np.empty(nx * ny)
    _check(_lib().mpm2p_field_white_noise(nx, ny, amp, seed, K.ctypes.data_as(_dp)))
    return K


def channels(nx, ny, lx, ly, seed, coverage=0.4, k_chan=1000.0, sd_chan=0.5, k_back=0.01, sd_back=1.0):
    K = np.empty(nx * ny)
    _check(_lib().mpm2p_field_channels(nx, ny, lx, ly, seed, coverage, k_chan, sd_chan, k_back, sd_back,
                                       K.ctypes.data_as(_dp)))
    return K


def save(path, nx, ny, K):
    K = np.ascontiguousarray(K, np.float64).ravel()
    _check(_lib().mpm2p_field_save(os.fsencode(path), nx, ny, K.ctypes.data_as(_dp)))


def save_text(path, nx, ny, K):
    K = np.ascontiguousarray(K, np.float64).ravel()
    _check(_lib().mpm2p_field_save_text(os.fsencode(path), nx, ny, K.ctypes.data_as(_dp)))


def load(path, nx, ny):
    K = np.empty(nx * ny)
    _check(_lib().mpm2p_field_load(os.fsencode(path), nx, ny, K.ctypes.data_as(_dp)))
    return K
