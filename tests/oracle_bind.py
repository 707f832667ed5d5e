"""Test-only binding of the CPU oracle (oracle/liboracle.so, prefix oracle_).

The oracle is the parity checker; only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs load it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2103_11050_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")

ORACLE_LD_SO = os.path.join(ORACLE_DIR, "liboracle_ld.so")

_LIBS = {}


def oracle_lib(extended: bool = False) -> _abi.Lib:
    """The oracle; extended=True loads the long-double build (accuracy yardstick)."""
    key = bool(extended)
    if key not in _LIBS:
        so = ORACLE_LD_SO if extended else ORACLE_SO
        if not os.path.exists(so):
            subprocess.run(["make", "-s", "-C", ORACLE_DIR, os.path.basename(so)], check=True)
        lib = _abi.load(so, "oracle_")
        d = lib.dll
        d.oracle_fine_solve.restype = C.c_int
        d.oracle_fine_solve.argtypes = [C.c_void_p, _abi._dp, _abi._dp, _abi._dp]
        d.oracle_gaussian_field.restype = C.c_int
        d.oracle_gaussian_field.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                            C.c_double, C.c_uint64, C.c_int32, C.c_double, _abi._dp]
        d.oracle_weak_residuals.restype = C.c_int
        d.oracle_weak_residuals.argtypes = [C.c_void_p, _abi._dp, _abi._dp]
        d.oracle_set_interface_solver.restype = None
        d.oracle_set_interface_solver.argtypes = [C.c_int32]
        d.oracle_set_threads.restype = None
        d.oracle_set_threads.argtypes = [C.c_int32]
        _LIBS[key] = lib
    return _LIBS[key]
