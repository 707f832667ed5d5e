"""ctypes mirror of include/mpm2p_b200.h (structs and function prototypes).

`load(path, prefix)` binds every entry point of a library that implements
the header under the given symbol prefix ("mpm2p_" for the CUDA product
library). The package itself only ever loads its own in-tree .so.
"""
from __future__ import annotations

import ctypes as C
import os

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class Problem(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("lx", C.c_double), ("ly", C.c_double),
        ("nsx", C.c_int32), ("nsy", C.c_int32),
        ("space_kind", C.c_int32), ("hbar_mode", C.c_int32), ("hbar_edges", C.c_int32),
        ("alpha_mode", C.c_int32), ("alpha", C.c_double), ("alpha_min", C.c_double),
        ("alpha_max", C.c_double), ("percentile_lo", C.c_double), ("percentile_hi", C.c_double),
        ("viscosity_ratio", C.c_double),
        ("K", _dp), ("q", _dp), ("bc_kind", _ip), ("bc_value", _dp),
        ("bc_beta", _dp), ("bc_robin_rhs", _dp),
    ]


class Split(C.Structure):
    _fields_ = [
        ("method", C.c_int32), ("cn", C.c_int32), ("eta", C.c_double), ("eta_mode", C.c_int32),
        ("cfl_safety", C.c_double), ("dt_cap", C.c_double), ("te", C.c_int64),
        ("pvi_max", C.c_double), ("stop_on_breakthrough", C.c_int32),
        ("max_steps_hard", C.c_int64), ("breakthrough_threshold", C.c_double),
        ("track_errors", C.c_int32), ("inflow_sat", C.c_double),
    ]


class Counters(C.Structure):
    _fields_ = [("homogeneous", C.c_int64), ("particular", C.c_int64), ("downscale", C.c_int64),
                ("fine", C.c_int64), ("interface_solves", C.c_int64)]


class StepRecord(C.Structure):
    _fields_ = [
        ("step", C.c_int64), ("pvi", C.c_double), ("epsilon", C.c_double), ("rebuilt", C.c_int32),
        ("flux_err", C.c_double), ("sat_err", C.c_double), ("bf_homog_cum", C.c_int64),
        ("bf_part_cum", C.c_int64), ("dt", C.c_double), ("wall_s", C.c_double),
        ("div_residual", C.c_double),
    ]


class RunRecord(C.Structure):
    _fields_ = [
        ("breakthrough_step", C.c_int64), ("breakthrough_pvi", C.c_double), ("te", C.c_int64),
        ("tm_updates", C.c_int64), ("tm_total", C.c_int64), ("nhat", C.c_int64),
        ("n_sub", C.c_int32), ("counters", Counters), ("max_div_residual", C.c_double),
        ("max_div_ratio", C.c_double), ("repair_warnings", C.c_int32), ("final_pvi", C.c_double),
        ("min_eps_margin", C.c_double), ("clamp_count", C.c_int64),
        ("interface_krylov", C.c_int32), ("interface_max_iterations", C.c_int32),
        ("interface_iterations", C.c_int64), ("min_rcond", C.c_double),
    ]


class DownscaleInfo(C.Structure):
    _fields_ = [("repair_max", C.c_double), ("flux_scale", C.c_double), ("repair_warning", C.c_int32),
                ("div_residual", C.c_double), ("div_scale", C.c_double)]


class Sizes(C.Structure):
    _fields_ = [
        ("cells", C.c_int32), ("faces", C.c_int32), ("bfaces", C.c_int32), ("n_sub", C.c_int32),
        ("n_interfaces", C.c_int32), ("skeleton_edges", C.c_int32), ("dim_flux", C.c_int32),
        ("dim_pressure", C.c_int32), ("nhat", C.c_int64), ("sub_nx", C.c_int32), ("sub_ny", C.c_int32),
        ("sub_faces", C.c_int32),
    ]


_vp = C.c_void_p
SNAPSHOT_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, _dp, _dp, _dp)  # mpm2p_snapshot_fn
PROTOTYPES = {
    "create": (C.c_int, [C.POINTER(Problem), C.POINTER(_vp)]),
    "destroy": (None, [_vp]),
    "last_error": (C.c_char_p, [_vp]),
    "create_error": (C.c_char_p, []),
    "get_sizes": (C.c_int, [_vp, C.POINTER(Sizes)]),
    "conductivity": (C.c_int, [_vp, _dp, _dp]),
    "max_fractional_flow_slope": (C.c_int, [_vp, _dp]),
    "cfl_timestep": (C.c_int, [_vp, _dp, C.c_double, C.c_double, _dp]),
    "upwind_step": (C.c_int, [_vp, _dp, C.c_double, _dp, C.c_double, _dp]),
    "injection_rate": (C.c_int, [_vp, _dp, C.c_double, _dp]),
    "max_outlet_saturation": (C.c_int, [_vp, _dp, _dp, _dp]),
    "divergence": (C.c_int, [_vp, _dp, _dp]),
    "fine_solve": (C.c_int, [_vp, _dp, _dp, _dp]),
    "fine_stats": (C.c_int, [_vp, C.POINTER(C.c_int32), _dp, _dp, _dp]),
    "epsilon": (C.c_int, [_vp, _dp, _dp, C.c_int32, _dp]),
    "compute_beta": (C.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "mrcm_solve": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp, C.POINTER(DownscaleInfo), C.POINTER(Counters)]),
    "mpm_update": (C.c_int, [_vp, _dp, _dp, _dp, _dp, C.POINTER(DownscaleInfo), C.POINTER(Counters)]),
    "interface_matrix": (C.c_int, [_vp, _dp]),
    # MRCM sub-steps (mrcm.hpp:77-136, 157-161)
    "compute_basis_set": (C.c_int, [_vp, _dp, _dp, _dp, C.POINTER(Counters)]),
    "restrict_physical_data": (C.c_int, [_vp, _dp, _ip, _dp, _dp, _dp]),
    "solve_particular": (C.c_int, [_vp, _dp, _ip, _dp, _dp, _dp, _dp, _dp, _dp, C.POINTER(Counters)]),
    "solve_interface": (C.c_int, [_vp, _dp, _dp, C.POINTER(Counters)]),
    "reconstruct": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
    "averaged_skeleton_flux": (C.c_int, [_vp, _dp, _dp]),
    "downscale": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp, C.POINTER(DownscaleInfo), C.POINTER(Counters)]),
    "weak_continuity_residuals": (C.c_int, [_vp, _dp, _dp, _dp, _dp]),
    "run": (C.c_int, [_vp, C.POINTER(Split), _dp, _dp, _dp, _dp, C.POINTER(StepRecord), C.c_int64,
                      C.POINTER(RunRecord)]),
    "run_snapshots": (C.c_int, [_vp, C.POINTER(Split), _dp, _dp, _dp, _dp, C.POINTER(StepRecord), C.c_int64,
                                C.POINTER(RunRecord), C.POINTER(C.c_int64), C.c_int64, SNAPSHOT_FN, _vp]),
    "run_begin": (C.c_int, [_vp, C.POINTER(Split), _dp, C.POINTER(StepRecord)]),
    "run_step": (C.c_int, [_vp, C.POINTER(StepRecord), C.POINTER(C.c_int32)]),
    "run_read": (C.c_int, [_vp, _dp, _dp, _dp]),
    "run_end": (C.c_int, [_vp, C.POINTER(RunRecord)]),
    "rcr": (C.c_double, [C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
}

# Instrumentation entry points (product library only).
INSTR_PROTOTYPES = {
    "set_device": (C.c_int, [C.c_int32]),
    "timer_record": (C.c_int, [_vp, C.c_int32]),
    "timer_elapsed": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp]),
    "flush_l2": (C.c_int, [_vp]),
    "profile_enable": (C.c_int, [_vp, C.c_int32]),
    "profile_report": (C.c_int, [_vp, C.c_char_p, C.c_int32]),
}

# Status codes (errors.hpp:9-24 mapped by the header).
OK, ECONFIG, ENUMERIC, ECAPACITY, ECUDA, EINTERNAL = 0, 2, 3, 4, 5, 6


class Lib:
    """A bound implementation of the header (one shared object + prefix)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.prefix = prefix
        self.dll = C.CDLL(path)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(self.dll, prefix + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)
        for name, (res, args) in INSTR_PROTOTYPES.items():
            fn = getattr(self.dll, prefix + name, None)
            if fn is not None:
                fn.restype = res
                fn.argtypes = args
                setattr(self, name, fn)

    def symbols(self):
        return [self.prefix + n for n in PROTOTYPES]


def load(path: str, prefix: str) -> Lib:
    return Lib(path, prefix)


def dptr(a):
    """numpy float64 array -> double* (or NULL for None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def iptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_ip)
