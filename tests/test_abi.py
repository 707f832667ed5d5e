"""The C-ABI library loads and exports every symbol include/mpm2p_b200.h
declares; the ctypes mirror matches the C struct layouts; the closed-form
decomposition tables the kernels use equal the reference-style tables of the
oracle, bit for bit. No GPU needed (no compute calls)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2103_11050_b200 import _abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpm2p_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mpm2p_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(api.LIB_PATH)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared()) >= 30


def test_oracle_exports_the_same_interface(oracle):
    skip = {"mpm2p_timer_record", "mpm2p_timer_elapsed", "mpm2p_flush_l2", "mpm2p_profile_enable",
            "mpm2p_profile_report", "mpm2p_set_device"}
    missing = [s for s in declared() if s not in skip and not hasattr(oracle.dll, "oracle_" + s[6:])]
    assert not missing, missing


def test_ctypes_struct_layout_matches_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "mpm2p_b200.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(mpm2p_problem),sizeof(mpm2p_split),sizeof(mpm2p_counters),sizeof(mpm2p_step_record),'
                   'sizeof(mpm2p_run_record),sizeof(mpm2p_downscale_info),sizeof(mpm2p_sizes),'
                   'offsetof(mpm2p_problem,K),offsetof(mpm2p_split,inflow_sat),offsetof(mpm2p_run_record,clamp_count));'
                   'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(_abi.Problem), C.sizeof(_abi.Split), C.sizeof(_abi.Counters), C.sizeof(_abi.StepRecord),
            C.sizeof(_abi.RunRecord), C.sizeof(_abi.DownscaleInfo), C.sizeof(_abi.Sizes),
            _abi.Problem.K.offset, _abi.Split.inflow_sat.offset, _abi.RunRecord.clamp_count.offset]
    assert got == want


def _tables(lib_fn, prob, s, nbe, maxh=512):
    edges = np.zeros(8 * nbe, np.int32)
    cols = np.zeros(maxh, np.int32)
    nh = C.c_int32()
    rc = lib_fn(C.byref(prob), s, edges.ctypes.data_as(C.POINTER(C.c_int32)),
                cols.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nh))
    assert rc == 0
    return edges.reshape(nbe, 8), cols[:nh.value]


@pytest.mark.parametrize("nx,ny,nsx,nsy,space,hbar", [
    (64, 64, 4, 4, api.SPACE_CONSTANT, api.HBAR_WHOLE),
    (16, 16, 2, 2, api.SPACE_CONSTANT, api.HBAR_PER_EDGE),
    (300, 50, 15, 5, api.SPACE_CONSTANT, api.HBAR_PER_EDGE),
    (220, 60, 11, 3, api.SPACE_LINEAR, api.HBAR_WHOLE),
    (12, 6, 3, 2, api.SPACE_CONSTANT, api.HBAR_HALF),
    (16, 8, 4, 1, api.SPACE_CONSTANT, api.HBAR_WHOLE),
    (8, 16, 1, 4, api.SPACE_LINEAR, api.HBAR_WHOLE),
    (12, 10, 1, 1, api.SPACE_CONSTANT, api.HBAR_WHOLE),
])
def test_layout_tables_bit_exact(oracle, nx, ny, nsx, nsy, space, hbar):
    gpu = C.CDLL(api.LIB_PATH)
    for f in (gpu.mpm2p_layout_tables, oracle.dll.oracle_layout_tables):
        f.restype = C.c_int
    K = np.ones(nx * ny)
    prob = api.Problem(nx, ny, float(nx) / 10, float(ny) / 10, nsx, nsy, K, api.pressure_drop(nx, ny),
                       space_kind=space, hbar_mode=hbar)
    cp, keep = prob.to_c()
    nbe = 2 * (nx // nsx + ny // nsy)
    for s in range(nsx * nsy):
        eg, cg = _tables(gpu.mpm2p_layout_tables, cp, s, nbe)
        eo, co = _tables(oracle.dll.oracle_layout_tables, cp, s, nbe)
        assert np.array_equal(eg, eo), s
        assert np.array_equal(cg, co), s


def test_indivisible_segment_is_a_config_error(oracle):
    """test_mrcm.cpp:207-210 (segment length 5 on 16-edge interfaces)."""
    nx = ny = 64
    prob = api.Problem(nx, ny, 1.0, 1.0, 4, 4, np.ones(nx * ny), api.pressure_drop(nx, ny),
                       hbar_mode=api.HBAR_SEGMENT, hbar_edges=5)
    with pytest.raises(api.ConfigError):
        api.Simulator(prob, oracle)
    cp, keep = prob.to_c()
    gpu = C.CDLL(api.LIB_PATH)
    e = np.zeros(8 * 32, np.int32)
    c = np.zeros(64, np.int32)
    n = C.c_int32()
    assert gpu.mpm2p_layout_tables(C.byref(cp), 0, e.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p),
                                   C.byref(n)) == _abi.ECONFIG
