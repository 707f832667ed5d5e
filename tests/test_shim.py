"""The C++ shim (shim/mrcmflow_b200.{hpp,cpp}): the reference's public C++
names and signatures (proj/include/mrcmflow/*.hpp) implemented on the C ABI.
CPU: it compiles against its header with the reference's signatures and
exports them. GPU: a reference-style caller (shim/example_run.cpp) drives
run() with snapshots, mrcm_solve, mpm_pressure_update and the sub-steps
through it, and gets the same answers as the Python mirror of the ABI."""
import os
import re
import subprocess

import numpy as np
import pytest

from cases import random_kappa, problem, rel_l2
from paper_2103_11050_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "shim")


def _build():
    subprocess.run(["make", "-s", "-C", SHIM], check=True)


def test_shim_builds_and_exports_reference_signatures():
    _build()
    out = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(SHIM, "libmrcmflow_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    for sig in [
        r"mrcmflow::run\(mrcmflow::RunInputs const&, std::vector<long, std::allocator<long> > const&, "
        r"std::function<void \(long, mrcmflow::SaturationField const&, mrcmflow::CellField const&, "
        r"mrcmflow::FaceField const&\)> const&\)",
        r"mrcmflow::mrcm_solve\(mrcmflow::CellField const&, std::shared_ptr<mrcmflow::DomainDecomposition const>, "
        r"std::shared_ptr<mrcmflow::InterfaceSpace const>, mrcmflow::RobinParameter const&, mrcmflow::CellField const&, "
        r"mrcmflow::BoundarySpec const&, mrcmflow::SolveCounters&\)",
        r"mrcmflow::mpm_pressure_update\(mrcmflow::PerturbationState const&, mrcmflow::CellField const&, "
        r"mrcmflow::CellField const&, mrcmflow::BoundarySpec const&, mrcmflow::SolveCounters&\)",
        r"mrcmflow::compute_beta\(mrcmflow::CellField const&, mrcmflow::DomainDecomposition const&, "
        r"mrcmflow::AlphaSpec const&\)",
        r"mrcmflow::epsilon\(mrcmflow::CellField const&, mrcmflow::CellField const&, mrcmflow::EpsilonMode\)",
        r"mrcmflow::cfl_timestep\(mrcmflow::FaceField const&, mrcmflow::FluidModel const&, "
        r"mrcmflow::CflPolicy const&\)",
        r"mrcmflow::upwind_step\(mrcmflow::SaturationField const&, mrcmflow::FaceField const&, double, "
        r"mrcmflow::FluidModel const&\)",
        r"mrcmflow::conductivity\(mrcmflow::CellField const&, mrcmflow::SaturationField const&, "
        r"mrcmflow::FluidModel const&\)",
        r"mrcmflow::compute_basis_set\(", r"mrcmflow::solve_particular\(", r"mrcmflow::solve_interface\(",
        r"mrcmflow::reconstruct\(", r"mrcmflow::weak_continuity_residuals\(",
    ]:
        assert re.search(sig, out), sig


@pytest.mark.gpu
def test_shim_run_matches_abi(tmp_path):
    _build()
    nx = ny = 64
    K = random_kappa(nx, ny, 9, 0.1, 10.0)
    kf = tmp_path / "K.bin"
    K.astype(np.float64).tofile(kf)
    of = tmp_path / "out.bin"
    te = 12
    res = subprocess.run([os.path.join(SHIM, "example_run"), str(kf), str(nx), str(ny), "4", "4", "5.0", str(te),
                          str(of)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    raw = np.fromfile(of, np.uint8)
    cells, faces = nx * ny, (nx + 1) * ny + nx * (ny + 1)
    off = 0

    def take(n, dt=np.float64):
        nonlocal off
        a = raw[off:off + n * np.dtype(dt).itemsize].view(dt)
        off += n * np.dtype(dt).itemsize
        return a
    s, p, u = take(cells), take(cells), take(faces)
    nrec = int(take(1, np.int64)[0])
    steps = take(2 * nrec).reshape(nrec, 2)
    nseen = int(take(1, np.int64)[0])
    seen = list(take(nseen, np.int64))
    u_mrcm, u_mpm = take(faces), take(faces)
    weak = take(2)
    prob = problem(nx, ny, 4, 4, K, M=5.0)
    sim = api.Simulator(prob)
    ref = sim.run(api.SplittingConfig(method=api.MPM2P, eta=0.01, te=te, cfl_safety=0.5))
    assert np.array_equal(s, ref.s_final) and np.array_equal(u, ref.u_final) and np.array_equal(p, ref.p_final)
    assert [int(x) for x in steps[:, 0]] == [x["rebuilt"] for x in ref.record.steps]
    assert list(steps[:, 1]) == [x["dt"] for x in ref.record.steps]
    assert seen == [0, 2, 5]
    g = api.Simulator(prob)
    gs = g.mrcm_solve(K)
    assert rel_l2(u_mrcm, gs.u) < 1e-12
    assert rel_l2(u_mpm, g.mpm_pressure_update(K * 1.05).u) < 1e-12
    assert max(weak) < 1e-8
