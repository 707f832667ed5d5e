"""Host-side mirror of the reference's C++ API for the MPM-2P / MRCM path.

Names, argument meaning and error behaviour follow proj/include/mrcmflow/
(simulation.hpp, mrcm.hpp, mpm.hpp, transport.hpp, robin.hpp): a `Simulator`
holds what `prepare()` builds (grid, decomposition, interface space, boundary
spec, fluid, alpha spec; config.cpp:568-611) and exposes `run`,
`mrcm_solve`, `mpm_pressure_update`, `compute_beta`, `epsilon`,
`cfl_timestep`, `upwind_step`, `conductivity`, ... Every call goes through the
C ABI of include/mpm2p_b200.h into hand-written sm_100a kernels; there is no
host fallback — constructing a Simulator without the CUDA library or a GPU
raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Optional

import numpy as np

from . import _abi
from ._abi import dptr, iptr

# enums (include/mpm2p_b200.h)
PRESSURE, FLUX, ROBIN = 0, 1, 2
SPACE_CONSTANT, SPACE_LINEAR = 0, 1
HBAR_WHOLE, HBAR_HALF, HBAR_PER_EDGE, HBAR_SEGMENT = 0, 1, 2, 3
ALPHA_UNIFORM, ALPHA_ADAPTIVE = 0, 1
EPS_RELATIVE, EPS_ABSOLUTE, EPS_MOBILITY = 0, 1, 2
FINE_REFERENCE, MRCM_EVERY_STEP, MPM2P, MPM2P_NO_UPDATES = 0, 1, 2, 3

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmpm2p_b200.so")


# errors.hpp:9-24
class ConfigError(RuntimeError):
    pass


class NumericError(RuntimeError):
    pass


class CapacityError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class InternalError(RuntimeError):
    pass


_ERRORS = {_abi.ECONFIG: ConfigError, _abi.ENUMERIC: NumericError, _abi.ECAPACITY: CapacityError,
           _abi.ECUDA: CudaError, _abi.EINTERNAL: InternalError}

_LIB = None


def product_lib() -> _abi.Lib:
    """The in-tree CUDA library; fails loudly when it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        _LIB = _abi.load(LIB_PATH, "mpm2p_")
    return _LIB


@dataclasses.dataclass
class BoundarySpec:
    """Per-face physical conditions in W(ny) E(ny) S(nx) N(nx) order (elliptic.hpp:33-55)."""
    kind: np.ndarray   # int32, PRESSURE, FLUX or ROBIN
    value: np.ndarray  # float64: pressure g, or outward normal velocity z
    beta: Optional[np.ndarray] = None       # Robin faces: -beta u.n_out + p_face = robin_rhs
    robin_rhs: Optional[np.ndarray] = None

    @staticmethod
    def uniform(nx: int, ny: int, w, e, s, n) -> "BoundarySpec":
        """BoundarySpec::uniform (elliptic.cpp:28-40); each side is (kind, value)."""
        kind = np.empty(2 * (nx + ny), np.int32)
        val = np.empty(2 * (nx + ny), np.float64)
        beta = np.zeros(2 * (nx + ny))
        rhs = np.zeros(2 * (nx + ny))
        for side, sl in ((w, slice(0, ny)), (e, slice(ny, 2 * ny)), (s, slice(2 * ny, 2 * ny + nx)),
                         (n, slice(2 * ny + nx, 2 * (nx + ny)))):
            kind[sl] = side[0]
            if side[0] == ROBIN:  # (ROBIN, beta, robin_rhs): FaceBc::robin (elliptic.hpp:27)
                val[sl] = 0.0
                beta[sl] = side[1]
                rhs[sl] = side[2]
            else:
                val[sl] = side[1]
        if np.any(kind == ROBIN):
            return BoundarySpec(kind, val, beta, rhs)
        return BoundarySpec(kind, val)

    def pure_neumann(self) -> bool:
        return bool(np.all(self.kind == FLUX))


def pressure_drop(nx, ny, pl=1.0, pr=0.0) -> BoundarySpec:  # config.cpp:528-529
    return BoundarySpec.uniform(nx, ny, (PRESSURE, pl), (PRESSURE, pr), (FLUX, 0.0), (FLUX, 0.0))


def unit_inflow(nx, ny) -> BoundarySpec:  # config.cpp:530-532
    return BoundarySpec.uniform(nx, ny, (FLUX, -1.0), (PRESSURE, 0.0), (FLUX, 0.0), (FLUX, 0.0))


@dataclasses.dataclass
class AlphaSpec:  # robin.hpp:15-22
    mode: int = ALPHA_UNIFORM
    alpha: float = 1.0
    alpha_min: float = 1e-2
    alpha_max: float = 1e2
    percentile_lo: float = 10.0
    percentile_hi: float = 90.0


@dataclasses.dataclass
class SplittingConfig:  # simulation.hpp:18-31
    method: int = MPM2P
    cn: int = 1
    eta: float = 0.01
    eta_mode: int = EPS_RELATIVE
    cfl_safety: float = 0.9
    dt_cap: float = 1.0
    te: int = 0
    pvi_max: float = 0.0
    stop_on_breakthrough: bool = False
    max_steps_hard: int = 50000
    breakthrough_threshold: float = 0.05
    track_errors: bool = False  # fine-reference shadow run + flux/saturation error records (simulation.cpp:133-150)


@dataclasses.dataclass
class Problem:
    """prepare()'s output without the splitting policy (RunInputs, simulation.hpp:99-110)."""
    nx: int
    ny: int
    lx: float
    ly: float
    nsx: int
    nsy: int
    K: np.ndarray
    bc: BoundarySpec
    viscosity_ratio: float = 1.0
    q: Optional[np.ndarray] = None
    space_kind: int = SPACE_CONSTANT
    hbar_mode: int = HBAR_WHOLE
    hbar_edges: int = 0
    alpha: AlphaSpec = dataclasses.field(default_factory=AlphaSpec)

    def to_c(self):
        K = np.ascontiguousarray(self.K, np.float64).ravel()
        q = None if self.q is None else np.ascontiguousarray(self.q, np.float64).ravel()
        kind = np.ascontiguousarray(self.bc.kind, np.int32)
        val = np.ascontiguousarray(self.bc.value, np.float64)
        rb = None if self.bc.beta is None else np.ascontiguousarray(self.bc.beta, np.float64)
        rr = None if self.bc.robin_rhs is None else np.ascontiguousarray(self.bc.robin_rhs, np.float64)
        keep = (K, q, kind, val, rb, rr)
        a = self.alpha
        p = _abi.Problem(self.nx, self.ny, self.lx, self.ly, self.nsx, self.nsy, self.space_kind, self.hbar_mode,
                         self.hbar_edges, a.mode, a.alpha, a.alpha_min, a.alpha_max, a.percentile_lo,
                         a.percentile_hi, self.viscosity_ratio, dptr(K), dptr(q), iptr(kind), dptr(val),
                         dptr(rb), dptr(rr))
        return p, keep


def split_to_c(sp: SplittingConfig, inflow_sat: float) -> _abi.Split:
    return _abi.Split(sp.method, sp.cn, sp.eta, sp.eta_mode, sp.cfl_safety, sp.dt_cap, sp.te, sp.pvi_max,
                      int(sp.stop_on_breakthrough), sp.max_steps_hard, sp.breakthrough_threshold,
                      int(sp.track_errors), inflow_sat)


@dataclasses.dataclass
class DownscaleInfo:
    repair_max: float
    flux_scale: float
    repair_warning: bool
    div_residual: float
    div_scale: float


@dataclasses.dataclass
class SolveCounters:  # mrcm.hpp:15-21
    homogeneous: int = 0
    particular: int = 0
    downscale: int = 0
    fine: int = 0
    interface_solves: int = 0


@dataclasses.dataclass
class GlobalSolution:  # mrcm.hpp:139-149
    p: np.ndarray
    u: np.ndarray
    coeffs: np.ndarray  # U_H then P_H
    info: DownscaleInfo
    counters: SolveCounters


@dataclasses.dataclass
class RunRecord:  # simulation.hpp:47-62
    steps: List[dict]
    breakthrough_step: int
    breakthrough_pvi: float
    te: int
    tm_updates: int
    tm_total: int
    nhat: int
    n_sub: int
    counters: SolveCounters
    max_div_residual: float
    max_div_ratio: float
    repair_warnings: int
    final_pvi: float
    min_eps_margin: float
    clamp_count: int
    interface_krylov: int = 0
    interface_max_iterations: int = 0
    interface_iterations: int = 0
    min_rcond: float = -1.0

    @property
    def update_steps(self):
        return [s["step"] for s in self.steps if s["rebuilt"]]


@dataclasses.dataclass
class RunResult:  # simulation.hpp:112-117
    record: RunRecord
    s_final: np.ndarray
    p_final: np.ndarray
    u_final: np.ndarray


def _step_dict(r: _abi.StepRecord) -> dict:
    return {f: getattr(r, f) for f, _ in _abi.StepRecord._fields_}


def _counters(c: _abi.Counters) -> SolveCounters:
    return SolveCounters(c.homogeneous, c.particular, c.downscale, c.fine, c.interface_solves)


def _record(steps, r: _abi.RunRecord) -> RunRecord:
    return RunRecord(steps, r.breakthrough_step, r.breakthrough_pvi, r.te, r.tm_updates, r.tm_total, r.nhat,
                     r.n_sub, _counters(r.counters), r.max_div_residual, r.max_div_ratio, r.repair_warnings,
                     r.final_pvi, r.min_eps_margin, r.clamp_count, r.interface_krylov,
                     r.interface_max_iterations, r.interface_iterations, r.min_rcond)


class Simulator:
    """One prepared problem bound to an implementation of the C ABI."""

    def __init__(self, problem: Problem, lib: Optional[_abi.Lib] = None):
        self.lib = lib if lib is not None else product_lib()
        self.problem = problem
        cp, self._keep = problem.to_c()
        h = C.c_void_p()
        rc = self.lib.create(C.byref(cp), C.byref(h))
        if rc != _abi.OK:
            msg = self.lib.create_error().decode()
            raise _ERRORS.get(rc, RuntimeError)(msg)
        self.h = h
        sz = _abi.Sizes()
        self.lib.get_sizes(self.h, C.byref(sz))
        self.sizes = sz
        self.cells, self.faces = sz.cells, sz.faces
        self.dim = sz.dim_flux + sz.dim_pressure

    def close(self):
        if getattr(self, "h", None):
            self.lib.destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        if rc != _abi.OK:
            raise _ERRORS.get(rc, RuntimeError)(self.lib.last_error(self.h).decode())

    @staticmethod
    def _f64(a, n):
        a = np.ascontiguousarray(a, np.float64).ravel()
        if a.size != n:
            raise ConfigError(f"expected {n} values, got {a.size}")
        return a

    # ---- transport (transport.hpp:41-50) ----
    def conductivity(self, s):
        s = self._f64(s, self.cells)
        out = np.empty(self.cells)
        self._check(self.lib.conductivity(self.h, dptr(s), dptr(out)))
        return out

    def max_fractional_flow_slope(self):
        v = C.c_double()
        self._check(self.lib.max_fractional_flow_slope(self.h, C.byref(v)))
        return v.value

    def cfl_timestep(self, u, safety=0.9, dt_cap=1.0):
        u = self._f64(u, self.faces)
        v = C.c_double()
        self._check(self.lib.cfl_timestep(self.h, dptr(u), safety, dt_cap, C.byref(v)))
        return v.value

    def upwind_step(self, s, inflow, u, dt):
        s = self._f64(s, self.cells)
        u = self._f64(u, self.faces)
        out = np.empty(self.cells)
        self._check(self.lib.upwind_step(self.h, dptr(s), inflow, dptr(u), dt, dptr(out)))
        return out

    def injection_rate(self, u, inflow=1.0):
        u = self._f64(u, self.faces)
        v = C.c_double()
        self._check(self.lib.injection_rate(self.h, dptr(u), inflow, C.byref(v)))
        return v.value

    def max_outlet_saturation(self, s, u):
        s = self._f64(s, self.cells)
        u = self._f64(u, self.faces)
        v = C.c_double()
        self._check(self.lib.max_outlet_saturation(self.h, dptr(s), dptr(u), C.byref(v)))
        return v.value

    def divergence(self, u):
        u = self._f64(u, self.faces)
        out = np.empty(self.cells)
        self._check(self.lib.divergence(self.h, dptr(u), dptr(out)))
        return out

    # ---- fine-reference solve (simulation.cpp:143-150; elliptic.cpp:245-250) ----
    def fine_solve(self, kappa):
        """solve_cell_centered on the whole grid: (p cells, u faces). Anchor cell 0
        iff every physical face is Flux. Device PCG (fine.cu), NumericError if it
        does not converge."""
        kappa = self._f64(kappa, self.cells)
        p = np.empty(self.cells)
        u = np.empty(self.faces)
        self._check(self.lib.fine_solve(self.h, dptr(kappa), dptr(p), dptr(u)))
        return p, u

    def fine_stats(self):
        """(iterations, relative residual, conservation_residual, residual_scale) of the last fine solve."""
        it = C.c_int32()
        rr, dr, ds = C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.fine_stats(self.h, C.byref(it), C.byref(rr), C.byref(dr), C.byref(ds)))
        return it.value, rr.value, dr.value, ds.value

    # ---- drift (mpm.hpp:20) ----
    def epsilon(self, kappa_n, kappa_m, mode=EPS_RELATIVE):
        a = self._f64(kappa_n, self.cells)
        b = self._f64(kappa_m, self.cells)
        v = C.c_double()
        self._check(self.lib.epsilon(self.h, dptr(a), dptr(b), mode, C.byref(v)))
        return v.value

    # ---- coupling (robin.hpp:37-38) ----
    def compute_beta(self, kappa):
        k = self._f64(kappa, self.cells)
        E = self.sizes.skeleton_edges
        bm, bp, al = np.empty(E), np.empty(E), np.empty(E)
        self._check(self.lib.compute_beta(self.h, dptr(k), dptr(bm), dptr(bp), dptr(al)))
        return bm, bp, al

    # ---- MRCM / MPM-2P (mrcm.hpp:151-153, mpm.hpp:53-55) ----
    def mrcm_solve(self, kappa, beta=None) -> GlobalSolution:
        k = self._f64(kappa, self.cells)
        bm = bp = None
        if beta is not None:
            bm = self._f64(beta[0], self.sizes.skeleton_edges)
            bp = self._f64(beta[1], self.sizes.skeleton_edges)
        p, u, co = np.empty(self.cells), np.empty(self.faces), np.empty(max(self.dim, 1))
        info, cnt = _abi.DownscaleInfo(), _abi.Counters()
        self._check(self.lib.mrcm_solve(self.h, dptr(k), dptr(bm), dptr(bp), dptr(p), dptr(u), dptr(co),
                                        C.byref(info), C.byref(cnt)))
        return GlobalSolution(p, u, co[:self.dim], DownscaleInfo(info.repair_max, info.flux_scale,
                              bool(info.repair_warning), info.div_residual, info.div_scale), _counters(cnt))

    def mpm_pressure_update(self, kappa_n) -> GlobalSolution:
        k = self._f64(kappa_n, self.cells)
        p, u, co = np.empty(self.cells), np.empty(self.faces), np.empty(max(self.dim, 1))
        info, cnt = _abi.DownscaleInfo(), _abi.Counters()
        self._check(self.lib.mpm_update(self.h, dptr(k), dptr(p), dptr(u), dptr(co), C.byref(info),
                                        C.byref(cnt)))
        return GlobalSolution(p, u, co[:self.dim], DownscaleInfo(info.repair_max, info.flux_scale,
                              bool(info.repair_warning), info.div_residual, info.div_scale), _counters(cnt))

    # ---- MRCM sub-steps (mrcm.hpp:77-136, 157-161) ----
    # LocalData / LocalSolution are dicts of per-subdomain arrays (subdomain-major):
    #   q, p: [n_sub, sub_nx*sub_ny]; u: [n_sub, sub_faces]; kind, value, beta,
    #   robin_rhs, boundary_p: [n_sub, 2(sub_nx+sub_ny)] (W, E, S, N)
    def _shapes(self):
        sz = self.sizes
        return sz.n_sub, sz.sub_nx * sz.sub_ny, sz.sub_faces, 2 * (sz.sub_nx + sz.sub_ny)

    def compute_basis_set(self, kappa, beta=None) -> SolveCounters:
        k = self._f64(kappa, self.cells)
        bm = bp = None
        if beta is not None:
            bm = self._f64(beta[0], self.sizes.skeleton_edges)
            bp = self._f64(beta[1], self.sizes.skeleton_edges)
        cnt = _abi.Counters()
        self._check(self.lib.compute_basis_set(self.h, dptr(k), dptr(bm), dptr(bp), C.byref(cnt)))
        return _counters(cnt)

    def restrict_physical_data(self) -> dict:
        ns, nc, nf, ne = self._shapes()
        d = {"q": np.empty((ns, nc)), "kind": np.empty((ns, ne), np.int32), "value": np.empty((ns, ne)),
             "beta": np.empty((ns, ne)), "robin_rhs": np.empty((ns, ne))}
        self._check(self.lib.restrict_physical_data(self.h, dptr(d["q"]), iptr(d["kind"]), dptr(d["value"]),
                                                    dptr(d["beta"]), dptr(d["robin_rhs"])))
        return d

    def solve_particular(self, data: dict):
        ns, nc, nf, ne = self._shapes()
        q = self._f64(data["q"], ns * nc)
        kind = np.ascontiguousarray(data["kind"], np.int32).ravel()
        val, beta, rr = (self._f64(data[k], ns * ne) for k in ("value", "beta", "robin_rhs"))
        out = {"p": np.empty((ns, nc)), "u": np.empty((ns, nf)), "boundary_p": np.empty((ns, ne))}
        cnt = _abi.Counters()
        self._check(self.lib.solve_particular(self.h, dptr(q), iptr(kind), dptr(val), dptr(beta), dptr(rr),
                                              dptr(out["p"]), dptr(out["u"]), dptr(out["boundary_p"]),
                                              C.byref(cnt)))
        return out, _counters(cnt)

    def solve_interface(self, particular: dict):
        ns, nc, nf, ne = self._shapes()
        u = self._f64(particular["u"], ns * nf)
        co = np.empty(max(self.dim, 1))
        cnt = _abi.Counters()
        self._check(self.lib.solve_interface(self.h, dptr(u), dptr(co), C.byref(cnt)))
        return co[:self.dim], _counters(cnt)

    def reconstruct(self, coeffs, particular: dict) -> dict:
        ns, nc, nf, ne = self._shapes()
        co = self._f64(coeffs, self.dim) if self.dim else np.zeros(1)
        p, u, bp = (self._f64(particular[k], n) for k, n in (("p", ns * nc), ("u", ns * nf),
                                                              ("boundary_p", ns * ne)))
        out = {"p": np.empty((ns, nc)), "u": np.empty((ns, nf)), "boundary_p": np.empty((ns, ne))}
        self._check(self.lib.reconstruct(self.h, dptr(co), dptr(p), dptr(u), dptr(bp), dptr(out["p"]),
                                         dptr(out["u"]), dptr(out["boundary_p"])))
        return out

    def averaged_skeleton_flux(self, recon: dict):
        ns, nc, nf, ne = self._shapes()
        u = self._f64(recon["u"], ns * nf)
        out = np.empty(max(self.sizes.skeleton_edges, 1))
        self._check(self.lib.averaged_skeleton_flux(self.h, dptr(u), dptr(out)))
        return out[:self.sizes.skeleton_edges]

    def downscale(self, kappa, recon: dict, skeleton_flux):
        ns, nc, nf, ne = self._shapes()
        k = self._f64(kappa, self.cells)
        p, u = self._f64(recon["p"], ns * nc), self._f64(recon["u"], ns * nf)
        fl = self._f64(skeleton_flux, self.sizes.skeleton_edges) if self.sizes.skeleton_edges else np.zeros(1)
        po, uo = np.empty(self.cells), np.empty(self.faces)
        info, cnt = _abi.DownscaleInfo(), _abi.Counters()
        self._check(self.lib.downscale(self.h, dptr(k), dptr(p), dptr(u), dptr(fl), dptr(po), dptr(uo),
                                       C.byref(info), C.byref(cnt)))
        return po, uo, DownscaleInfo(info.repair_max, info.flux_scale, bool(info.repair_warning),
                                     info.div_residual, info.div_scale), _counters(cnt)

    def weak_continuity_residuals(self, recon: dict):
        ns, nc, nf, ne = self._shapes()
        u, bp = self._f64(recon["u"], ns * nf), self._f64(recon["boundary_p"], ns * ne)
        fj, pj = C.c_double(), C.c_double()
        self._check(self.lib.weak_continuity_residuals(self.h, dptr(u), dptr(bp), C.byref(fj), C.byref(pj)))
        return fj.value, pj.value

    def interface_matrix(self):
        M = np.empty((self.dim, self.dim))
        self._check(self.lib.interface_matrix(self.h, dptr(M)))
        return M

    # ---- driver (simulation.hpp:127-128) ----
    def run(self, split: SplittingConfig, s0=None, inflow_sat=1.0, max_records=None, snapshot_steps=(),
            snap=None) -> RunResult:
        """run(in, snapshot_steps, snap) (simulation.hpp:119-128): snap(step, s, p, u)
        is called with copies of the fields after each listed step's record."""
        s0 = np.zeros(self.cells) if s0 is None else self._f64(s0, self.cells)
        cs = split_to_c(split, inflow_sat)
        n_rec = max_records or (split.te if split.te > 0 else split.max_steps_hard) + 1
        recs = (_abi.StepRecord * n_rec)()
        rr = _abi.RunRecord()
        s, p, u = np.empty(self.cells), np.empty(self.cells), np.empty(self.faces)
        if snap is not None and len(snapshot_steps):
            cells, faces = self.cells, self.faces

            def _cb(_user, step, sp_, pp_, up_):
                snap(int(step), np.ctypeslib.as_array(sp_, (cells,)).copy(),
                     np.ctypeslib.as_array(pp_, (cells,)).copy(), np.ctypeslib.as_array(up_, (faces,)).copy())
            cb = _abi.SNAPSHOT_FN(_cb)
            want = np.ascontiguousarray(snapshot_steps, np.int64)
            self._check(self.lib.run_snapshots(self.h, C.byref(cs), dptr(s0), dptr(s), dptr(p), dptr(u), recs, n_rec,
                                               C.byref(rr), want.ctypes.data_as(C.POINTER(C.c_int64)), want.size,
                                               cb, None))
        else:
            self._check(self.lib.run(self.h, C.byref(cs), dptr(s0), dptr(s), dptr(p), dptr(u), recs, n_rec,
                                     C.byref(rr)))
        steps = [_step_dict(recs[i]) for i in range(min(rr.te, n_rec))]
        return RunResult(_record(steps, rr), s, p, u)

    def run_begin(self, split: SplittingConfig, s0=None, inflow_sat=1.0):
        s0 = np.zeros(self.cells) if s0 is None else self._f64(s0, self.cells)
        self._split = split_to_c(split, inflow_sat)
        first = _abi.StepRecord()
        self._check(self.lib.run_begin(self.h, C.byref(self._split), dptr(s0), C.byref(first)))
        self._steps = [_step_dict(first)]
        return self._steps[0]

    def run_step(self):
        r = _abi.StepRecord()
        done = C.c_int32()
        self._check(self.lib.run_step(self.h, C.byref(r), C.byref(done)))
        if done.value:
            return None
        d = _step_dict(r)
        self._steps.append(d)
        return d

    def run_read(self):
        s, p, u = np.empty(self.cells), np.empty(self.cells), np.empty(self.faces)
        self._check(self.lib.run_read(self.h, dptr(s), dptr(p), dptr(u)))
        return s, p, u

    def run_end(self) -> RunRecord:
        rr = _abi.RunRecord()
        self._check(self.lib.run_end(self.h, C.byref(rr)))
        return _record(self._steps, rr)


def rcr(nhat, n, te, tm, lib: Optional[_abi.Lib] = None) -> float:  # simulation.cpp:11-19
    if te <= 0:
        raise ConfigError("rcr: te must be positive")
    if nhat < 0 or n < 0 or tm < 0:
        raise ConfigError("rcr: negative counter")
    if tm > te:
        raise ConfigError("rcr: tm exceeds te")
    frac = (te - tm) / te
    bf = 1.0 - 2.0 * n / (nhat + 2 * n)
    return frac * bf * 100.0
