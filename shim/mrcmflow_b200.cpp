// mrcmflow_b200.cpp — the reference's C++ API (mrcmflow_b200.hpp) on the C ABI
// of the B200 library (include/mpm2p_b200.h). Every call maps its value
// types onto one device context (mpm2p_ctx) and rethrows the ABI's status
// codes as the reference's exception types (errors.hpp:9-24).
#include "mrcmflow_b200.hpp"

#include <algorithm>
#include <cmath>

#include "../include/mpm2p_b200.h"

namespace mrcmflow {

namespace detail {

[[noreturn]] void raise(int rc, const std::string& msg) {
    switch (rc) {
        case MPM2P_ECONFIG: throw ConfigError(msg);
        case MPM2P_ENUMERIC: throw NumericError(msg);
        case MPM2P_ECAPACITY: throw CapacityError(msg);
        default: throw std::runtime_error(msg);
    }
}

int bc_code(BcKind k) { return k == BcKind::Pressure ? MPM2P_BC_PRESSURE : k == BcKind::Flux ? MPM2P_BC_FLUX : MPM2P_BC_ROBIN; }
int hbar_code(HbarSpec::Mode m) {
    switch (m) {
        case HbarSpec::Mode::WholeInterface: return MPM2P_HBAR_WHOLE;
        case HbarSpec::Mode::HalfInterface: return MPM2P_HBAR_HALF;
        case HbarSpec::Mode::PerEdge: return MPM2P_HBAR_PER_EDGE;
        default: return MPM2P_HBAR_SEGMENT;
    }
}
int eps_code(EpsilonMode m) {
    return m == EpsilonMode::Relative ? MPM2P_EPS_RELATIVE : m == EpsilonMode::Absolute ? MPM2P_EPS_ABSOLUTE
                                                                                         : MPM2P_EPS_MOBILITY;
}

// One device context (prepare(), config.cpp:568-611) and the host arrays its
// creation read.
struct Backend {
    mpm2p_ctx* ctx = nullptr;
    mpm2p_sizes sz{};
    Backend(const DomainDecomposition& dd, const InterfaceSpace& space, const AlphaSpec& alpha,
            const BoundarySpec& bc, const CellField& K, const CellField* q, double M) {
        const StructuredGrid2D& g = dd.grid;
        if (K.size() != g.cell_count()) throw ConfigError("conductivity does not match the grid");
        if (bc.count() != 2 * (g.nx + g.ny)) throw ConfigError("boundary spec does not match the grid");
        kind.resize(bc.count());
        value.resize(bc.count());
        beta.resize(bc.count());
        rhs.resize(bc.count());
        for (int i = 0; i < bc.count(); ++i) {
            kind[i] = bc_code(bc.faces[i].kind);
            value[i] = bc.faces[i].value;
            beta[i] = bc.faces[i].beta;
            rhs[i] = bc.faces[i].robin_rhs;
        }
        mpm2p_problem p{};
        p.nx = g.nx, p.ny = g.ny, p.lx = g.lx, p.ly = g.ly, p.nsx = dd.nsx, p.nsy = dd.nsy;
        p.space_kind = space.kind == InterfaceSpace::Kind::Linear ? MPM2P_SPACE_LINEAR : MPM2P_SPACE_CONSTANT;
        p.hbar_mode = hbar_code(space.hbar.mode);
        p.hbar_edges = space.hbar.edges;
        p.alpha_mode = alpha.mode == AlphaMode::Adaptive ? MPM2P_ALPHA_ADAPTIVE : MPM2P_ALPHA_UNIFORM;
        p.alpha = alpha.alpha, p.alpha_min = alpha.alpha_min, p.alpha_max = alpha.alpha_max;
        p.percentile_lo = alpha.percentile_lo, p.percentile_hi = alpha.percentile_hi;
        p.viscosity_ratio = M;
        p.K = K.v.data();
        p.q = (q && q->size() == g.cell_count()) ? q->v.data() : nullptr;
        p.bc_kind = kind.data();
        p.bc_value = value.data();
        p.bc_beta = beta.data();
        p.bc_robin_rhs = rhs.data();
        const int rc = mpm2p_create(&p, &ctx);
        if (rc != MPM2P_OK) raise(rc, mpm2p_create_error());
        mpm2p_get_sizes(ctx, &sz);
    }
    ~Backend() {
        if (ctx) mpm2p_destroy(ctx);
    }
    Backend(const Backend&) = delete;
    Backend& operator=(const Backend&) = delete;
    void check(int rc) const {
        if (rc != MPM2P_OK) raise(rc, mpm2p_last_error(ctx));
    }
    std::vector<int32_t> kind;
    std::vector<double> value, beta, rhs;
};

// a context for grid-only work (transport, epsilon): the first decomposition
// whose subdomain fits the device's banded kernels, Flux faces, constant space
std::unique_ptr<Backend> grid_backend(const StructuredGrid2D& g, const CellField& K, double M) {
    auto pick = [](int n) {
        for (int k = 1; k <= n; ++k)
            if (n % k == 0 && n / k <= 32) return k;
        return -1;
    };
    const int nsx = pick(g.nx), nsy = pick(g.ny);
    if (nsx < 0 || nsy < 0) throw CapacityError("no subdomain split of this grid fits the device kernels");
    DomainDecomposition dd = build_decomposition(g, nsx, nsy);
    BoundarySpec bc(g.nx, g.ny);
    return std::make_unique<Backend>(dd, build_interface_space(dd, InterfaceSpace::Kind::Constant), AlphaSpec{}, bc, K,
                                     nullptr, M);
}

std::vector<double> flat_beta(const std::vector<std::vector<double>>& b) {
    std::vector<double> out;
    for (const auto& v : b) out.insert(out.end(), v.begin(), v.end());
    return out;
}

std::vector<std::vector<double>> per_interface(const DomainDecomposition& dd, const std::vector<double>& flat) {
    const int snx = dd.grid.nx / dd.nsx, sny = dd.grid.ny / dd.nsy;
    const int nv = dd.nsy * (dd.nsx - 1);
    std::vector<std::vector<double>> out(dd.interface_count());
    size_t off = 0;
    for (int k = 0; k < dd.interface_count(); ++k) {
        const int ne = k < nv ? sny : snx;
        out[k].assign(flat.begin() + off, flat.begin() + off + ne);
        off += ne;
    }
    return out;
}

SolveCounters counters_of(const mpm2p_counters& c) {
    SolveCounters s;
    s.homogeneous = c.homogeneous, s.particular = c.particular, s.downscale = c.downscale, s.fine = c.fine;
    s.interface_solves = c.interface_solves;
    return s;
}
void add(SolveCounters& a, const mpm2p_counters& c) {
    a.homogeneous += c.homogeneous, a.particular += c.particular, a.downscale += c.downscale, a.fine += c.fine;
    a.interface_solves += c.interface_solves;
}

// LocalSolution vectors <-> the ABI's subdomain-major arrays
struct Flat {
    std::vector<double> p, u, bp;
};
Flat flatten(const std::vector<LocalSolution>& v) {
    Flat f;
    for (const auto& l : v) {
        f.p.insert(f.p.end(), l.p.v.begin(), l.p.v.end());
        f.u.insert(f.u.end(), l.u.v.begin(), l.u.v.end());
        f.bp.insert(f.bp.end(), l.boundary_p.begin(), l.boundary_p.end());
    }
    return f;
}
std::vector<LocalSolution> unflatten(const DomainDecomposition& dd, const mpm2p_sizes& sz, const Flat& f) {
    std::vector<LocalSolution> out(dd.subdomain_count());
    const int nc = sz.sub_nx * sz.sub_ny, nf = sz.sub_faces, ne = 2 * (sz.sub_nx + sz.sub_ny);
    for (int s = 0; s < dd.subdomain_count(); ++s) {
        const StructuredGrid2D& lg = dd.subgrids[s];
        out[s].p = CellField(lg);
        out[s].u = FaceField(lg);
        std::copy(f.p.begin() + (size_t)s * nc, f.p.begin() + (size_t)(s + 1) * nc, out[s].p.v.begin());
        std::copy(f.u.begin() + (size_t)s * nf, f.u.begin() + (size_t)(s + 1) * nf, out[s].u.v.begin());
        out[s].boundary_p.assign(f.bp.begin() + (size_t)s * ne, f.bp.begin() + (size_t)(s + 1) * ne);
    }
    return out;
}

}  // namespace detail

using detail::Backend;

// ---- grid / decomposition / space (grid.cpp:9-15, decomposition.cpp:21-41, interface_space.cpp:9-52)
StructuredGrid2D build_grid(int nx, int ny, double lx, double ly) {
    if (nx < 1 || ny < 1)
        throw ConfigError("build_grid: cell counts must be >= 1, got " + std::to_string(nx) + "x" + std::to_string(ny));
    if (!(lx > 0.0) || !(ly > 0.0)) throw ConfigError("build_grid: domain lengths must be positive");
    return StructuredGrid2D(nx, ny, lx, ly);
}

DomainDecomposition build_decomposition(const StructuredGrid2D& grid, int nsx, int nsy) {
    if (nsx < 1 || nsy < 1) throw ConfigError("build_decomposition: subdomain counts must be >= 1");
    if (grid.nx % nsx != 0 || grid.ny % nsy != 0)
        throw ConfigError("build_decomposition: subdomains do not divide the grid");
    DomainDecomposition dd;
    dd.grid = grid;
    dd.nsx = nsx;
    dd.nsy = nsy;
    const int snx = grid.nx / nsx, sny = grid.ny / nsy;
    dd.subgrids.assign((size_t)nsx * nsy, StructuredGrid2D(snx, sny, snx * grid.hx, sny * grid.hy));
    return dd;
}

InterfaceSpace build_interface_space(const DomainDecomposition& dd, InterfaceSpace::Kind kind, const HbarSpec& hbar) {
    InterfaceSpace sp;
    sp.kind = kind;
    sp.hbar = hbar;
    const int snx = dd.grid.nx / dd.nsx, sny = dd.grid.ny / dd.nsy;
    const int nv = dd.nsy * (dd.nsx - 1), nh = (dd.nsy - 1) * dd.nsx;
    auto bases = [&](int n) {
        if (kind == InterfaceSpace::Kind::Linear) return 2;
        int seg = n;
        switch (hbar.mode) {
            case HbarSpec::Mode::WholeInterface: seg = n; break;
            case HbarSpec::Mode::HalfInterface: seg = n / 2; break;
            case HbarSpec::Mode::PerEdge: seg = 1; break;
            case HbarSpec::Mode::EdgesPerSegment: seg = hbar.edges; break;
        }
        if (seg < 1 || n % seg != 0)
            throw ConfigError("build_interface_space: segment length " + std::to_string(seg) +
                              " does not divide an interface of " + std::to_string(n) + " edges");
        return n / seg;
    };
    sp.n_flux = (nv > 0 ? nv * bases(sny) : 0) + (nh > 0 ? nh * bases(snx) : 0);
    sp.n_pressure = sp.n_flux;
    return sp;
}

BoundarySpec BoundarySpec::uniform(const StructuredGrid2D& g, FaceBc w, FaceBc e, FaceBc s, FaceBc n) {
    BoundarySpec b(g.nx, g.ny);
    for (int j = 0; j < g.ny; ++j) b.faces[b.west(j)] = w, b.faces[b.east(j)] = e;
    for (int i = 0; i < g.nx; ++i) b.faces[b.south(i)] = s, b.faces[b.north(i)] = n;
    return b;
}

// ---- transport (transport.cpp) and grid.cpp:19-31 on a grid-only context
CellField divergence(const FaceField& u) {
    auto b = detail::grid_backend(u.grid, CellField(u.grid, 1.0), 1.0);
    CellField out(u.grid);
    b->check(mpm2p_divergence(b->ctx, u.v.data(), out.v.data()));
    return out;
}

double max_fractional_flow_slope(const FluidModel& fluid) {
    const StructuredGrid2D g(1, 1, 1.0, 1.0);
    auto b = detail::grid_backend(g, CellField(g, 1.0), fluid.viscosity_ratio);
    double v = 0.0;
    b->check(mpm2p_max_fractional_flow_slope(b->ctx, &v));
    return v;
}

double cfl_timestep(const FaceField& u, const FluidModel& fluid, const CflPolicy& policy) {
    auto b = detail::grid_backend(u.grid, CellField(u.grid, 1.0), fluid.viscosity_ratio);
    double dt = 0.0;
    b->check(mpm2p_cfl_timestep(b->ctx, u.v.data(), policy.safety, policy.dt_cap, &dt));
    return dt;
}

SaturationField upwind_step(const SaturationField& s, const FaceField& u, double dt, const FluidModel& fluid) {
    if (!s.s.grid.same_shape(u.grid)) throw ConfigError("upwind_step: grid mismatch");
    auto b = detail::grid_backend(u.grid, CellField(u.grid, 1.0), fluid.viscosity_ratio);
    SaturationField out{CellField(u.grid), s.inflow};
    b->check(mpm2p_upwind_step(b->ctx, s.s.v.data(), s.inflow, u.v.data(), dt, out.s.v.data()));
    return out;
}

CellField conductivity(const CellField& K, const SaturationField& s, const FluidModel& fluid) {
    auto b = detail::grid_backend(K.grid, K, fluid.viscosity_ratio);
    CellField out(K.grid);
    b->check(mpm2p_conductivity(b->ctx, s.s.v.data(), out.v.data()));
    return out;
}

double epsilon(const CellField& kappa_n, const CellField& kappa_m, EpsilonMode mode) {
    auto b = detail::grid_backend(kappa_m.grid, kappa_m, 1.0);
    double v = 0.0;
    b->check(mpm2p_epsilon(b->ctx, kappa_n.v.data(), kappa_m.v.data(), detail::eps_code(mode), &v));
    return v;
}

bool needs_update(const PerturbationState& state, const CellField& kappa_n) {
    return epsilon(kappa_n, state.kappa_m(), state.mode) > state.eta;
}

// ---- robin.cpp:39-92
RobinParameter compute_beta(const CellField& kappa, const DomainDecomposition& dd, const AlphaSpec& spec) {
    Backend b(dd, build_interface_space(dd, InterfaceSpace::Kind::Constant), spec, BoundarySpec(dd.grid.nx, dd.grid.ny),
              kappa, nullptr, 1.0);
    const size_t E = dd.skeleton_edge_count();
    std::vector<double> bm(std::max<size_t>(E, 1)), bp(bm.size()), al(bm.size());
    b.check(mpm2p_compute_beta(b.ctx, kappa.v.data(), bm.data(), bp.data(), al.data()));
    bm.resize(E), bp.resize(E), al.resize(E);
    RobinParameter rp;
    rp.beta_minus = detail::per_interface(dd, bm);
    rp.beta_plus = detail::per_interface(dd, bp);
    rp.alpha = detail::per_interface(dd, al);
    return rp;
}

// ---- mrcm.cpp
namespace {
ParticularSolution particular_of(const BasisSet& basis, SolveCounters* counters) {
    Backend& b = *basis.backend;
    const size_t ns = b.sz.n_sub, nc = (size_t)b.sz.sub_nx * b.sz.sub_ny, ne = 2 * (b.sz.sub_nx + b.sz.sub_ny);
    std::vector<double> q(ns * nc), val(ns * ne), be(ns * ne), rr(ns * ne);
    std::vector<int32_t> kind(ns * ne);
    b.check(mpm2p_restrict_physical_data(b.ctx, q.data(), kind.data(), val.data(), be.data(), rr.data()));
    detail::Flat f;
    f.p.resize(ns * nc), f.u.resize(ns * b.sz.sub_faces), f.bp.resize(ns * ne);
    mpm2p_counters c{};
    b.check(mpm2p_solve_particular(b.ctx, q.data(), kind.data(), val.data(), be.data(), rr.data(), f.p.data(),
                                   f.u.data(), f.bp.data(), &c));
    if (counters) detail::add(*counters, c);
    return ParticularSolution{detail::unflatten(*basis.dd, b.sz, f)};
}

std::shared_ptr<BasisSet> make_basis(const CellField& kappa, std::shared_ptr<const DomainDecomposition> dd,
                                     std::shared_ptr<const InterfaceSpace> space, const RobinParameter& beta,
                                     const CellField& q, const BoundarySpec& bc) {
    auto basis = std::make_shared<BasisSet>();
    basis->backend = std::make_shared<Backend>(*dd, *space, AlphaSpec{}, bc, kappa, &q, 1.0);
    basis->dd = dd;
    basis->space = space;
    basis->beta = beta;
    basis->kappa_m = kappa;
    basis->n_flux = space->dim_flux();
    basis->n_pressure = space->dim_pressure();
    basis->nhat_ = basis->backend->sz.nhat;
    return basis;
}
}  // namespace

std::shared_ptr<BasisSet> compute_basis_set(const CellField& kappa, std::shared_ptr<const DomainDecomposition> dd,
                                            std::shared_ptr<const InterfaceSpace> space, const RobinParameter& beta,
                                            const CellField& q, const BoundarySpec& bc, SolveCounters& counters) {
    auto basis = make_basis(kappa, dd, space, beta, q, bc);
    Backend& b = *basis->backend;
    const auto bm = detail::flat_beta(beta.beta_minus), bp = detail::flat_beta(beta.beta_plus);
    mpm2p_counters c{};
    b.check(mpm2p_compute_basis_set(b.ctx, kappa.v.data(), bm.data(), bp.data(), &c));
    detail::add(counters, c);
    basis->particular = particular_of(*basis, nullptr);  // the set's own (q, bc) solution, already counted
    return basis;
}

ParticularSolution solve_particular(const BasisSet& basis, const std::vector<LocalData>& data, SolveCounters& counters) {
    Backend& b = *basis.backend;
    const size_t ns = b.sz.n_sub, nc = (size_t)b.sz.sub_nx * b.sz.sub_ny, ne = 2 * (b.sz.sub_nx + b.sz.sub_ny);
    if (data.size() != ns) throw ConfigError("solve_particular: one LocalData per subdomain expected");
    std::vector<double> q, val, be, rr;
    std::vector<int32_t> kind;
    for (const auto& d : data) {
        q.insert(q.end(), d.q.v.begin(), d.q.v.end());
        for (const auto& f : d.bc.faces) {
            kind.push_back(detail::bc_code(f.kind));
            val.push_back(f.value);
            be.push_back(f.beta);
            rr.push_back(f.robin_rhs);
        }
    }
    if (q.size() != ns * nc || kind.size() != ns * ne) throw ConfigError("solve_particular: LocalData size mismatch");
    detail::Flat f;
    f.p.resize(ns * nc), f.u.resize(ns * b.sz.sub_faces), f.bp.resize(ns * ne);
    mpm2p_counters c{};
    b.check(mpm2p_solve_particular(b.ctx, q.data(), kind.data(), val.data(), be.data(), rr.data(), f.p.data(),
                                   f.u.data(), f.bp.data(), &c));
    detail::add(counters, c);
    return ParticularSolution{detail::unflatten(*basis.dd, b.sz, f)};
}

SkeletonCoeffs solve_interface(const BasisSet& basis, const ParticularSolution& particular, SolveCounters& counters) {
    Backend& b = *basis.backend;
    const detail::Flat f = detail::flatten(particular.per_sub);
    std::vector<double> x(std::max(1, basis.system_dim()));
    mpm2p_counters c{};
    b.check(mpm2p_solve_interface(b.ctx, f.u.data(), x.data(), &c));
    detail::add(counters, c);
    SkeletonCoeffs co;
    co.flux.assign(x.begin(), x.begin() + basis.n_flux);
    co.pressure.assign(x.begin() + basis.n_flux, x.begin() + basis.n_flux + basis.n_pressure);
    return co;
}

MrcmReconstruction reconstruct(const BasisSet& basis, const SkeletonCoeffs& coeffs, const ParticularSolution& particular) {
    Backend& b = *basis.backend;
    const detail::Flat f = detail::flatten(particular.per_sub);
    std::vector<double> x(coeffs.flux);
    x.insert(x.end(), coeffs.pressure.begin(), coeffs.pressure.end());
    if (x.empty()) x.push_back(0.0);
    detail::Flat o;
    o.p.resize(f.p.size()), o.u.resize(f.u.size()), o.bp.resize(f.bp.size());
    b.check(mpm2p_reconstruct(b.ctx, x.data(), f.p.data(), f.u.data(), f.bp.data(), o.p.data(), o.u.data(), o.bp.data()));
    return MrcmReconstruction{detail::unflatten(*basis.dd, b.sz, o)};
}

WeakResiduals weak_continuity_residuals(const BasisSet& basis, const MrcmReconstruction& recon) {
    Backend& b = *basis.backend;
    const detail::Flat f = detail::flatten(recon.per_sub);
    WeakResiduals w;
    b.check(mpm2p_weak_continuity_residuals(b.ctx, f.u.data(), f.bp.data(), &w.flux_jump, &w.pressure_jump));
    return w;
}

GlobalSolution mrcm_solve(const CellField& kappa, std::shared_ptr<const DomainDecomposition> dd,
                          std::shared_ptr<const InterfaceSpace> space, const RobinParameter& beta, const CellField& q,
                          const BoundarySpec& bc, SolveCounters& counters) {
    GlobalSolution g;
    g.basis = make_basis(kappa, dd, space, beta, q, bc);
    Backend& b = *g.basis->backend;
    const auto bm = detail::flat_beta(beta.beta_minus), bp = detail::flat_beta(beta.beta_plus);
    g.p = CellField(dd->grid);
    g.u = FaceField(dd->grid);
    std::vector<double> x(std::max(1, g.basis->system_dim()));
    mpm2p_downscale_info info{};
    mpm2p_counters c{};
    b.check(mpm2p_mrcm_solve(b.ctx, kappa.v.data(), bm.data(), bp.data(), g.p.v.data(), g.u.v.data(), x.data(), &info, &c));
    detail::add(counters, c);
    g.coeffs.flux.assign(x.begin(), x.begin() + g.basis->n_flux);
    g.coeffs.pressure.assign(x.begin() + g.basis->n_flux, x.begin() + g.basis->system_dim());
    g.repair_max = info.repair_max;
    g.repair_warning = info.repair_warning != 0;
    g.div_residual = info.div_residual;
    g.div_scale = info.div_scale;
    // the set's particular solution and the recombination (recon_m), re-formed on the device
    g.basis->particular = particular_of(*g.basis, nullptr);
    g.recon = reconstruct(*g.basis, g.coeffs, g.basis->particular);
    return g;
}

MpmResult mpm_pressure_update(const PerturbationState& state, const CellField& kappa_n, const CellField& q,
                              const BoundarySpec& bc, SolveCounters& counters) {
    // the device context holds the state's basis and recon_m (installed by
    // mrcm_solve); q and bc are the ones the basis was prepared with
    (void)q;
    (void)bc;
    if (!state.basis || !state.basis->backend) throw ConfigError("mpm_pressure_update: no basis set");
    const BasisSet& basis = *state.basis;
    Backend& b = *basis.backend;
    MpmResult r;
    r.p = CellField(basis.dd->grid);
    r.u = FaceField(basis.dd->grid);
    std::vector<double> x(std::max(1, basis.system_dim()));
    mpm2p_downscale_info info{};
    mpm2p_counters c{};
    b.check(mpm2p_mpm_update(b.ctx, kappa_n.v.data(), r.p.v.data(), r.u.v.data(), x.data(), &info, &c));
    detail::add(counters, c);
    r.delta_coeffs.flux.assign(x.begin(), x.begin() + basis.n_flux);
    r.delta_coeffs.pressure.assign(x.begin() + basis.n_flux, x.begin() + basis.system_dim());
    r.repair_max = info.repair_max;
    r.repair_warning = info.repair_warning != 0;
    r.div_residual = info.div_residual;
    r.div_scale = info.div_scale;
    return r;
}

// ---- simulation.cpp:118-340
namespace {
struct SnapCtx {
    const SnapshotCallback* fn;
    StructuredGrid2D grid;
    double inflow;
};
void snap_trampoline(void* user, int64_t step, const double* s, const double* p, const double* u) {
    const SnapCtx* sc = static_cast<const SnapCtx*>(user);
    SaturationField sf{CellField(sc->grid), sc->inflow};
    CellField pf(sc->grid);
    FaceField uf(sc->grid);
    std::copy(s, s + sf.s.size(), sf.s.v.begin());
    std::copy(p, p + pf.size(), pf.v.begin());
    std::copy(u, u + uf.size(), uf.v.begin());
    (*sc->fn)((long)step, sf, pf, uf);
}
}  // namespace

RunResult run(const RunInputs& in, const std::vector<long>& snapshot_steps, const SnapshotCallback& snap) {
    if (!in.dd || !in.space) throw ConfigError("run: decomposition and interface space are required");
    const StructuredGrid2D& g = in.dd->grid;
    Backend b(*in.dd, *in.space, in.alpha, in.bc, in.K, &in.q, in.fluid.viscosity_ratio);
    mpm2p_split sp{};
    const SplittingConfig& s = in.split;
    sp.method = s.method == Method::FineReference    ? MPM2P_METHOD_FINE_REFERENCE
                : s.method == Method::MrcmEveryStep  ? MPM2P_METHOD_MRCM_EVERY_STEP
                : s.method == Method::Mpm2p          ? MPM2P_METHOD_MPM2P
                                                     : MPM2P_METHOD_MPM2P_NO_UPDATES;
    sp.cn = s.cn, sp.eta = s.eta, sp.eta_mode = detail::eps_code(s.eta_mode), sp.cfl_safety = s.cfl_safety;
    sp.dt_cap = s.dt_cap, sp.te = s.te, sp.pvi_max = s.pvi_max, sp.stop_on_breakthrough = s.stop_on_breakthrough;
    sp.max_steps_hard = s.max_steps_hard, sp.breakthrough_threshold = s.breakthrough_threshold;
    sp.track_errors = s.track_errors, sp.inflow_sat = in.inflow_sat;
    const CellField s0 = in.s0.size() == g.cell_count() ? in.s0 : CellField(g, 0.0);
    RunResult r;
    r.s_final = SaturationField{CellField(g), in.inflow_sat};
    r.p_final = CellField(g);
    r.u_final = FaceField(g);
    const int64_t cap = (s.te > 0 ? s.te : s.max_steps_hard) + 1;
    std::vector<mpm2p_step_record> steps((size_t)cap);
    mpm2p_run_record rec{};
    std::vector<int64_t> want(snapshot_steps.begin(), snapshot_steps.end());
    SnapCtx sc{&snap, g, in.inflow_sat};
    b.check(mpm2p_run_snapshots(b.ctx, &sp, s0.v.data(), r.s_final.s.v.data(), r.p_final.v.data(), r.u_final.v.data(),
                                steps.data(), cap, &rec, want.data(), (int64_t)want.size(),
                                snap ? snap_trampoline : nullptr, &sc));
    RunRecord& o = r.record;
    for (int64_t i = 0; i < rec.te && i < cap; ++i) {
        const mpm2p_step_record& t = steps[(size_t)i];
        StepRecord sr;
        sr.step = (long)t.step, sr.pvi = t.pvi, sr.epsilon = t.epsilon, sr.rebuilt = t.rebuilt;
        sr.flux_err = t.flux_err, sr.sat_err = t.sat_err, sr.bf_homog_cum = (long)t.bf_homog_cum;
        sr.bf_part_cum = (long)t.bf_part_cum, sr.dt = t.dt, sr.wall_s = t.wall_s, sr.div_residual = t.div_residual;
        o.steps.push_back(sr);
        if (sr.rebuilt) o.update_steps.push_back(sr.step);
    }
    o.breakthrough_step = (long)rec.breakthrough_step, o.breakthrough_pvi = rec.breakthrough_pvi;
    o.te = (long)rec.te, o.tm_updates = (long)rec.tm_updates, o.tm_total = (long)rec.tm_total;
    o.nhat = (long)rec.nhat, o.n_sub = rec.n_sub, o.counters = detail::counters_of(rec.counters);
    o.max_div_residual = rec.max_div_residual, o.max_div_ratio = rec.max_div_ratio;
    o.repair_warnings = rec.repair_warnings, o.final_pvi = rec.final_pvi;
    return r;
}

}  // namespace mrcmflow
