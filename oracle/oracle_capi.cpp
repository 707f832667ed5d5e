// CPU ORACLE — TEST INFRASTRUCTURE ONLY. C ABI over the restatement, with the
// same signatures as include/mpm2p_b200.h (prefix oracle_ instead of mpm2p_),
// so parity tests call both implementations identically.
#include <new>
#include <algorithm>
#include <cstring>
#include <string>

#include "../include/mpm2p_b200.h"
#include "mrcm_oracle.hpp"

using namespace orc;

struct oracle_ctx {
    std::shared_ptr<const Decomp> dd;
    std::shared_ptr<const Space> space;
    BoundarySpec bc;
    Vec K, q;
    AlphaSpec alpha;
    double M = 1.0;
    std::string err;
    PerturbationState state;  // installed by oracle_mrcm_solve
    std::unique_ptr<Runner> runner;
    int64_t clamp_base = 0;
    double fine_div_res = 0.0, fine_div_scale = 1.0;  // last oracle_fine_solve
};

namespace {
thread_local std::string g_create_err;

template <typename F>
int guarded(oracle_ctx* ctx, F&& fn) {
    try {
        fn();
        return MPM2P_OK;
    } catch (const ConfigError& e) {
        if (ctx) ctx->err = e.what();
        else g_create_err = e.what();
        return MPM2P_ECONFIG;
    } catch (const NumericError& e) {
        if (ctx) ctx->err = e.what();
        else g_create_err = e.what();
        return MPM2P_ENUMERIC;
    } catch (const CapacityError& e) {
        if (ctx) ctx->err = e.what();
        else g_create_err = e.what();
        return MPM2P_ECAPACITY;
    } catch (const std::bad_alloc& e) {
        if (ctx) ctx->err = e.what();
        else g_create_err = e.what();
        return MPM2P_ECAPACITY;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        else g_create_err = e.what();
        return MPM2P_EINTERNAL;
    }
}

void copy_out(double* dst, const Vec& v) {
    if (dst)
        for (size_t i = 0; i < v.size(); ++i) dst[i] = (double)v[i];
}

Vec flatten(const std::vector<Vec>& vv) {
    Vec out;
    for (const auto& v : vv) out.insert(out.end(), v.begin(), v.end());
    return out;
}

void fill_info(mpm2p_downscale_info* info, const DownscaleResult& ds) {
    if (!info) return;
    info->repair_max = ds.repair_max;
    info->flux_scale = ds.flux_scale;
    info->repair_warning = ds.repair_warning ? 1 : 0;
    info->div_residual = ds.div_residual;
    info->div_scale = ds.div_scale;
}

void fill_counters(mpm2p_counters* c, const SolveCounters& s) {
    if (!c) return;
    c->homogeneous = s.homogeneous;
    c->particular = s.particular;
    c->downscale = s.downscale;
    c->fine = s.fine;
    c->interface_solves = s.interface_solves;
}

void fill_step(mpm2p_step_record* o, const StepRecord& s) {
    o->step = s.step;
    o->pvi = s.pvi;
    o->epsilon = s.epsilon;
    o->rebuilt = s.rebuilt;
    o->flux_err = s.flux_err;
    o->sat_err = s.sat_err;
    o->bf_homog_cum = s.bf_homog_cum;
    o->bf_part_cum = s.bf_part_cum;
    o->dt = s.dt;
    o->wall_s = s.wall_s;
    o->div_residual = s.div_residual;
}

void fill_run(mpm2p_run_record* o, const RunRecord& r, int64_t clamps) {
    o->breakthrough_step = r.breakthrough_step;
    o->breakthrough_pvi = r.breakthrough_pvi;
    o->te = r.te;
    o->tm_updates = r.tm_updates;
    o->tm_total = r.tm_total;
    o->nhat = r.nhat;
    o->n_sub = r.n_sub;
    fill_counters(&o->counters, r.counters);
    o->max_div_residual = r.max_div_residual;
    o->max_div_ratio = r.max_div_ratio;
    o->repair_warnings = r.repair_warnings;
    o->final_pvi = r.final_pvi;
    o->min_eps_margin = r.min_eps_margin;
    o->clamp_count = clamps;
    o->interface_krylov = 0;
    o->interface_max_iterations = 0;
    o->interface_iterations = 0;
    o->min_rcond = -1.0;
}

RunInputs make_inputs(const oracle_ctx* ctx, const mpm2p_split* sp, const double* s0) {
    RunInputs in;
    in.dd = ctx->dd;
    in.K = ctx->K;
    in.q = ctx->q;
    in.M = ctx->M;
    in.bc = ctx->bc;
    in.space = ctx->space;
    in.alpha = ctx->alpha;
    Split& s = in.split;
    s.method = sp->method;
    s.cn = sp->cn;
    s.eta = sp->eta;
    s.eta_mode = sp->eta_mode;
    s.cfl_safety = sp->cfl_safety;
    s.dt_cap = sp->dt_cap;
    s.te = (long)sp->te;
    s.pvi_max = sp->pvi_max;
    s.stop_on_breakthrough = sp->stop_on_breakthrough != 0;
    s.max_steps_hard = (long)sp->max_steps_hard;
    s.breakthrough_threshold = sp->breakthrough_threshold;
    s.track_errors = sp->track_errors != 0;
    in.inflow_sat = sp->inflow_sat;
    const int n = ctx->dd->grid.cells();
    in.s0.assign(s0, s0 + n);
    return in;
}

RobinParameter beta_from(const oracle_ctx* ctx, const Vec& kappa, const double* bm, const double* bp) {
    if (!bm || !bp) return compute_beta(kappa, *ctx->dd, ctx->alpha);
    RobinParameter rp;
    const Decomp& dd = *ctx->dd;
    rp.beta_minus.resize(dd.n_iface());
    rp.beta_plus.resize(dd.n_iface());
    rp.alpha.resize(dd.n_iface());
    size_t off = 0;
    for (int k = 0; k < dd.n_iface(); ++k) {
        const size_t n = dd.ifaces[k].faces.size();
        rp.beta_minus[k].assign(bm + off, bm + off + n);
        rp.beta_plus[k].assign(bp + off, bp + off + n);
        rp.alpha[k].assign(n, 0.0);
        off += n;
    }
    return rp;
}
}  // namespace

extern "C" {

int oracle_create(const mpm2p_problem* p, oracle_ctx** out) {
    *out = nullptr;
    auto ctx = new oracle_ctx();
    const int rc = guarded(nullptr, [&] {
        const Grid g = build_grid(p->nx, p->ny, p->lx, p->ly);
        auto dd = std::make_shared<Decomp>(build_decomposition(g, p->nsx, p->nsy));
        HbarSpec hb{p->hbar_mode, p->hbar_edges};
        ctx->space = std::make_shared<Space>(build_interface_space(*dd, p->space_kind, hb));
        ctx->dd = dd;
        ctx->K.assign(p->K, p->K + g.cells());
        ctx->q = p->q ? Vec(p->q, p->q + g.cells()) : Vec(g.cells(), 0.0);
        ctx->bc = BoundarySpec(g.nx, g.ny);
        for (int i = 0; i < ctx->bc.count(); ++i) {
            ctx->bc.faces[i].kind = p->bc_kind[i];
            ctx->bc.faces[i].value = p->bc_value[i];
            if (p->bc_kind[i] != Pressure && p->bc_kind[i] != Flux && p->bc_kind[i] != Robin)
                throw ConfigError("problem: unknown boundary kind");
            if (p->bc_kind[i] == Robin) {  // FaceBc::robin(beta, rhs) (elliptic.hpp:27)
                if (!p->bc_beta || !p->bc_robin_rhs) throw ConfigError("problem: Robin faces need bc_beta and bc_robin_rhs");
                ctx->bc.faces[i].value = 0.0;
                ctx->bc.faces[i].beta = p->bc_beta[i];
                ctx->bc.faces[i].robin_rhs = p->bc_robin_rhs[i];
            }
        }
        ctx->alpha.mode = p->alpha_mode;
        ctx->alpha.alpha = p->alpha;
        ctx->alpha.alpha_min = p->alpha_min;
        ctx->alpha.alpha_max = p->alpha_max;
        ctx->alpha.pct_lo = p->percentile_lo;
        ctx->alpha.pct_hi = p->percentile_hi;
        ctx->M = p->viscosity_ratio;
    });
    if (rc != MPM2P_OK) {
        delete ctx;
        return rc;
    }
    *out = ctx;
    return rc;
}

void oracle_destroy(oracle_ctx* ctx) { delete ctx; }
const char* oracle_last_error(const oracle_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
const char* oracle_create_error(void) { return g_create_err.c_str(); }

int oracle_get_sizes(const oracle_ctx* ctx, mpm2p_sizes* o) {
    const Decomp& dd = *ctx->dd;
    o->cells = dd.grid.cells();
    o->faces = dd.grid.faces();
    o->bfaces = 2 * (dd.grid.nx + dd.grid.ny);
    o->n_sub = dd.n_sub();
    o->n_interfaces = dd.n_iface();
    o->skeleton_edges = dd.skeleton_edges();
    o->dim_flux = ctx->space->dim_flux();
    o->dim_pressure = ctx->space->dim_pres();
    int64_t nhat = 0;
    for (int s = 0; s < dd.n_sub(); ++s) {
        std::vector<int> inc;
        for (const auto& e : dd.sub_boundary[s])
            if (e.on_skeleton && std::find(inc.begin(), inc.end(), e.iface) == inc.end()) inc.push_back(e.iface);
        for (int k : inc) nhat += 2 * (int64_t)ctx->space->flux_by_iface[k].size();
    }
    o->nhat = nhat;
    o->sub_nx = dd.subs[0].nx;
    o->sub_ny = dd.subs[0].ny;
    const Grid& lg0 = dd.subgrids[0];
    o->sub_faces = lg0.faces();
    return MPM2P_OK;
}

int oracle_conductivity(oracle_ctx* ctx, const double* s, double* kappa) {
    return guarded(ctx, [&] {
        const int n = ctx->dd->grid.cells();
        copy_out(kappa, conductivity(ctx->K, Vec(s, s + n), ctx->M));
    });
}

int oracle_max_fractional_flow_slope(oracle_ctx* ctx, double* out) {
    return guarded(ctx, [&] { *out = max_fractional_flow_slope(ctx->M); });
}

int oracle_cfl_timestep(oracle_ctx* ctx, const double* u, double safety, double dt_cap, double* dt) {
    return guarded(ctx, [&] {
        const Grid& g = ctx->dd->grid;
        *dt = cfl_timestep(g, Vec(u, u + g.faces()), ctx->M, safety, dt_cap);
    });
}

int oracle_upwind_step(oracle_ctx* ctx, const double* s, double inflow, const double* u, double dt, double* s_out) {
    return guarded(ctx, [&] {
        const Grid& g = ctx->dd->grid;
        copy_out(s_out, upwind_step(g, Vec(s, s + g.cells()), inflow, Vec(u, u + g.faces()), dt, ctx->M));
    });
}

int oracle_injection_rate(oracle_ctx* ctx, const double* u, double inflow, double* out) {
    return guarded(ctx, [&] {
        const Grid& g = ctx->dd->grid;
        *out = injection_rate(g, Vec(u, u + g.faces()), inflow, ctx->M);
    });
}

int oracle_max_outlet_saturation(oracle_ctx* ctx, const double* s, const double* u, double* out) {
    return guarded(ctx, [&] {
        const Grid& g = ctx->dd->grid;
        *out = max_outlet_saturation(g, Vec(s, s + g.cells()), Vec(u, u + g.faces()));
    });
}

int oracle_divergence(oracle_ctx* ctx, const double* u, double* div) {
    return guarded(ctx, [&] {
        const Grid& g = ctx->dd->grid;
        copy_out(div, divergence(g, Vec(u, u + g.faces())));
    });
}

int oracle_epsilon(oracle_ctx* ctx, const double* kn, const double* km, int32_t mode, double* out) {
    return guarded(ctx, [&] {
        const Grid& g = ctx->dd->grid;
        const int n = g.cells();
        *out = epsilon(g, Vec(kn, kn + n), Vec(km, km + n), mode);
    });
}

int oracle_compute_beta(oracle_ctx* ctx, const double* kappa, double* bm, double* bp, double* alpha) {
    return guarded(ctx, [&] {
        const int n = ctx->dd->grid.cells();
        const RobinParameter rp = compute_beta(Vec(kappa, kappa + n), *ctx->dd, ctx->alpha);
        copy_out(bm, flatten(rp.beta_minus));
        copy_out(bp, flatten(rp.beta_plus));
        copy_out(alpha, flatten(rp.alpha));
    });
}

int oracle_mrcm_solve(oracle_ctx* ctx, const double* kappa, const double* bm, const double* bp, double* p,
                      double* u, double* coeffs, mpm2p_downscale_info* info, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        const int n = ctx->dd->grid.cells();
        const Vec k(kappa, kappa + n);
        const RobinParameter rp = beta_from(ctx, k, bm, bp);
        SolveCounters c;
        GlobalSolution sol = mrcm_solve(k, ctx->dd, ctx->space, rp, ctx->q, ctx->bc, c);
        copy_out(p, sol.ds.p);
        copy_out(u, sol.ds.u);
        if (coeffs) {
            copy_out(coeffs, sol.coeffs.flux);
            copy_out(coeffs + sol.coeffs.flux.size(), sol.coeffs.pres);
        }
        fill_info(info, sol.ds);
        fill_counters(counters, c);
        ctx->state.basis = sol.basis;
        ctx->state.recon_m = std::move(sol.recon);
    });
}

int oracle_mpm_update(oracle_ctx* ctx, const double* kappa_n, double* p, double* u, double* dcoeffs,
                      mpm2p_downscale_info* info, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("mpm_update: no basis installed (call mrcm_solve first)");
        const int n = ctx->dd->grid.cells();
        SolveCounters c;
        MpmResult r = mpm_pressure_update(ctx->state, Vec(kappa_n, kappa_n + n), ctx->q, ctx->bc, c);
        copy_out(p, r.ds.p);
        copy_out(u, r.ds.u);
        if (dcoeffs) {
            copy_out(dcoeffs, r.delta.flux);
            copy_out(dcoeffs + r.delta.flux.size(), r.delta.pres);
        }
        fill_info(info, r.ds);
        fill_counters(counters, c);
    });
}

int oracle_interface_matrix(oracle_ctx* ctx, double* M) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("interface_matrix: no basis installed");
        copy_out(M, ctx->state.basis->dense_matrix());
    });
}

int oracle_run(oracle_ctx* ctx, const mpm2p_split* sp, const double* s0, double* s_final, double* p_final,
               double* u_final, mpm2p_step_record* steps, int64_t max_steps, mpm2p_run_record* rec) {
    return guarded(ctx, [&] {
        const int64_t c0 = clamp_count();
        RunResult r = run(make_inputs(ctx, sp, s0));
        copy_out(s_final, r.s_final);
        copy_out(p_final, r.p_final);
        copy_out(u_final, r.u_final);
        if (steps)
            for (int64_t i = 0; i < (int64_t)r.rec.steps.size() && i < max_steps; ++i) fill_step(&steps[i], r.rec.steps[i]);
        if (rec) fill_run(rec, r.rec, clamp_count() - c0);
    });
}

int oracle_run_snapshots(oracle_ctx* ctx, const mpm2p_split* sp, const double* s0, double* s_final, double* p_final,
                         double* u_final, mpm2p_step_record* steps, int64_t max_steps, mpm2p_run_record* rec,
                         const int64_t* snapshot_steps, int64_t n_snapshots, mpm2p_snapshot_fn snap, void* user) {
    return guarded(ctx, [&] {
        const int64_t c0 = clamp_count();
        Runner r(make_inputs(ctx, sp, s0));
        std::vector<double> hs, hp, hu;
        auto maybe_snap = [&]() {  // simulation.cpp:224-226
            if (!snap || !snapshot_steps) return;
            const int64_t n = r.record().steps.back().step;
            if (std::find(snapshot_steps, snapshot_steps + n_snapshots, n) == snapshot_steps + n_snapshots) return;
            hs.assign(r.s().begin(), r.s().end());
            hp.assign(r.p().begin(), r.p().end());
            hu.assign(r.u().begin(), r.u().end());
            snap(user, n, hs.data(), hp.data(), hu.data());
        };
        r.begin();
        maybe_snap();
        while (r.step()) maybe_snap();
        copy_out(s_final, r.s());
        copy_out(p_final, r.p());
        copy_out(u_final, r.u());
        RunResult res = r.finish();
        if (steps)
            for (int64_t i = 0; i < (int64_t)res.rec.steps.size() && i < max_steps; ++i) fill_step(&steps[i], res.rec.steps[i]);
        if (rec) fill_run(rec, res.rec, clamp_count() - c0);
    });
}

int oracle_run_begin(oracle_ctx* ctx, const mpm2p_split* sp, const double* s0, mpm2p_step_record* first) {
    return guarded(ctx, [&] {
        ctx->clamp_base = clamp_count();
        ctx->runner = std::make_unique<Runner>(make_inputs(ctx, sp, s0));
        ctx->runner->begin();
        if (first) fill_step(first, ctx->runner->record().steps.back());
    });
}

int oracle_run_step(oracle_ctx* ctx, mpm2p_step_record* out, int32_t* done) {
    return guarded(ctx, [&] {
        if (!ctx->runner) throw ConfigError("run_step: run_begin not called");
        const bool did = ctx->runner->step();
        *done = did ? 0 : 1;
        if (did && out) fill_step(out, ctx->runner->record().steps.back());
    });
}

int oracle_run_read(oracle_ctx* ctx, double* s, double* p, double* u) {
    return guarded(ctx, [&] {
        if (!ctx->runner) throw ConfigError("run_read: run_begin not called");
        copy_out(s, ctx->runner->s());
        copy_out(p, ctx->runner->p());
        copy_out(u, ctx->runner->u());
    });
}

int oracle_run_end(oracle_ctx* ctx, mpm2p_run_record* rec) {
    return guarded(ctx, [&] {
        if (!ctx->runner) throw ConfigError("run_end: run_begin not called");
        RunResult r = ctx->runner->finish();
        if (rec) fill_run(rec, r.rec, clamp_count() - ctx->clamp_base);
        ctx->runner.reset();
    });
}

double oracle_rcr(int64_t nhat, int64_t n, int64_t te, int64_t tm) {
    try {
        return rcr((long)nhat, (long)n, (long)te, (long)tm);
    } catch (...) {
        return -1.0;
    }
}

// ---- oracle-only helpers (test infrastructure) --------------------------
/* The undecomposed fine solve (simulation.cpp:143-150), for equivalence tests. */
int oracle_fine_solve(oracle_ctx* ctx, const double* kappa, double* p, double* u) {
    return guarded(ctx, [&] {
        const Grid& g = ctx->dd->grid;
        const int anchor = ctx->bc.pure_neumann() ? 0 : -1;
        LocalSolution s = solve_cell_centered(g, Vec(kappa, kappa + g.cells()), ctx->q, ctx->bc, anchor);
        ctx->fine_div_res = conservation_residual(g, s, ctx->q);
        ctx->fine_div_scale = residual_scale(g, s, ctx->q);
        copy_out(p, s.p);
        copy_out(u, s.u);
    });
}

/* Mirror of mpm2p_fine_stats: a direct solve reports 0 iterations and 0
 * residual; conservation_residual / residual_scale of the last solve. */
int oracle_fine_stats(oracle_ctx* ctx, int32_t* iterations, double* relres, double* div_residual,
                      double* div_scale) {
    return guarded(ctx, [&] {
        if (iterations) *iterations = 0;
        if (relres) *relres = 0.0;
        if (div_residual) *div_residual = ctx->fine_div_res;
        if (div_scale) *div_scale = ctx->fine_div_scale;
    });
}

/* Restated GaussianSampler (fields_io.cpp:25-85). */
int oracle_gaussian_field(int32_t nx, int32_t ny, double lx, double ly, double delta, double mean_coeff,
                          uint64_t seed, int32_t range_norm, double range_target, double* out) {
    return guarded(nullptr, [&] {
        const Grid g = build_grid(nx, ny, lx, ly);
        copy_out(out, gaussian_field(g, delta, mean_coeff, seed, range_norm != 0, range_target));
    });
}

// ---- MRCM sub-steps (mrcm.hpp:77-136) over the per-subdomain C-ABI layouts
namespace {
std::vector<LocalSolution> locals_in(const oracle_ctx* ctx, const double* p, const double* u, const double* bp) {
    const Decomp& dd = *ctx->dd;
    std::vector<LocalSolution> out(dd.n_sub());
    size_t oc = 0, of = 0, oe = 0;
    for (int s = 0; s < dd.n_sub(); ++s) {
        const Grid& lg = dd.subgrids[s];
        const size_t ne = dd.sub_boundary[s].size();
        out[s].p = p ? Vec(p + oc, p + oc + lg.cells()) : Vec(lg.cells(), 0.0);
        out[s].u = u ? Vec(u + of, u + of + lg.faces()) : Vec(lg.faces(), 0.0);
        out[s].boundary_p = bp ? Vec(bp + oe, bp + oe + ne) : Vec(ne, 0.0);
        oc += lg.cells(), of += lg.faces(), oe += ne;
    }
    return out;
}
void locals_out(const std::vector<LocalSolution>& v, double* p, double* u, double* bp) {
    size_t oc = 0, of = 0, oe = 0;
    for (const auto& l : v) {
        if (p) copy_out(p + oc, l.p);
        if (u) copy_out(u + of, l.u);
        if (bp) copy_out(bp + oe, l.boundary_p);
        oc += l.p.size(), of += l.u.size(), oe += l.boundary_p.size();
    }
}
}  // namespace

int oracle_compute_basis_set(oracle_ctx* ctx, const double* kappa, const double* bm, const double* bp,
                             mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        const int n = ctx->dd->grid.cells();
        const Vec k(kappa, kappa + n);
        const RobinParameter rp = beta_from(ctx, k, bm, bp);
        SolveCounters c;
        ctx->state.basis.reset();
        ctx->state.recon_m.clear();
        ctx->state.basis = compute_basis_set(k, ctx->dd, ctx->space, rp, ctx->q, ctx->bc, c);
        fill_counters(counters, c);
    });
}

int oracle_restrict_physical_data(oracle_ctx* ctx, double* q_local, int32_t* kind, double* val, double* beta,
                                  double* rhs) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("restrict_physical_data: no basis installed");
        const auto data = restrict_physical_data(*ctx->dd, ctx->state.basis->beta, ctx->q, ctx->bc);
        size_t oc = 0, oe = 0;
        for (const auto& d : data) {
            if (q_local) copy_out(q_local + oc, d.q);
            for (const auto& f : d.bc.faces) {
                if (kind) kind[oe] = f.kind;
                if (val) val[oe] = (double)f.value;
                if (beta) beta[oe] = (double)f.beta;
                if (rhs) rhs[oe] = (double)f.robin_rhs;
                ++oe;
            }
            oc += d.q.size();
        }
    });
}

int oracle_solve_particular(oracle_ctx* ctx, const double* q_local, const int32_t* kind, const double* val,
                            const double* beta, const double* rhs, double* p, double* u, double* bp,
                            mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("solve_particular: no basis installed");
        const Decomp& dd = *ctx->dd;
        std::vector<LocalData> data(dd.n_sub());
        size_t oc = 0, oe = 0;
        for (int s = 0; s < dd.n_sub(); ++s) {
            const Grid& lg = dd.subgrids[s];
            data[s].q = Vec(q_local + oc, q_local + oc + lg.cells());
            data[s].bc = BoundarySpec(lg.nx, lg.ny);
            for (auto& f : data[s].bc.faces) {
                f.kind = kind[oe];
                f.value = val[oe];
                f.beta = beta[oe];
                f.robin_rhs = rhs[oe];
                ++oe;
            }
            oc += lg.cells();
        }
        SolveCounters c;
        locals_out(solve_particular(*ctx->state.basis, data, c), p, u, bp);
        fill_counters(counters, c);
    });
}

int oracle_solve_interface(oracle_ctx* ctx, const double* u_local, double* coeffs, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("solve_interface: no basis installed");
        SolveCounters c;
        const SkeletonCoeffs co = solve_interface(*ctx->state.basis, locals_in(ctx, nullptr, u_local, nullptr), c);
        if (coeffs) {
            copy_out(coeffs, co.flux);
            copy_out(coeffs + co.flux.size(), co.pres);
        }
        fill_counters(counters, c);
    });
}

int oracle_reconstruct(oracle_ctx* ctx, const double* coeffs, const double* p, const double* u, const double* bp,
                       double* po, double* uo, double* bpo) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("reconstruct: no basis installed");
        const BasisSet& b = *ctx->state.basis;
        SkeletonCoeffs co;
        co.flux = Vec(coeffs, coeffs + b.n_flux);
        co.pres = Vec(coeffs + b.n_flux, coeffs + b.n_flux + b.n_pres);
        locals_out(reconstruct(b, co, locals_in(ctx, p, u, bp)), po, uo, bpo);
    });
}

int oracle_averaged_skeleton_flux(oracle_ctx* ctx, const double* u_local, double* flux) {
    return guarded(ctx, [&] {
        copy_out(flux, flatten(averaged_skeleton_flux(*ctx->dd, locals_in(ctx, nullptr, u_local, nullptr))));
    });
}

int oracle_downscale(oracle_ctx* ctx, const double* kappa, const double* p_local, const double* u_local,
                     const double* flux, double* p, double* u, mpm2p_downscale_info* info, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        const Decomp& dd = *ctx->dd;
        std::vector<Vec> skel(dd.n_iface());
        size_t off = 0;
        for (int k = 0; k < dd.n_iface(); ++k) {
            const size_t ne = dd.ifaces[k].faces.size();
            skel[k] = Vec(flux + off, flux + off + ne);
            off += ne;
        }
        SolveCounters c;
        const int n = dd.grid.cells();
        const DownscaleResult ds =
            downscale(dd, Vec(kappa, kappa + n), ctx->q, ctx->bc, locals_in(ctx, p_local, u_local, nullptr), skel, c);
        copy_out(p, ds.p);
        copy_out(u, ds.u);
        fill_info(info, ds);
        fill_counters(counters, c);
    });
}

int oracle_weak_continuity_residuals(oracle_ctx* ctx, const double* u_local, const double* bp_local, double* fj, double* pj) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("weak_continuity_residuals: no basis installed");
        const WeakResiduals w = weak_continuity_residuals(*ctx->state.basis, locals_in(ctx, nullptr, u_local, bp_local));
        if (fj) *fj = w.flux_jump;
        if (pj) *pj = w.pressure_jump;
    });
}

/* weak_continuity_residuals (mrcm.cpp:459-483) of the installed reconstruction. */
int oracle_weak_residuals(oracle_ctx* ctx, double* flux_jump, double* pressure_jump) {
    return guarded(ctx, [&] {
        if (!ctx->state.basis) throw ConfigError("weak_residuals: no basis installed");
        WeakResiduals w = weak_continuity_residuals(*ctx->state.basis, ctx->state.recon_m);
        *flux_jump = w.flux_jump;
        *pressure_jump = w.pressure_jump;
    });
}

int64_t oracle_clamp_count(void) { return clamp_count(); }

/* 0: natural elimination order (default), 1: reversed — an equally exact
 * direct solve with different rounding, used to measure solver-noise floors. */
void oracle_set_elimination_order(int32_t order) { set_elimination_order(order); }
// 0 auto (dense LU up to 16,384 unknowns, banded LU above), 1 dense, 2 banded
void oracle_set_interface_solver(int32_t mode) { set_interface_solver(mode); }
// threads for the per-subdomain loops (default 1, the reference's single thread)
void oracle_set_threads(int32_t n) { set_threads(n); }

/* Decomposition tables built the reference's way (decomposition.cpp:35-132,
 * mrcm.cpp:157-189), same layout as mpm2p_layout_tables. */
int oracle_layout_tables(const mpm2p_problem* p, int32_t s, int32_t* edges, int32_t* hom_cols, int32_t* n_hom) {
    return guarded(nullptr, [&] {
        const Grid g = build_grid(p->nx, p->ny, p->lx, p->ly);
        const Decomp dd = build_decomposition(g, p->nsx, p->nsy);
        const Space sp = build_interface_space(dd, p->space_kind, HbarSpec{p->hbar_mode, p->hbar_edges});
        if (s < 0 || s >= dd.n_sub()) throw ConfigError("layout_tables: subdomain out of range");
        auto gbc = [&](int f) {  // mrcm.cpp:14-28
            if (g.is_vface(f)) {
                const int i = f % (g.nx + 1), j = f / (g.nx + 1);
                return i == 0 ? j : (i == g.nx ? g.ny + j : -1);
            }
            const int fh = f - g.vcount(), i = fh % g.nx, j = fh / g.nx;
            return j == 0 ? 2 * g.ny + i : (j == g.ny ? 2 * g.ny + g.nx + i : -1);
        };
        const auto& E = dd.sub_boundary[s];
        for (size_t idx = 0; idx < E.size(); ++idx) {
            const BoundaryEdge& e = E[idx];
            int32_t* o = edges + 8 * idx;
            o[0] = e.side;
            o[1] = e.local_cell;
            o[2] = e.local_face;
            o[3] = e.global_face;
            o[4] = e.iface;
            o[5] = e.pos;
            o[6] = e.on_skeleton ? -1 : gbc(e.global_face);
            o[7] = e.sign > 0 ? 1 : -1;
        }
        std::vector<int> inc;
        for (const auto& e : E)
            if (e.on_skeleton && std::find(inc.begin(), inc.end(), e.iface) == inc.end()) inc.push_back(e.iface);
        std::sort(inc.begin(), inc.end());
        int h = 0;
        for (int k : inc) for (int b : sp.flux_by_iface[k]) hom_cols[h++] = b;
        for (int k : inc) for (int b : sp.pres_by_iface[k]) hom_cols[h++] = sp.dim_flux() + b;
        *n_hom = h;
    });
}

}  // extern "C"
