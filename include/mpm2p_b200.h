/*
 * mpm2p_b200.h — C ABI of the B200-native MPM-2P / MRCM velocity-update and
 * saturation-update path.
 *
 * The reference (arxiv/paper_2103_11050, C++ library `mrcmflow`) has no FFI:
 * its boundary is the C++ API in proj/include/mrcmflow/ (*.hpp), called by
 * run() (proj/src/simulation.cpp:118-340) and by its tests. Every entry point
 * below replaces one of those C++ functions; the citation on each names the
 * reference declaration it stands in for. Arrays are plain host pointers in
 * the reference layouts:
 *   - cells row-major c = j*nx + i                        (grid.hpp:9-13)
 *   - faces: vertical f = j*(nx+1)+i, then horizontal
 *            (nx+1)*ny + j*nx + i, values = normal flux in +x/+y
 *   - boundary faces in BoundarySpec order W(ny) E(ny) S(nx) N(nx)
 *                                                          (elliptic.hpp:30-44)
 *   - skeleton edges flattened interface-major (interfaces: vertical ones
 *     sy-major, then horizontal; decomposition.cpp:28-56), position-minor
 *   - interface coefficients: U_H (flux bases) then P_H (pressure bases)
 *                                                          (mrcm.hpp:24-27)
 * No torch/CUDA types appear in any signature. The library never retains a
 * host pointer past the call that received it.
 *
 * Error convention (errors.hpp:9-24, mrcmflow_main.cpp:119-129): every call
 * returns 0 on success, MPM2P_ECONFIG (ConfigError), MPM2P_ENUMERIC
 * (NumericError), MPM2P_ECAPACITY (CapacityError, also a failed host
 * allocation), MPM2P_ECUDA or MPM2P_EINTERNAL; the message
 * is available from mpm2p_last_error(ctx).
 *
 * The CPU oracle (oracle/, test infrastructure only) exports the same
 * functions with the prefix `oracle_` instead of `mpm2p_`.
 */
#ifndef MPM2P_B200_H
#define MPM2P_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MPM2P_OK = 0,
    MPM2P_ECONFIG = 2,   /* ConfigError   (errors.hpp:9-12)  */
    MPM2P_ENUMERIC = 3,  /* NumericError  (errors.hpp:14-17) */
    MPM2P_ECAPACITY = 4, /* CapacityError (errors.hpp:19-22) */
    MPM2P_ECUDA = 5,     /* CUDA runtime failure (no reference counterpart) */
    MPM2P_EINTERNAL = 6  /* unexpected exception inside the library (a bug, never a config problem) */
};

/* BcKind (elliptic.hpp:13) */
enum { MPM2P_BC_PRESSURE = 0, MPM2P_BC_FLUX = 1, MPM2P_BC_ROBIN = 2 };
/* InterfaceSpace::Kind (interface_space.hpp:34) */
enum { MPM2P_SPACE_CONSTANT = 0, MPM2P_SPACE_LINEAR = 1 };
/* HbarSpec::Mode (interface_space.hpp:12) */
enum { MPM2P_HBAR_WHOLE = 0, MPM2P_HBAR_HALF = 1, MPM2P_HBAR_PER_EDGE = 2, MPM2P_HBAR_SEGMENT = 3 };
/* AlphaMode (robin.hpp:11) */
enum { MPM2P_ALPHA_UNIFORM = 0, MPM2P_ALPHA_ADAPTIVE = 1 };
/* EpsilonMode (mpm.hpp:15) */
enum { MPM2P_EPS_RELATIVE = 0, MPM2P_EPS_ABSOLUTE = 1, MPM2P_EPS_MOBILITY = 2 };
/* Method (simulation.hpp:13) */
enum {
    MPM2P_METHOD_FINE_REFERENCE = 0,
    MPM2P_METHOD_MRCM_EVERY_STEP = 1,
    MPM2P_METHOD_MPM2P = 2,
    MPM2P_METHOD_MPM2P_NO_UPDATES = 3
};

/* Everything RunInputs carries except the splitting policy and s0
 * (simulation.hpp:99-110), plus the decomposition/space/alpha knobs that
 * prepare() turns into shared objects (config.cpp:568-611). */
typedef struct mpm2p_problem {
    int32_t nx, ny;          /* build_grid (grid.cpp:9)            */
    double lx, ly;
    int32_t nsx, nsy;        /* build_decomposition (decomposition.cpp:21) */
    int32_t space_kind;      /* build_interface_space (interface_space.cpp:9) */
    int32_t hbar_mode, hbar_edges;
    int32_t alpha_mode;      /* AlphaSpec (robin.hpp:15-22)        */
    double alpha, alpha_min, alpha_max, percentile_lo, percentile_hi;
    double viscosity_ratio;  /* FluidModel M = mu_o/mu_w (transport.hpp:11-13) */
    const double* K;         /* permeability, nx*ny                */
    const double* q;         /* sources nx*ny, or NULL for zero     */
    const int32_t* bc_kind;  /* 2(nx+ny) BcKind                     */
    const double* bc_value;  /* 2(nx+ny) Pressure g / Flux z (outward) */
    /* FaceBc::beta / FaceBc::robin_rhs of physical Robin faces
     * (-beta u.n_out + p_face = robin_rhs, elliptic.hpp:16-28), 2(nx+ny)
     * each; read only where bc_kind == MPM2P_BC_ROBIN. NULL when the spec has
     * no Robin face. */
    const double* bc_beta;
    const double* bc_robin_rhs;
} mpm2p_problem;

/* SplittingConfig (simulation.hpp:18-31) + RunInputs::inflow_sat. */
typedef struct mpm2p_split {
    int32_t method;
    int32_t cn;
    double eta;
    int32_t eta_mode;
    double cfl_safety, dt_cap;
    int64_t te;
    double pvi_max;
    int32_t stop_on_breakthrough;
    int64_t max_steps_hard;
    double breakthrough_threshold;
    int32_t track_errors;   /* RunInputs::track_errors: a fine-reference shadow run (fine.cu) */
    double inflow_sat;
} mpm2p_split;

/* SolveCounters (mrcm.hpp:15-21) — exact integers. */
typedef struct mpm2p_counters {
    int64_t homogeneous, particular, downscale, fine, interface_solves;
} mpm2p_counters;

/* StepRecord (simulation.hpp:33-45). */
typedef struct mpm2p_step_record {
    int64_t step;
    double pvi, epsilon;
    int32_t rebuilt;
    double flux_err, sat_err;
    int64_t bf_homog_cum, bf_part_cum;
    double dt, wall_s, div_residual;
} mpm2p_step_record;

/* RunRecord (simulation.hpp:47-62) plus the decision-margin log (H4). */
typedef struct mpm2p_run_record {
    int64_t breakthrough_step;
    double breakthrough_pvi;
    int64_t te, tm_updates, tm_total, nhat;
    int32_t n_sub;
    mpm2p_counters counters;
    double max_div_residual, max_div_ratio;
    int32_t repair_warnings;
    double final_pvi;
    double min_eps_margin;  /* min over decisions of |eps - eta| / eta (bit-exactness guard) */
    int64_t clamp_count;    /* clamp_count() (transport.hpp:24-26) */
    /* Interface-solve diagnostics of this implementation (no reference
     * counterpart; the oracle writes zeros): interface_krylov = 0 dense
     * inverse, 1 MINRES, 2 direct block-tridiagonal; MINRES iteration counts. */
    int32_t interface_krylov, interface_max_iterations;
    int64_t interface_iterations;
    double min_rcond;  /* smallest interface-matrix rcond over the run's rebuilds (dense path; -1 otherwise) */
} mpm2p_run_record;

/* DownscaleResult diagnostics (mrcm.hpp:122-130). */
typedef struct mpm2p_downscale_info {
    double repair_max, flux_scale;
    int32_t repair_warning;
    double div_residual, div_scale;
} mpm2p_downscale_info;

/* Derived sizes (grid.hpp:22-25, decomposition.hpp:40-44, interface_space.hpp:37-38). */
typedef struct mpm2p_sizes {
    int32_t cells, faces, bfaces;
    int32_t n_sub, n_interfaces, skeleton_edges;
    int32_t dim_flux, dim_pressure;
    int64_t nhat;             /* homogeneous solves per rebuild (BasisSet::nhat) */
    int32_t sub_nx, sub_ny;
    int32_t sub_faces;        /* local faces per subdomain: (sub_nx+1) sub_ny + sub_nx (sub_ny+1) */
} mpm2p_sizes;

typedef struct mpm2p_ctx mpm2p_ctx;

/* ---- context ---------------------------------------------------------- */
/* prepare() (config.cpp:568-611): grid, decomposition, interface space and
 * boundary spec. Copies K/q/bc to the device. */
int mpm2p_create(const mpm2p_problem* prob, mpm2p_ctx** out);
void mpm2p_destroy(mpm2p_ctx* ctx);
const char* mpm2p_last_error(const mpm2p_ctx* ctx);
/* Message of the last failed mpm2p_create (no context exists then). */
const char* mpm2p_create_error(void);
int mpm2p_get_sizes(const mpm2p_ctx* ctx, mpm2p_sizes* out);

/* ---- transport (transport.cpp) ---------------------------------------- */
/* CellField conductivity(K, s, fluid)              transport.hpp:50  */
int mpm2p_conductivity(mpm2p_ctx* ctx, const double* s, double* kappa);
/* double max_fractional_flow_slope(fluid)          transport.hpp:22  */
int mpm2p_max_fractional_flow_slope(mpm2p_ctx* ctx, double* out);
/* double cfl_timestep(u, fluid, policy)            transport.hpp:41  */
int mpm2p_cfl_timestep(mpm2p_ctx* ctx, const double* u, double safety, double dt_cap, double* dt);
/* SaturationField upwind_step(s, u, dt, fluid)     transport.hpp:46-47 */
int mpm2p_upwind_step(mpm2p_ctx* ctx, const double* s, double inflow, const double* u, double dt,
                      double* s_out);
/* double injection_rate(u, inflow_sat, fluid)      simulation.hpp:96 */
int mpm2p_injection_rate(mpm2p_ctx* ctx, const double* u, double inflow, double* out);
/* double max_outlet_saturation(s, u)               simulation.hpp:93 */
int mpm2p_max_outlet_saturation(mpm2p_ctx* ctx, const double* s, const double* u, double* out);
/* CellField divergence(u)                          grid.hpp:79       */
int mpm2p_divergence(mpm2p_ctx* ctx, const double* u, double* div);

/* ---- fine-reference solve (simulation.cpp:143-150) ----------------------- */
/* LocalSolution solve_cell_centered(grid, kappa, q, bc, anchor)  elliptic.hpp
 * (elliptic.cpp:245-250) on the whole grid: p (cells) and u (faces) of the
 * undecomposed 5-point problem, anchor cell 0 iff every physical face is
 * Flux. Device path: two-level-Schwarz PCG to ||r|| <= 1e-13 ||b|| (fine.cu);
 * NumericError if it does not converge. Bumps SolveCounters::fine. */
int mpm2p_fine_solve(mpm2p_ctx* ctx, const double* kappa, double* p, double* u);
/* Diagnostics of the last fine solve (no reference counterpart): PCG
 * iterations, final relative residual, and conservation_residual /
 * residual_scale of its velocity (elliptic.cpp:252-267). Any pointer may be NULL. */
int mpm2p_fine_stats(mpm2p_ctx* ctx, int32_t* iterations, double* relres, double* div_residual,
                     double* div_scale);

/* ---- drift test (mpm.cpp:9-29) ----------------------------------------- */
/* double epsilon(kappa_n, kappa_m, mode)           mpm.hpp:20        */
int mpm2p_epsilon(mpm2p_ctx* ctx, const double* kappa_n, const double* kappa_m, int32_t mode,
                  double* out);

/* ---- coupling (robin.cpp) ---------------------------------------------- */
/* RobinParameter compute_beta(kappa, dd, spec)     robin.hpp:37-38
 * Outputs flattened per skeleton edge (interface-major), may be NULL. */
int mpm2p_compute_beta(mpm2p_ctx* ctx, const double* kappa, double* beta_minus,
                       double* beta_plus, double* alpha);

/* ---- MRCM / MPM-2P (mrcm.cpp, mpm.cpp) --------------------------------- */
/* GlobalSolution mrcm_solve(kappa, dd, space, beta, q, bc, counters)  mrcm.hpp:151-153
 * beta_minus/beta_plus NULL => compute_beta(kappa) with the problem's AlphaSpec.
 * Installs the basis and recon_m as the context's PerturbationState
 * (mpm.hpp:26-33) for later mpm2p_mpm_update calls. Output pointers may be NULL. */
int mpm2p_mrcm_solve(mpm2p_ctx* ctx, const double* kappa, const double* beta_minus,
                     const double* beta_plus, double* p, double* u, double* coeffs,
                     mpm2p_downscale_info* info, mpm2p_counters* counters);
/* MpmResult mpm_pressure_update(state, kappa_n, q, bc, counters)      mpm.hpp:53-55 */
int mpm2p_mpm_update(mpm2p_ctx* ctx, const double* kappa_n, double* p, double* u,
                     double* delta_coeffs, mpm2p_downscale_info* info, mpm2p_counters* counters);
/* BasisSet::iface_matrix (mrcm.hpp:68), dense dim x dim row-major. */
int mpm2p_interface_matrix(mpm2p_ctx* ctx, double* M);

/* ---- MRCM sub-steps (mrcm.hpp:77-136, 157-161) ---------------------------
 * Per-subdomain layouts (subdomain-major, s = sy*nsx + sx):
 *   cells     [n_sub][sub_nx*sub_ny]  local row-major r = jj*sub_nx + ii
 *   faces     [n_sub][sub_faces]      local faces: vertical (sub_nx+1)*sub_ny,
 *                                     then horizontal; global orientation
 *   edges     [n_sub][2(sub_nx+sub_ny)] boundary edges W, E, S, N (the local
 *                                     BoundarySpec order, elliptic.hpp:30-44)
 * LocalData = (q cells, edge kind / value / beta / robin_rhs);
 * LocalSolution = (p cells, u faces, boundary_p edges). */

/* std::shared_ptr<BasisSet> compute_basis_set(kappa, dd, space, beta, q, bc, counters)
 *                                                       mrcm.hpp:77-81
 * Factors every subdomain operator, solves the homogeneous and particular
 * problems, assembles and factors the interface matrix (rcond guard), and
 * installs the result as the context's basis. beta_minus/beta_plus NULL =>
 * compute_beta(kappa) with the problem's AlphaSpec. */
int mpm2p_compute_basis_set(mpm2p_ctx* ctx, const double* kappa, const double* beta_minus,
                            const double* beta_plus, mpm2p_counters* counters);
/* std::vector<LocalData> restrict_physical_data(dd, beta, q, bc)   mrcm.hpp:85-87
 * With the installed basis's beta. */
int mpm2p_restrict_physical_data(mpm2p_ctx* ctx, double* q_local, int32_t* kind_local, double* value_local,
                                 double* beta_local, double* robin_rhs_local);
/* ParticularSolution solve_particular(basis, data, counters)        mrcm.hpp:91-92
 * NumericError if the edges' kinds / betas differ from the factorization's. */
int mpm2p_solve_particular(mpm2p_ctx* ctx, const double* q_local, const int32_t* kind_local,
                           const double* value_local, const double* beta_local, const double* robin_rhs_local,
                           double* p_local, double* u_local, double* bp_local, mpm2p_counters* counters);
/* SkeletonCoeffs solve_interface(basis, particular, counters)       mrcm.hpp:95-96
 * u_local: the particular solution's face velocities. coeffs: U_H then P_H. */
int mpm2p_solve_interface(mpm2p_ctx* ctx, const double* u_local, double* coeffs, mpm2p_counters* counters);
/* MrcmReconstruction reconstruct(basis, coeffs, particular)         mrcm.hpp:100-101 */
int mpm2p_reconstruct(mpm2p_ctx* ctx, const double* coeffs, const double* p_local, const double* u_local,
                      const double* bp_local, double* p_out, double* u_out, double* bp_out);
/* std::vector<std::vector<double>> averaged_skeleton_flux(dd, recon) mrcm.hpp:105-106
 * flux per skeleton edge, interface-major (vertical interfaces first). */
int mpm2p_averaged_skeleton_flux(mpm2p_ctx* ctx, const double* u_local, double* flux);
/* DownscaleResult downscale(dd, kappa_current, q, bc, recon, skeleton_flux, counters)
 *                                                       mrcm.hpp:122-126 */
int mpm2p_downscale(mpm2p_ctx* ctx, const double* kappa, const double* p_local, const double* u_local,
                    const double* flux, double* p, double* u, mpm2p_downscale_info* info,
                    mpm2p_counters* counters);
/* WeakResiduals weak_continuity_residuals(basis, recon)             mrcm.hpp:157-161 */
int mpm2p_weak_continuity_residuals(mpm2p_ctx* ctx, const double* u_local, const double* bp_local, double* flux_jump,
                         double* pressure_jump);

/* ---- the driver (simulation.cpp:118-340) ------------------------------- */
/* RunResult run(in, snapshot_steps, snap)          simulation.hpp:127-128
 * steps may be NULL; otherwise it receives up to max_steps records. */
int mpm2p_run(mpm2p_ctx* ctx, const mpm2p_split* split, const double* s0, double* s_final,
              double* p_final, double* u_final, mpm2p_step_record* steps, int64_t max_steps,
              mpm2p_run_record* rec);
/* RunResult run(in, snapshot_steps, snap) with snapshots   simulation.hpp:119-128
 * SnapshotCallback: called on the calling thread after each step record whose
 * step is listed (the initial solve is step 0; simulation.cpp:207-227), with
 * host copies of s, p, u that are valid only during the call. */
typedef void (*mpm2p_snapshot_fn)(void* user, int64_t step, const double* s, const double* p, const double* u);
int mpm2p_run_snapshots(mpm2p_ctx* ctx, const mpm2p_split* split, const double* s0, double* s_final,
                        double* p_final, double* u_final, mpm2p_step_record* steps, int64_t max_steps,
                        mpm2p_run_record* rec, const int64_t* snapshot_steps, int64_t n_snapshots,
                        mpm2p_snapshot_fn snap, void* user);
/* The same loop, one Algorithm-1 iteration per call (inputs stay resident in
 * HBM). run_begin performs the initial solve and writes its record. */
int mpm2p_run_begin(mpm2p_ctx* ctx, const mpm2p_split* split, const double* s0,
                    mpm2p_step_record* first);
int mpm2p_run_step(mpm2p_ctx* ctx, mpm2p_step_record* out, int32_t* done);
int mpm2p_run_read(mpm2p_ctx* ctx, double* s, double* p, double* u);
int mpm2p_run_end(mpm2p_ctx* ctx, mpm2p_run_record* rec);

/* ---- cost model (simulation.cpp:11-28) --------------------------------- */
double mpm2p_rcr(int64_t nhat, int64_t n, int64_t te, int64_t tm);

/* ---- instrumentation (no reference counterpart; used by bench.py) ------ */
/* Host-only dump of the decomposition tables the kernels compute in closed
 * form (decomposition.cpp:101-129, mrcm.cpp:157-189): per boundary edge of
 * subdomain s, 8 ints {side, local_cell, local_face, global_face, interface,
 * pos, global BC index, sign}; hom_cols gets the n_hom interface-system
 * columns of s's homogeneous solves in order. Needs no GPU. */
int mpm2p_layout_tables(const mpm2p_problem* prob, int32_t s, int32_t* edges, int32_t* hom_cols,
                        int32_t* n_hom);
/* Selects the CUDA device for contexts created afterwards on this thread. */
int mpm2p_set_device(int32_t device);
/* Records CUDA event `slot` (0..15) on the context's stream. */
int mpm2p_timer_record(mpm2p_ctx* ctx, int32_t slot);
/* Device time between two recorded events (waits for `b`). */
int mpm2p_timer_elapsed(mpm2p_ctx* ctx, int32_t a, int32_t b, double* ms);
/* Writes a buffer larger than L2 (126 MB) on the context's stream. */
int mpm2p_flush_l2(mpm2p_ctx* ctx);
/* Per-kernel CUDA-event timing of every launch on the context's stream. */
int mpm2p_profile_enable(mpm2p_ctx* ctx, int32_t enable);
/* "name count total_ms" lines for every profiled kernel; resets the totals. */
int mpm2p_profile_report(mpm2p_ctx* ctx, char* buf, int32_t buflen);

#ifdef __cplusplus
}
#endif

#endif /* MPM2P_B200_H */
