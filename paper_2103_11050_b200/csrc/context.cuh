// context.cuh — device-resident state of one simulation (the B200 stand-in
// for RunInputs + BasisSet + PerturbationState + the driver's fields,
// proj/include/mrcmflow/{simulation,mrcm,mpm}.hpp) and the kernel launchers.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "layout.cuh"

namespace mpm2p {

// Per-step device scalars (one 256-byte block read back once per step).
struct Scalars {
    double dt, pvi, inj, eps_pending, eps, slope;
    double repair_max, flux_scale, div_residual, div_scale;
    double outlet_max, rcond, min_margin;
    double eps_num_hi, eps_num_lo, eps_den_hi, eps_den_lo;
    unsigned err;
    int any_flow;
    int rebuild_next;
    int repair_warning;
    long long clamp;
    long long kr_iters_total;  // MINRES iterations (K7), summed over solves
    int kr_iters_max, kr_solves;
    double dt_next, inj_next;  // next step's cfl_timestep / injection_rate (k_ds_u_div with CflNext)
    int any_next;
    int fine_iters;            // PCG iterations of the last fine solve (fine.cu)
    double fine_relres;        // its final ||r|| / ||b||
    long long fine_iters_total;
    double dt_main;            // track_errors: cfl_timestep of u_main (sub-cycling, simulation.cpp:270-272)
    double flux_err, sat_err;  // track_errors records (simulation.cpp:30-59,210-215)
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        if (count == n && p) return;
        release();
        n = count;
        if (count) CK(cudaMalloc(&p, count * sizeof(T)));
    }
    void zero(cudaStream_t st) {
        if (p) CK(cudaMemsetAsync(p, 0, n * sizeof(T), st));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    operator T*() const { return p; }
};

struct Ctx {
    Layout L;
    cudaStream_t st = nullptr;
    std::string err;
    int num_sms = 148;

    // problem (host copies for validation/readback)
    double M = 1.0;
    int alpha_mode = 0;
    double alpha = 1, alpha_min = 1e-2, alpha_max = 1e2, pct_lo = 10, pct_hi = 90;
    std::vector<int> bc_kind_h;
    bool grounded = false;
    bool anchor_m = false;  // rebuild-time operator is pure Neumann (1x1, all-flux)
    bool repair_active = false;
    int max_rhs = 1;        // 1 + max homogeneous solves per subdomain
    int dim = 0;            // interface system dimension (2 * dim_flux)

    // static data
    DevBuf<double> K, q, bc_value, rb_beta, rb_rhs, qsum_sub, ground, Linv;
    DevBuf<int4> homtab;  // Layout::hom(s, h) for every (subdomain, homogeneous function)
    DevBuf<int> bc_kind;
    // transport / driver state
    DevBuf<double> s, s2, u, p, kappa_n, kappa_m, lam_reb, T;
    // rebuild cache (BasisSet)
    DevBuf<double> beta_m, beta_p, alpha_e, face_kappa, sort_keys;
    DevBuf<unsigned char> sort_tmp;
    size_t sort_tmp_bytes = 0;
    DevBuf<double> BDm, BWm, BSm, Dm, Lcm, Lrm;
    DevBuf<double> HU, HB, HP;
    DevBuf<double> pm, bpm, pmsum;
    // interface system (CSR pattern built once; values per rebuild)
    DevBuf<int> csr_ptr, csr_col, csr_row, csr_tpos;  // tpos[z]: position of the transposed entry
    DevBuf<double> csr_val, Mdense, Minv, gj_work, gj_col, gj_row, gj_krow;
    DevBuf<int> gj_piv, gj_aux;
    DevBuf<double> gj_pp;     // ping-pong GJ: two padded copies + two 32 x 32 pivot inverses
    DevBuf<double> irhs, icoef, ires, idelta;
    int nnz = 0;
    // K7 Krylov interface solve (dimension above the dense limit, or forced by
    // MPM2P_IFACE=krylov): K = J M in CSR, Jacobi preconditioner, MINRES work.
    bool use_krylov = false;
    double krylov_tol = 1e-13;
    int krylov_maxit = 20000;
    DevBuf<int> k_ptr, k_col;
    DevBuf<double> k_val, kr_pinv, kr_work;
    // K7b direct block-tridiagonal interface solve (blocktri.cu): the default
    // above the dense limit; MPM2P_IFACE=blocktri forces it, =krylov selects MINRES
    bool use_blocktri = false;
    bool rhs_w = true;  // per-edge + per-cell MPM-2P right-hand side (k_mpm_edges, k_mpm_rhs_w); MPM2P_RHS_W=0: k_mpm_rhs_sub
    // block-tridiagonal interface solve (blocktri.cu): block of each unknown,
    // its position in the block, block sizes; the cyclic-reduction plan
    int bt_nblk = 0;
    std::vector<int> bt_sz;
    DevBuf<int> bt_blk, bt_loc, bt_bsz;
    DevBuf<double> bt_y, bt_x;  // padded block-order work vectors
    std::shared_ptr<void> cr_plan;
    DevBuf<double> hg_x, hg_y, hg_z, hg_xi, hg_state;  // rcond estimate (bt_rcond)
    // per-solve scratch
    DevBuf<double> X, PU, PB, PS, GZ, WU, ET, RU, RS, skel, resid, delta, corr;
    // MPM-2P edge data owned by the MPM path (GZ / ET are the downscale's scratch): g' / z', the edge's rhs term,
    // and the static pressure drop p^m - p^m_face of the last rebuild
    DevBuf<double> MGZ, MET, PD;
    bool mpm_static_ok = false;  // MGZ / MET / PD hold the last rebuild's static entries (launch_rebuild)
    // downscale
    DevBuf<double> BDd, BWd, BSd, Dd, Lrd, Xd;
    // split downscale (latency regime): the kappa_n operator is factored on a
    // side stream (st2) while the particular / interface / recon chain runs;
    // only the two sweeps stay on the critical path
    bool ds_split = false;
    bool sep_repair = false;  // separable repair solve (sep_repair_setup) instead of the dense inverse
    DevBuf<double> sep_qx, sep_qy, sep_lam, sep_z1, sep_z2;
    bool rhs_sub = true;  // k_mpm_rhs_sub, one CTA per subdomain (MPM2P_RHS_SUB=0: one thread per cell)
    int kappa_col = -1;        // k_kappa_col: -1 auto (long row segments), 1 always, 0 never (MPM2P_KAPPA_COL)
    int hom_group = 8;         // homogeneous solves per warp in the rebuild (k_hom_solve_rm); 1: k_hom_solve_r (MPM2P_HOM_GROUP)
    int upwind_col = -1;       // k_upwind_col: -1 auto (long row segments), 1 always, 0 never (MPM2P_UPWIND_COL)
    bool upwind_tiled = true;  // k_upwind_tile (MPM2P_UPWIND_TILE=0: one thread per cell, k_upwind)
    bool ds_pending = false;  // a forked factor awaits its join (ev_join)
    cudaStream_t st2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    DevBuf<double> Lcd, ds_midb, ds_sinv, ds_yscr;
    // scalars and reduction workspace
    DevBuf<Scalars> sc;
    DevBuf<double> red;
    DevBuf<unsigned> red_count;
    Scalars* sc_host = nullptr;  // pinned

    int iface_sym = -1;  // J*M symmetric (pivot-free inverse)? -1 unknown
    // per-run CUDA graphs of one driver step (MPM-2P reuse / MRCM rebuild)
    bool use_graphs = true;
    // The driver's steps take dt from the previous pressure update's k_ds_u_div
    // (CflNext) instead of a separate k_cfl pass.
    bool cfl_fused = false;
    double cfl_safety = 0.0, cfl_dt_cap = 0.0, cfl_inflow = 0.0;
    std::unordered_map<const void*, int> occ;
    // fine-reference solve (fine.cu): global transmissibilities, blocked band
    // rows / factors of the block-Jacobi preconditioner, CG vectors (blocked
    // order; f_x is the warm start), coarse operator and its inverse
    DevBuf<double> f_T, f_BD, f_BW, f_BS, f_D, f_Lc, f_Lr, f_b, f_x, f_r, f_p, f_q, f_y;
    DevBuf<double> f_A0, f_A0i, f_c0, f_e, f_part;
    // coarse space above 4,096 subdomains (or MPM2P_FINE_COARSE=cr): block-
    // tridiagonal by subdomain rows, solved by cyclic reduction inside the PCG
    bool f_cr = false;
    std::shared_ptr<void> f_cr_plan;
    DevBuf<double> f_cy, f_cx;
    bool f_ready = false, f_warm = false;
    int f_anchor = -1;
    double f_tol = 1e-13;
    // track_errors / fine-reference runs: reference saturation (ping-pong),
    // its conductivity and the fine solution (simulation.cpp:133-150)
    DevBuf<double> t_sref, t_sref2, t_kref, t_uref, t_pref;  // resident blocks / SM per grid-stride kernel (TPB threads)
    bool trans_fresh = false;  // T already matches kappa_n (set by the driver's fused k_kappa)
    bool refine = true;        // one refinement step in MPM-2P interface solves (decided per rebuild from rcond)
    bool force_refine = false; // MPM2P_REFINE=1: always refine
    bool never_refine = false; // MPM2P_REFINE=0: never (accuracy experiments)
    double refine_rcond = 1e-8;  // refine when rcond <= this (cond >= 1e8; C3 yes, C1/C2/C4 no)
    bool pdl = false;  // programmatic dependent launch between kernels (MPM2P_PDL=1; measured neutral on C2)
    bool no_regband = false;  // MPM2P_NO_REGBAND=1: generic shared-memory band kernels only
    bool no_twist = false;    // MPM2P_NO_TWIST=1: one-sided register-window band solves
    bool kappa_checked = false;  // the current kappa came from the driver's k_kappa (already guarded)
    int ds_blk = -1;          // fused downscale on the DMMA blocked solver (band_blk.cuh): -1 auto (B = 24, 32), 0/1 (MPM2P_DS_BLK)
    bool twist_ok = false;    // two-sided band solves enabled for this problem (latency-bound regime)
    bool twist_store = false; // rebuild factor stored in the two-sided layout (band_twist.cuh)
    bool blk_split = false;   // B = 32 with few subdomains per SM: the blocked downscale factor on the side stream, sweeps after the join (MPM2P_BLK_SPLIT)
    DevBuf<double> Gd;        // its pivot-block inverses (8 doubles per cell)
    DevBuf<double> tw_midb, tw_sinv;  // per subdomain: bottom middle multipliers, middle S^-1 (B x B)
    // one graph per (branch, saturation-buffer parity): the upwind ping-pong
    // swaps s/s2 instead of copying, so the captured pointers alternate
    cudaGraphExec_t g_mpm[2][2] = {}, g_rebuild[2] = {};  // mpm: [parity][refine]
    long long gd_mpm[6] = {}, gd_rebuild[6] = {};  // counter / launch deltas per replay
    int s_par = 0;                                 // parity of the s/s2 pointer swap
    const double* outlet_s = nullptr;              // set during driver steps: k_divres also probes the outlet
    void drop_graphs() {
        for (int i = 0; i < 2; ++i) {
            for (int r = 0; r < 2; ++r) {
                if (g_mpm[i][r]) cudaGraphExecDestroy(g_mpm[i][r]);
                g_mpm[i][r] = nullptr;
            }
            if (g_rebuild[i]) cudaGraphExecDestroy(g_rebuild[i]);
            g_rebuild[i] = nullptr;
        }
    }
    bool has_basis = false;
    bool has_factor = false;
    double rcond = 0.0;

    // counters (exact integers, SolveCounters mrcm.hpp:15-21)
    long long c_hom = 0, c_part = 0, c_down = 0, c_fine = 0, c_iface = 0;
    long long nhat = 0;

    // instrumentation: per-kernel CUDA-event timing on this stream, user timers
    bool profiling = false;
    long long launch_count = 0;  // kernels launched on this context (all launches go through PROF)
    struct Pending { const char* name; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    std::vector<std::string> prof_names;
    std::vector<double> prof_ms;
    std::vector<long long> prof_count;
    cudaEvent_t timers[16] = {};
    bool graph_timing = false;  // MPM2P_GRAPH_TIMING=1: timers 14 / 15 bracket each step's graph replay
    DevBuf<unsigned char> flush_buf;

    cudaEvent_t take_event() {
        if (event_pool.empty()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    // Folds finished kernel timings into the per-name totals (stream must be idle).
    void resolve_profile() {
        for (auto& p : pending) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p.a, p.b));
            size_t i = 0;
            while (i < prof_names.size() && prof_names[i] != p.name) ++i;
            if (i == prof_names.size()) {
                prof_names.emplace_back(p.name);
                prof_ms.push_back(0.0);
                prof_count.push_back(0);
            }
            prof_ms[i] += ms;
            prof_count[i] += 1;
            event_pool.push_back(p.a);
            event_pool.push_back(p.b);
        }
        pending.clear();
    }
};

// Kernel launch on the context's stream with programmatic stream
// serialisation when enabled (every kernel begins with pdl_begin()).
// MPM2P_PDL=1 turns it on; on C2 it measured neutral (launch gaps are not
// the bottleneck), so it is off by default.
template <typename... KArgs, typename... Args>
inline void launch_k(const Ctx& c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = c.pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// Grid for a grid-stride reduction kernel of 256-thread blocks over `work`
// items: one wave of resident blocks (at most 8 per SM, which the reduction
// partial buffer c.red is sized for), never more blocks than items need.
// Per-device cache of a launch attribute / occupancy figure: function
// attributes and occupancy are properties of the device, so a process with
// contexts on several devices keeps one value per device ordinal.
struct DeviceCache {
    std::atomic<int> v[64];
    DeviceCache() {
        for (auto& x : v) x.store(-1);
    }
    std::atomic<int>& at() {
        int d = 0;
        cudaGetDevice(&d);
        return v[d & 63];
    }
};

template <typename... KArgs>
inline int red_blocks(Ctx& c, void (*kern)(KArgs...), long long work) {
    int& n = c.occ[(const void*)kern];
    if (n == 0) {
        int b = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0));
        n = b < 1 ? 1 : (b > 8 ? 8 : b);
    }
    const int need = cdiv(work, 256);
    return need < n * c.num_sms ? (need < 1 ? 1 : need) : n * c.num_sms;
}

// RAII scope recording CUDA events around one kernel launch when profiling.
struct ProfScope {
    Ctx& c;
    const char* name;
    cudaEvent_t a = nullptr;
    ProfScope(Ctx& cc, const char* n) : c(cc), name(n) {
        ++c.launch_count;
        if (c.profiling) {
            a = c.take_event();
            CK(cudaEventRecord(a, c.st));
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = c.take_event();
            cudaEventRecord(b, c.st);
            c.pending.push_back({name, a, b});
        }
    }
};
#define PROF(c, name) ::mpm2p::ProfScope prof_scope_##__LINE__((c), (name))

// ---- launchers (transport.cu) ----------------------------------------------
void launch_max_slope(Ctx& c);
void launch_cfl(Ctx& c, const double* u, double safety, double dt_cap);
void launch_inj_pvi(Ctx& c, const double* u, double inflow, int cn, bool add_pvi);
void launch_upwind(Ctx& c, const double* s_in, double* s_out, const double* u, double inflow, bool take_next = false,
                   int inj_cn = 0, int sub = 1);
void launch_track_errors(Ctx& c, const double* u, const double* ur, const double* s, const double* sr);
void launch_save_dt_main(Ctx& c);  // sc->dt_main = sc->dt
void launch_conductivity(Ctx& c, const double* s, double* kappa, int eps_mode, bool want_eps);
void launch_cfl_inj(Ctx& c, const double* u, double safety, double dt_cap, double inflow, int cn);
void launch_conductivity_decide(Ctx& c, const double* s, double* kappa, int eps_mode, int rebuilt, int method,
                                double eta);
void launch_outlet(Ctx& c, const double* s, const double* u);
void launch_lambda(Ctx& c, const double* s, double* lam);
void launch_divergence(Ctx& c, const double* u, double* div);
void launch_decide(Ctx& c, int rebuilt, int method, double eta, int step);
void launch_epsilon_fields(Ctx& c, const double* kn, const double* km, int mode);

// ---- launchers (solver.cu) -------------------------------------------------
void launch_trans(Ctx& c, const double* kappa);
void launch_beta(Ctx& c, const double* kappa);
void launch_rebuild(Ctx& c, const double* kappa, bool compute_beta = true);  // basis + interface matrix + recon_m + downscale
void launch_mpm(Ctx& c, const double* kappa_n);       // MPM-2P update + downscale
void launch_basis_core(Ctx& c, const double* kappa);  // compute_basis_set with beta and T in place (X, traces, interface factor)
bool particular_solve_x(Ctx& c);                      // particular solve in place on X[s][0] with the cached factor
void interface_solve(Ctx& c, bool refine);            // c.PU -> c.irhs -> c.icoef (mrcm.cpp:254-268)
void downscale(Ctx& c, const double* kappa, bool skel_given = false);  // c.RU, c.RS (+ c.skel) -> p, u (mrcm.cpp:306-439)
void ds_factor_fork(Ctx& c);                          // split downscale: factor on the side stream
// ---- MRCM sub-steps (substeps.cu; mrcm.hpp:77-136,157-161), device arrays in the C-ABI layouts
int sub_local_faces(const Layout& L);
void sub_restrict(Ctx& c, double* qL, int* kindL, double* valL, double* betaL, double* rhsL);
void sub_solve_particular(Ctx& c, const double* qL, const int* kindL, const double* valL, const double* betaL,
                          const double* rhsL, double* pL, double* uL, double* bpL);
void sub_solve_interface(Ctx& c, const double* uL);  // -> c.icoef
void sub_reconstruct(Ctx& c, const double* coef, const double* pL, const double* uL, const double* bpL, double* pO,
                     double* uO, double* bpO);
void sub_skeleton_flux(Ctx& c, const double* uL, double* flux);
void sub_downscale(Ctx& c, const double* kappa, const double* pL, const double* uL, const double* flux);
void sub_weak_residuals(Ctx& c, const double* uL, const double* bpL, double* out2);
void launch_setup_static(Ctx& c);                     // qsum, ground, repair operator inverse
bool sep_repair_setup(Ctx& c);                        // separable repair operator (before the Linv allocation)
void configure_kernels();

// ---- launchers (dense.cu) --------------------------------------------------
// In-place Gauss-Jordan inverse with partial pivoting of an n x n row-major
// matrix A into Ainv; returns the 1-norm reciprocal condition number.
double dense_inverse(Ctx& c, const double* A, double* Ainv, int n);
// Stream-ordered variant: writes rcond to rcond_dev and sets err_bit in the
// device error word when rcond <= threshold (no host synchronisation).
void dense_inverse_async(Ctx& c, const double* A, double* Ainv, int n, double* rcond_dev, unsigned err_bit,
                         double threshold);
// Interface inverse straight from the CSR operator (K = J M built padded,
// ping-pong GJ, M^-1 and the device rcond guard). Returns false when K is
// not symmetric (the caller then takes the pivoted dense path).
bool interface_inverse_csr(Ctx& c, double* rcond_dev, unsigned err_bit, double threshold);
// Interface matrix: pivot-free blocked GJ on K = J M (symmetric quasi-definite).
void interface_inverse_async(Ctx& c, const double* M, double* Minv, int n, double* rcond_dev, unsigned err_bit,
                             double threshold);
// SPD matrix (repair Laplacian): pivot-free blocked GJ; returns rcond.
double spd_inverse(Ctx& c, const double* A, double* Ainv, int n);
void block_gj_inplace_pub(Ctx& c, double* W, int n);  // SPD / quasi-definite, pivot-free, in place
// ---- fine-reference solve (fine.cu) ------------------------------------------
void fine_setup(Ctx& c);
void fine_solve(Ctx& c, const double* kappa, double* p, double* u, bool cold = false);
void launch_gemv(Ctx& c, const double* A, const double* x, double* y, int n);
void launch_gemv_acc(Ctx& c, const double* A, const double* x, double* y, int n);  // y += A x
void launch_csr_residual(Ctx& c, const int* ptr, const int* col, const double* val, const double* x,
                         const double* b, double* r, int n);
void launch_axpy(Ctx& c, double* y, const double* x, int n);

// ---- launchers (krylov.cu) -------------------------------------------------
constexpr int DENSE_IFACE_MAX = 16384;  // above this the interface solve is MINRES
void krylov_setup(Ctx& c, const std::vector<int>& mptr, const std::vector<int>& mcol);
void krylov_prepare(Ctx& c);                                  // after assembly
void krylov_solve(Ctx& c, const double* rhs, double* x);      // x = M^-1 rhs

// ---- launchers (blocktri.cu) ----------------------------------------------
void bt_setup(Ctx& c);                                    // block layout and buffers (once)
void bt_factor(Ctx& c);                                   // block LDL^T with explicit S_j^-1 (each rebuild)
void bt_solve(Ctx& c, const double* rhs, double* x);      // x = M^-1 rhs
void bt_rcond(Ctx& c, double threshold, unsigned err_bit);  // Hager/Higham rcond guard (each rebuild)
// generic cyclic-reduction systems (blocktri.cu): nb blocks of S x S (S % 64 == 0)
struct CrView {
    double* D;    // nb diagonal blocks, to fill (after cr_zero)
    double* Up0;  // nb upper coupling blocks K[j][j+1], to fill (the lower ones are their transposes)
    int nb, S;
    const void* jobs;    // GemvJob array of the solve
    const int2* phases;  // (first, count) per solve phase
    int nphase;
};
std::shared_ptr<void> cr_create(Ctx& c, int nb, int S, double* y, double* x);  // solve: y (overwritten) -> x
CrView cr_view(const std::shared_ptr<void>& plan);
void cr_zero(Ctx& c, const std::shared_ptr<void>& plan);
void cr_factor(Ctx& c, const std::shared_ptr<void>& plan, unsigned err_bit);

}  // namespace mpm2p
