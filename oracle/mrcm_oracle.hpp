// ============================================================================
// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain C++17 restatement (no Eigen) of the reference's MPM-2P / MRCM
// velocity-update and saturation-update path (arxiv/paper_2103_11050,
// proj/src/{grid,decomposition,elliptic,robin,interface_space,mrcm,mpm,
// transport,simulation}.cpp and the prepare/BC/IC semantics of config.cpp).
// Every function cites the reference file:line it follows.
//
// It is the parity CHECKER for the CUDA path and the `cpu_baseline` arm of
// bench.py. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it. The product library never links it.
//
// Eigen (>=3.3, unpinned; absent here) is replaced by exact direct solvers:
// banded LDL^T for the 5-point local/fine systems (Eigen SimplicialLDLT+AMD,
// elliptic.cpp:97-98,143-149), dense partial-pivot LU with a Hager/Higham
// 1-norm rcond estimate (Eigen PartialPivLU::rcond, mrcm.cpp:226-238), and
// banded LDL^T for the downscale repair Laplacian (Eigen dense LDLT,
// mrcm.cpp:372). Results agree with the Eigen build to solver roundoff; the
// pins are the reference's own known answers and proj/test_output.txt.
// ============================================================================
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// errors.hpp:9-24
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };

// Scalar type of the restatement: double (the reference's), or long double
// in the extended-precision build (liboracle_ld.so, -DORACLE_LONG_DOUBLE) used
// only to measure how far double-precision answers sit from the exact one.
#ifdef ORACLE_LONG_DOUBLE
using Real = long double;
#else
using Real = double;
#endif
using Vec = std::vector<Real>;

// grid.hpp:14-43
struct Grid {
    int nx = 0, ny = 0;
    Real lx = 0, ly = 0, hx = 0, hy = 0;
    Grid() = default;
    Grid(int nx_, int ny_, Real lx_, Real ly_)
        : nx(nx_), ny(ny_), lx(lx_), ly(ly_), hx(lx_ / nx_), hy(ly_ / ny_) {}
    int cells() const { return nx * ny; }
    int vcount() const { return (nx + 1) * ny; }
    int hcount() const { return nx * (ny + 1); }
    int faces() const { return vcount() + hcount(); }
    int cell(int i, int j) const { return j * nx + i; }
    int vface(int i, int j) const { return j * (nx + 1) + i; }
    int hface(int i, int j) const { return vcount() + j * nx + i; }
    bool is_vface(int f) const { return f < vcount(); }
    Real cx(int i) const { return (i + 0.5) * hx; }
    Real cy(int j) const { return (j + 0.5) * hy; }
    Real vol() const { return hx * hy; }
    Real area(int f) const { return is_vface(f) ? hy : hx; }
    bool same_shape(const Grid& o) const { return nx == o.nx && ny == o.ny && lx == o.lx && ly == o.ly; }
};
Grid build_grid(int nx, int ny, Real lx, Real ly);       // grid.cpp:9-15
Vec divergence(const Grid& g, const Vec& u);                  // grid.cpp:19-31

// decomposition.hpp:11-70
enum Side { West = 0, East = 1, South = 2, North = 3 };
inline Real side_sign(int s) { return (s == East || s == North) ? 1.0 : -1.0; }
struct Rect { int i0, j0, nx, ny; };
struct Interface { int minus = -1, plus = -1; bool vertical = true; std::vector<int> faces; };
struct BoundaryEdge {
    int global_face = -1, local_face = -1, local_cell = -1, side = 0;
    Real sign = 0.0;
    bool on_skeleton = false;
    int iface = -1, pos = -1;
};
struct Decomp {
    Grid grid;
    int nsx = 0, nsy = 0;
    std::vector<Rect> subs;
    std::vector<Grid> subgrids;
    std::vector<Interface> ifaces;
    std::vector<std::vector<BoundaryEdge>> sub_boundary;
    int n_sub() const { return nsx * nsy; }
    int n_iface() const { return (int)ifaces.size(); }
    int skeleton_edges() const;
    Real coarse_h() const;
    Vec restrict_cells(const Vec& global, int s) const;
};
Decomp build_decomposition(const Grid& g, int nsx, int nsy);  // decomposition.cpp:21-132

// elliptic.hpp:13-64
enum BcKind { Pressure = 0, Flux = 1, Robin = 2 };
struct FaceBc { int kind = Flux; Real value = 0, beta = 0, robin_rhs = 0; };
struct BoundarySpec {
    int nx = 0, ny = 0;
    std::vector<FaceBc> faces;
    BoundarySpec() = default;
    BoundarySpec(int nx_, int ny_) : nx(nx_), ny(ny_), faces(2 * (nx_ + ny_)) {}
    int count() const { return (int)faces.size(); }
    bool pure_neumann() const {
        for (const auto& f : faces) if (f.kind != Flux) return false;
        return true;
    }
};
struct LocalSolution { Vec p, u, boundary_p; };

Vec transmissibility(const Grid& g, const Vec& kappa);  // elliptic.cpp:44-61

// Banded symmetric LDL^T (half-bandwidth w, natural ordering).
struct BandLDLT {
    int n = 0, w = 0;
    Vec L;  // row r: entries for columns r-w .. r-1 at [r*w + (c - r + w)]
    Vec D;
    bool rev = false;
    void factor(const Vec& band);  // band: [r*(w+1) + (c - r + w)], c in [r-w, r]
    void solve(Vec& x) const;
    void solve_natural(Vec& x) const;
};
void set_elimination_order(int order);  // 0 natural, 1 reversed (all banded solves)

// CellCenteredSolver (elliptic.hpp:74-103, elliptic.cpp:68-243)
class LocalSolver {
public:
    explicit LocalSolver(const Grid& g) : g_(g) {}
    void factorize(const Vec& kappa, const BoundarySpec& bc, int anchor = -1);
    LocalSolution solve(const Vec& q, const BoundarySpec& bc) const;
    const Grid& grid() const { return g_; }
private:
    Grid g_;
    Vec trans_;
    BoundarySpec bc_struct_;
    int anchor_ = -1;
    BandLDLT ldlt_;
};
LocalSolution solve_cell_centered(const Grid& g, const Vec& kappa, const Vec& q,
                                  const BoundarySpec& bc, int anchor = -1);
Real conservation_residual(const Grid& g, const LocalSolution& sol, const Vec& q);
Real residual_scale(const Grid& g, const LocalSolution& sol, const Vec& q);

// interface_space.hpp:11-48
struct HbarSpec { int mode = 0; int edges = 0; };  // 0 whole, 1 half, 2 per-edge, 3 segment
struct InterfaceBasis { int iface = -1; Vec values; };
struct Space {
    int kind = 0;  // 0 constant, 1 linear
    std::vector<InterfaceBasis> flux, pres;
    std::vector<std::vector<int>> flux_by_iface, pres_by_iface;
    int dim_flux() const { return (int)flux.size(); }
    int dim_pres() const { return (int)pres.size(); }
};
Space build_interface_space(const Decomp& dd, int kind, HbarSpec hbar);

// robin.hpp:15-38
struct AlphaSpec {
    int mode = 0;  // 0 uniform, 1 adaptive
    Real alpha = 1.0, alpha_min = 1e-2, alpha_max = 1e2, pct_lo = 10.0, pct_hi = 90.0;
};
struct RobinParameter {
    std::vector<Vec> beta_minus, beta_plus, alpha;
    Real beta(int k, int pos, bool minus) const { return minus ? beta_minus[k][pos] : beta_plus[k][pos]; }
};
RobinParameter compute_beta(const Vec& kappa, const Decomp& dd, const AlphaSpec& spec);

// Dense partial-pivot LU (stand-in for Eigen::PartialPivLU).
struct DenseLU {
    int n = 0;
    Vec A;  // packed LU, row-major
    std::vector<int> perm;
    void compute(const Vec& M, int n);
    Vec solve(const Vec& b) const;
    Vec solve_transposed(const Vec& b) const;
    Real rcond(const Vec& M) const;  // Hager/Higham 1-norm estimate
};

// Banded partial-pivot LU of a row- and column-permuted sparse matrix
// (the LAPACK dgbtrf/dgbtrs algorithm, column-major band storage). The
// interface matrix is solved with it above kDenseInterfaceMax unknowns, where
// the reference's dense PartialPivLU (mrcm.cpp:198,226-238) would need a
// dim^2 matrix (C5: 34 GB, 1.8e14 flop). With the unknowns ordered by the
// interfaces' position in the subdomain grid (vertical interfaces of subdomain
// row j, then the horizontal ones above it) M is banded (C5: bandwidth ~510).
// Same mathematics as the dense LU: agreement at solver roundoff.
struct BandLU {
    int n = 0, kl = 0, ku = 0, ld = 0;
    std::vector<int> prow, pcol;  // A'(i, j) = M(prow[i], pcol[j])
    Vec AB;                       // A'(i, j) at AB[j * ld + kl + ku + i - j]
    std::vector<int> ipiv;
    bool singular = false;
    void init(int n, std::vector<int> prow, std::vector<int> pcol, int kl, int ku);
    Real& at(int i, int j) { return AB[(size_t)j * ld + kl + ku + i - j]; }
    Real get(int i, int j) const { return AB[(size_t)j * ld + kl + ku + i - j]; }
    void factor();
    Vec solve(const Vec& b) const;             // M x = b (original ordering)
    Vec solve_transposed(const Vec& b) const;  // M^T x = b
    Real rcond(Real anorm) const;          // Hager/Higham 1-norm estimate
};
constexpr int kDenseInterfaceMax = 16384;
void set_interface_solver(int mode);  // 0 auto (dense up to kDenseInterfaceMax), 1 dense, 2 banded
int interface_solver_mode();
void set_threads(int n);              // per-subdomain loops (default 1: the reference is single-threaded)

// mrcm.hpp:15-153
struct SolveCounters { long homogeneous = 0, particular = 0, downscale = 0, fine = 0, interface_solves = 0; };
struct SkeletonCoeffs { Vec flux, pres; };
struct LocalData { Vec q; BoundarySpec bc; };
struct BasisSet {
    struct Hom { int col; LocalSolution sol; };
    struct Sub { LocalSolver solver; BoundarySpec bc_struct; std::vector<Hom> hom; };
    std::shared_ptr<const Decomp> dd;
    std::shared_ptr<const Space> space;
    RobinParameter beta;
    Vec kappa_m;
    std::vector<Sub> subs;
    Vec M;  // dense interface matrix, row-major (dense solver only)
    DenseLU lu;
    bool banded = false;
    BandLU blu;  // banded solver (large interface systems)
    Vec dense_matrix() const;  // M, re-assembled when the banded solver holds it
    std::vector<LocalSolution> particular;
    int n_flux = 0, n_pres = 0;
    int dim() const { return n_flux + n_pres; }
    long nhat() const { long n = 0; for (const auto& s : subs) n += (long)s.hom.size(); return n; }
};
std::vector<LocalData> restrict_physical_data(const Decomp& dd, const RobinParameter& beta,
                                              const Vec& q, const BoundarySpec& bc);
std::shared_ptr<BasisSet> compute_basis_set(const Vec& kappa, std::shared_ptr<const Decomp> dd,
                                            std::shared_ptr<const Space> space,
                                            const RobinParameter& beta, const Vec& q,
                                            const BoundarySpec& bc, SolveCounters& c);
std::vector<LocalSolution> solve_particular(const BasisSet& b, const std::vector<LocalData>& data,
                                            SolveCounters& c);
SkeletonCoeffs solve_interface(const BasisSet& b, const std::vector<LocalSolution>& part,
                               SolveCounters& c);
std::vector<LocalSolution> reconstruct(const BasisSet& b, const SkeletonCoeffs& co,
                                       const std::vector<LocalSolution>& part);
std::vector<Vec> averaged_skeleton_flux(const Decomp& dd, const std::vector<LocalSolution>& recon);
struct DownscaleResult {
    Vec p, u;
    Real repair_max = 0, flux_scale = 0;
    bool repair_warning = false;
    Real div_residual = 0, div_scale = 1;
};
DownscaleResult downscale(const Decomp& dd, const Vec& kappa, const Vec& q, const BoundarySpec& bc,
                          const std::vector<LocalSolution>& recon, const std::vector<Vec>& skel,
                          SolveCounters& c);
struct GlobalSolution {
    std::shared_ptr<BasisSet> basis;
    SkeletonCoeffs coeffs;
    std::vector<LocalSolution> recon;
    DownscaleResult ds;
};
GlobalSolution mrcm_solve(const Vec& kappa, std::shared_ptr<const Decomp> dd,
                          std::shared_ptr<const Space> space, const RobinParameter& beta,
                          const Vec& q, const BoundarySpec& bc, SolveCounters& c);
struct WeakResiduals { Real flux_jump = 0, pressure_jump = 0; };
WeakResiduals weak_continuity_residuals(const BasisSet& b, const std::vector<LocalSolution>& recon);

// mpm.hpp:15-55
enum EpsMode { EpsRelative = 0, EpsAbsolute = 1, EpsMobility = 2 };
Real epsilon(const Grid& g, const Vec& kn, const Vec& km, int mode);
struct PerturbationState {
    std::shared_ptr<const BasisSet> basis;
    std::vector<LocalSolution> recon_m;
    Real eta = 0.01;
    int mode = EpsRelative;
};
struct MpmResult { SkeletonCoeffs delta; std::vector<LocalSolution> recon_n; DownscaleResult ds; };
MpmResult mpm_pressure_update(const PerturbationState& st, const Vec& kappa_n, const Vec& q,
                              const BoundarySpec& bc, SolveCounters& c);

// transport.hpp:11-50
int64_t clamp_count();
void reset_clamp_count();
Real total_mobility(Real s, Real M);
Real fractional_flow(Real s, Real M);
Real max_fractional_flow_slope(Real M);
Real cfl_timestep(const Grid& g, const Vec& u, Real M, Real safety, Real dt_cap);
Vec upwind_step(const Grid& g, const Vec& s, Real inflow, const Vec& u, Real dt, Real M);
Vec conductivity(const Vec& K, const Vec& s, Real M);

// simulation.hpp:13-128
enum Method { FineReference = 0, MrcmEveryStep = 1, Mpm2p = 2, Mpm2pNoUpdates = 3 };
struct Split {
    int method = Mpm2p, cn = 1;
    Real eta = 0.01;
    int eta_mode = EpsRelative;
    Real cfl_safety = 0.9, dt_cap = 1.0;
    long te = 0;
    Real pvi_max = 0.0;
    bool stop_on_breakthrough = false;
    long max_steps_hard = 50000;
    Real breakthrough_threshold = 0.05;
    bool track_errors = true;
};
struct StepRecord {
    long step = 0; Real pvi = 0, epsilon = 0; int rebuilt = 0;
    Real flux_err = 0, sat_err = 0; long bf_homog_cum = 0, bf_part_cum = 0;
    Real dt = 0, wall_s = 0, div_residual = 0;
};
struct RunRecord {
    std::vector<StepRecord> steps;
    std::vector<long> update_steps;
    long breakthrough_step = -1; Real breakthrough_pvi = -1.0;
    long te = 0, tm_updates = 0, tm_total = 0, nhat = 0; int n_sub = 0;
    SolveCounters counters;
    Real max_div_residual = 0, max_div_ratio = 0; int repair_warnings = 0;
    Real final_pvi = 0;
    Real min_eps_margin = INFINITY;
};
struct RunInputs {
    std::shared_ptr<const Decomp> dd;
    Vec K, q;
    Real M = 1.0;
    BoundarySpec bc;
    std::shared_ptr<const Space> space;
    AlphaSpec alpha;
    Split split;
    Vec s0;
    Real inflow_sat = 1.0;
};
struct RunResult { RunRecord rec; Vec s_final, p_final, u_final; };
Real rcr(long nhat, long n, long te, long tm);
Real relative_flux_error(const Grid& g, const Vec& u, const Vec& u_ref);
Real relative_sat_error(const Vec& s, const Vec& s_ref);
Real max_outlet_saturation(const Grid& g, const Vec& s, const Vec& u);
Real injection_rate(const Grid& g, const Vec& u, Real inflow, Real M);

// The Algorithm-1 driver, split into begin/step for the step-wise ABI.
class Runner {
public:
    explicit Runner(const RunInputs& in);
    void begin();
    bool step();  // one loop iteration; false when a stop condition held (no work done)
    RunResult finish();
    const RunInputs& in() const { return in_; }
    const RunRecord& record() const { return rec_; }
    const Vec& s() const { return s_main_; }
    const Vec& p() const { return p_main_; }
    const Vec& u() const { return u_main_; }
private:
    void rebuild(const Vec& kappa);
    void reuse(const Vec& kappa);
    LocalSolution fine_solve(const Vec& kappa);
    Real drift(const Vec& kappa_n);
    void note(Real dres, Real dscale, bool warn);
    void record_step(int rebuilt, Real eps, Real dt, Real wall);
    void breakthrough_check();
    RunInputs in_;
    RunRecord rec_;
    bool multiscale_ = true, track_ = false;
    Vec q_, s_main_, s_ref_, p_main_, u_main_, p_ref_, u_ref_, lambda_rebuild_;
    PerturbationState state_;
    std::unique_ptr<LocalSolver> fine_;
    int fine_anchor_ = -1;
    Real pvi_ = 0, eps_ = 0, step_div_ = 0;
    long n_ = 0, ell_ = 0;
};
RunResult run(const RunInputs& in);

// fields_io.cpp:25-116 (test-only restatement, used to pin the slab study)
Vec gaussian_field(const Grid& g, Real delta, Real mean_coeff, uint64_t seed, bool range_norm,
                   Real range_target);
Vec load_cell_field(const std::string& path, const Grid& g);
void save_cell_field(const std::string& path, const Grid& g, const Vec& f);

// config.cpp:525-538
BoundarySpec preset_bc(const Grid& g, int preset);  // 0 pressure-drop, 1 unit-inflow, 2 finger

}  // namespace orc
