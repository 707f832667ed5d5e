// mrcmflow_b200.hpp — the C++ face of the B200 path: the reference library's
// public names and signatures (proj/include/mrcmflow/{grid,elliptic,
// decomposition,interface_space,robin,transport,mrcm,mpm,simulation,errors}
// .hpp) implemented on the C ABI of include/mpm2p_b200.h (mrcmflow_b200.cpp).
//
// A maintainer switches the reference's callers (run(), its tests, tools) to
// the GPU by compiling them against this header instead of the Eigen-based
// one and linking libmrcmflow_b200 + libmpm2p_b200.so. Value types keep the
// reference's field names and layouts (CellField / FaceField / BoundarySpec /
// SplittingConfig / StepRecord / RunRecord / RunInputs / RunResult ...).
// Types whose reference members are Eigen factorizations (BasisSet, the
// coefficient vectors) hold the device context instead; their public fields
// are the reference's where they carry data callers read.
//
// Not provided here: the reference's CLI/config/report/VTK layers and the
// field generator (outside the hot path).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace mrcmflow {

// ---- errors.hpp:9-24
class ConfigError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class NumericError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class CapacityError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// ---- grid.hpp:14-79
struct StructuredGrid2D {
    int nx = 0, ny = 0;
    double lx = 0.0, ly = 0.0;
    double hx = 0.0, hy = 0.0;
    StructuredGrid2D() = default;
    StructuredGrid2D(int nx_, int ny_, double lx_, double ly_)
        : nx(nx_), ny(ny_), lx(lx_), ly(ly_), hx(lx_ / nx_), hy(ly_ / ny_) {}
    int cell_count() const { return nx * ny; }
    int vface_count() const { return (nx + 1) * ny; }
    int hface_count() const { return nx * (ny + 1); }
    int face_count() const { return vface_count() + hface_count(); }
    int cell(int i, int j) const { return j * nx + i; }
    int vface(int i, int j) const { return j * (nx + 1) + i; }
    int hface(int i, int j) const { return vface_count() + j * nx + i; }
    bool is_vface(int f) const { return f < vface_count(); }
    double cell_volume() const { return hx * hy; }
    double face_area(int f) const { return is_vface(f) ? hy : hx; }
    bool same_shape(const StructuredGrid2D& o) const { return nx == o.nx && ny == o.ny && lx == o.lx && ly == o.ly; }
};
StructuredGrid2D build_grid(int nx, int ny, double lx, double ly);

struct CellField {
    StructuredGrid2D grid;
    std::vector<double> v;
    CellField() = default;
    explicit CellField(const StructuredGrid2D& g, double init = 0.0) : grid(g), v(g.cell_count(), init) {}
    double& operator()(int i, int j) { return v[grid.cell(i, j)]; }
    double operator()(int i, int j) const { return v[grid.cell(i, j)]; }
    double& operator[](int c) { return v[c]; }
    double operator[](int c) const { return v[c]; }
    int size() const { return static_cast<int>(v.size()); }
};
struct FaceField {
    StructuredGrid2D grid;
    std::vector<double> v;
    FaceField() = default;
    explicit FaceField(const StructuredGrid2D& g, double init = 0.0) : grid(g), v(g.face_count(), init) {}
    double& operator[](int f) { return v[f]; }
    double operator[](int f) const { return v[f]; }
    int size() const { return static_cast<int>(v.size()); }
};
CellField divergence(const FaceField& u);

// ---- elliptic.hpp:13-64
enum class BcKind { Pressure, Flux, Robin };
struct FaceBc {
    BcKind kind = BcKind::Flux;
    double value = 0.0;
    double beta = 0.0;
    double robin_rhs = 0.0;
    static FaceBc pressure(double g) { return {BcKind::Pressure, g, 0.0, 0.0}; }
    static FaceBc flux(double z) { return {BcKind::Flux, z, 0.0, 0.0}; }
    static FaceBc robin(double beta, double rhs) { return {BcKind::Robin, 0.0, beta, rhs}; }
};
struct BoundarySpec {
    int nx = 0, ny = 0;
    std::vector<FaceBc> faces;
    BoundarySpec() = default;
    BoundarySpec(int nx_, int ny_) : nx(nx_), ny(ny_), faces(2 * (nx_ + ny_)) {}
    int count() const { return static_cast<int>(faces.size()); }
    int west(int j) const { return j; }
    int east(int j) const { return ny + j; }
    int south(int i) const { return 2 * ny + i; }
    int north(int i) const { return 2 * ny + nx + i; }
    bool pure_neumann() const {
        for (const auto& f : faces)
            if (f.kind != BcKind::Flux) return false;
        return true;
    }
    static BoundarySpec uniform(const StructuredGrid2D& g, FaceBc w, FaceBc e, FaceBc s, FaceBc n);
};
struct LocalSolution {
    CellField p;
    FaceField u;
    std::vector<double> boundary_p;
};

// ---- decomposition.hpp:48-70 (the tables live on the device; closed form there)
struct DomainDecomposition {
    StructuredGrid2D grid;
    int nsx = 0, nsy = 0;
    std::vector<StructuredGrid2D> subgrids;
    int subdomain_count() const { return nsx * nsy; }
    int interface_count() const { return nsy * (nsx - 1) + (nsy - 1) * nsx; }
    int skeleton_edge_count() const {
        return nsy * (nsx - 1) * (grid.ny / nsy) + (nsy - 1) * nsx * (grid.nx / nsx);
    }
    double coarse_h() const { return std::max(grid.lx / nsx, grid.ly / nsy); }
};
DomainDecomposition build_decomposition(const StructuredGrid2D& grid, int nsx, int nsy);

// ---- interface_space.hpp:11-48
struct HbarSpec {
    enum class Mode { WholeInterface, HalfInterface, PerEdge, EdgesPerSegment };
    Mode mode = Mode::WholeInterface;
    int edges = 0;
    static HbarSpec whole() { return {Mode::WholeInterface, 0}; }
    static HbarSpec half() { return {Mode::HalfInterface, 0}; }
    static HbarSpec per_edge() { return {Mode::PerEdge, 0}; }
    static HbarSpec segment_edges(int n) { return {Mode::EdgesPerSegment, n}; }
};
struct InterfaceSpace {
    enum class Kind { Constant, Linear };
    Kind kind = Kind::Constant;
    HbarSpec hbar;  // kept to rebuild the space on the device
    int n_flux = 0, n_pressure = 0;
    int dim_flux() const { return n_flux; }
    int dim_pressure() const { return n_pressure; }
};
InterfaceSpace build_interface_space(const DomainDecomposition& dd, InterfaceSpace::Kind kind,
                                     const HbarSpec& hbar = HbarSpec::whole());

// ---- robin.hpp:9-38
enum class AlphaMode { Uniform, Adaptive };
struct AlphaSpec {
    AlphaMode mode = AlphaMode::Uniform;
    double alpha = 1.0;
    double alpha_min = 1e-2;
    double alpha_max = 1e2;
    double percentile_lo = 10.0;
    double percentile_hi = 90.0;
};
struct RobinParameter {
    std::vector<std::vector<double>> beta_minus;
    std::vector<std::vector<double>> beta_plus;
    std::vector<std::vector<double>> alpha;
    double beta(int interface_id, int pos, bool minus_side) const {
        return minus_side ? beta_minus[interface_id][pos] : beta_plus[interface_id][pos];
    }
};
RobinParameter compute_beta(const CellField& kappa, const DomainDecomposition& dd, const AlphaSpec& spec);

// ---- transport.hpp:9-52
struct FluidModel {
    double viscosity_ratio = 1.0;
};
double max_fractional_flow_slope(const FluidModel& fluid);
struct SaturationField {
    CellField s;
    double inflow = 1.0;
};
struct CflPolicy {
    double safety = 0.9;
    double dt_cap = 1.0;
};
double cfl_timestep(const FaceField& u, const FluidModel& fluid, const CflPolicy& policy);
SaturationField upwind_step(const SaturationField& s, const FaceField& u, double dt, const FluidModel& fluid);
CellField conductivity(const CellField& K, const SaturationField& s, const FluidModel& fluid);

// ---- mrcm.hpp:15-161
struct SolveCounters {
    long homogeneous = 0;
    long particular = 0;
    long downscale = 0;
    long fine = 0;
    long interface_solves = 0;
};
struct SkeletonCoeffs {  // Eigen::VectorXd in the reference
    std::vector<double> flux;      // U_H
    std::vector<double> pressure;  // P_H
};
struct MrcmReconstruction {
    std::vector<LocalSolution> per_sub;
};
struct ParticularSolution {
    std::vector<LocalSolution> per_sub;
};
struct LocalData {
    CellField q;
    BoundarySpec bc;
};
namespace detail {
struct Backend;  // one device context (mpm2p_ctx)
}
class BasisSet {  // the factorizations live on the device, in `backend`
public:
    std::shared_ptr<const DomainDecomposition> dd;
    std::shared_ptr<const InterfaceSpace> space;
    RobinParameter beta;
    CellField kappa_m;
    ParticularSolution particular;  // for the (q, bc) the set was built with
    int n_flux = 0, n_pressure = 0;
    long nhat_ = 0;
    std::shared_ptr<detail::Backend> backend;
    int system_dim() const { return n_flux + n_pressure; }
    long nhat() const { return nhat_; }
};
std::shared_ptr<BasisSet> compute_basis_set(const CellField& kappa, std::shared_ptr<const DomainDecomposition> dd,
                                            std::shared_ptr<const InterfaceSpace> space, const RobinParameter& beta,
                                            const CellField& q, const BoundarySpec& bc, SolveCounters& counters);
ParticularSolution solve_particular(const BasisSet& basis, const std::vector<LocalData>& data,
                                    SolveCounters& counters);
SkeletonCoeffs solve_interface(const BasisSet& basis, const ParticularSolution& particular, SolveCounters& counters);
MrcmReconstruction reconstruct(const BasisSet& basis, const SkeletonCoeffs& coeffs,
                               const ParticularSolution& particular);
struct DownscaleResult {
    CellField p;
    FaceField u;
    double repair_max = 0.0;
    double flux_scale = 0.0;
    bool repair_warning = false;
    double div_residual = 0.0;
    double div_scale = 1.0;
};
struct GlobalSolution {
    std::shared_ptr<BasisSet> basis;
    SkeletonCoeffs coeffs;
    MrcmReconstruction recon;
    CellField p;
    FaceField u;
    double repair_max = 0.0;
    bool repair_warning = false;
    double div_residual = 0.0;
    double div_scale = 1.0;
};
GlobalSolution mrcm_solve(const CellField& kappa, std::shared_ptr<const DomainDecomposition> dd,
                          std::shared_ptr<const InterfaceSpace> space, const RobinParameter& beta,
                          const CellField& q, const BoundarySpec& bc, SolveCounters& counters);
struct WeakResiduals {
    double flux_jump = 0.0;
    double pressure_jump = 0.0;
};
WeakResiduals weak_continuity_residuals(const BasisSet& basis, const MrcmReconstruction& recon);

// ---- mpm.hpp:15-55
enum class EpsilonMode { Relative, Absolute, Mobility };
double epsilon(const CellField& kappa_n, const CellField& kappa_m, EpsilonMode mode);
struct PerturbationState {
    std::shared_ptr<const BasisSet> basis;
    MrcmReconstruction recon_m;
    double eta = 0.01;
    EpsilonMode mode = EpsilonMode::Relative;
    const CellField& kappa_m() const { return basis->kappa_m; }
};
bool needs_update(const PerturbationState& state, const CellField& kappa_n);
struct MpmResult {
    SkeletonCoeffs delta_coeffs;
    MrcmReconstruction recon_n;
    CellField p;
    FaceField u;
    double repair_max = 0.0;
    bool repair_warning = false;
    double div_residual = 0.0;
    double div_scale = 1.0;
};
MpmResult mpm_pressure_update(const PerturbationState& state, const CellField& kappa_n, const CellField& q,
                              const BoundarySpec& bc, SolveCounters& counters);

// ---- simulation.hpp:13-128
enum class Method { FineReference, MrcmEveryStep, Mpm2p, Mpm2pNoUpdates };
struct SplittingConfig {
    Method method = Method::Mpm2p;
    int cn = 1;
    double eta = 0.01;
    EpsilonMode eta_mode = EpsilonMode::Relative;
    double cfl_safety = 0.9;
    double dt_cap = 1.0;
    long te = 0;
    double pvi_max = 0.0;
    bool stop_on_breakthrough = false;
    long max_steps_hard = 50000;
    double breakthrough_threshold = 0.05;
    bool track_errors = true;
};
struct StepRecord {
    long step = 0;
    double pvi = 0.0;
    double epsilon = 0.0;
    int rebuilt = 0;
    double flux_err = 0.0;
    double sat_err = 0.0;
    long bf_homog_cum = 0;
    long bf_part_cum = 0;
    double dt = 0.0;
    double wall_s = 0.0;
    double div_residual = 0.0;
};
struct RunRecord {
    std::vector<StepRecord> steps;
    std::vector<long> update_steps;
    long breakthrough_step = -1;
    double breakthrough_pvi = -1.0;
    long te = 0;
    long tm_updates = 0;
    long tm_total = 0;
    long nhat = 0;
    int n_sub = 0;
    SolveCounters counters;
    double max_div_residual = 0.0;
    double max_div_ratio = 0.0;
    int repair_warnings = 0;
    double final_pvi = 0.0;
};
struct RunInputs {
    std::shared_ptr<const DomainDecomposition> dd;
    CellField K;
    CellField q;
    FluidModel fluid;
    BoundarySpec bc;
    std::shared_ptr<const InterfaceSpace> space;
    AlphaSpec alpha;
    SplittingConfig split;
    CellField s0;
    double inflow_sat = 1.0;
};
struct RunResult {
    RunRecord record;
    SaturationField s_final;
    CellField p_final;
    FaceField u_final;
};
using SnapshotCallback =
    std::function<void(long step, const SaturationField& s, const CellField& p, const FaceField& u)>;
RunResult run(const RunInputs& in, const std::vector<long>& snapshot_steps = {}, const SnapshotCallback& snap = nullptr);

}  // namespace mrcmflow
