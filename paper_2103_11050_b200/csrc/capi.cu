// capi.cu — context setup (prepare(), config.cpp:568-611), the Algorithm-1
// driver (run(), proj/src/simulation.cpp:118-340) as a host state machine
// over the device kernels, and the extern "C" boundary of
// include/mpm2p_b200.h. Exceptions map to the reference's error classes
// (errors.hpp:9-24) as status codes.
#include <new>
#include <algorithm>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "../../include/mpm2p_b200.h"
#include "band.cuh"
#include "context.cuh"

using namespace mpm2p;

namespace {

thread_local std::string g_create_err;

struct Driver {
    mpm2p_split sp{};
    long long n = 0, ell = 0;
    bool active = false;
    int rebuild_next = 0;
    mpm2p_run_record rec{};
    std::vector<mpm2p_step_record> steps;
    long long tm_total = 0;
    double min_rcond = -1.0;
    // FineReference method (every velocity from the fine solve) / track_errors
    // (a fine-reference shadow run beside the multiscale one); both run eagerly
    bool fine_ref = false, track = false;
};

}  // namespace

struct mpm2p_ctx {
    Ctx c;
    Driver d;
    std::unique_ptr<DevBuf<double>> scratch_a, scratch_b, scratch_c;
};

namespace {

template <typename F>
int guarded(mpm2p_ctx* ctx, F&& fn) {
    std::string* err = ctx ? &ctx->c.err : &g_create_err;
    try {
        fn();
        return MPM2P_OK;
    } catch (const ConfigError& e) {
        *err = e.what();
        return MPM2P_ECONFIG;
    } catch (const NumericError& e) {
        *err = e.what();
        return MPM2P_ENUMERIC;
    } catch (const CapacityError& e) {
        *err = e.what();
        return MPM2P_ECAPACITY;
    } catch (const CudaError& e) {
        *err = e.what();
        return MPM2P_ECUDA;
    } catch (const std::bad_alloc& e) {  // host allocation: out of capacity, not a bad config
        *err = std::string("host allocation failed: ") + e.what();
        return MPM2P_ECAPACITY;
    } catch (const std::exception& e) {  // anything else is an implementation fault, not the caller's config
        *err = std::string("internal error: ") + e.what();
        return MPM2P_EINTERNAL;
    }
}

// Large transfers from / to pageable host memory go through pinned staging:
// a pageable cudaMemcpy runs through the driver's bounce buffer with one host
// thread (C5's final s, p, u: 0.54 GB in ~112 ms). Two pinned 16 MB buffers
// per device, shared by the process's contexts; the device copies are
// pipelined against a multi-threaded host memcpy.
struct HostStage {
    std::mutex mu;
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2];
    bool ready = false;
};
constexpr size_t STAGE_BYTES = size_t(16) << 20;
constexpr size_t STAGE_MIN = size_t(8) << 20;  // smaller transfers: the plain copy
constexpr int STAGE_DEVICES = 64;

HostStage* host_stage() {  // the calling thread's current device, nullptr if unusable
    static HostStage stages[STAGE_DEVICES];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= STAGE_DEVICES) return nullptr;
    HostStage& h = stages[dev];
    std::lock_guard<std::mutex> g(h.mu);
    if (!h.ready) {
        for (int k = 0; k < 2; ++k) {
            CK(cudaMallocHost(&h.buf[k], STAGE_BYTES));
            CK(cudaEventCreateWithFlags(&h.ev[k], cudaEventDisableTiming));
        }
        h.ready = true;
    }
    return &h;
}

bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
    const int nt = (int)std::max<size_t>(1, std::min<size_t>(8, bytes >> 20));
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int t = 0; t < nt; ++t) {
        const size_t b0 = bytes * t / nt, b1 = bytes * (t + 1) / nt;
        std::memcpy(static_cast<char*>(dst) + b0, static_cast<const char*>(src) + b0, b1 - b0);
    }
}

void upload(Ctx& c, double* dst, const double* src, size_t n) {
    const size_t bytes = n * sizeof(double);
    HostStage* h = bytes >= STAGE_MIN && !host_pinned(src) ? host_stage() : nullptr;
    if (!h) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.st));
        return;
    }
    std::lock_guard<std::mutex> g(h->mu);
    const size_t nch = (bytes + STAGE_BYTES - 1) / STAGE_BYTES;
    for (size_t k = 0; k < nch; ++k) {
        const int b = (int)(k & 1);
        const size_t off = k * STAGE_BYTES, len = std::min(STAGE_BYTES, bytes - off);
        if (k >= 2) CK(cudaEventSynchronize(h->ev[b]));  // chunk k-2 has left this buffer
        par_memcpy(h->buf[b], reinterpret_cast<const char*>(src) + off, len);
        CK(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + off, h->buf[b], len, cudaMemcpyHostToDevice, c.st));
        CK(cudaEventRecord(h->ev[b], c.st));
    }
    CK(cudaStreamSynchronize(c.st));  // the staging buffers are reused by the next transfer
}
void download(Ctx& c, double* dst, const double* src, size_t n) {
    if (!dst) return;
    const size_t bytes = n * sizeof(double);
    HostStage* h = bytes >= STAGE_MIN && !host_pinned(dst) ? host_stage() : nullptr;
    if (!h) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.st));
        return;
    }
    std::lock_guard<std::mutex> g(h->mu);
    const size_t nch = (bytes + STAGE_BYTES - 1) / STAGE_BYTES;
    auto issue = [&](size_t k) {
        const int b = (int)(k & 1);
        const size_t off = k * STAGE_BYTES, len = std::min(STAGE_BYTES, bytes - off);
        CK(cudaMemcpyAsync(h->buf[b], reinterpret_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, c.st));
        CK(cudaEventRecord(h->ev[b], c.st));
    };
    issue(0);
    if (nch > 1) issue(1);
    for (size_t k = 0; k < nch; ++k) {
        const int b = (int)(k & 1);
        const size_t off = k * STAGE_BYTES, len = std::min(STAGE_BYTES, bytes - off);
        CK(cudaEventSynchronize(h->ev[b]));
        par_memcpy(reinterpret_cast<char*>(dst) + off, h->buf[b], len);
        if (k + 2 < nch) issue(k + 2);
    }
}

// Reads the per-step scalars back and raises the reference's exceptions for
// any guard the device tripped.
const Scalars& sync_scalars(Ctx& c) {
    CK(cudaMemcpyAsync(c.sc_host, c.sc.p, sizeof(Scalars), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    if (c.profiling) c.resolve_profile();
    const unsigned e = c.sc_host->err;
    if (e) {
        CK(cudaMemsetAsync(&c.sc.p->err, 0, sizeof(unsigned), c.st));
        if (e & ERR_CFL) throw NumericError("upwind_step: saturation left [0,1]; CFL condition violated");
        if (e & ERR_KAPPA) throw NumericError("CellCenteredSolver: conductivity must be positive and finite");
        if (e & ERR_ROBIN_BETA) throw ConfigError("CellCenteredSolver: Robin face requires beta > 0");
        if (e & ERR_PIVOT) throw NumericError("CellCenteredSolver: direct solve failed");
        if (e & ERR_STRUCT) throw NumericError("CellCenteredSolver: boundary structure changed since factorization");
        if (e & ERR_EPS_ZERO) throw NumericError("epsilon: zero reference norm in relative mode");
        if (e & ERR_TRACK_ZERO) throw NumericError("relative_flux_error: zero reference norm");
        if (e & ERR_FINE_NOCONV)
            throw NumericError("CellCenteredSolver: fine-grid PCG did not converge (relres " +
                               std::to_string(c.sc_host->fine_relres) + ")");
        if (e & ERR_SINGULAR)
            throw NumericError("compute_basis_set: interface matrix is numerically singular (rcond=" +
                               std::to_string(c.sc_host->rcond) + ")");
        throw NumericError("device error word " + std::to_string(e));
    }
    return *c.sc_host;
}

void reset_scalars(Ctx& c) {
    Scalars z{};
    z.min_margin = INFINITY;
    z.div_scale = 1.0;
    const double slope = c.sc_host ? c.sc_host->slope : 0.0;
    CK(cudaMemcpyAsync(c.sc.p, &z, sizeof(Scalars), cudaMemcpyHostToDevice, c.st));
    CK(cudaStreamSynchronize(c.st));
    (void)slope;
    launch_max_slope(c);
}

// CSR pattern of the interface matrix: row r (psi rows, then phi rows) couples
// to every basis of every interface that shares a subdomain with r's interface.
void build_csr(Ctx& c) {
    const Layout& L = c.L;
    const int np = L.dim_flux;
    std::vector<int> ptr(1, 0), col;
    ptr.reserve(2 * (size_t)np + 1);
    col.reserve(2 * (size_t)np * 16);
    for (int R = 0; R < 2 * np; ++R) {
        const int rb = R < np ? R : R - np;
        const int k = L.basis_iface(rb);
        int nb[8], nn = 0;  // interfaces incident to either side's subdomain, ascending, distinct
        for (int s : {L.iface_minus(k), L.iface_plus(k)}) {
            int inc[4];
            const int ni = L.incident(s, inc);
            for (int a = 0; a < ni; ++a) nb[nn++] = inc[a];
        }
        for (int a = 1; a < nn; ++a)  // insertion sort of <= 8 entries
            for (int b = a; b > 0 && nb[b - 1] > nb[b]; --b) std::swap(nb[b - 1], nb[b]);
        nn = (int)(std::unique(nb, nb + nn) - nb);
        for (int a = 0; a < nn; ++a)
            for (int t = 0; t < L.iface_nb(nb[a]); ++t) col.push_back(L.iface_first_basis(nb[a]) + t);
        for (int a = 0; a < nn; ++a)
            for (int t = 0; t < L.iface_nb(nb[a]); ++t) col.push_back(np + L.iface_first_basis(nb[a]) + t);
        ptr.push_back((int)col.size());
    }
    c.nnz = (int)col.size();
    // transposed positions (the pattern is structurally symmetric): tpos[z] for
    // z = (i, j) is the index of (j, i) in row j
    std::vector<int> tpos(col.size(), -1);
    for (int r = 0; r + 1 < (int)ptr.size(); ++r)
        for (int z = ptr[r]; z < ptr[r + 1]; ++z) {
            const int j = col[z];
            for (int z2 = ptr[j]; z2 < ptr[j + 1]; ++z2)
                if (col[z2] == r) {
                    tpos[z] = z2;
                    break;
                }
            if (tpos[z] < 0) throw ConfigError("interface system: CSR pattern is not symmetric");
        }
    c.csr_tpos.alloc(std::max<size_t>(tpos.size(), 1));
    if (!tpos.empty())
        CK(cudaMemcpyAsync(c.csr_tpos.p, tpos.data(), tpos.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    c.csr_ptr.alloc(ptr.size());
    std::vector<int> rowv(col.size());
    for (size_t r = 0; r + 1 < ptr.size(); ++r)
        for (int z = ptr[r]; z < ptr[r + 1]; ++z) rowv[z] = (int)r;
    c.csr_row.alloc(std::max<size_t>(rowv.size(), 1));
    if (!rowv.empty()) CK(cudaMemcpyAsync(c.csr_row.p, rowv.data(), rowv.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    c.csr_col.alloc(std::max<size_t>(col.size(), 1));
    c.csr_val.alloc(std::max<size_t>(col.size(), 1));
    CK(cudaMemcpyAsync(c.csr_ptr.p, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    if (!col.empty()) CK(cudaMemcpyAsync(c.csr_col.p, col.data(), col.size() * sizeof(int), cudaMemcpyHostToDevice, c.st));
    CK(cudaStreamSynchronize(c.st));
    if (c.use_krylov || c.use_blocktri) krylov_setup(c, ptr, col);  // K = J M in CSR
    if (c.use_blocktri) bt_setup(c);
}

// Grid, decomposition and interface-space sizes with the reference's
// validation (grid.cpp:9-15, decomposition.cpp:35-41, interface_space.cpp:9-52).
Layout make_layout(const mpm2p_problem* P) {
    Layout L{};
    if (P->nx < 1 || P->ny < 1)
        throw ConfigError("build_grid: cell counts must be >= 1, got " + std::to_string(P->nx) + "x" + std::to_string(P->ny));
    if (!(P->lx > 0.0) || !(P->ly > 0.0)) throw ConfigError("build_grid: domain lengths must be positive");
    if (P->nsx < 1 || P->nsy < 1) throw ConfigError("build_decomposition: subdomain counts must be >= 1");
    if (P->nx % P->nsx != 0 || P->ny % P->nsy != 0)
        throw ConfigError("build_decomposition: subdomains do not divide the grid");
    L.nx = P->nx;
    L.ny = P->ny;
    L.lx = P->lx;
    L.ly = P->ly;
    L.hx = P->lx / P->nx;
    L.hy = P->ly / P->ny;
    {
        int e;
        const bool px = std::frexp(L.hx, &e) == 0.5, py = std::frexp(L.hy, &e) == 0.5;
        const double v = L.hx * L.hy;
        L.pow2 = px && py && std::isnormal(v) && std::isnormal(1.0 / v) && std::isnormal(1.0 / L.hx) &&
                 std::isnormal(1.0 / L.hy);
        L.inv_hx = 1.0 / L.hx;
        L.inv_hy = 1.0 / L.hy;
        L.inv_vol = 1.0 / v;
    }
    L.nsx = P->nsx;
    L.nsy = P->nsy;
    L.snx = P->nx / P->nsx;
    L.sny = P->ny / P->nsy;
    L.n_sub = P->nsx * P->nsy;
    L.NV = P->nsy * (P->nsx - 1);
    L.NH = (P->nsy - 1) * P->nsx;
    L.n_iface = L.NV + L.NH;
    L.nbe = 2 * (L.snx + L.sny);
    L.ncs = L.snx * L.sny;
    if (L.snx > BAND_MAX)
        throw CapacityError("subdomain width " + std::to_string(L.snx) + " exceeds the banded kernel limit of " +
                            std::to_string(BAND_MAX) + " cells");
    // interface space (interface_space.cpp:9-52)
    L.space_kind = P->space_kind;
    if (P->space_kind == MPM2P_SPACE_LINEAR) {
        L.nbv = L.nbh = 2;
        L.segv = L.segh = 0;
    } else {
        auto seg_of = [&](int n) {
            int seg = n;
            switch (P->hbar_mode) {
                case MPM2P_HBAR_WHOLE: seg = n; break;
                case MPM2P_HBAR_HALF: seg = n / 2; break;
                case MPM2P_HBAR_PER_EDGE: seg = 1; break;
                case MPM2P_HBAR_SEGMENT: seg = P->hbar_edges; break;
                default: throw ConfigError("build_interface_space: unknown hbar mode");
            }
            if (seg < 1 || n % seg != 0)
                throw ConfigError("build_interface_space: segment length " + std::to_string(seg) +
                                  " does not divide an interface of " + std::to_string(n) + " edges");
            return seg;
        };
        L.segv = L.NV > 0 ? seg_of(L.sny) : 1;
        L.segh = L.NH > 0 ? seg_of(L.snx) : 1;
        L.nbv = L.NV > 0 ? L.sny / L.segv : 0;
        L.nbh = L.NH > 0 ? L.snx / L.segh : 0;
    }
    L.dim_flux = L.NV * L.nbv + L.NH * L.nbh;
    L.max_hom = 0;
    for (int s = 0; s < L.n_sub; ++s) L.max_hom = std::max(L.max_hom, L.n_hom(s));
    return L;
}

void create_ctx(mpm2p_ctx* ctx, const mpm2p_problem* P) {
    Ctx& c = ctx->c;
    if (!P->K || !P->bc_kind || !P->bc_value) throw ConfigError("problem: K and the boundary spec are required");
    c.L = make_layout(P);
    const Layout& L = c.L;
    c.nhat = 0;
    for (int s = 0; s < L.n_sub; ++s) c.nhat += L.n_hom(s);
    c.max_rhs = 1 + L.max_hom;
    c.dim = 2 * L.dim_flux;
    c.M = P->viscosity_ratio;
    c.alpha_mode = P->alpha_mode;
    c.alpha = P->alpha;
    c.alpha_min = P->alpha_min;
    c.alpha_max = P->alpha_max;
    c.pct_lo = P->percentile_lo;
    c.pct_hi = P->percentile_hi;
    // boundary spec
    const int nb = L.bfaces();
    c.bc_kind_h.assign(P->bc_kind, P->bc_kind + nb);
    bool pure_neumann = true;
    bool any_robin = false;
    for (int i = 0; i < nb; ++i) {
        const int k = c.bc_kind_h[i];
        if (k != BC_PRESSURE && k != BC_FLUX && k != BC_ROBIN) throw ConfigError("problem: unknown boundary kind");
        if (k == BC_ROBIN) {  // FaceBc::robin(beta, rhs) (elliptic.hpp:27)
            if (!P->bc_beta || !P->bc_robin_rhs)
                throw ConfigError("problem: Robin faces need bc_beta and bc_robin_rhs");
            any_robin = true;
        }
        if (k != BC_FLUX) pure_neumann = false;  // BoundarySpec::pure_neumann (elliptic.hpp:46-50)
        if (k == BC_PRESSURE) c.grounded = true;  // only Pressure faces absorb repair residual (mrcm.cpp:333-336)
    }
    c.anchor_m = (L.n_iface == 0) && pure_neumann;
    c.repair_active = L.n_sub > 1 || c.grounded;
    if (const char* e = std::getenv("MPM2P_NO_GRAPHS")) c.use_graphs = e[0] != 0 && e[0] == '0';
    if (const char* e = std::getenv("MPM2P_NO_REGBAND")) c.no_regband = e[0] == '1';
    if (const char* e = std::getenv("MPM2P_NO_TWIST")) c.no_twist = e[0] == '1';
    if (const char* e = std::getenv("MPM2P_DS_BLK")) c.ds_blk = std::atoi(e);
    if (const char* e = std::getenv("MPM2P_PDL")) c.pdl = e[0] == '1';
    if (const char* e = std::getenv("MPM2P_GRAPH_TIMING")) c.graph_timing = e[0] == '1';
    if (const char* e = std::getenv("MPM2P_UPWIND_TILE")) c.upwind_tiled = e[0] != '0';
    if (const char* e = std::getenv("MPM2P_UPWIND_COL")) c.upwind_col = std::atoi(e);
    if (const char* e = std::getenv("MPM2P_KAPPA_COL")) c.kappa_col = std::atoi(e);
    if (const char* e = std::getenv("MPM2P_HOM_GROUP")) c.hom_group = std::atoi(e);
    if (const char* e = std::getenv("MPM2P_RHS_SUB")) c.rhs_sub = e[0] != '0';
    if (const char* e = std::getenv("MPM2P_REFINE")) {  // 1: always refine, 0: never (experiments)
        c.force_refine = e[0] == '1';
        c.never_refine = e[0] == '0';
    }
    c.refine = true;
    // interface solver: dense inverse up to DENSE_IFACE_MAX, direct block-
    // tridiagonal above; MPM2P_IFACE = dense | blocktri | krylov overrides
    c.use_blocktri = c.dim > DENSE_IFACE_MAX;
    c.use_krylov = false;
    if (const char* e = std::getenv("MPM2P_IFACE")) {
        if (std::strcmp(e, "krylov") == 0) {
            c.use_krylov = c.dim > 0;
            c.use_blocktri = false;
        } else if (std::strcmp(e, "blocktri") == 0) {
            c.use_blocktri = c.dim > 0;
        } else if (std::strcmp(e, "dense") == 0) {
            c.use_blocktri = false;
        }
    }

    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, dev));
    // per-edge + per-cell right-hand side where the subdomains outnumber the
    // resident warps (C5: 457 -> 334 us); with few subdomains (C2) one CTA per
    // subdomain saves a launch (105 vs 109 us per MPM-2P step)
    c.rhs_w = L.n_sub > 8 * c.num_sms;
    if (const char* e = std::getenv("MPM2P_RHS_W")) c.rhs_w = e[0] != '0';
    CK(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
    configure_kernels();
    const size_t cells = L.cells(), faces = L.faces(), ns = L.n_sub, nbe = L.nbe, ncs = L.ncs;
    const size_t skel = std::max(1, L.skeleton_edges());
    c.K.alloc(cells);
    c.q.alloc(cells);
    c.bc_value.alloc(nb);
    c.bc_kind.alloc(nb);
    c.qsum_sub.alloc(ns);
    c.ground.alloc(ns);
    c.sep_repair = c.repair_active && sep_repair_setup(c);
    if (c.repair_active && !c.sep_repair) c.Linv.alloc(ns * ns);
    c.s.alloc(cells);
    c.s2.alloc(cells);
    c.u.alloc(faces);
    c.p.alloc(cells);
    c.kappa_n.alloc(cells);
    c.kappa_m.alloc(cells);
    c.lam_reb.alloc(cells);
    c.T.alloc(faces);
    c.beta_m.alloc(skel);
    c.beta_p.alloc(skel);
    c.alpha_e.alloc(skel);
    c.face_kappa.alloc(skel);
    c.sort_keys.alloc(skel);
    if (c.alpha_mode == MPM2P_ALPHA_ADAPTIVE && L.skeleton_edges() > 0) {
        CK(cub::DeviceRadixSort::SortKeys(nullptr, c.sort_tmp_bytes, c.face_kappa.p, c.sort_keys.p,
                                          L.skeleton_edges(), 0, 64, c.st));
        c.sort_tmp.alloc(std::max<size_t>(c.sort_tmp_bytes, 1));
    }
    const size_t B = L.snx;
    c.BDm.alloc(ns * ncs);
    c.BWm.alloc(ns * ncs);
    c.BSm.alloc(ns * ncs);
    c.Dm.alloc(ns * ncs);
    c.Lcm.alloc(ns * ncs * B);
    c.Lrm.alloc(ns * ncs * B);
    const size_t hmax = std::max(1, L.max_hom);
    c.HU.alloc(ns * hmax * nbe);
    c.HB.alloc(ns * hmax * nbe);
    c.HP.alloc(ns * hmax);
    c.pm.alloc(cells);
    c.bpm.alloc(ns * nbe);
    c.pmsum.alloc(ns);
    const size_t dim = std::max(1, c.dim);
    if (c.dim > 0 && !c.use_krylov && !c.use_blocktri)
        c.Minv.alloc((size_t)c.dim * c.dim);  // dense M only on the pivoted fallback
    c.irhs.alloc(dim);
    c.icoef.alloc(dim);
    c.ires.alloc(dim);
    c.idelta.alloc(dim);
    c.X.alloc(ns * c.max_rhs * ncs);
    c.PU.alloc(ns * nbe);
    c.PB.alloc(ns * nbe);
    c.PS.alloc(ns);
    c.GZ.alloc(ns * nbe);
    c.WU.alloc(ns * nbe);
    c.ET.alloc(ns * nbe);
    c.MGZ.alloc(ns * nbe);
    c.MET.alloc(ns * nbe);
    c.PD.alloc(ns * nbe);
    c.RU.alloc(ns * nbe);
    c.RS.alloc(ns);
    c.skel.alloc(skel);
    c.resid.alloc(ns);
    c.delta.alloc(ns);
    c.corr.alloc(std::max(1, L.n_iface));
    c.BDd.alloc(ns * ncs);
    c.BWd.alloc(ns * ncs);
    c.BSd.alloc(ns * ncs);
    c.Dd.alloc(ns * ncs);
    c.Lrd.alloc(ns * ncs * B);
    c.Xd.alloc(ns * ncs);
    // two-sided band solves: even widths <= 16 with at least 3 rows of cells
    // two-sided solves pay off where the local solves are latency-bound (few
    // subdomains per SM); with many subdomains the one-warp kernels keep
    // higher occupancy (C5: 16,384 subdomains)
    c.twist_ok = !c.no_regband && !c.no_twist && L.sny >= 3 && L.n_sub <= 8 * c.num_sms;
    if (const char* e = std::getenv("MPM2P_TWIST")) c.twist_ok = !c.no_regband && L.sny >= 3 && e[0] == '1';
    c.twist_store = c.twist_ok &&
                    (L.snx == 4 || L.snx == 8 || L.snx == 10 || L.snx == 12 || L.snx == 16 || L.snx == 20 ||
                     L.snx == 24 || L.snx == 32);
    if (c.twist_store) {
        c.tw_midb.alloc(ns * B * B);
        c.tw_sinv.alloc(ns * B * B);
    }
    // B <= 20: at B = 32 (C4) the stored two-sided factor doubles the
    // downscale's factor traffic and the side-stream factor competes with the
    // particular solve (measured C4 362 -> 400 us per step; C2 140 -> 127, C3 202 -> 165)
    c.ds_split = c.twist_store && L.snx <= 20;
    if (const char* e = std::getenv("MPM2P_DS_SPLIT")) c.ds_split = c.ds_split && e[0] != '0';
    c.blk_split = !c.ds_split && c.twist_ok && L.snx == 32 && c.ds_blk != 0;
    if (const char* e = std::getenv("MPM2P_BLK_SPLIT")) {
        if (e[0] == '1' && c.twist_ok && L.snx % 8 == 0 && L.snx >= 16 && L.snx <= 32 && c.ds_blk != 0) {
            c.blk_split = true;  // forced: instead of the two-sided split below B = 32
            c.ds_split = false;
        } else {
            c.blk_split = c.blk_split && e[0] != '0';
        }
    }
    if (c.blk_split) c.Gd.alloc((size_t)L.n_sub * L.ncs * 8);
    if (c.ds_split || c.blk_split) {
        CK(cudaStreamCreateWithFlags(&c.st2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
    }
    if (c.ds_split) {
        c.Lcd.alloc(ns * ncs * B);
        c.ds_midb.alloc(ns * B * B);
        c.ds_sinv.alloc(ns * B * B);
        c.ds_yscr.alloc(ns * ncs);
        c.ds_yscr.zero(c.st);
    }
    c.sc.alloc(1);
    c.red.alloc(16 * 8 * (size_t)c.num_sms + 4096);  // <= 16 values x 8 resident blocks / SM (red_blocks)
    c.red_count.alloc(1);
    CK(cudaMallocHost(&c.sc_host, sizeof(Scalars)));
    std::memset(c.sc_host, 0, sizeof(Scalars));
    c.red_count.zero(c.st);
    c.delta.zero(c.st);
    upload(c, c.K, P->K, cells);
    if (P->q) upload(c, c.q, P->q, cells);
    else c.q.zero(c.st);
    upload(c, c.bc_value, P->bc_value, nb);
    CK(cudaMemcpyAsync(c.bc_kind.p, P->bc_kind, nb * sizeof(int), cudaMemcpyHostToDevice, c.st));
    c.rb_beta.alloc(nb);
    c.rb_rhs.alloc(nb);
    if (any_robin) {
        std::vector<double> rb(nb, 0.0), rr(nb, 0.0);
        for (int i = 0; i < nb; ++i)
            if (c.bc_kind_h[i] == BC_ROBIN) {
                rb[i] = P->bc_beta[i];
                rr[i] = P->bc_robin_rhs[i];
            }
        upload(c, c.rb_beta, rb.data(), nb);
        upload(c, c.rb_rhs, rr.data(), nb);
        CK(cudaStreamSynchronize(c.st));
    } else {
        c.rb_beta.zero(c.st);
        c.rb_rhs.zero(c.st);
    }
    c.L.rb_beta = c.rb_beta.p;
    c.L.rb_rhs = c.rb_rhs.p;
    if (L.max_hom > 0) {  // static (interface, basis, flux?, column) table of the homogeneous functions
        std::vector<int4> tab((size_t)L.n_sub * L.max_hom, make_int4(0, 0, 0, 0));
        for (int sd = 0; sd < L.n_sub; ++sd)
            for (int h = 0; h < L.n_hom(sd); ++h) {
                int k, t, col;
                bool fl;
                L.hom(sd, h, k, t, fl, col);
                tab[(size_t)sd * L.max_hom + h] = make_int4(k, t, fl ? 1 : 0, col);
            }
        c.homtab.alloc(tab.size());
        CK(cudaMemcpyAsync(c.homtab.p, tab.data(), tab.size() * sizeof(int4), cudaMemcpyHostToDevice, c.st));
        CK(cudaStreamSynchronize(c.st));
        c.L.homtab = c.homtab.p;
    }
    if (c.dim > 0) build_csr(c);
    reset_scalars(c);
    launch_setup_static(c);
    CK(cudaStreamSynchronize(c.st));
}

// ---- driver (simulation.cpp:118-340) ----------------------------------------
void fill_counters(const Ctx& c, mpm2p_counters* o) {
    o->homogeneous = c.c_hom;
    o->particular = c.c_part;
    o->downscale = c.c_down;
    o->fine = c.c_fine;
    o->interface_solves = c.c_iface;
}

void note(Driver& d, const Scalars& s) {  // simulation.cpp:176-181
    d.rec.max_div_residual = std::max(d.rec.max_div_residual, s.div_residual);
    d.rec.max_div_ratio = std::max(d.rec.max_div_ratio, s.div_residual / s.div_scale);
    if (s.repair_warning) ++d.rec.repair_warnings;
}

mpm2p_step_record make_record(const Ctx& c, const Driver& d, const Scalars& s, int rebuilt, double dt, double wall) {
    mpm2p_step_record r{};
    r.step = d.n;
    r.pvi = s.pvi;
    r.epsilon = s.eps;
    r.rebuilt = rebuilt;
    r.bf_homog_cum = c.c_hom;
    r.bf_part_cum = c.c_part;
    r.dt = dt;
    r.wall_s = wall;
    r.div_residual = s.div_residual;
    return r;
}

// After a rebuild on the dense path: record rcond and decide whether the MPM
// steps using this inverse need the refinement step. A GEMV with the explicit
// inverse is accurate to ~cond * eps; refinement against the CSR operator is
// kept only when rcond <= Ctx::refine_rcond (1e-8), e.g. C3's channelised
// field (rcond 4e-10). C1/C2/C4 (rcond >= 2e-7) pass the 1e-8 parity bar with
// no refinement at all (MPM2P_REFINE=0).
void note_rcond(Ctx& c, Driver& d, double rcond) {
    if (c.use_krylov || c.dim == 0) return;
    if (d.min_rcond < 0.0 || rcond < d.min_rcond) d.min_rcond = rcond;
    if (c.use_blocktri) return;  // direct block solves: no refinement step
    c.refine = !c.never_refine && (c.force_refine || !(rcond > c.refine_rcond));
}

void breakthrough_check(Driver& d, const Scalars& s) {  // simulation.cpp:253-259
    if (d.rec.breakthrough_step >= 0) return;
    if (s.outlet_max > d.sp.breakthrough_threshold) {
        d.rec.breakthrough_step = d.n - 1;
        d.rec.breakthrough_pvi = s.pvi;
    }
}

// ---- fine-reference / track_errors runs (simulation.cpp:133-150,232-329) ----
// Eager (no graphs): the sub-cycling count of track_errors depends on both
// CFL steps (simulation.cpp:268-272), decided on the host each step. The
// multiscale branch, the transport and every record field are the same
// kernels as the graph path; the fine solves are fine.cu's PCG.
void swap_sat(Ctx& c) {
    std::swap(c.s.p, c.s2.p);
    c.s_par ^= 1;
}

void fine_record_extras(const Driver& d, const Scalars& s, mpm2p_step_record& r) {
    if (d.track) {
        r.flux_err = s.flux_err;
        r.sat_err = s.sat_err;
    }
    if (d.fine_ref) r.epsilon = 0.0;
}

void fine_run_begin(Ctx& c, Driver& d, mpm2p_step_record* first, std::chrono::steady_clock::time_point t0) {
    const mpm2p_split& sp = d.sp;
    const size_t nc = c.L.cells(), nf = c.L.faces();
    if (d.track) {
        c.t_sref.alloc(nc);
        c.t_sref2.alloc(nc);
        c.t_kref.alloc(nc);
        c.t_uref.alloc(nf);
        c.t_pref.alloc(nc);
        CK(cudaMemcpyAsync(c.t_sref.p, c.s.p, nc * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    }
    launch_conductivity(c, c.s, c.kappa_n, -1, false);  // k0
    if (d.fine_ref) {
        fine_solve(c, c.kappa_n, c.p, c.u, true);  // p_main = p_ref, u_main = u_ref (simulation.cpp:241-249)
    } else {
        fine_solve(c, c.kappa_n, c.t_pref, c.t_uref, true);
        launch_rebuild(c, c.kappa_n);
        launch_lambda(c, c.s, c.lam_reb);
    }
    launch_outlet(c, c.s, c.u);
    CK(cudaMemcpyAsync(&c.sc.p->eps_pending, &sp.eta, sizeof(double), cudaMemcpyHostToDevice, c.st));
    launch_decide(c, 0, sp.method, sp.eta, 0);
    if (d.track) launch_track_errors(c, c.u, c.t_uref, c.s, c.t_sref);
    const Scalars& s = sync_scalars(c);
    note(d, s);
    if (!d.fine_ref) note_rcond(c, d, s.rcond);
    Scalars s_rec = s;
    s_rec.eps = 0.0;
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    mpm2p_step_record r = make_record(c, d, s_rec, 1, 0.0, wall);
    fine_record_extras(d, s_rec, r);
    d.steps.push_back(r);
    d.tm_total = 1;
    if (first) *first = r;
    d.n = 1;
    d.rebuild_next = s.rebuild_next;
    breakthrough_check(d, s);
    d.active = true;
}

bool fine_run_step(Ctx& c, Driver& d, mpm2p_step_record* out) {
    const mpm2p_split& sp = d.sp;
    const auto t0 = std::chrono::steady_clock::now();
    const int rebuilt = d.fine_ref ? 1 : d.rebuild_next;
    if (!d.fine_ref && rebuilt) ++d.ell;
    const double* usched = d.track ? c.t_uref.p : c.u.p;  // simulation.cpp:266
    int sub = 1;
    if (d.track) {
        launch_cfl(c, c.u, sp.cfl_safety, sp.dt_cap);
        launch_save_dt_main(c);
    }
    launch_cfl(c, usched, sp.cfl_safety, sp.dt_cap);
    launch_inj_pvi(c, usched, sp.inflow_sat, sp.cn, true);  // pvi += inj dt / pore, cn times
    if (d.track) {  // simulation.cpp:268-272
        const Scalars& sc = sync_scalars(c);
        const double dt = sc.dt, dtm = sc.dt_main;
        if (dt > dtm * (1.0 + 1e-12)) sub = (int)std::ceil(dt / dtm - 1e-12);
    }
    c.outlet_s = nullptr;
    for (int k = 0; k < sp.cn; ++k) {
        for (int j = 0; j < sub; ++j) {
            launch_upwind(c, c.s, c.s2, c.u, sp.inflow_sat, false, 0, sub);
            swap_sat(c);
        }
        if (d.track) {
            launch_upwind(c, c.t_sref, c.t_sref2, c.t_uref, sp.inflow_sat);
            std::swap(c.t_sref.p, c.t_sref2.p);
        }
    }
    try {
        if (d.fine_ref) {
            launch_conductivity(c, c.s, c.kappa_n, -1, false);
            fine_solve(c, c.kappa_n, c.p, c.u);
            launch_outlet(c, c.s, c.u);
        } else {
            launch_conductivity_decide(c, c.s, c.kappa_n, sp.eta_mode, rebuilt, sp.method, sp.eta);
            launch_conductivity(c, c.t_sref, c.t_kref, -1, false);
            fine_solve(c, c.t_kref, c.t_pref, c.t_uref);  // u_ref, p_ref (simulation.cpp:281-285)
            c.outlet_s = c.s;
            if (rebuilt) {
                launch_rebuild(c, c.kappa_n);
                launch_lambda(c, c.s, c.lam_reb);
            } else {
                launch_mpm(c, c.kappa_n);
            }
            launch_track_errors(c, c.u, c.t_uref, c.s, c.t_sref);
        }
    } catch (...) {
        c.outlet_s = nullptr;
        c.trans_fresh = false;
        c.kappa_checked = false;
        throw;
    }
    c.outlet_s = nullptr;
    c.trans_fresh = false;
        c.kappa_checked = false;
    const Scalars& s = sync_scalars(c);
    note(d, s);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    mpm2p_step_record r = make_record(c, d, s, rebuilt, s.dt, wall);
    fine_record_extras(d, s, r);
    d.steps.push_back(r);
    if (rebuilt) {
        ++d.tm_total;
        if (!d.fine_ref) note_rcond(c, d, s.rcond);
    }
    if (out) *out = r;
    d.rebuild_next = d.fine_ref ? 0 : s.rebuild_next;
    ++d.n;
    breakthrough_check(d, s);
    return true;
}

void run_begin(mpm2p_ctx* ctx, const mpm2p_split* sp, const double* s0, mpm2p_step_record* first) {
    Ctx& c = ctx->c;
    Driver& d = ctx->d;
    if (sp->cn < 1) throw ConfigError("run: cn must be >= 1");
    if (sp->te <= 0 && sp->pvi_max <= 0.0 && !sp->stop_on_breakthrough)
        throw ConfigError("run: no stop condition configured");
    if (sp->method == MPM2P_METHOD_MPM2P && sp->eta < 0.0) throw ConfigError("run: negative eta");
    if (!s0) throw ConfigError("run: initial saturation grid mismatch");
    const bool multiscale = sp->method != MPM2P_METHOD_FINE_REFERENCE;  // simulation.cpp:131-133
    if (!multiscale || sp->track_errors) fine_setup(c);  // capacity / width checks before any state changes
    d = Driver{};
    d.sp = *sp;
    d.fine_ref = !multiscale;
    d.track = sp->track_errors != 0 && multiscale;
    d.rec.breakthrough_step = -1;
    d.rec.breakthrough_pvi = -1.0;
    d.rec.n_sub = c.L.n_sub;
    d.rec.min_eps_margin = INFINITY;
    c.c_hom = c.c_part = c.c_down = c.c_fine = c.c_iface = 0;
    c.drop_graphs();
    c.cfl_fused = false;
    reset_scalars(c);
    const auto t0 = std::chrono::steady_clock::now();
    upload(c, c.s, s0, c.L.cells());
    if (d.fine_ref || d.track) {
        fine_run_begin(c, d, first, t0);
        return;
    }
    // every pressure update of the run also forms the next step's CFL dt
    c.cfl_fused = true;
    c.cfl_safety = sp->cfl_safety;
    c.cfl_dt_cap = sp->dt_cap;
    c.cfl_inflow = sp->inflow_sat;
    launch_conductivity(c, c.s, c.kappa_n, -1, false);
    launch_rebuild(c, c.kappa_n);
    launch_lambda(c, c.s, c.lam_reb);
    launch_outlet(c, c.s, c.u);
    // epsilon_0 = eta: the first branch check reuses (simulation.cpp:205)
    CK(cudaMemcpyAsync(&c.sc.p->eps_pending, &sp->eta, sizeof(double), cudaMemcpyHostToDevice, c.st));
    launch_decide(c, 0, sp->method, sp->eta, 0);
    const Scalars& s = sync_scalars(c);
    note(d, s);
    note_rcond(c, d, s.rcond);
    Scalars s_rec = s;
    s_rec.eps = 0.0;
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    mpm2p_step_record r = make_record(c, d, s_rec, 1, 0.0, wall);
    d.steps.push_back(r);
    d.tm_total = 1;
    if (first) *first = r;
    d.n = 1;
    d.rebuild_next = s.rebuild_next;
    breakthrough_check(d, s);
    d.active = true;
}

bool run_step(mpm2p_ctx* ctx, mpm2p_step_record* out) {
    Ctx& c = ctx->c;
    Driver& d = ctx->d;
    const mpm2p_split& sp = d.sp;
    if (!d.active) throw ConfigError("run_step: run_begin not called");
    if (sp.te > 0 && d.n >= sp.te) return false;
    if (sp.pvi_max > 0.0 && c.sc_host->pvi >= sp.pvi_max) return false;
    if (sp.stop_on_breakthrough && d.rec.breakthrough_step >= 0) return false;
    if (d.n >= sp.max_steps_hard) return false;
    if (d.fine_ref || d.track) return fine_run_step(c, d, out);
    const auto t0 = std::chrono::steady_clock::now();
    const int rebuilt = d.rebuild_next;
    if (rebuilt) ++d.ell;
    // One Algorithm-1 iteration is a fixed kernel sequence per branch; it is
    // captured once per run as a CUDA graph (MPM-2P reuse / MRCM rebuild) and
    // replayed, so the device runs the ~30 kernels back to back. Profiling
    // mode launches them eagerly so each kernel can be timed.
    // cn upwind sub-steps ping-pong between s and s2; the step's saturation
    // ends in `cur` and the buffers are swapped afterwards (no copy)
    double* cur = (sp.cn % 2 == 1) ? c.s2.p : c.s.p;
    auto body = [&] {
        // cfl_timestep + injection_rate of this step were formed by the previous
        // pressure update's k_ds_u_div (c.cfl_fused); the first sub-step promotes them
        for (int k = 0; k < sp.cn; ++k) {
            launch_upwind(c, k % 2 == 0 ? c.s : c.s2, k % 2 == 0 ? c.s2 : c.s, c.u, sp.inflow_sat, k == 0, sp.cn);
        }
        launch_conductivity_decide(c, cur, c.kappa_n, sp.eta_mode, rebuilt, sp.method, sp.eta);
        c.outlet_s = cur;  // the step's last k_divres also takes max_outlet_saturation
        if (rebuilt) {
            launch_rebuild(c, c.kappa_n);
            launch_lambda(c, cur, c.lam_reb);
        } else {
            launch_mpm(c, c.kappa_n);
        }
        c.outlet_s = nullptr;
        c.trans_fresh = false;
        c.kappa_checked = false;
    };
    if (c.profiling || !c.use_graphs) {
        try {
            body();
        } catch (...) {
            c.outlet_s = nullptr;
            c.trans_fresh = false;
        c.kappa_checked = false;
            throw;
        }
    } else {
        cudaGraphExec_t& g = rebuilt ? c.g_rebuild[c.s_par] : c.g_mpm[c.s_par][c.refine ? 1 : 0];
        long long* delta = rebuilt ? c.gd_rebuild : c.gd_mpm;
        if (!g) {
            const long long before[5] = {c.c_hom, c.c_part, c.c_down, c.c_fine, c.c_iface};
            const long long launches_before = c.launch_count;
            CK(cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal));
            try {
                body();
            } catch (...) {
                c.outlet_s = nullptr;
                c.trans_fresh = false;
        c.kappa_checked = false;
                cudaGraph_t dummy = nullptr;
                cudaStreamEndCapture(c.st, &dummy);
                if (dummy) cudaGraphDestroy(dummy);
                throw;
            }
            cudaGraph_t graph = nullptr;
            CK(cudaStreamEndCapture(c.st, &graph));
            CK(cudaGraphInstantiate(&g, graph, 0));
            CK(cudaGraphDestroy(graph));
            const long long after[5] = {c.c_hom, c.c_part, c.c_down, c.c_fine, c.c_iface};
            for (int i = 0; i < 5; ++i) delta[i] = after[i] - before[i];
            delta[5] = c.launch_count - launches_before;
            c.c_hom = before[0];
            c.c_part = before[1];
            c.c_down = before[2];
            c.c_fine = before[3];
            c.c_iface = before[4];
            c.launch_count = launches_before;
        }
        if (c.graph_timing) {  // device time of the replay alone (timer slots 14 / 15)
            for (int t = 14; t < 16; ++t)
                if (!c.timers[t]) CK(cudaEventCreate(&c.timers[t]));
            CK(cudaEventRecord(c.timers[14], c.st));
        }
        CK(cudaGraphLaunch(g, c.st));
        if (c.graph_timing) CK(cudaEventRecord(c.timers[15], c.st));
        c.c_hom += delta[0];
        c.c_part += delta[1];
        c.c_down += delta[2];
        c.c_fine += delta[3];
        c.c_iface += delta[4];
        c.launch_count += delta[5];
    }
    if (sp.cn % 2 == 1) {
        std::swap(c.s.p, c.s2.p);
        c.s_par ^= 1;
    }
    const Scalars& s = sync_scalars(c);
    note(d, s);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    mpm2p_step_record r = make_record(c, d, s, rebuilt, s.dt, wall);
    d.steps.push_back(r);
    if (rebuilt) {
        ++d.tm_total;
        note_rcond(c, d, s.rcond);
    }
    if (out) *out = r;
    d.rebuild_next = s.rebuild_next;
    ++d.n;
    breakthrough_check(d, s);
    return true;
}

void run_end(mpm2p_ctx* ctx, mpm2p_run_record* out) {
    Ctx& c = ctx->c;
    Driver& d = ctx->d;
    if (!d.active) throw ConfigError("run_end: run_begin not called");
    d.rec.te = d.n;
    d.rec.tm_updates = d.ell;
    d.rec.tm_total = d.tm_total;
    d.rec.nhat = c.nhat;
    fill_counters(c, &d.rec.counters);
    d.rec.final_pvi = c.sc_host->pvi;
    d.rec.min_eps_margin = c.sc_host->min_margin;
    d.rec.clamp_count = c.sc_host->clamp;
    d.rec.interface_krylov = c.use_krylov ? 1 : (c.use_blocktri ? 2 : 0);
    d.rec.interface_max_iterations = c.sc_host->kr_iters_max;
    d.rec.interface_iterations = c.sc_host->kr_iters_total;
    d.rec.min_rcond = d.min_rcond;
    if (out) *out = d.rec;
    d.active = false;
    c.cfl_fused = false;
}

DevBuf<double>& scratch(std::unique_ptr<DevBuf<double>>& b, size_t n) {
    if (!b) b = std::make_unique<DevBuf<double>>();
    if (b->n < n) b->alloc(n);
    return *b;
}

void fill_info(const Scalars& s, mpm2p_downscale_info* info) {
    if (!info) return;
    info->repair_max = s.repair_max;
    info->flux_scale = s.flux_scale;
    info->repair_warning = s.repair_warning;
    info->div_residual = s.div_residual;
    info->div_scale = s.div_scale;
}

}  // namespace

extern "C" {

int mpm2p_create(const mpm2p_problem* prob, mpm2p_ctx** out) {
    *out = nullptr;
    auto* ctx = new mpm2p_ctx();
    const int rc = guarded(nullptr, [&] { create_ctx(ctx, prob); });
    if (rc != MPM2P_OK) {
        mpm2p_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return rc;
}

void mpm2p_destroy(mpm2p_ctx* ctx) {
    if (!ctx) return;
    if (ctx->c.st) cudaStreamSynchronize(ctx->c.st);
    if (ctx->c.sc_host) cudaFreeHost(ctx->c.sc_host);
    for (auto& p : ctx->c.pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : ctx->c.event_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->c.timers)
        if (e) cudaEventDestroy(e);
    ctx->c.drop_graphs();
    if (ctx->c.ev_fork) cudaEventDestroy(ctx->c.ev_fork);
    if (ctx->c.ev_join) cudaEventDestroy(ctx->c.ev_join);
    cudaStream_t st = ctx->c.st, st2 = ctx->c.st2;
    delete ctx;
    if (st) cudaStreamDestroy(st);
    if (st2) cudaStreamDestroy(st2);
}

const char* mpm2p_last_error(const mpm2p_ctx* ctx) { return ctx ? ctx->c.err.c_str() : g_create_err.c_str(); }
const char* mpm2p_create_error(void) { return g_create_err.c_str(); }

int mpm2p_get_sizes(const mpm2p_ctx* ctx, mpm2p_sizes* o) {
    const Layout& L = ctx->c.L;
    o->cells = L.cells();
    o->faces = L.faces();
    o->bfaces = L.bfaces();
    o->n_sub = L.n_sub;
    o->n_interfaces = L.n_iface;
    o->skeleton_edges = L.skeleton_edges();
    o->dim_flux = L.dim_flux;
    o->dim_pressure = L.dim_flux;
    o->nhat = ctx->c.nhat;
    o->sub_nx = L.snx;
    o->sub_ny = L.sny;
    o->sub_faces = sub_local_faces(L);
    return MPM2P_OK;
}

int mpm2p_conductivity(mpm2p_ctx* ctx, const double* s, double* kappa) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const size_t n = c.L.cells();
        auto& a = scratch(ctx->scratch_a, n);
        auto& b = scratch(ctx->scratch_b, n);
        upload(c, a, s, n);
        launch_conductivity(c, a, b, -1, false);
        download(c, kappa, b, n);
        sync_scalars(c);
    });
}

int mpm2p_max_fractional_flow_slope(mpm2p_ctx* ctx, double* out) {
    return guarded(ctx, [&] {
        launch_max_slope(ctx->c);
        *out = sync_scalars(ctx->c).slope;
    });
}

int mpm2p_cfl_timestep(mpm2p_ctx* ctx, const double* u, double safety, double dt_cap, double* dt) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        auto& a = scratch(ctx->scratch_a, c.L.faces());
        upload(c, a, u, c.L.faces());
        launch_cfl(c, a, safety, dt_cap);
        *dt = sync_scalars(c).dt;
    });
}

int mpm2p_upwind_step(mpm2p_ctx* ctx, const double* s, double inflow, const double* u, double dt, double* s_out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const size_t n = c.L.cells(), f = c.L.faces();
        auto& a = scratch(ctx->scratch_a, n);
        auto& b = scratch(ctx->scratch_b, n);
        auto& uu = scratch(ctx->scratch_c, f);
        upload(c, a, s, n);
        upload(c, uu, u, f);
        CK(cudaMemcpyAsync(&c.sc.p->dt, &dt, sizeof(double), cudaMemcpyHostToDevice, c.st));
        launch_upwind(c, a, b, uu, inflow);
        sync_scalars(c);
        download(c, s_out, b, n);
        CK(cudaStreamSynchronize(c.st));
    });
}

int mpm2p_injection_rate(mpm2p_ctx* ctx, const double* u, double inflow, double* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        auto& a = scratch(ctx->scratch_a, c.L.faces());
        upload(c, a, u, c.L.faces());
        launch_inj_pvi(c, a, inflow, 0, false);
        *out = sync_scalars(c).inj;
    });
}

int mpm2p_max_outlet_saturation(mpm2p_ctx* ctx, const double* s, const double* u, double* out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        auto& a = scratch(ctx->scratch_a, c.L.cells());
        auto& b = scratch(ctx->scratch_b, c.L.faces());
        upload(c, a, s, c.L.cells());
        upload(c, b, u, c.L.faces());
        launch_outlet(c, a, b);
        *out = sync_scalars(c).outlet_max;
    });
}

int mpm2p_fine_solve(mpm2p_ctx* ctx, const double* kappa, double* p, double* u) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        auto& a = scratch(ctx->scratch_a, c.L.cells());
        auto& pb = scratch(ctx->scratch_b, c.L.cells());
        auto& ub = scratch(ctx->scratch_c, c.L.faces());
        upload(c, a, kappa, c.L.cells());
        fine_solve(c, a, pb, ub, true);
        download(c, p, pb, c.L.cells());
        download(c, u, ub, c.L.faces());
        sync_scalars(c);
    });
}

int mpm2p_fine_stats(mpm2p_ctx* ctx, int32_t* iterations, double* relres, double* div_residual,
                     double* div_scale) {
    return guarded(ctx, [&] {
        const Scalars& s = sync_scalars(ctx->c);
        if (iterations) *iterations = s.fine_iters;
        if (relres) *relres = s.fine_relres;
        if (div_residual) *div_residual = s.div_residual;
        if (div_scale) *div_scale = s.div_scale;
    });
}

int mpm2p_divergence(mpm2p_ctx* ctx, const double* u, double* div) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        auto& a = scratch(ctx->scratch_a, c.L.faces());
        auto& b = scratch(ctx->scratch_b, c.L.cells());
        upload(c, a, u, c.L.faces());
        launch_divergence(c, a, b);
        download(c, div, b, c.L.cells());
        sync_scalars(c);
    });
}

int mpm2p_epsilon(mpm2p_ctx* ctx, const double* kn, const double* km, int32_t mode, double* out) {
    return guarded(ctx, [&] {
        if (mode == MPM2P_EPS_MOBILITY)
            throw ConfigError("epsilon: mobility mode needs saturation fields, not conductivities");
        Ctx& c = ctx->c;
        const size_t n = c.L.cells();
        auto& a = scratch(ctx->scratch_a, n);
        auto& b = scratch(ctx->scratch_b, n);
        upload(c, a, kn, n);
        upload(c, b, km, n);
        launch_epsilon_fields(c, a, b, mode);
        *out = sync_scalars(c).eps_pending;
    });
}

int mpm2p_compute_beta(mpm2p_ctx* ctx, const double* kappa, double* bm, double* bp, double* alpha) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const size_t n = c.L.cells(), E = c.L.skeleton_edges();
        auto& a = scratch(ctx->scratch_a, n);
        upload(c, a, kappa, n);
        launch_beta(c, a);
        sync_scalars(c);
        if (E) {
            download(c, bm, c.beta_m, E);
            download(c, bp, c.beta_p, E);
            download(c, alpha, c.alpha_e, E);
        }
        CK(cudaStreamSynchronize(c.st));
    });
}

int mpm2p_mrcm_solve(mpm2p_ctx* ctx, const double* kappa, const double* bm, const double* bp, double* p, double* u,
                     double* coeffs, mpm2p_downscale_info* info, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        c.trans_fresh = false;  // a caller's kappa: T and the kappa guard are formed here
        c.kappa_checked = false;
        const Layout& L = c.L;
        c.c_hom = c.c_part = c.c_down = c.c_fine = c.c_iface = 0;
        upload(c, c.kappa_n, kappa, L.cells());
        const bool given = bm && bp;
        if (given && L.skeleton_edges() > 0) {
            upload(c, c.beta_m, bm, L.skeleton_edges());
            upload(c, c.beta_p, bp, L.skeleton_edges());
        }
        launch_rebuild(c, c.kappa_n, !given);
        const Scalars& s = sync_scalars(c);
        download(c, p, c.p, L.cells());
        download(c, u, c.u, L.faces());
        if (coeffs && c.dim > 0) download(c, coeffs, c.icoef, c.dim);
        CK(cudaStreamSynchronize(c.st));
        fill_info(s, info);
        if (counters) fill_counters(c, counters);
    });
}

int mpm2p_mpm_update(mpm2p_ctx* ctx, const double* kappa_n, double* p, double* u, double* dcoeffs,
                     mpm2p_downscale_info* info, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        c.trans_fresh = false;  // a caller's kappa: T and the kappa guard are formed here
        c.kappa_checked = false;
        const Layout& L = c.L;
        if (!c.has_basis) throw ConfigError("mpm_update: no basis installed (call mrcm_solve first)");
        c.c_hom = c.c_part = c.c_down = c.c_fine = c.c_iface = 0;
        upload(c, c.kappa_n, kappa_n, L.cells());
        launch_mpm(c, c.kappa_n);
        const Scalars& s = sync_scalars(c);
        download(c, p, c.p, L.cells());
        download(c, u, c.u, L.faces());
        if (dcoeffs && c.dim > 0) download(c, dcoeffs, c.icoef, c.dim);
        CK(cudaStreamSynchronize(c.st));
        fill_info(s, info);
        if (counters) fill_counters(c, counters);
    });
}

int mpm2p_interface_matrix(mpm2p_ctx* ctx, double* M) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (!c.has_basis) throw ConfigError("interface_matrix: no basis installed");
        if (c.dim > 0 && M) {  // the operator lives in CSR: scatter its values
            std::vector<int> ptr(c.dim + 1), col(c.nnz);
            std::vector<double> val(c.nnz);
            CK(cudaMemcpyAsync(ptr.data(), c.csr_ptr.p, ptr.size() * sizeof(int), cudaMemcpyDeviceToHost, c.st));
            CK(cudaMemcpyAsync(col.data(), c.csr_col.p, col.size() * sizeof(int), cudaMemcpyDeviceToHost, c.st));
            CK(cudaMemcpyAsync(val.data(), c.csr_val.p, val.size() * sizeof(double), cudaMemcpyDeviceToHost, c.st));
            CK(cudaStreamSynchronize(c.st));
            std::fill(M, M + (size_t)c.dim * c.dim, 0.0);
            for (int r = 0; r < c.dim; ++r)
                for (int z = ptr[r]; z < ptr[r + 1]; ++z) M[(size_t)r * c.dim + col[z]] = val[z];
        }
        CK(cudaStreamSynchronize(c.st));
    });
}

// ---- MRCM sub-steps (substeps.cu) ------------------------------------------
namespace {
struct LocalBufs {  // device copies of the per-subdomain C-ABI arrays
    DevBuf<double> q, val, beta, rhs, p, u, bp, p2, u2, bp2, flux;
    DevBuf<int> kind;
};
void need_basis(const Ctx& c, const char* fn) {
    if (!c.has_basis) throw ConfigError(std::string(fn) + ": no basis installed (compute_basis_set or mrcm_solve first)");
}
void up_cells(Ctx& c, DevBuf<double>& d, const double* h, size_t n, const char* what) {
    if (!h) throw ConfigError(std::string("missing ") + what);
    d.alloc(std::max<size_t>(n, 1));
    upload(c, d, h, n);
}
}  // namespace

int mpm2p_compute_basis_set(mpm2p_ctx* ctx, const double* kappa, const double* bm, const double* bp,
                            mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        c.trans_fresh = false;  // a caller's kappa: T and the kappa guard are formed here
        c.kappa_checked = false;
        const Layout& L = c.L;
        c.c_hom = c.c_part = c.c_down = c.c_fine = c.c_iface = 0;
        upload(c, c.kappa_n, kappa, L.cells());
        const bool given = bm && bp;
        if (given && L.skeleton_edges() > 0) {
            upload(c, c.beta_m, bm, L.skeleton_edges());
            upload(c, c.beta_p, bp, L.skeleton_edges());
        }
        if (!given) launch_beta(c, c.kappa_n);
        c.trans_fresh = false;
        c.kappa_checked = false;
        launch_trans(c, c.kappa_n);
        launch_basis_core(c, c.kappa_n);
        sync_scalars(c);
        c.has_basis = true;
        c.mpm_static_ok = false;  // p^m of this basis is not known here: the MPM-2P edge data are formed per call
        if (counters) fill_counters(c, counters);
    });
}

int mpm2p_restrict_physical_data(mpm2p_ctx* ctx, double* q_local, int32_t* kind_local, double* value_local,
                                 double* beta_local, double* rhs_local) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const Layout& L = c.L;
        need_basis(c, "restrict_physical_data");
        const size_t nc = (size_t)L.n_sub * L.ncs, ne = (size_t)L.n_sub * L.nbe;
        LocalBufs b;
        b.q.alloc(nc), b.kind.alloc(ne), b.val.alloc(ne), b.beta.alloc(ne), b.rhs.alloc(ne);
        sub_restrict(c, b.q, b.kind, b.val, b.beta, b.rhs);
        download(c, q_local, b.q, nc);
        if (kind_local) CK(cudaMemcpyAsync(kind_local, b.kind.p, ne * sizeof(int), cudaMemcpyDeviceToHost, c.st));
        download(c, value_local, b.val, ne);
        download(c, beta_local, b.beta, ne);
        download(c, rhs_local, b.rhs, ne);
        sync_scalars(c);
    });
}

int mpm2p_solve_particular(mpm2p_ctx* ctx, const double* q_local, const int32_t* kind_local, const double* value_local,
                           const double* beta_local, const double* rhs_local, double* p_local, double* u_local,
                           double* bp_local, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const Layout& L = c.L;
        need_basis(c, "solve_particular");
        c.c_hom = c.c_part = c.c_down = c.c_fine = c.c_iface = 0;
        const size_t nc = (size_t)L.n_sub * L.ncs, ne = (size_t)L.n_sub * L.nbe;
        const size_t nf = (size_t)L.n_sub * sub_local_faces(L);
        LocalBufs b;
        up_cells(c, b.q, q_local, nc, "q_local");
        if (!kind_local) throw ConfigError("missing kind_local");
        b.kind.alloc(ne);
        CK(cudaMemcpyAsync(b.kind.p, kind_local, ne * sizeof(int), cudaMemcpyHostToDevice, c.st));
        up_cells(c, b.val, value_local, ne, "value_local");
        up_cells(c, b.beta, beta_local, ne, "beta_local");
        up_cells(c, b.rhs, rhs_local, ne, "robin_rhs_local");
        b.p.alloc(nc), b.u.alloc(nf), b.bp.alloc(ne);
        sub_solve_particular(c, b.q, b.kind, b.val, b.beta, b.rhs, b.p, b.u, b.bp);
        sync_scalars(c);
        download(c, p_local, b.p, nc);
        download(c, u_local, b.u, nf);
        download(c, bp_local, b.bp, ne);
        CK(cudaStreamSynchronize(c.st));
        if (counters) fill_counters(c, counters);
    });
}

int mpm2p_solve_interface(mpm2p_ctx* ctx, const double* u_local, double* coeffs, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const Layout& L = c.L;
        need_basis(c, "solve_interface");
        c.c_hom = c.c_part = c.c_down = c.c_fine = c.c_iface = 0;
        LocalBufs b;
        up_cells(c, b.u, u_local, (size_t)L.n_sub * sub_local_faces(L), "u_local");
        sub_solve_interface(c, b.u);
        sync_scalars(c);
        if (coeffs && c.dim > 0) download(c, coeffs, c.icoef, c.dim);
        CK(cudaStreamSynchronize(c.st));
        if (counters) fill_counters(c, counters);
    });
}

int mpm2p_reconstruct(mpm2p_ctx* ctx, const double* coeffs, const double* p_local, const double* u_local,
                      const double* bp_local, double* p_out, double* u_out, double* bp_out) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const Layout& L = c.L;
        need_basis(c, "reconstruct");
        const size_t nc = (size_t)L.n_sub * L.ncs, ne = (size_t)L.n_sub * L.nbe;
        const size_t nf = (size_t)L.n_sub * sub_local_faces(L);
        LocalBufs b;
        up_cells(c, b.p, p_local, nc, "p_local");
        up_cells(c, b.u, u_local, nf, "u_local");
        up_cells(c, b.bp, bp_local, ne, "bp_local");
        DevBuf<double> co;
        co.alloc(std::max(1, c.dim));
        if (c.dim > 0) up_cells(c, co, coeffs, c.dim, "coeffs");
        b.p2.alloc(nc), b.u2.alloc(nf), b.bp2.alloc(ne);
        sub_reconstruct(c, co, b.p, b.u, b.bp, b.p2, b.u2, b.bp2);
        sync_scalars(c);
        download(c, p_out, b.p2, nc);
        download(c, u_out, b.u2, nf);
        download(c, bp_out, b.bp2, ne);
        CK(cudaStreamSynchronize(c.st));
    });
}

int mpm2p_averaged_skeleton_flux(mpm2p_ctx* ctx, const double* u_local, double* flux) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const Layout& L = c.L;
        LocalBufs b;
        up_cells(c, b.u, u_local, (size_t)L.n_sub * sub_local_faces(L), "u_local");
        b.flux.alloc(std::max(1, L.skeleton_edges()));
        sub_skeleton_flux(c, b.u, b.flux);
        download(c, flux, b.flux, L.skeleton_edges());
        sync_scalars(c);
    });
}

int mpm2p_downscale(mpm2p_ctx* ctx, const double* kappa, const double* p_local, const double* u_local,
                    const double* flux, double* p, double* u, mpm2p_downscale_info* info, mpm2p_counters* counters) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        c.trans_fresh = false;  // a caller's kappa: T and the kappa guard are formed here
        c.kappa_checked = false;
        const Layout& L = c.L;
        c.c_hom = c.c_part = c.c_down = c.c_fine = c.c_iface = 0;
        LocalBufs b;
        up_cells(c, b.p, p_local, (size_t)L.n_sub * L.ncs, "p_local");
        up_cells(c, b.u, u_local, (size_t)L.n_sub * sub_local_faces(L), "u_local");
        b.flux.alloc(std::max(1, L.skeleton_edges()));
        if (L.skeleton_edges() > 0) up_cells(c, b.flux, flux, L.skeleton_edges(), "skeleton flux");
        upload(c, c.kappa_n, kappa, L.cells());
        sub_downscale(c, c.kappa_n, b.p, b.u, b.flux);
        const Scalars& s = sync_scalars(c);
        download(c, p, c.p, L.cells());
        download(c, u, c.u, L.faces());
        CK(cudaStreamSynchronize(c.st));
        fill_info(s, info);
        if (counters) fill_counters(c, counters);
    });
}

int mpm2p_weak_continuity_residuals(mpm2p_ctx* ctx, const double* u_local, const double* bp_local, double* flux_jump,
                         double* pressure_jump) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const Layout& L = c.L;
        need_basis(c, "weak_continuity_residuals");
        LocalBufs b;
        up_cells(c, b.u, u_local, (size_t)L.n_sub * sub_local_faces(L), "u_local");
        up_cells(c, b.bp, bp_local, (size_t)L.n_sub * L.nbe, "bp_local");
        DevBuf<double> out;
        out.alloc(2);
        sub_weak_residuals(c, b.u, b.bp, out);
        double h[2];
        CK(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, c.st));
        sync_scalars(c);
        if (flux_jump) *flux_jump = h[0];
        if (pressure_jump) *pressure_jump = h[1];
    });
}

int mpm2p_run(mpm2p_ctx* ctx, const mpm2p_split* sp, const double* s0, double* s_final, double* p_final,
              double* u_final, mpm2p_step_record* steps, int64_t max_steps, mpm2p_run_record* rec) {
    return guarded(ctx, [&] {
        run_begin(ctx, sp, s0, nullptr);
        while (run_step(ctx, nullptr)) {
        }
        Ctx& c = ctx->c;
        download(c, s_final, c.s, c.L.cells());
        download(c, p_final, c.p, c.L.cells());
        download(c, u_final, c.u, c.L.faces());
        CK(cudaStreamSynchronize(c.st));
        if (steps)
            for (int64_t i = 0; i < (int64_t)ctx->d.steps.size() && i < max_steps; ++i) steps[i] = ctx->d.steps[i];
        run_end(ctx, rec);
    });
}

int mpm2p_run_begin(mpm2p_ctx* ctx, const mpm2p_split* sp, const double* s0, mpm2p_step_record* first) {
    return guarded(ctx, [&] { run_begin(ctx, sp, s0, first); });
}

int mpm2p_run_step(mpm2p_ctx* ctx, mpm2p_step_record* out, int32_t* done) {
    return guarded(ctx, [&] { *done = run_step(ctx, out) ? 0 : 1; });
}

int mpm2p_run_snapshots(mpm2p_ctx* ctx, const mpm2p_split* sp, const double* s0, double* s_final, double* p_final,
                        double* u_final, mpm2p_step_record* steps, int64_t max_steps, mpm2p_run_record* rec,
                        const int64_t* snapshot_steps, int64_t n_snapshots, mpm2p_snapshot_fn snap, void* user) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const std::set<int64_t> want(snapshot_steps, snapshot_steps + (snapshot_steps ? n_snapshots : 0));
        std::vector<double> hs, hp, hu;
        auto maybe_snap = [&]() {  // simulation.cpp:224-226, after the step's record
            if (!snap || want.empty()) return;
            const int64_t n = ctx->d.steps.back().step;
            if (!want.count(n)) return;
            hs.resize(c.L.cells()), hp.resize(c.L.cells()), hu.resize(c.L.faces());
            download(c, hs.data(), c.s, c.L.cells());
            download(c, hp.data(), c.p, c.L.cells());
            download(c, hu.data(), c.u, c.L.faces());
            CK(cudaStreamSynchronize(c.st));
            snap(user, n, hs.data(), hp.data(), hu.data());
        };
        run_begin(ctx, sp, s0, nullptr);
        maybe_snap();
        while (run_step(ctx, nullptr)) maybe_snap();
        download(c, s_final, c.s, c.L.cells());
        download(c, p_final, c.p, c.L.cells());
        download(c, u_final, c.u, c.L.faces());
        CK(cudaStreamSynchronize(c.st));
        if (steps)
            for (int64_t i = 0; i < (int64_t)ctx->d.steps.size() && i < max_steps; ++i) steps[i] = ctx->d.steps[i];
        run_end(ctx, rec);
    });
}

int mpm2p_run_read(mpm2p_ctx* ctx, double* s, double* p, double* u) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        download(c, s, c.s, c.L.cells());
        download(c, p, c.p, c.L.cells());
        download(c, u, c.u, c.L.faces());
        CK(cudaStreamSynchronize(c.st));
    });
}

int mpm2p_run_end(mpm2p_ctx* ctx, mpm2p_run_record* rec) {
    return guarded(ctx, [&] { run_end(ctx, rec); });
}

int mpm2p_timer_record(mpm2p_ctx* ctx, int32_t slot) {
    return guarded(ctx, [&] {
        if (slot < 0 || slot >= 16) throw ConfigError("timer slot out of range");
        Ctx& c = ctx->c;
        if (!c.timers[slot]) CK(cudaEventCreate(&c.timers[slot]));
        CK(cudaEventRecord(c.timers[slot], c.st));
    });
}

int mpm2p_timer_elapsed(mpm2p_ctx* ctx, int32_t a, int32_t b, double* ms) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        if (a < 0 || a >= 16 || b < 0 || b >= 16 || !c.timers[a] || !c.timers[b])
            throw ConfigError("timer slot not recorded");
        CK(cudaEventSynchronize(c.timers[b]));
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, c.timers[a], c.timers[b]));
        *ms = f;
    });
}

// Host-only introspection of the closed-form decomposition (no GPU needed):
// per boundary edge of subdomain s, 8 ints: side, local_cell, local_face,
// global_face, interface (-1 physical), pos, global BC index, sign (+1/-1);
// then per homogeneous solve of s its interface-system column.
int mpm2p_layout_tables(const mpm2p_problem* prob, int32_t s, int32_t* edges, int32_t* hom_cols, int32_t* n_hom) {
    return guarded(nullptr, [&] {
        const Layout L = make_layout(prob);
        if (s < 0 || s >= L.n_sub) throw ConfigError("layout_tables: subdomain out of range");
        for (int idx = 0; idx < L.nbe; ++idx) {
            const EdgeInfo e = L.edge(s, idx);
            int32_t* o = edges + 8 * idx;
            o[0] = e.side;
            o[1] = e.local_cell;
            o[2] = e.local_face;
            o[3] = e.global_face;
            o[4] = e.iface;
            o[5] = e.pos;
            o[6] = e.gbc;
            o[7] = e.sign > 0 ? 1 : -1;
        }
        const int nh = L.n_hom(s);
        *n_hom = nh;
        for (int h = 0; h < nh; ++h) {
            int k, t, col;
            bool fl;
            L.hom(s, h, k, t, fl, col);
            hom_cols[h] = col;
        }
    });
}

int mpm2p_set_device(int32_t device) {
    return guarded(nullptr, [&] { CK(cudaSetDevice(device)); });
}

int mpm2p_flush_l2(mpm2p_ctx* ctx) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        const size_t bytes = (size_t)256 << 20;
        if (c.flush_buf.n < bytes) c.flush_buf.alloc(bytes);
        CK(cudaMemsetAsync(c.flush_buf.p, c.flush_buf.n & 0xff, bytes, c.st));
    });
}

int mpm2p_profile_enable(mpm2p_ctx* ctx, int32_t enable) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        CK(cudaStreamSynchronize(c.st));
        c.resolve_profile();
        c.profiling = enable != 0;
    });
}

int mpm2p_profile_report(mpm2p_ctx* ctx, char* buf, int32_t buflen) {
    return guarded(ctx, [&] {
        Ctx& c = ctx->c;
        CK(cudaStreamSynchronize(c.st));
        c.resolve_profile();
        std::string out = "__launches__ " + std::to_string(c.launch_count) + " 0\n";
        for (size_t i = 0; i < c.prof_names.size(); ++i)
            out += c.prof_names[i] + " " + std::to_string(c.prof_count[i]) + " " + std::to_string(c.prof_ms[i]) + "\n";
        c.prof_names.clear();
        c.prof_ms.clear();
        c.prof_count.clear();
        if (buf && buflen > 0) {
            std::strncpy(buf, out.c_str(), (size_t)buflen - 1);
            buf[buflen - 1] = '\0';
        }
    });
}

double mpm2p_rcr(int64_t nhat, int64_t n, int64_t te, int64_t tm) {  // simulation.cpp:11-19
    if (te <= 0 || nhat < 0 || n < 0 || tm < 0 || tm > te) return -1.0;
    const double frac = (double)(te - tm) / (double)te;
    const double bf = 1.0 - 2.0 * (double)n / (double)(nhat + 2 * n);
    return frac * bf * 100.0;
}

}  // extern "C"
