// example_run.cpp — a reference-style caller of the shim: builds a problem the
// way proj/src/config.cpp:prepare() does and calls mrcmflow::run with
// snapshots, then mrcm_solve / mpm_pressure_update and the sub-step chain.
// usage: example_run K.bin nx ny nsx nsy M te out.bin
// K.bin: nx*ny doubles; out.bin: s_final, p_final, u_final, then per step
// (rebuilt, dt), the snapshot steps seen, and the sub-step chain's u.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "mrcmflow_b200.hpp"

using namespace mrcmflow;

int main(int argc, char** argv) {
    if (argc < 9) {
        std::fprintf(stderr, "usage: %s K.bin nx ny nsx nsy M te out.bin\n", argv[0]);
        return 2;
    }
    const int nx = std::atoi(argv[2]), ny = std::atoi(argv[3]), nsx = std::atoi(argv[4]), nsy = std::atoi(argv[5]);
    const double M = std::atof(argv[6]);
    const long te = std::atol(argv[7]);
    try {
        const StructuredGrid2D g = build_grid(nx, ny, 1.0, 1.0);
        CellField K(g);
        FILE* f = std::fopen(argv[1], "rb");
        if (!f || std::fread(K.v.data(), sizeof(double), K.v.size(), f) != K.v.size()) return 3;
        std::fclose(f);
        RunInputs in;
        in.dd = std::make_shared<DomainDecomposition>(build_decomposition(g, nsx, nsy));
        in.K = K;
        in.q = CellField(g, 0.0);
        in.fluid.viscosity_ratio = M;
        in.bc = BoundarySpec::uniform(g, FaceBc::pressure(1.0), FaceBc::pressure(0.0), FaceBc::flux(0.0), FaceBc::flux(0.0));
        in.space = std::make_shared<InterfaceSpace>(build_interface_space(*in.dd, InterfaceSpace::Kind::Constant));
        in.split.method = Method::Mpm2p;
        in.split.eta = 0.01;
        in.split.te = te;
        in.split.cfl_safety = 0.5;
        in.split.track_errors = false;
        in.s0 = CellField(g, 0.0);
        std::vector<long> seen;
        const RunResult r = run(in, {0, 2, 5}, [&](long n, const SaturationField&, const CellField&, const FaceField&) {
            seen.push_back(n);
        });
        // one MRCM solve and one MPM-2P update through the library API, then the sub-steps
        SolveCounters cnt;
        const RobinParameter beta = compute_beta(K, *in.dd, in.alpha);
        const GlobalSolution gs = mrcm_solve(K, in.dd, in.space, beta, in.q, in.bc, cnt);
        PerturbationState st;
        st.basis = gs.basis;
        st.recon_m = gs.recon;
        CellField kn = K;
        for (double& v : kn.v) v *= 1.05;
        const MpmResult mr = mpm_pressure_update(st, kn, in.q, in.bc, cnt);
        const auto basis = compute_basis_set(K, in.dd, in.space, beta, in.q, in.bc, cnt);
        const SkeletonCoeffs co = solve_interface(*basis, basis->particular, cnt);
        const MrcmReconstruction rec = reconstruct(*basis, co, basis->particular);
        const WeakResiduals w = weak_continuity_residuals(*basis, rec);
        FILE* o = std::fopen(argv[8], "wb");
        std::fwrite(r.s_final.s.v.data(), sizeof(double), r.s_final.s.v.size(), o);
        std::fwrite(r.p_final.v.data(), sizeof(double), r.p_final.v.size(), o);
        std::fwrite(r.u_final.v.data(), sizeof(double), r.u_final.v.size(), o);
        const long nrec = (long)r.record.steps.size();
        std::fwrite(&nrec, sizeof(long), 1, o);
        for (const auto& s : r.record.steps) {
            const double row[2] = {(double)s.rebuilt, s.dt};
            std::fwrite(row, sizeof(double), 2, o);
        }
        const long ns = (long)seen.size();
        std::fwrite(&ns, sizeof(long), 1, o);
        std::fwrite(seen.data(), sizeof(long), seen.size(), o);
        std::fwrite(gs.u.v.data(), sizeof(double), gs.u.v.size(), o);
        std::fwrite(mr.u.v.data(), sizeof(double), mr.u.v.size(), o);
        const double wr[2] = {w.flux_jump, w.pressure_jump};
        std::fwrite(wr, sizeof(double), 2, o);
        std::fclose(o);
        std::printf("ok te=%ld rebuilds=%ld snapshots=%ld weak=%.3e/%.3e\n", r.record.te, r.record.tm_total, ns,
                    w.flux_jump, w.pressure_jump);
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "ConfigError: %s\n", e.what());
        return 2;
    } catch (const NumericError& e) {
        std::fprintf(stderr, "NumericError: %s\n", e.what());
        return 3;
    } catch (const CapacityError& e) {
        std::fprintf(stderr, "CapacityError: %s\n", e.what());
        return 4;
    }
    return 0;
}
