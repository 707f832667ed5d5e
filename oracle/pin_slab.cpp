// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
// Reproduces the reference acceptance slab study (proj/tests/acceptance.cpp:
// 122-164, run_slab_study(303)) with the restated oracle and prints the
// numbers proj/test_output.txt:7-22 records, as one JSON object. This pins
// the oracle against the reference's own recorded run.
#include <cstdio>
#include <string>

#include "mrcm_oracle.hpp"

using namespace orc;

namespace {
// preset("gaussian-slab") (config.cpp:443-462) + prepare (config.cpp:568-611)
RunInputs slab(const Vec& K, int method, double eta, int mode, int hbar_mode, long te, bool stop_bt) {
    const Grid g = build_grid(64, 64, 1.0, 1.0);
    RunInputs in;
    auto dd = std::make_shared<Decomp>(build_decomposition(g, 4, 4));
    in.dd = dd;
    in.space = std::make_shared<Space>(build_interface_space(*dd, 0, HbarSpec{hbar_mode, 0}));
    in.K = K;
    in.q = Vec(g.cells(), 0.0);
    in.M = 40.0;
    in.bc = preset_bc(g, 0);
    in.split.method = method;
    in.split.eta = eta;
    in.split.eta_mode = mode;
    in.split.cn = 1;
    in.split.te = te;
    in.split.stop_on_breakthrough = stop_bt;
    in.split.max_steps_hard = 8000;
    in.s0 = Vec(g.cells(), 0.0);
    in.inflow_sat = 1.0;
    return in;
}
}  // namespace

int main(int argc, char** argv) {
    const uint64_t seed = argc > 1 ? std::stoull(argv[1]) : 303;
    const Grid g = build_grid(64, 64, 1.0, 1.0);
    const Vec K = gaussian_field(g, 2.5, 0.8, seed, true, 2.7631021115928548);
    RunResult fine = run(slab(K, FineReference, 0.01, EpsMobility, 0, 0, true));
    const long bt = fine.rec.breakthrough_step;
    const long te = bt + 1;
    auto go = [&](int method, double eta, int mode, int hb) {
        return run(slab(K, method, eta, mode, hb, te, false));
    };
    RunResult mpm_h = go(Mpm2p, 0.01, EpsRelative, 0);
    RunResult mrcm_h = go(MrcmEveryStep, 0.01, EpsRelative, 0);
    RunResult mpm_h2 = go(Mpm2p, 0.01, EpsRelative, 1);
    RunResult eta05 = go(Mpm2p, 0.05, EpsRelative, 0);
    RunResult frozen = go(Mpm2pNoUpdates, 0.01, EpsRelative, 0);
    RunResult mob = go(Mpm2p, 0.01, EpsMobility, 0);
    double worst_div = 0.0;
    for (const RunResult* r : {&mpm_h, &mrcm_h, &mpm_h2}) worst_div = std::max(worst_div, r->rec.max_div_ratio);
    auto last = [](const RunResult& r) { return r.rec.steps.back(); };
    std::printf("{\"seed\": %llu, \"bt_step\": %ld, \"bt_pvi\": %.10g, \"te\": %ld,\n", (unsigned long long)seed, bt,
                fine.rec.breakthrough_pvi, mpm_h.rec.te);
    std::printf(" \"rebuilds\": {\"mrcm\": %ld, \"relative\": %ld, \"eta05\": %ld, \"frozen\": %ld, \"mobility\": %ld, \"h2\": %ld},\n",
                mrcm_h.rec.tm_total, mpm_h.rec.tm_total, eta05.rec.tm_total, frozen.rec.tm_total, mob.rec.tm_total,
                mpm_h2.rec.tm_total);
    std::printf(" \"flux_err\": {\"mrcm\": %.10g, \"relative\": %.10g, \"eta05\": %.10g, \"frozen\": %.10g, \"mobility\": %.10g, \"h2\": %.10g},\n",
                last(mrcm_h).flux_err, last(mpm_h).flux_err, last(eta05).flux_err, last(frozen).flux_err,
                last(mob).flux_err, last(mpm_h2).flux_err);
    std::printf(" \"sat_err\": {\"relative\": %.10g, \"h2\": %.10g},\n", last(mpm_h).sat_err, last(mpm_h2).sat_err);
    std::printf(" \"max_div_ratio\": %.6g, \"nhat\": %ld, \"rcr\": %.10g,\n", worst_div, mpm_h.rec.nhat,
                rcr(mpm_h.rec.nhat, mpm_h.rec.n_sub, mpm_h.rec.te, mpm_h.rec.tm_total));
    std::printf(" \"min_eps_margin_relative\": %.6g, \"min_eps_margin_mobility\": %.6g}\n", mpm_h.rec.min_eps_margin,
                mob.rec.min_eps_margin);
    return 0;
}
