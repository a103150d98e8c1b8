// Drop-in usage from C++: the reference's own call sequence (ProblemSpec ->
// GapToothEngine -> cpi::run), with `patchdyn::` replaced by `pdb200::`.
// Builds BASELINE config 1 the way a reference user would (identity map,
// cdr_coefficients, sin(pi x) sin(pi y), homogeneous Dirichlet data), runs it
// on the B200 and writes the final macro field (raw float64) to argv[2].
//
//   dropin_c1 <fast|exact> <out.bin> [linear_cache: off|auto|on]
// The BASELINE pin is linear_cache = off (the micro-solve is the hot path);
// the reference's own default, auto, takes GapToothEngine::step's
// linear-response shortcut for this problem (gaptooth.cpp:213-224).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>

#include "gaptooth_b200.hpp"

int main(int argc, char** argv) {
    using namespace pdb200;
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <fast|exact> <out.bin>\n", argv[0]);
        return 2;
    }
    problems::ProblemSpec p;
    p.name = "diffusion-square";
    p.mapping = geometry::identity_map();
    auto one = [](double, double, double) { return 1.0; };
    auto zero3 = [](double, double, double) { return 0.0; };
    auto zero2 = [](double, double) { return 0.0; };
    p.physical = geometry::cdr_coefficients(one, one, zero3, zero3, zero3);
    p.initial = [](double xi, double eta) { return std::sin(M_PI * xi) * std::sin(M_PI * eta); };
    p.exact = [](double xi, double eta, double t) {
        return std::exp(-2.0 * M_PI * M_PI * 1.0 * t) * std::sin(M_PI * xi) * std::sin(M_PI * eta);
    };
    p.bcW = p.bcE = p.bcS = p.bcN = zero2;
    p.source_zero = true;
    p.coeffs_xi_independent = true;

    // configs/c1_diffusion.cfg pins: N = 19, h = 0.2 Delta, 7x7 nodes, dt = 0.2 d^2/D, K = 20, Dt = 5 tau
    cpi::SchemeConfig cfg;
    cfg.N_xi = cfg.N_eta = 19;
    cfg.nx = cfg.ny = 6;
    cfg.nt = 20;
    cfg.Nt = 200;
    cfg.k = 0;
    cfg.h_xi = cfg.h_eta = 0.2 * ((1.0 - 0.0) / 19);
    const double d = cfg.h_xi / cfg.nx;
    cfg.tau = cfg.nt * (0.2 * d * d / 1.0);
    cfg.T = cfg.Nt * (5.0 * cfg.tau);
    cfg.solver = cpi::SchemeConfig::Solver::Explicit;
    cfg.mode = std::strcmp(argv[1], "exact") == 0 ? PD_MODE_EXACT : PD_MODE_FAST;
    const char* lc = argc > 3 ? argv[3] : "off";
    cfg.linear_cache = std::strcmp(lc, "auto") == 0 ? cpi::SchemeConfig::LinearCache::Auto
                       : std::strcmp(lc, "on") == 0 ? cpi::SchemeConfig::LinearCache::On
                                                    : cpi::SchemeConfig::LinearCache::Off;

    try {
        const gaptooth::GapToothEngine engine(p, cfg);
        const cpi::RunResult res = cpi::run(engine);
        std::ofstream f(argv[2], std::ios::binary);
        f.write(reinterpret_cast<const char*>(res.final_field.U.data()),
                static_cast<std::streamsize>(res.final_field.U.size() * sizeof(double)));
        std::printf("kernel_family=%s linear_cache=%d steps=%zu max_pct_err=%.12f\n",
                    engine.kernel_family() == PD_MODE_FAST ? "fast" : "exact", int(engine.uses_linear_cache()),
                    res.times.size(), res.max_pct_err);
    } catch (const Error& e) {
        std::fprintf(stderr, "error %d: %s\n", e.status, e.what());
        return 3;
    }
    return 0;
}
