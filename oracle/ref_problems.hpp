// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Builds the reference's own ProblemSpec / SchemeConfig objects
// (proj/include/patchdyn/problems.hpp:17-41, scheme_config.hpp:9-37) for the
// BASELINE configs, using only the reference's public API, so that the
// unmodified reference (compiled from /root/reference by oracle/Makefile into
// oracle/_ref/) can be run on exactly the problems the B200 engine runs.
// The formulas are written textually identical to the product's host builder
// (paper_2405_08764_b200/csrc/host/problems.cpp) so both produce bit-identical
// coefficient samples; tests pin that.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <random>
#include <vector>

#include "patchdyn/cpi.hpp"
#include "patchdyn/errors.hpp"
#include "patchdyn/gaptooth.hpp"
#include "patchdyn/geometry.hpp"
#include "patchdyn/problems.hpp"
#include "patchdyn_b200.h"

namespace refshim {

using namespace patchdyn;

// Seeded macro field of configs 4/5: mt19937_64(seed), i-major
// node order, double(x >> 11) * 2^-53, then `sweeps` Jacobi sweeps on the
// interior with the boundary fixed, each sweep from a copy.
inline std::vector<double> seeded_field(int Nxi, int Neta, uint64_t seed, int sweeps) {
    const int n2 = Neta + 1;
    std::vector<double> U(static_cast<size_t>(Nxi + 1) * n2);
    std::mt19937_64 rng(seed);
    for (int i = 0; i <= Nxi; ++i)
        for (int j = 0; j <= Neta; ++j)
            U[static_cast<size_t>(i) * n2 + j] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    for (int s = 0; s < sweeps; ++s) {
        const std::vector<double> V = U;
        for (int i = 1; i < Nxi; ++i)
            for (int j = 1; j < Neta; ++j)
                U[static_cast<size_t>(i) * n2 + j] =
                    0.25 * (V[static_cast<size_t>(i - 1) * n2 + j] + V[static_cast<size_t>(i + 1) * n2 + j] +
                            V[static_cast<size_t>(i) * n2 + j - 1] + V[static_cast<size_t>(i) * n2 + j + 1]);
    }
    return U;
}

struct Built {
    problems::ProblemSpec spec;
    cpi::SchemeConfig cfg;
    std::shared_ptr<std::vector<double>> table; // node-indexed IC (configs 4/5)
};

inline cpi::SchemeConfig scheme_from(const pd_problem_desc& d) {
    cpi::SchemeConfig s;
    s.N_xi = d.N_xi;
    s.N_eta = d.N_eta;
    s.Nt = d.Nt;
    s.T = d.T;
    s.tau = d.tau;
    s.k = d.k;
    s.h_xi = d.h_xi;
    s.h_eta = d.h_eta;
    s.nx = d.nx;
    s.ny = d.ny;
    s.nt = d.nt;
    s.solver = d.solver == PD_SOLVER_ADI ? cpi::SchemeConfig::Solver::ADI : cpi::SchemeConfig::Solver::Explicit;
    s.upwind.order = d.upwind_order == PD_UPWIND_FOUR    ? microsim::UpwindOrder::Four
                     : d.upwind_order == PD_UPWIND_THREE ? microsim::UpwindOrder::Three
                                                         : microsim::UpwindOrder::Two;
    s.upwind.r = d.upwind_r;
    s.bc_type = d.bc_type == PD_BC_DIRICHLET ? cpi::SchemeConfig::BCType::Dirichlet
              : d.bc_type == PD_BC_ROBIN     ? cpi::SchemeConfig::BCType::Robin
                                             : cpi::SchemeConfig::BCType::Neumann;
    s.robin_w1 = d.robin_w1;
    s.robin_w2 = d.robin_w2;
    s.quadrature = d.quadrature == PD_QUAD_SIMPSON ? cpi::SchemeConfig::Quadrature::Simpson
                                                   : cpi::SchemeConfig::Quadrature::Trapezoid;
    s.linear_cache = cpi::SchemeConfig::LinearCache::Off; // B3: the direct path is the hot path
    return s;
}

// Problem specs.  `d` must be the RESOLVED description (pd_problem_resolved).
inline Built build(const pd_problem_desc& d) {
    Built b;
    b.cfg = scheme_from(d);
    problems::ProblemSpec& p = b.spec;
    auto zero3 = [](double, double, double) { return 0.0; };
    auto zero2 = [](double, double) { return 0.0; };
    switch (d.problem) {
        case PD_PROBLEM_DIFFUSION_SQUARE: {
            const double D = d.eps;
            p.name = "diffusion-square";
            p.mapping = geometry::identity_map();
            auto Dfn = [D](double, double, double) { return D; };
            p.physical = geometry::cdr_coefficients(Dfn, Dfn, zero3, zero3, zero3);
            p.initial = [](double xi, double eta) { return std::sin(M_PI * xi) * std::sin(M_PI * eta); };
            p.exact = [D](double xi, double eta, double t) {
                return std::exp(-2.0 * M_PI * M_PI * D * t) * std::sin(M_PI * xi) * std::sin(M_PI * eta);
            };
            p.bcW = p.bcE = p.bcS = p.bcN = zero2;
            p.coeffs_time_independent = true;
            p.source_zero = true;
            p.coeffs_xi_independent = true;
            break;
        }
        case PD_PROBLEM_CDR_TANH: {
            const double beta = d.beta, eps = d.eps, vel = d.vel, om = d.omega;
            const double tb = std::tanh(beta);
            auto X = [beta, tb](double s) { return 1.0 - std::tanh(beta * (1.0 - s)) / tb; };
            auto Xp = [beta, tb](double s) {
                const double th = std::tanh(beta * (1.0 - s));
                return beta * (1.0 - th * th) / tb;
            };
            auto Xpp = [beta, tb](double s) {
                const double th = std::tanh(beta * (1.0 - s));
                return 2.0 * beta * beta * th * (1.0 - th * th) / tb;
            };
            p.name = "cdr-tanh";
            p.mapping = geometry::user_analytic_map(
                [X](double xi, double eta) { return geometry::PhysPoint{X(xi), X(eta)}; },
                [Xp](double xi, double eta) { return geometry::InverseMetrics{Xp(xi), 0.0, 0.0, Xp(eta)}; },
                [Xpp](double xi, double eta) {
                    return geometry::SecondDerivs{Xpp(xi), 0.0, 0.0, 0.0, 0.0, Xpp(eta)};
                });
            auto Dfn = [eps](double, double, double) { return eps; };
            auto Vfn = [vel](double, double, double) { return vel; };
            p.physical = geometry::cdr_coefficients(Dfn, Dfn, Vfn, Vfn, zero3);
            p.physical.omega = [om](double, double, double) { return om; };
            auto ex = [X, eps](double xi, double eta, double t) {
                return std::exp(-t) * (1.0 - std::exp((X(xi) - 1.0) / eps)) *
                       (1.0 - std::exp((X(eta) - 1.0) / eps));
            };
            p.exact = ex;
            p.initial = [ex](double xi, double eta) { return ex(xi, eta, 0.0); };
            p.bcW = [ex](double eta, double t) { return ex(0.0, eta, t); };
            p.bcE = [ex](double eta, double t) { return ex(1.0, eta, t); };
            p.bcS = [ex](double xi, double t) { return ex(xi, 0.0, t); };
            p.bcN = [ex](double xi, double t) { return ex(xi, 1.0, t); };
            p.coeffs_time_independent = true;
            p.source_zero = true;
            p.coeffs_xi_independent = false;
            break;
        }
        case PD_PROBLEM_ANNULUS_NONAXI: {
            const double D = d.eps;
            p.name = "annulus-nonaxi";
            p.mapping = geometry::polar_map();
            p.a = 0.0;
            p.b = 2.0 * M_PI;
            p.c = 1.0;
            p.d = 2.0;
            p.periodic_xi = true;
            auto Dfn = [D](double, double, double) { return D; };
            p.physical = geometry::cdr_coefficients(Dfn, Dfn, zero3, zero3, zero3);
            p.initial = [](double th, double r) {
                return (r - 1.0) * (2.0 - r) * (1.0 + 0.5 * std::cos(2.0 * th) + 0.25 * std::sin(3.0 * th));
            };
            p.bcS = p.bcN = zero2;
            p.coeffs_time_independent = true;
            p.source_zero = true;
            p.coeffs_xi_independent = true;
            break;
        }
        case PD_PROBLEM_SHEAR_CDR: {
            const double A = d.amp, eps = d.eps, om = d.omega;
            p.name = "shear-cdr";
            p.mapping = geometry::user_analytic_map(
                [A](double xi, double eta) {
                    return geometry::PhysPoint{xi + A * std::sin(2.0 * M_PI * eta),
                                               eta + A * std::sin(2.0 * M_PI * xi)};
                },
                [A](double xi, double eta) {
                    return geometry::InverseMetrics{1.0, 2.0 * M_PI * A * std::cos(2.0 * M_PI * eta),
                                                    2.0 * M_PI * A * std::cos(2.0 * M_PI * xi), 1.0};
                },
                [A](double xi, double eta) {
                    return geometry::SecondDerivs{0.0, 0.0, -4.0 * M_PI * M_PI * A * std::sin(2.0 * M_PI * eta),
                                                  -4.0 * M_PI * M_PI * A * std::sin(2.0 * M_PI * xi), 0.0, 0.0};
                });
            auto Dfn = [eps](double, double, double) { return eps; };
            auto vx = [](double, double y, double) { return std::sin(M_PI * y); };
            auto vy = [](double x, double, double) { return std::cos(M_PI * x); };
            p.physical = geometry::cdr_coefficients(Dfn, Dfn, vx, vy, zero3);
            p.physical.omega = [om](double, double, double) { return om; };
            b.table = std::make_shared<std::vector<double>>(
                seeded_field(d.N_xi, d.N_eta, d.seed, d.jacobi_sweeps));
            auto tab = b.table;
            const int Nxi = d.N_xi, Neta = d.N_eta;
            const double dxi = 1.0 / Nxi, deta = 1.0 / Neta;
            auto at = [tab, Neta](int i, int j) { return (*tab)[static_cast<size_t>(i) * (Neta + 1) + j]; };
            auto ii = [dxi](double xi) { return static_cast<int>(std::lround(xi / dxi)); };
            auto jj = [deta](double eta) { return static_cast<int>(std::lround(eta / deta)); };
            p.initial = [at, ii, jj](double xi, double eta) { return at(ii(xi), jj(eta)); };
            p.bcW = [at, jj](double eta, double) { return at(0, jj(eta)); };
            p.bcE = [at, jj, Nxi](double eta, double) { return at(Nxi, jj(eta)); };
            p.bcS = [at, ii](double xi, double) { return at(ii(xi), 0); };
            p.bcN = [at, ii, Neta](double xi, double) { return at(ii(xi), Neta); };
            p.coeffs_time_independent = true;
            p.source_zero = true;
            p.coeffs_xi_independent = false;
            break;
        }
        case PD_PROBLEM_REF_ANNULUS:
            p = problems::problem2_annulus();
            break;
        case PD_PROBLEM_REF_CDR:
            p = problems::problem1_constant(d.lambda);
            break;
        case PD_PROBLEM_REF_CDR_VAR:
            p = problems::problem1_variable(d.lambda);
            break;
        case PD_PROBLEM_STEADY: {
            p.name = "steady";
            p.mapping = geometry::identity_map();
            auto one = [](double, double, double) { return 1.0; };
            p.physical = geometry::cdr_coefficients(one, one, zero3, zero3, zero3);
            p.initial = [](double xi, double eta) { return xi + eta; };
            p.exact = [](double xi, double eta, double) { return xi + eta; };
            p.bcW = [](double eta, double) { return eta; };
            p.bcE = [](double eta, double) { return 1.0 + eta; };
            p.bcS = [](double xi, double) { return xi; };
            p.bcN = [](double xi, double) { return 1.0 + xi; };
            p.coeffs_time_independent = true;
            p.source_zero = true;
            p.coeffs_xi_independent = true;
            break;
        }
        case PD_PROBLEM_PULSED_CDR: { // time-dependent coefficients + a general source
            const double eps = d.eps, vel = d.vel, om = d.omega; // om: pulsation frequency
            p.name = "pulsed-cdr";
            p.mapping = geometry::identity_map();
            auto Dfn = [eps, om](double, double, double t) { return eps * (1.0 + 0.5 * std::sin(om * t)); };
            auto vx = [vel, om](double, double, double t) { return vel * std::cos(om * t); };
            auto vy = [vel](double, double, double) { return 0.5 * vel; };
            auto f = [om](double x, double y, double t) { return std::sin(M_PI * x) * std::cos(M_PI * y + om * t); };
            p.physical = geometry::cdr_coefficients(Dfn, Dfn, vx, vy, f);
            p.initial = [](double xi, double eta) { return std::sin(M_PI * xi) * std::sin(M_PI * eta); };
            p.bcW = p.bcE = p.bcS = p.bcN = zero2;
            p.coeffs_time_independent = false;
            p.source_zero = false;
            p.source_separable = false;
            break;
        }
        default:
            throw ValidationError("unknown problem kind");
    }
    return b;
}

} // namespace refshim
