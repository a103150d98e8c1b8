// Problem factory, pin resolution and coefficient-table builder (host).
// See problems.hpp.  Built with -ffp-contract=off -fopenmp.
#include "problems.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <sstream>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace pdb200 {

// ---------------------------------------------------------------------------
// Problems.  The formulas for the BASELINE configs are written exactly as in
// oracle/ref_problems.hpp (which feeds the same specs to the unmodified
// reference), so both sides sample bit-identical coefficients.
// ---------------------------------------------------------------------------
namespace problems {

std::vector<double> seeded_field(int Nxi, int Neta, uint64_t seed, int sweeps) {
    const size_t n2 = static_cast<size_t>(Neta) + 1;
    std::vector<double> U((static_cast<size_t>(Nxi) + 1) * n2);
    std::mt19937_64 gen(seed);
    for (int i = 0; i <= Nxi; ++i)
        for (int j = 0; j <= Neta; ++j) U[i * n2 + j] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    std::vector<double> V;
    for (int s = 0; s < sweeps; ++s) {
        V = U; // each sweep reads a copy; boundary nodes stay fixed
        for (int i = 1; i < Nxi; ++i)
            for (int j = 1; j < Neta; ++j)
                U[i * n2 + j] = 0.25 * (V[(i - 1) * n2 + j] + V[(i + 1) * n2 + j] + V[i * n2 + j - 1] +
                                        V[i * n2 + j + 1]);
    }
    return U;
}

namespace {
using geometry::InverseMetrics;
using geometry::PhysPoint;
using geometry::SecondDerivs;
auto zero3 = [](double, double, double) { return 0.0; };
auto zero2 = [](double, double) { return 0.0; };

ProblemSpec ref_cdr(double lambda, bool variable) {
    // problems::problem1_constant / problem1_variable  proj/src/problems.cpp:19-75
    // (lambda-stretched CDR, exact e^{x+y+t}, separable source
    // (c0 x + 10y - 1) e^{x+y} * e^t; variable: D = 1 + x, c0 = 8)
    if (!(lambda >= 0.0 && lambda < 1.0)) {
        std::ostringstream os;
        os << "stretching parameter must lie in [0,1), got " << lambda;
        throw InvalidStretch(os.str());
    }
    ProblemSpec p;
    p.name = variable ? "cdr-var" : "cdr-const";
    p.mapping = lambda == 0.0 ? geometry::identity_map() : geometry::stretched_map(lambda);
    auto Dx = [variable](double x, double, double) { return variable ? 1.0 + x : 1.0; };
    auto vx = [](double x, double, double) { return 10.0 * x; };
    auto vy = [](double, double y, double) { return 10.0 * y; };
    const double c0 = variable ? 8.0 : 10.0;
    auto src = [c0](double x, double y, double t) { return (c0 * x + 10.0 * y - 1.0) * std::exp(x + y + t); };
    p.physical = geometry::cdr_coefficients(Dx, Dx, vx, vy, src);
    const geometry::Mapping m = p.mapping;
    p.initial = [m](double xi, double eta) {
        const PhysPoint q = m.forward(xi, eta);
        return std::exp(q.x + q.y);
    };
    p.exact = [m](double xi, double eta, double t) {
        const PhysPoint q = m.forward(xi, eta);
        return std::exp(q.x + q.y + t);
    };
    p.bcW = [m](double eta, double t) { return std::exp(m.forward(0, eta).y + t); };
    p.bcE = [m](double eta, double t) { return std::exp(1.0 + m.forward(1, eta).y + t); };
    p.bcS = [m](double xi, double t) { return std::exp(m.forward(xi, 0).x + t); };
    p.bcN = [m](double xi, double t) { return std::exp(m.forward(xi, 1).x + 1.0 + t); };
    p.coeffs_time_independent = true;
    p.source_zero = false;
    p.source_separable = true;
    p.source_spatial = [m, c0](double xi, double eta) {
        const PhysPoint q = m.forward(xi, eta);
        return (c0 * q.x + 10.0 * q.y - 1.0) * std::exp(q.x + q.y);
    };
    p.source_time = [](double t) { return std::exp(t); };
    p.coeffs_xi_independent = false;
    return p;
}
} // namespace

ProblemSpec from_desc(const pd_problem_desc& d) {
    ProblemSpec p;
    switch (d.problem) {
        case PD_PROBLEM_DIFFUSION_SQUARE: { // config 1
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
            p.source_zero = true;
            p.coeffs_xi_independent = true;
            return p;
        }
        case PD_PROBLEM_CDR_TANH: { // config 2
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
                [X](double xi, double eta) { return PhysPoint{X(xi), X(eta)}; },
                [Xp](double xi, double eta) { return InverseMetrics{Xp(xi), 0.0, 0.0, Xp(eta)}; },
                [Xpp](double xi, double eta) { return SecondDerivs{Xpp(xi), 0.0, 0.0, 0.0, 0.0, Xpp(eta)}; });
            auto Dfn = [eps](double, double, double) { return eps; };
            auto Vfn = [vel](double, double, double) { return vel; };
            p.physical = geometry::cdr_coefficients(Dfn, Dfn, Vfn, Vfn, zero3);
            p.physical.omega = [om](double, double, double) { return om; };
            auto ex = [X, eps](double xi, double eta, double t) {
                return std::exp(-t) * (1.0 - std::exp((X(xi) - 1.0) / eps)) * (1.0 - std::exp((X(eta) - 1.0) / eps));
            };
            p.exact = ex;
            p.initial = [ex](double xi, double eta) { return ex(xi, eta, 0.0); };
            p.bcW = [ex](double eta, double t) { return ex(0.0, eta, t); };
            p.bcE = [ex](double eta, double t) { return ex(1.0, eta, t); };
            p.bcS = [ex](double xi, double t) { return ex(xi, 0.0, t); };
            p.bcN = [ex](double xi, double t) { return ex(xi, 1.0, t); };
            p.source_zero = true;
            return p;
        }
        case PD_PROBLEM_ANNULUS_NONAXI: { // config 3 (reference orientation)
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
            p.source_zero = true;
            p.coeffs_xi_independent = true;
            return p;
        }
        case PD_PROBLEM_SHEAR_CDR: { // configs 4/5: x = xi + A sin 2pi eta, y = eta + A sin 2pi xi
            const double A = d.amp, eps = d.eps, om = d.omega;
            p.name = "shear-cdr";
            p.mapping = geometry::user_analytic_map(
                [A](double xi, double eta) {
                    return PhysPoint{xi + A * std::sin(2.0 * M_PI * eta), eta + A * std::sin(2.0 * M_PI * xi)};
                },
                [A](double xi, double eta) {
                    return InverseMetrics{1.0, 2.0 * M_PI * A * std::cos(2.0 * M_PI * eta),
                                          2.0 * M_PI * A * std::cos(2.0 * M_PI * xi), 1.0};
                },
                [A](double xi, double eta) {
                    return SecondDerivs{0.0, 0.0, -4.0 * M_PI * M_PI * A * std::sin(2.0 * M_PI * eta),
                                        -4.0 * M_PI * M_PI * A * std::sin(2.0 * M_PI * xi), 0.0, 0.0};
                });
            auto Dfn = [eps](double, double, double) { return eps; };
            auto vx = [](double, double y, double) { return std::sin(M_PI * y); };
            auto vy = [](double x, double, double) { return std::cos(M_PI * x); };
            p.physical = geometry::cdr_coefficients(Dfn, Dfn, vx, vy, zero3);
            p.physical.omega = [om](double, double, double) { return om; };
            // initial / boundary data live on the macro nodes; looked up by index
            auto tab = std::make_shared<std::vector<double>>(seeded_field(d.N_xi, d.N_eta, d.seed, d.jacobi_sweeps));
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
            p.source_zero = true;
            return p;
        }
        case PD_PROBLEM_REF_ANNULUS: { // problems::problem2_annulus  proj/src/problems.cpp:110-138
            p.name = "annulus";
            p.mapping = geometry::polar_map();
            p.a = 0.0;
            p.b = 2.0 * M_PI;
            p.c = 1.0;
            p.d = 2.0;
            p.periodic_xi = true;
            auto one = [](double, double, double) { return 1.0; };
            p.physical = geometry::cdr_coefficients(one, one, zero3, zero3, zero3);
            p.initial = [](double th, double r) { return (r - 1.0) * (2.0 - r) * std::sin(th); };
            p.bcS = p.bcN = zero2;
            p.source_zero = true;
            p.coeffs_xi_independent = true;
            return p;
        }
        case PD_PROBLEM_REF_CDR:
            return ref_cdr(d.lambda, false);
        case PD_PROBLEM_REF_CDR_VAR:
            return ref_cdr(d.lambda, true);
        case PD_PROBLEM_STEADY: { // harmonic u = x + y  (proj/tests/test_gaptooth.cpp:32-49)
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
            p.source_zero = true;
            p.coeffs_xi_independent = true;
            return p;
        }
        case PD_PROBLEM_PULSED_CDR: { // time-dependent coefficients + general source (as oracle/ref_problems.hpp)
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
            return p;
        }
        default:
            throw ValidationError("unknown problem kind " + std::to_string(d.problem));
    }
}
} // namespace problems

// ---------------------------------------------------------------------------
// Scheme
// ---------------------------------------------------------------------------
namespace cpi {

void SchemeConfig::validate(double xi_extent, double eta_extent) const {
    auto fail = [](const std::string& m) { throw ValidationError(m); };
    if (N_xi < 2 || N_eta < 2) fail("coarse grid needs at least 2 intervals per direction");
    if (Nt < 1) fail("Nt must be at least 1");
    if (!(T > 0)) fail("final time T must be positive");
    if (!(tau > 0)) fail("gap-tooth horizon tau must be positive");
    if (k < 0) fail("k must be non-negative");
    if (!((k + 1) * tau < dt())) {
        std::ostringstream msg;
        msg << "(k+1)*tau = " << (k + 1) * tau << " must stay below the macro step dt = " << dt();
        fail(msg.str());
    }
    if (!(h_xi > 0 && h_eta > 0)) fail("patch extents must be positive");
    if (h_xi > xi_extent / N_xi * (1.0 + 1e-12)) fail("h_xi exceeds the coarse spacing (patches must not overlap)");
    if (h_eta > eta_extent / N_eta * (1.0 + 1e-12)) fail("h_eta exceeds the coarse spacing (patches must not overlap)");
    if (nx < 2 || ny < 2) fail("micro resolution needs nx, ny >= 2");
    if (nt < 1) fail("micro time steps nt must be >= 1");
    if (quadrature == Quadrature::Simpson && (nx % 2 != 0 || ny % 2 != 0))
        fail("Simpson restriction needs even nx and ny");
    if (bc_type == BCType::Robin && robin_w1 == 0.0 && robin_w2 == 0.0)
        fail("robin patch conditions need nonzero weights");
}

SchemeConfig scheme_from_desc(const pd_problem_desc& d) {
    SchemeConfig s;
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
    s.solver = d.solver == PD_SOLVER_ADI ? SchemeConfig::Solver::ADI : SchemeConfig::Solver::Explicit;
    s.upwind.order = d.upwind_order == PD_UPWIND_FOUR    ? microsim::UpwindOrder::Four
                     : d.upwind_order == PD_UPWIND_THREE ? microsim::UpwindOrder::Three
                                                         : microsim::UpwindOrder::Two;
    s.upwind.r = d.upwind_r;
    s.bc_type = d.bc_type == PD_BC_DIRICHLET ? SchemeConfig::BCType::Dirichlet
              : d.bc_type == PD_BC_ROBIN     ? SchemeConfig::BCType::Robin
                                             : SchemeConfig::BCType::Neumann;
    s.robin_w1 = d.robin_w1;
    s.robin_w2 = d.robin_w2;
    s.quadrature = d.quadrature == PD_QUAD_SIMPSON ? SchemeConfig::Quadrature::Simpson
                                                   : SchemeConfig::Quadrature::Trapezoid;
    s.mode = d.mode;
    s.linear_cache = SchemeConfig::LinearCache::Off; // BASELINE pin: the micro-solve is the hot path
    return s;
}
} // namespace cpi

// ---------------------------------------------------------------------------
// Tables
// ---------------------------------------------------------------------------
void EngineTables::relink() {
    desc.npatches = static_cast<int32_t>(patch_ij.size() / 2);
    desc.patch_ij = patch_ij.data();
    desc.coeff_set = coeff_set.empty() ? nullptr : coeff_set.data();
    desc.coeffs = coeffs.empty() ? nullptr : coeffs.data();
    desc.source_spatial = source_spatial.empty() ? nullptr : source_spatial.data();
}

EngineTables build_tables(const problems::ProblemSpec& p, const cpi::SchemeConfig& cfg, int threads, bool sample) {
    // time-dependent coefficients: the table is the t = 0 sample (the reference's
    // co0_, microsim.cpp:217); the sampled step entries supply later ones.  General
    // sources: PD_SOURCE_GENERAL, supplied per micro step the same way.
    EngineTables t;
    pd_engine_desc& d = t.desc;
    d.a = p.a;
    d.b = p.b;
    d.c = p.c;
    d.d = p.d;
    d.Nxi = cfg.N_xi;
    d.Neta = cfg.N_eta;
    d.periodic_xi = p.periodic_xi;
    d.nx = cfg.nx;
    d.ny = cfg.ny;
    d.nt = cfg.nt;
    d.k = cfg.k;
    d.tau = cfg.tau;
    d.dt_macro = cfg.dt();
    d.h_xi = cfg.h_xi;
    d.h_eta = cfg.h_eta;
    d.bc_type = cfg.bc_type == cpi::SchemeConfig::BCType::Dirichlet ? PD_BC_DIRICHLET
              : cfg.bc_type == cpi::SchemeConfig::BCType::Robin     ? PD_BC_ROBIN
                                                                    : PD_BC_NEUMANN;
    d.robin_w1 = cfg.robin_w1;
    d.robin_w2 = cfg.robin_w2;
    d.quadrature = cfg.quadrature == cpi::SchemeConfig::Quadrature::Simpson ? PD_QUAD_SIMPSON : PD_QUAD_TRAPEZOID;
    d.source_kind = p.source_zero ? PD_SOURCE_ZERO : p.source_separable ? PD_SOURCE_SEPARABLE : PD_SOURCE_GENERAL;
    d.l = p.physical.l;
    d.mode = cfg.mode;
    d.solver = cfg.solver == cpi::SchemeConfig::Solver::ADI ? PD_SOLVER_ADI : PD_SOLVER_EXPLICIT;
    d.upwind_order = cfg.upwind.order == microsim::UpwindOrder::Four    ? PD_UPWIND_FOUR
                     : cfg.upwind.order == microsim::UpwindOrder::Three ? PD_UPWIND_THREE
                                                                        : PD_UPWIND_TWO;
    d.upwind_r = cfg.upwind.r;
    if (d.l == 0.0) throw ValidationError("time-derivative multiplier l must be nonzero");

    // patch list: j outer, i inner (gaptooth.cpp:251-280)
    const int i_lo = p.periodic_xi ? 0 : 1, i_hi = cfg.N_xi - 1;
    for (int j = 1; j <= cfg.N_eta - 1; ++j)
        for (int i = i_lo; i <= i_hi; ++i) {
            t.patch_ij.push_back(i);
            t.patch_ij.push_back(j);
        }
    const int P = static_cast<int>(t.patch_ij.size() / 2);
    // one integrator per eta-row when the reference shares them (gaptooth.cpp:254-266)
    const bool share_rows = p.coeffs_time_independent && p.coeffs_xi_independent && p.source_zero;
    std::vector<int> set_i, set_j;
    if (share_rows) {
        for (int j = 1; j <= cfg.N_eta - 1; ++j) {
            set_i.push_back(i_lo);
            set_j.push_back(j);
        }
        t.coeff_set.resize(P);
        for (int q = 0; q < P; ++q) t.coeff_set[q] = t.patch_ij[2 * q + 1] - 1;
    } else {
        for (int q = 0; q < P; ++q) {
            set_i.push_back(t.patch_ij[2 * q]);
            set_j.push_back(t.patch_ij[2 * q + 1]);
        }
    }
    const int S = static_cast<int>(set_i.size());
    d.ncoeff_sets = S;
    const int n1 = cfg.nx + 1, n2 = cfg.ny + 1;
    const size_t N = static_cast<size_t>(n1) * n2;
    if (!sample) {
        t.relink();
        return t;
    }
    t.coeffs.assign(static_cast<size_t>(S) * PD_NCOEF * N, 0.0);
    if (p.source_separable) t.source_spatial.assign(static_cast<size_t>(S) * N, 0.0);

    // CoarseGrid::xi/eta (gaptooth.hpp:21-24) and make_micro_grid (microsim.cpp:18-24)
    const double Dxi = (p.b - p.a) / cfg.N_xi, Deta = (p.d - p.c) / cfg.N_eta;
    const double mdxi = cfg.h_xi / cfg.nx, mdeta = cfg.h_eta / cfg.ny;
    const double l = p.physical.l;
    double m_ac = 0.0, m_apc = 0.0, m_b = 0.0;
    int err_status = 0;
    std::string err_msg;
#ifdef _OPENMP
    const int nth = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for num_threads(nth) schedule(dynamic, 4) reduction(max : m_ac, m_apc, m_b)
#endif
    for (int s = 0; s < S; ++s) {
        try {
            const double xc = p.a + Dxi * set_i[s], ec = p.c + Deta * set_j[s];
            // PatchIntegrator node coordinates  microsim.cpp:208-209, microsim.hpp:97-98
            const double xi0 = xc - 0.5 * mdxi * cfg.nx, eta0 = ec - 0.5 * mdeta * cfg.ny;
            double* o = t.coeffs.data() + static_cast<size_t>(s) * PD_NCOEF * N;
            for (int i = 0; i < n1; ++i)
                for (int j = 0; j < n2; ++j) {
                    const double xi = xi0 + i * mdxi, eta = eta0 + j * mdeta;
                    const geometry::TransformedCoefficients tc =
                        geometry::transform_coefficients(p.mapping, p.physical, xi, eta, 0.0);
                    const size_t k = static_cast<size_t>(i) * n2 + j;
                    // solver form  microsim.cpp:245-249 (+ B = -b/l).  The reference
                    // ignores |b| <= 1e-12 (microsim.cpp:239); so does the table.
                    const double A = -tc.a / l, B = std::abs(tc.b) > 1e-12 ? -tc.b / l : 0.0, Cc = -tc.c / l;
                    o[PD_COEF_A * N + k] = A;
                    o[PD_COEF_B * N + k] = B;
                    o[PD_COEF_C * N + k] = Cc;
                    o[PD_COEF_VX * N + k] = tc.d / l;
                    o[PD_COEF_VY * N + k] = tc.e / l;
                    o[PD_COEF_W * N + k] = tc.f / l;
                    m_ac = std::max({m_ac, std::abs(A), std::abs(Cc)});
                    m_apc = std::max(m_apc, std::abs(A) + std::abs(Cc));
                    m_b = std::max(m_b, std::abs(B));
                    if (p.source_separable)
                        t.source_spatial[static_cast<size_t>(s) * N + k] = p.source_spatial(xi, eta);
                }
        } catch (const Error& e) {
#ifdef _OPENMP
#pragma omp critical
#endif
            {
                if (!err_status) {
                    err_status = e.status;
                    err_msg = e.what();
                }
            }
        }
    }
    if (err_status) {
        if (err_status == PD_NON_POSITIVE_JACOBIAN) throw NonPositiveJacobian(err_msg);
        throw Error(err_status, err_msg);
    }
    t.max_abs_ac = m_ac;
    t.max_a_plus_c = m_apc;
    t.max_abs_b = m_b;
    if (m_b > 0.0 && d.bc_type == PD_BC_ROBIN)
        throw MixedTermUnsupported("mixed-derivative term with Robin patch conditions is not defined");
    t.relink();
    return t;
}

// Time-dependent coefficients / general sources: the per-micro-step samples the
// reference's PatchIntegrator takes inside integrate (sample_coeffs(t_co) and
// sample_source(t_co), microsim.cpp:537-542, 265-281), for every coefficient
// set, at the set's node coordinates (same arithmetic as build_tables).
void sample_substep(const problems::ProblemSpec& p, const cpi::SchemeConfig& cfg, const EngineTables& t, double t0,
                    double* coeff_steps, double* source_steps, int threads) {
    const int S = t.desc.ncoeff_sets, n1 = cfg.nx + 1, n2 = cfg.ny + 1;
    const size_t N = static_cast<size_t>(n1) * n2;
    const double Dxi = (p.b - p.a) / cfg.N_xi, Deta = (p.d - p.c) / cfg.N_eta;
    const double mdxi = cfg.h_xi / cfg.nx, mdeta = cfg.h_eta / cfg.ny;
    const double l = p.physical.l, dt = cfg.tau / cfg.nt;
    const double dmin = std::min(mdxi, mdeta);
    // the set -> representative patch map of build_tables: row sharing never
    // applies here (it needs time-independent coefficients and no source)
    int err_status = 0;
    std::string err_msg;
#ifdef _OPENMP
    const int nth = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for num_threads(nth) schedule(dynamic, 4)
#endif
    for (int s = 0; s < S; ++s) {
        try {
            const int pi = t.patch_ij[2 * s], pj = t.patch_ij[2 * s + 1];
            const double xc = p.a + Dxi * pi, ec = p.c + Deta * pj;
            const double xi0 = xc - 0.5 * mdxi * cfg.nx, eta0 = ec - 0.5 * mdeta * cfg.ny;
            for (int step = 0; step < cfg.nt; ++step) {
                const double tc = t0 + step * dt; // explicit scheme (microsim.cpp:535-537)
                double mx = 0.0;
                for (int i = 0; i < n1; ++i)
                    for (int j = 0; j < n2; ++j) {
                        const double xi = xi0 + i * mdxi, eta = eta0 + j * mdeta;
                        const size_t k = static_cast<size_t>(i) * n2 + j;
                        if (coeff_steps) {
                            const geometry::TransformedCoefficients tc2 =
                                geometry::transform_coefficients(p.mapping, p.physical, xi, eta, tc);
                            double* o = coeff_steps + (static_cast<size_t>(step) * S + s) * PD_NCOEF * N;
                            const double A = -tc2.a / l, Cc = -tc2.c / l;
                            o[PD_COEF_A * N + k] = A;
                            o[PD_COEF_B * N + k] = std::abs(tc2.b) > 1e-12 ? -tc2.b / l : 0.0;
                            o[PD_COEF_C * N + k] = Cc;
                            o[PD_COEF_VX * N + k] = tc2.d / l;
                            o[PD_COEF_VY * N + k] = tc2.e / l;
                            o[PD_COEF_W * N + k] = tc2.f / l;
                            mx = std::max({mx, std::abs(A), std::abs(Cc)});
                        }
                        if (source_steps) {
                            const geometry::PhysPoint q = p.mapping.forward(xi, eta);
                            source_steps[(static_cast<size_t>(step) * S + s) * N + k] = p.physical.phi(q.x, q.y, tc) / l;
                        }
                    }
                // the explicit guard of every sample  microsim.cpp:253-262
                if (coeff_steps && cfg.solver == cpi::SchemeConfig::Solver::Explicit &&
                    mx * dt / (dmin * dmin) > 0.5 + 1e-12) {
                    std::ostringstream msg;
                    msg << "explicit micro scheme diffusive stability number " << mx * dt / (dmin * dmin)
                        << " exceeds 0.5 at t = " << tc;
                    throw StabilityViolation(msg.str());
                }
            }
        } catch (const Error& e) {
#ifdef _OPENMP
#pragma omp critical
#endif
            {
                if (!err_status) {
                    err_status = e.status;
                    err_msg = e.what();
                }
            }
        }
    }
    if (err_status) throw Error(err_status, err_msg);
}

void check_stability(const EngineTables& t, const cpi::SchemeConfig& cfg) {
    if (cfg.solver != cpi::SchemeConfig::Solver::Explicit) return; // guard of the explicit scheme only
    const double mdxi = cfg.h_xi / cfg.nx, mdeta = cfg.h_eta / cfg.ny;
    const double dt = cfg.tau / cfg.nt;
    const double dmin = std::min(mdxi, mdeta);
    const double number = t.max_abs_ac * dt / (dmin * dmin);
    if (number > 0.5 + 1e-12) {
        std::ostringstream msg;
        msg << "explicit micro scheme diffusive stability number " << number << " exceeds 0.5";
        throw StabilityViolation(msg.str());
    }
}

} // namespace pdb200
