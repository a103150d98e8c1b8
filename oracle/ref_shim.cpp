// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference (proj/src/*.cpp compiled from
// /root/reference by oracle/Makefile into oracle/_ref/libpatchdyn_ref.so).
// Every numerical result returned here is computed by reference code:
//   GapToothEngine::step_direct / initial_field / refresh_boundary
//       proj/src/gaptooth.cpp:284-375
//   cpi::projective_step / cpi::run               proj/src/cpi.cpp:58-216
//   PatchIntegrator::integrate (step_explicit)    proj/src/microsim.cpp:509-564
//   build_stencil / neumann_edge_slopes / dirichlet_edge_values / lift /
//   restrict_average                              proj/src/gaptooth.cpp:74-194
//   transform_coefficients                        proj/src/geometry.cpp:93-125
// The shim only marshals arrays and maps exceptions to pd_status codes.
#include <chrono>
#include <cstring>
#include <string>

#include "ref_problems.hpp"

using namespace patchdyn;

namespace {

thread_local std::string g_err;

int map_exception(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const NonPositiveJacobian*>(&e)) return PD_NON_POSITIVE_JACOBIAN;
    if (dynamic_cast<const MixedTermUnsupported*>(&e)) return PD_MIXED_TERM_UNSUPPORTED;
    if (dynamic_cast<const StabilityViolation*>(&e)) return PD_STABILITY_VIOLATION;
    if (dynamic_cast<const IndexOutOfRange*>(&e)) return PD_INDEX_OUT_OF_RANGE;
    if (dynamic_cast<const ShapeMismatch*>(&e)) return PD_SHAPE_MISMATCH;
    if (dynamic_cast<const MacroInstability*>(&e)) return PD_MACRO_INSTABILITY;
    if (dynamic_cast<const MacroPatchError*>(&e)) return PD_MACRO_PATCH_ERROR;
    if (dynamic_cast<const ValidationError*>(&e)) return PD_VALIDATION_ERROR;
    return PD_VALIDATION_ERROR + 1000;
}

struct RefEngine {
    refshim::Built built;
    std::unique_ptr<gaptooth::GapToothEngine> eng;
};

gaptooth::CoarseField field_from(const RefEngine& r, const double* U) {
    gaptooth::CoarseField F = r.eng->initial_field();
    std::memcpy(F.U.data(), U, F.U.size() * sizeof(double));
    return F;
}

microsim::EdgeCondition edge_from(int kind, const double* val, const double* slope, int len,
                                  double w1, double w2) {
    std::vector<double> v(val, val + len), s(slope, slope + len);
    if (kind == PD_EDGE_DIRICHLET) return microsim::dirichlet_edge(v);
    if (kind == PD_EDGE_ROBIN) return microsim::robin_edge(w1, w2, v, s);
    return microsim::neumann_edge(s);
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_engine_create(const pd_problem_desc* d, void** out) {
    try {
        auto r = std::make_unique<RefEngine>();
        r->built = refshim::build(*d);
        r->eng = std::make_unique<gaptooth::GapToothEngine>(r->built.spec, r->built.cfg);
        *out = r.release();
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// linear_cache: 0 Auto, 1 On, 2 Off (SchemeConfig::LinearCache, scheme_config.hpp:30-31)
int ref_engine_create_lc(const pd_problem_desc* d, int linear_cache, void** out) {
    try {
        auto r = std::make_unique<RefEngine>();
        r->built = refshim::build(*d);
        r->built.cfg.linear_cache = linear_cache == 0   ? cpi::SchemeConfig::LinearCache::Auto
                                    : linear_cache == 1 ? cpi::SchemeConfig::LinearCache::On
                                                        : cpi::SchemeConfig::LinearCache::Off;
        r->eng = std::make_unique<gaptooth::GapToothEngine>(r->built.spec, r->built.cfg);
        *out = r.release();
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_initial_field(void* h, double* U) {
    auto* r = static_cast<RefEngine*>(h);
    gaptooth::CoarseField F = r->eng->initial_field();
    r->eng->refresh_boundary(F, 0.0);
    std::memcpy(U, F.U.data(), F.U.size() * sizeof(double));
    return 0;
}

int ref_refresh_boundary(void* h, double* U, double t) {
    auto* r = static_cast<RefEngine*>(h);
    gaptooth::CoarseField F = field_from(*r, U);
    r->eng->refresh_boundary(F, t);
    std::memcpy(U, F.U.data(), F.U.size() * sizeof(double));
    return 0;
}

int ref_step_direct(void* h, const double* Uin, double* Uout, double t) {
    auto* r = static_cast<RefEngine*>(h);
    try {
        const gaptooth::CoarseField F = field_from(*r, Uin);
        const gaptooth::CoarseField G = r->eng->step_direct(F, t);
        std::memcpy(Uout, G.U.data(), G.U.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// GapToothEngine::step (linear-response path when the engine enabled it)
int ref_step(void* h, const double* Uin, double* Uout, double t) {
    auto* r = static_cast<RefEngine*>(h);
    try {
        const gaptooth::CoarseField F = field_from(*r, Uin);
        const gaptooth::CoarseField G = r->eng->step(F, t);
        std::memcpy(Uout, G.U.data(), G.U.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

int ref_projective_step(void* h, const double* Uin, double* Uout, double t) {
    auto* r = static_cast<RefEngine*>(h);
    try {
        const gaptooth::CoarseField F = field_from(*r, Uin);
        const gaptooth::CoarseField G = cpi::projective_step(*r->eng, F, t);
        std::memcpy(Uout, G.U.data(), G.U.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// Full cpi::run (cpi.cpp:134-216): final field, max % error, wall seconds.
int ref_run(void* h, double* Ufinal, double* max_pct_err, double* seconds) {
    auto* r = static_cast<RefEngine*>(h);
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const cpi::RunResult res = cpi::run(*r->eng);
        const auto t1 = std::chrono::steady_clock::now();
        std::memcpy(Ufinal, res.final_field.U.data(), res.final_field.U.size() * sizeof(double));
        if (max_pct_err) *max_pct_err = res.max_pct_err;
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// nsteps projective steps from U at t0 = n0*dt (cpi.cpp:175-178 loop body
// without the diagnostics); wall seconds of the loop.
int ref_steps(void* h, double* U, int n0, int nsteps, double* seconds) {
    auto* r = static_cast<RefEngine*>(h);
    try {
        gaptooth::CoarseField F = field_from(*r, U);
        const double dt = r->eng->config().dt();
        const auto t0 = std::chrono::steady_clock::now();
        for (int n = n0; n < n0 + nsteps; ++n) F = cpi::projective_step(*r->eng, F, n * dt);
        const auto t1 = std::chrono::steady_clock::now();
        std::memcpy(U, F.U.data(), F.U.size() * sizeof(double));
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// Per-node solver-form coefficients exactly as PatchIntegrator samples them
// (microsim.cpp:204-252): node coordinates from a reference PatchIntegrator
// (node_xi/node_eta, microsim.hpp:97-98) and geometry::transform_coefficients.
// out: [npatch][6][n1][n2] for the listed patch centres (A,B,C,Vx,Vy,W with
// B = -b/l, which the reference itself would reject).
int ref_sample_coeffs(void* h, int npatch, const int* patch_ij, double* out) {
    auto* r = static_cast<RefEngine*>(h);
    const auto& g = r->eng->grid();
    const auto& mg = r->eng->micro_grid();
    const auto map = r->built.spec.mapping;
    const auto phys = r->built.spec.physical;
    const double l = phys.l;
    const int n1 = mg.nx + 1, n2 = mg.ny + 1;
    microsim::CoeffSampler zero = [](double, double, double) {
        geometry::TransformedCoefficients tc{};
        tc.a = -1.0;
        tc.c = -1.0;
        return tc;
    };
    try {
        for (int p = 0; p < npatch; ++p) {
            const double xc = g.xi(patch_ij[2 * p]), ec = g.eta(patch_ij[2 * p + 1]);
            const microsim::PatchIntegrator pi(xc, ec, mg, l, zero, true, microsim::SourceSpec{},
                                               microsim::PatchIntegrator::Scheme::ADI);
            double* o = out + static_cast<size_t>(p) * 6 * n1 * n2;
            for (int i = 0; i < n1; ++i)
                for (int j = 0; j < n2; ++j) {
                    const auto tc = geometry::transform_coefficients(map, phys, pi.node_xi(i), pi.node_eta(j), 0.0);
                    const size_t k = static_cast<size_t>(i) * n2 + j, N = static_cast<size_t>(n1) * n2;
                    o[0 * N + k] = -tc.a / l;
                    o[1 * N + k] = std::abs(tc.b) > 1e-12 ? -tc.b / l : 0.0; // dropped below the reference's 1e-12 tolerance (microsim.cpp:239)
                    o[2 * N + k] = -tc.c / l;
                    o[3 * N + k] = tc.d / l;
                    o[4 * N + k] = tc.e / l;
                    o[5 * N + k] = tc.f / l;
                }
        }
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// Same sampling without a GapToothEngine (whose constructor rejects b != 0):
// the problem spec from refshim::build, CoarseGrid::xi/eta and PatchIntegrator
// node coordinates, geometry::transform_coefficients.  Used for config 4/5.
int ref_sample_coeffs_desc(const pd_problem_desc* d, int npatch, const int* patch_ij, double* out) {
    try {
        const refshim::Built b = refshim::build(*d);
        gaptooth::CoarseGrid g{b.spec.a, b.spec.b, b.spec.c, b.spec.d, d->N_xi, d->N_eta};
        const microsim::MicroGrid mg = microsim::make_micro_grid(d->h_xi, d->h_eta, d->tau, d->nx, d->ny, d->nt);
        const double l = b.spec.physical.l;
        const int n1 = mg.nx + 1, n2 = mg.ny + 1;
        microsim::CoeffSampler zero = [](double, double, double) {
            geometry::TransformedCoefficients tc{};
            tc.a = -1.0;
            tc.c = -1.0;
            return tc;
        };
        for (int p = 0; p < npatch; ++p) {
            const microsim::PatchIntegrator pi(g.xi(patch_ij[2 * p]), g.eta(patch_ij[2 * p + 1]), mg, l, zero, true,
                                               microsim::SourceSpec{}, microsim::PatchIntegrator::Scheme::ADI);
            double* o = out + static_cast<size_t>(p) * 6 * n1 * n2;
            const size_t N = static_cast<size_t>(n1) * n2;
            for (int i = 0; i < n1; ++i)
                for (int j = 0; j < n2; ++j) {
                    const auto tc = geometry::transform_coefficients(b.spec.mapping, b.spec.physical, pi.node_xi(i),
                                                                     pi.node_eta(j), 0.0);
                    const size_t k = static_cast<size_t>(i) * n2 + j;
                    o[0 * N + k] = -tc.a / l;
                    o[1 * N + k] = std::abs(tc.b) > 1e-12 ? -tc.b / l : 0.0;
                    o[2 * N + k] = -tc.c / l;
                    o[3 * N + k] = tc.d / l;
                    o[4 * N + k] = tc.e / l;
                    o[5 * N + k] = tc.f / l;
                }
        }
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// The problem's computational domain, xi-periodicity and row sharing (ProblemSpec
// a, b, c, d, periodic_xi, structure hints; problems.hpp:17-41): what the pin
// resolution (h = h_frac * Delta, the metric dt rule) needs.  flags[2].
int ref_problem_domain(const pd_problem_desc* d, double* abcd, int* periodic) {
    try {
        const refshim::Built b = refshim::build(*d);
        abcd[0] = b.spec.a;
        abcd[1] = b.spec.b;
        abcd[2] = b.spec.c;
        abcd[3] = b.spec.d;
        // periodic_xi, and whether the engine shares one integrator per eta-row
        // (gaptooth.cpp:254-266: time- and xi-independent coefficients, no source)
        periodic[0] = b.spec.periodic_xi ? 1 : 0;
        periodic[1] = b.spec.coeffs_time_independent && b.spec.coeffs_xi_independent && b.spec.source_zero;
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// Neighbour indices through the reference's build_stencil (gaptooth.cpp:74-104):
// the field holds each node's flat index, so the gathered values ARE the indices.
int ref_neighbours(void* h, int npatch, const int* patch_ij, int* out) {
    auto* r = static_cast<RefEngine*>(h);
    try {
        gaptooth::CoarseField F = r->eng->initial_field();
        for (size_t k = 0; k < F.U.size(); ++k) F.U.raw()[k] = static_cast<double>(k);
        for (int p = 0; p < npatch; ++p) {
            const gaptooth::StencilPoly s = gaptooth::build_stencil(F, patch_ij[2 * p], patch_ij[2 * p + 1]);
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) out[9 * p + 3 * a + b] = static_cast<int>(s.vals[a][b]);
        }
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// PatchIntegrator::integrate (explicit) with constant solver-form coefficients
// coef[5] = {A, C, Vx, Vy, W} (the test fixture const_coeffs of
// proj/tests/test_microsim.cpp:18-30) or, when coef_table != NULL, a
// per-node table [5][n1][n2] looked up by node index.
int ref_integrate(const double* coef, const double* coef_table, int nx, int ny, int nt, double h_xi,
                  double h_eta, double tau, double xi_c, double eta_c, const int* kinds,
                  const double* values, const double* slopes, const double* robin_w, double t0,
                  const double* u0, double* uT) {
    try {
        const microsim::MicroGrid g = microsim::make_micro_grid(h_xi, h_eta, tau, nx, ny, nt);
        const int n1 = nx + 1, n2 = ny + 1, L = std::max(n1, n2);
        const double xi0 = xi_c - 0.5 * g.dxi * g.nx, eta0 = eta_c - 0.5 * g.deta * g.ny;
        microsim::CoeffSampler cs;
        if (coef_table) {
            cs = [=](double xi, double eta, double) {
                const int i = static_cast<int>(std::lround((xi - xi0) / g.dxi));
                const int j = static_cast<int>(std::lround((eta - eta0) / g.deta));
                const size_t N = static_cast<size_t>(n1) * n2, k = static_cast<size_t>(i) * n2 + j;
                geometry::TransformedCoefficients tc{};
                tc.a = -coef_table[0 * N + k];
                tc.c = -coef_table[1 * N + k];
                tc.d = coef_table[2 * N + k];
                tc.e = coef_table[3 * N + k];
                tc.f = coef_table[4 * N + k];
                return tc;
            };
        } else {
            const double A = coef[0], C = coef[1], Vx = coef[2], Vy = coef[3], W = coef[4];
            cs = [=](double, double, double) {
                geometry::TransformedCoefficients tc{};
                tc.a = -A;
                tc.c = -C;
                tc.d = Vx;
                tc.e = Vy;
                tc.f = W;
                return tc;
            };
        }
        microsim::PatchProblem p;
        p.xi_c = xi_c;
        p.eta_c = eta_c;
        p.h_xi = h_xi;
        p.h_eta = h_eta;
        p.t0 = t0;
        p.l = 1.0;
        p.coeffs = cs;
        p.source.zero = true;
        p.initial = Field2D(n1, n2);
        std::memcpy(p.initial.data(), u0, sizeof(double) * n1 * n2);
        for (int e = 0; e < 4; ++e) {
            const int len = (e == PD_EDGE_E || e == PD_EDGE_W) ? n2 : n1;
            p.edges[e] = edge_from(kinds[e], values + e * L, slopes + e * L, len, robin_w[2 * e],
                                   robin_w[2 * e + 1]);
        }
        const Field2D u = microsim::step_explicit(p, g);
        std::memcpy(uT, u.data(), sizeof(double) * n1 * n2);
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// Lifting chain for one stencil of macro values vals[3][3] centred at
// (xi_c, eta_c) with macro spacings (dxi, deta): u0 [n1][n2] plus edge slope
// and value profiles [4][L] in E,W,N,S order (gaptooth.cpp:110-168).
int ref_lift(const double* vals, double xi_c, double eta_c, double dxi, double deta, double h_xi,
             double h_eta, int nx, int ny, double* u0, double* slopes, double* values) {
    try {
        gaptooth::StencilPoly s;
        s.xi_c = xi_c;
        s.eta_c = eta_c;
        s.dxi = dxi;
        s.deta = deta;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) s.vals[a][b] = vals[3 * a + b];
        const microsim::MicroGrid g = microsim::make_micro_grid(h_xi, h_eta, 1.0, nx, ny, 1);
        const Field2D u = gaptooth::lift(s, h_xi, h_eta, g);
        std::memcpy(u0, u.data(), sizeof(double) * (nx + 1) * (ny + 1));
        const int L = std::max(nx, ny) + 1;
        const gaptooth::EdgeProfiles sl = gaptooth::neumann_edge_slopes(s, h_xi, h_eta, nx, ny);
        const gaptooth::EdgeProfiles va = gaptooth::dirichlet_edge_values(s, h_xi, h_eta, nx, ny);
        const std::vector<double>* S[4] = {&sl.E, &sl.W, &sl.N, &sl.S};
        const std::vector<double>* V[4] = {&va.E, &va.W, &va.N, &va.S};
        for (int e = 0; e < 4; ++e) {
            for (size_t k = 0; k < S[e]->size(); ++k) slopes[e * L + k] = (*S[e])[k];
            for (size_t k = 0; k < V[e]->size(); ++k) values[e * L + k] = (*V[e])[k];
        }
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

double ref_restrict(const double* u, int n1, int n2, int simpson) {
    Field2D f(n1, n2);
    std::memcpy(f.data(), u, sizeof(double) * n1 * n2);
    return gaptooth::restrict_average(f, simpson ? cpi::SchemeConfig::Quadrature::Simpson
                                                 : cpi::SchemeConfig::Quadrature::Trapezoid);
}

} // extern "C"
