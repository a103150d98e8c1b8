// Host-side problem / scheme types and the coefficient-table builder.
//
// Same shapes as the reference's ProblemSpec (proj/include/patchdyn/problems.hpp:
// 17-41), SchemeConfig (scheme_config.hpp:9-37) and Field2D (field.hpp:10-39)
// so the drop-in API reads like the reference.  build_tables() is the
// B200 framework's version of what the GapToothEngine constructor does on the
// host (gaptooth.cpp:200-282 + PatchIntegrator::sample_coeffs,
// microsim.cpp:204-263): the patch list, row sharing, and per-node solver-form
// coefficients, flattened into the pd_engine_desc tables the device consumes.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "geometry.hpp"
#include "patchdyn_b200.h"

namespace pdb200 {

class Field2D {
public:
    Field2D() = default;
    Field2D(int n1, int n2, double fill = 0.0) : n1_(n1), n2_(n2), v_(static_cast<size_t>(n1) * n2, fill) {}
    int n1() const { return n1_; }
    int n2() const { return n2_; }
    size_t size() const { return v_.size(); }
    double& operator()(int i, int j) { return v_[static_cast<size_t>(i) * n2_ + j]; }
    double operator()(int i, int j) const { return v_[static_cast<size_t>(i) * n2_ + j]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    std::vector<double>& raw() { return v_; }
    const std::vector<double>& raw() const { return v_; }
    bool same_shape(const Field2D& o) const { return n1_ == o.n1_ && n2_ == o.n2_; }

private:
    int n1_ = 0, n2_ = 0;
    std::vector<double> v_;
};

namespace problems {
struct ProblemSpec {
    std::string name;
    geometry::Mapping mapping;
    geometry::PhysicalCoefficients physical;
    double a = 0, b = 1, c = 0, d = 1;
    double T = 1.0;
    bool periodic_xi = false;
    std::function<double(double, double)> initial;
    std::function<double(double, double)> bcW, bcE, bcS, bcN;
    std::function<double(double, double, double)> exact;
    bool coeffs_time_independent = true;
    bool source_zero = false;
    bool source_separable = false;
    std::function<double(double, double)> source_spatial;
    std::function<double(double)> source_time;
    bool coeffs_xi_independent = false;
    bool has_exact() const { return static_cast<bool>(exact); }
};

// The reference benchmark problems and the BASELINE configs, from a
// pd_problem_desc (see include/patchdyn_b200.h).
ProblemSpec from_desc(const pd_problem_desc& d);
// seeded U[0,1) macro field + Jacobi smoothing of configs 4/5
std::vector<double> seeded_field(int Nxi, int Neta, uint64_t seed, int sweeps);
} // namespace problems

namespace microsim {
// UpwindSpec  proj/include/patchdyn/microsim.hpp:43-48 (ADI convection stencils)
enum class UpwindOrder { Two, Three, Four };
struct UpwindSpec {
    UpwindOrder order = UpwindOrder::Two;
    double r = 0.5; // modification weight of the four-point scheme
};
} // namespace microsim

namespace cpi {
struct SchemeConfig {
    int N_xi = 10, N_eta = 10;
    int Nt = 1000;
    double T = 1.0;
    double tau = 1e-6;
    int k = 0;
    double h_xi = 1e-3, h_eta = 1e-3;
    int nx = 10, ny = 10, nt = 2;
    enum class Solver { ADI, Explicit };
    Solver solver = Solver::ADI; // the reference's default (scheme_config.hpp:19-20)
    microsim::UpwindSpec upwind{};
    enum class BCType { Neumann, Dirichlet, Robin };
    BCType bc_type = BCType::Neumann;
    double robin_w1 = 1.0, robin_w2 = 1.0;
    enum class Quadrature { Trapezoid, Simpson };
    Quadrature quadrature = Quadrature::Trapezoid;
    // linear-response shortcut of GapToothEngine::step (scheme_config.hpp:30-31);
    // the reference's default is Auto, the BASELINE configs pin Off
    enum class LinearCache { Auto, On, Off };
    LinearCache linear_cache = LinearCache::Auto;
    int mode = PD_MODE_FAST;
    double dt() const { return T / Nt; }
    // SchemeConfig::validate  proj/src/cpi.cpp:11-44
    void validate(double xi_extent, double eta_extent) const;
};
SchemeConfig scheme_from_desc(const pd_problem_desc& d);
} // namespace cpi

// Host tables behind one pd_engine_desc.  `desc` points into the vectors.
struct EngineTables {
    pd_engine_desc desc{};
    std::vector<int32_t> patch_ij, coeff_set;
    std::vector<double> coeffs, source_spatial;
    double max_abs_ac = 0.0;   // max(|A|,|C|): the reference's guard numerator
    double max_a_plus_c = 0.0; // max(|A|+|C|): the dt pin denominator
    double max_abs_b = 0.0;
    void relink();
};

// Samples the solver-form coefficients for every patch (or every eta-row when
// the reference would share integrators across the row).  Does not check the
// explicit stability guard (that needs the final dt; see check_stability).
// sample = false: patch list and set map only (coefficients generated on the
// device, pd_coeffgen.cu); the maxima then come from the generator.
EngineTables build_tables(const problems::ProblemSpec& p, const cpi::SchemeConfig& cfg, int threads,
                          bool sample = true);
// PatchIntegrator's explicit guard  microsim.cpp:253-262
void check_stability(const EngineTables& t, const cpi::SchemeConfig& cfg);
// Per-micro-step samples of one substep from t0 (time-dependent coefficients,
// general sources; microsim.cpp:537-542, 265-281): coeff_steps [nt][sets][6][N],
// source_steps [nt][sets][N], either may be null.  Throws StabilityViolation.
void sample_substep(const problems::ProblemSpec& p, const cpi::SchemeConfig& cfg, const EngineTables& t, double t0,
                    double* coeff_steps, double* source_steps, int threads = 0);

} // namespace pdb200
