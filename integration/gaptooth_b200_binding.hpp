// Reference-side binding of the B200 engine (compiled).
//
// What a maintainer of the reference (/root/reference/proj, namespace
// patchdyn) adds to route the gap-tooth hot path through the C-ABI
// (include/patchdyn_b200.h) while the reference keeps everything around it:
// the reference's own GapToothEngine stays the owner of the problem, the
// scheme, the coarse grid, the micro grid, initial_field and refresh_boundary
// (gaptooth.hpp:83-123); this class takes its patch list (the constructor's
// order, gaptooth.cpp:251-280, with the same row sharing, :254-266) and the
// coefficients sampled by the reference's own transform_coefficients at the
// reference's own PatchIntegrator node coordinates (microsim.cpp:204-263) and
// hands them to pd_engine_create.  step_direct / projective_step / run then
// replace GapToothEngine::step_direct (gaptooth.cpp:360-375),
// cpi::projective_step (cpi.cpp:58-77) and cpi::run's loop (cpi.cpp:134-216).
//
// Only public reference API is used (grid(), config(), problem(),
// micro_grid(), initial_field(), refresh_boundary(), PatchIntegrator's public
// constructor and node_xi/node_eta, geometry::transform_coefficients), so it
// compiles against the unmodified headers: -I proj/include -I <repo>/include.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <sstream>
#include <vector>

#include "patchdyn/cpi.hpp"
#include "patchdyn/errors.hpp"
#include "patchdyn/gaptooth.hpp"
#include "patchdyn/geometry.hpp"
#include "patchdyn/microsim.hpp"
#include "patchdyn_b200.h"

namespace patchdyn::b200 {

// pd_status -> the reference's exception classes (errors.hpp:9-61)
inline void throw_status(int st, const pd_engine* e) {
    if (st == PD_OK) return;
    const std::string m = pd_last_error(e);
    switch (st) {
        case PD_MACRO_INSTABILITY: throw MacroInstability(m);
        case PD_MACRO_PATCH_ERROR: throw MacroPatchError(m);
        case PD_STABILITY_VIOLATION: throw StabilityViolation(m);
        case PD_MIXED_TERM_UNSUPPORTED: throw MixedTermUnsupported(m);
        case PD_SHAPE_MISMATCH: throw ShapeMismatch(m);
        default: throw ValidationError(std::string(pd_status_name(st)) + ": " + m);
    }
}

class DeviceGapTooth {
public:
    // mode: PD_MODE_FAST (register-blocked kernels, within 1e-11 after a full
    // run) or PD_MODE_EXACT (the reference's operation order, bit-identical)
    explicit DeviceGapTooth(const gaptooth::GapToothEngine& ref, int32_t mode = PD_MODE_FAST) : ref_(ref) {
        const gaptooth::CoarseGrid& g = ref.grid();
        const cpi::SchemeConfig& cfg = ref.config();
        const problems::ProblemSpec& pr = ref.problem();
        const microsim::MicroGrid& mg = ref.micro_grid();
        if (!pr.coeffs_time_independent)
            throw ValidationError("B200 binding: time-dependent coefficients stay on the reference path");
        if (!pr.source_zero && !pr.source_separable)
            throw ValidationError("B200 binding: general sources stay on the reference path");
        // patch list in the constructor's order  gaptooth.cpp:251-280
        const int i_lo = pr.periodic_xi ? 0 : 1, i_hi = g.Nxi - 1;
        const bool share_rows = pr.coeffs_time_independent && pr.coeffs_xi_independent && pr.source_zero;
        std::vector<int> set_i, set_j;
        for (int j = 1; j <= g.Neta - 1; ++j) {
            if (share_rows) {
                set_i.push_back(i_lo);
                set_j.push_back(j);
            }
            for (int i = i_lo; i <= i_hi; ++i) {
                pij_.push_back(i);
                pij_.push_back(j);
                if (share_rows) {
                    cset_.push_back(j - 1);
                } else {
                    set_i.push_back(i);
                    set_j.push_back(j);
                }
            }
        }
        // coefficients at the reference's node coordinates  microsim.cpp:208-209, 245-249
        const int n1 = mg.nx + 1, n2 = mg.ny + 1;
        const size_t N = static_cast<size_t>(n1) * n2;
        const double l = pr.physical.l;
        microsim::CoeffSampler probe = [](double, double, double) {
            geometry::TransformedCoefficients tc{};
            tc.a = tc.c = -1.0;
            return tc;
        };
        coef_.assign(set_i.size() * PD_NCOEF * N, 0.0);
        if (pr.source_separable) src_.assign(set_i.size() * N, 0.0);
        for (size_t s = 0; s < set_i.size(); ++s) {
            const microsim::PatchIntegrator node(g.xi(set_i[s]), g.eta(set_j[s]), mg, l, probe, true,
                                                 microsim::SourceSpec{}, microsim::PatchIntegrator::Scheme::ADI);
            double* o = coef_.data() + s * PD_NCOEF * N;
            for (int i = 0; i < n1; ++i)
                for (int j = 0; j < n2; ++j) {
                    const auto tc = geometry::transform_coefficients(pr.mapping, pr.physical, node.node_xi(i),
                                                                     node.node_eta(j), 0.0);
                    const size_t k = static_cast<size_t>(i) * n2 + j;
                    o[PD_COEF_A * N + k] = -tc.a / l;
                    o[PD_COEF_B * N + k] = std::abs(tc.b) > 1e-12 ? -tc.b / l : 0.0;
                    o[PD_COEF_C * N + k] = -tc.c / l;
                    o[PD_COEF_VX * N + k] = tc.d / l;
                    o[PD_COEF_VY * N + k] = tc.e / l;
                    o[PD_COEF_W * N + k] = tc.f / l;
                    if (pr.source_separable) src_[s * N + k] = pr.source_spatial(node.node_xi(i), node.node_eta(j));
                }
        }
        pd_engine_desc d{};
        d.a = g.a;
        d.b = g.b;
        d.c = g.c;
        d.d = g.d;
        d.Nxi = g.Nxi;
        d.Neta = g.Neta;
        d.periodic_xi = pr.periodic_xi ? 1 : 0;
        d.nx = mg.nx;
        d.ny = mg.ny;
        d.nt = mg.nt;
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
        d.npatches = static_cast<int32_t>(pij_.size() / 2);
        d.patch_ij = pij_.data();
        d.ncoeff_sets = static_cast<int32_t>(set_i.size());
        d.coeff_set = cset_.empty() ? nullptr : cset_.data();
        d.coeffs = coef_.data();
        d.source_kind = pr.source_zero ? PD_SOURCE_ZERO : PD_SOURCE_SEPARABLE;
        d.source_spatial = src_.empty() ? nullptr : src_.data();
        d.l = l;
        d.mode = mode;
        d.solver = cfg.solver == cpi::SchemeConfig::Solver::ADI ? PD_SOLVER_ADI : PD_SOLVER_EXPLICIT;
        d.upwind_order = cfg.upwind.order == microsim::UpwindOrder::Four    ? PD_UPWIND_FOUR
                         : cfg.upwind.order == microsim::UpwindOrder::Three ? PD_UPWIND_THREE
                                                                            : PD_UPWIND_TWO;
        d.upwind_r = cfg.upwind.r;
        throw_status(pd_engine_create(&d, &dev_), nullptr);
        perim_ = pd_perimeter_len(g.Nxi, g.Neta);
    }
    ~DeviceGapTooth() { pd_engine_destroy(dev_); }
    DeviceGapTooth(const DeviceGapTooth&) = delete;
    DeviceGapTooth& operator=(const DeviceGapTooth&) = delete;

    const gaptooth::GapToothEngine& reference() const { return ref_; }
    pd_engine* device() const { return dev_; }
    int32_t mode() const { return pd_engine_mode(dev_); }

    // refresh_boundary's values at t as a perimeter array [S][N][W][E]
    // (pd_perimeter_len), taken from the reference's own refresh_boundary
    void perimeter(double t, double* out) const {
        gaptooth::CoarseField F = ref_.initial_field();
        ref_.refresh_boundary(F, t);
        const int N1 = F.grid.Nxi, N2 = F.grid.Neta;
        double* S = out;
        double* Nn = out + (N1 + 1);
        double* W = out + 2 * (N1 + 1);
        double* E = W + (N2 + 1);
        for (int i = 0; i <= N1; ++i) {
            S[i] = F.U(i, 0);
            Nn[i] = F.U(i, N2);
        }
        for (int j = 0; j <= N2; ++j) {
            W[j] = F.U(0, j);
            E[j] = F.U(N1, j);
        }
    }

    // source time factors time(t0 + s dt)/l of the k+1 substeps (microsim.cpp:272-277)
    std::vector<double> source_factors(double t) const {
        const problems::ProblemSpec& pr = ref_.problem();
        const cpi::SchemeConfig& cfg = ref_.config();
        std::vector<double> f;
        if (!pr.source_separable) return f;
        const microsim::MicroGrid& mg = ref_.micro_grid();
        for (int m = 0; m <= cfg.k; ++m)
            for (int s = 0; s < mg.nt; ++s) f.push_back(pr.source_time((t + m * cfg.tau) + s * mg.dt) / pr.physical.l);
        return f;
    }

    // GapToothEngine::step_direct  gaptooth.cpp:360-375
    gaptooth::CoarseField step_direct(const gaptooth::CoarseField& F, double t) const {
        gaptooth::CoarseField out = F;
        std::vector<double> src = source_factors(t);
        throw_status(pd_gaptooth_step(dev_, F.U.data(), out.U.data(), t, nullptr, src.empty() ? nullptr : src.data()),
                     dev_);
        ref_.refresh_boundary(out, t + ref_.config().tau);
        return out;
    }

    // cpi::projective_step  cpi.cpp:58-77 (k+1 substeps + extrapolation on the device)
    gaptooth::CoarseField projective_step(const gaptooth::CoarseField& U, double t) const {
        const cpi::SchemeConfig& cfg = ref_.config();
        std::vector<double> bnd = boundary_rows(t);
        std::vector<double> src = source_factors(t);
        gaptooth::CoarseField out = U;
        throw_status(pd_projective_step(dev_, U.U.data(), out.U.data(), t, bnd.data(), src.empty() ? nullptr : src.data()),
                     dev_);
        (void)cfg;
        return out;
    }

    // cpi::run  cpi.cpp:134-216 without probes / snapshots / progress: the whole
    // macro loop in one pd_run_exact call (blow-up guard and the per-step
    // max_percent_error on the device)
    cpi::RunResult run() const {
        const cpi::SchemeConfig& cfg = ref_.config();
        const problems::ProblemSpec& pr = ref_.problem();
        const gaptooth::CoarseGrid& g = ref_.grid();
        const double dt = cfg.dt();
        gaptooth::CoarseField U = ref_.initial_field();
        ref_.refresh_boundary(U, 0.0);
        std::vector<double> bnd, src;
        for (int n = 0; n < cfg.Nt; ++n) {
            const std::vector<double> b = boundary_rows(n * dt);
            bnd.insert(bnd.end(), b.begin(), b.end());
            const std::vector<double> f = source_factors(n * dt);
            src.insert(src.end(), f.begin(), f.end());
        }
        const bool has_exact = pr.has_exact();
        const size_t NF = U.U.size();
        std::vector<double> exact, err;
        if (has_exact) { // max_percent_error's sampling  cpi.cpp:79-94
            exact.assign(NF * static_cast<size_t>(cfg.Nt), 0.0);
            err.assign(static_cast<size_t>(cfg.Nt), 0.0);
            const int i_lo = pr.periodic_xi ? 0 : 1;
            for (int n = 0; n < cfg.Nt; ++n) {
                double* ex = exact.data() + NF * static_cast<size_t>(n);
                for (int i = i_lo; i <= g.Nxi - 1; ++i)
                    for (int j = 1; j <= g.Neta - 1; ++j)
                        ex[static_cast<size_t>(i) * (g.Neta + 1) + j] = pr.exact(g.xi(i), g.eta(j), (n + 1) * dt);
            }
        }
        pd_run_stats st{};
        throw_status(pd_run_exact(dev_, U.U.data(), cfg.Nt, 0.0, bnd.data(), src.empty() ? nullptr : src.data(),
                                  has_exact ? exact.data() : nullptr, has_exact ? err.data() : nullptr, &st),
                     dev_);
        cpi::RunResult res;
        for (int n = 0; n < cfg.Nt; ++n) res.times.push_back((n + 1) * dt);
        for (double e : err) {
            res.step_max_pct_err.push_back(e);
            res.max_pct_err = std::max(res.max_pct_err, e);
        }
        res.final_field = std::move(U);
        return res;
    }

private:
    // [k+2][perimeter]: refresh values at t+(m+1)tau (m = 0..k) and at t+dt
    std::vector<double> boundary_rows(double t) const {
        const cpi::SchemeConfig& cfg = ref_.config();
        std::vector<double> b(static_cast<size_t>(cfg.k + 2) * perim_);
        for (int m = 0; m <= cfg.k; ++m) perimeter((t + m * cfg.tau) + cfg.tau, b.data() + m * perim_);
        perimeter(t + cfg.dt(), b.data() + (cfg.k + 1) * perim_);
        return b;
    }

    const gaptooth::GapToothEngine& ref_;
    pd_engine* dev_ = nullptr;
    size_t perim_ = 0;
    std::vector<int32_t> pij_, cset_;
    std::vector<double> coef_, src_;
};

} // namespace patchdyn::b200
