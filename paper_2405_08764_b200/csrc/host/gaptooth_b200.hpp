// Drop-in C++ operator interface over the B200 C-ABI.
//
// Same names and call shapes as the reference's gap-tooth / CPI layer so a
// reference user switches namespaces (patchdyn:: -> pdb200::):
//   GapToothEngine(problem, cfg)         proj/include/patchdyn/gaptooth.hpp:85
//   initial_field / refresh_boundary     gaptooth.hpp:87-88 (gaptooth.cpp:284-310)
//   step / step_direct                   gaptooth.hpp:91,100 (gaptooth.cpp:360-375)
//   cpi::projective_step                 proj/include/patchdyn/cpi.hpp:19-20 (cpi.cpp:58-77)
//   cpi::run                             cpi.hpp:45 (cpi.cpp:134-216)
// Mesh/metric setup stays on the host (build_tables samples
// transform_coefficients exactly like PatchIntegrator::sample_coeffs); the
// per-patch micro-solve, lifting, restriction and the projective axpy run in
// the sm_100a kernels behind pd_engine_* (include/patchdyn_b200.h).
// Errors surface as the reference's exception types (pdb200::Error family).
#pragma once

#include <algorithm>
#include <cmath>
#include <functional>
#include <memory>
#include <sstream>
#include <utility>
#include <vector>

#include "patchdyn_b200.h"
#include "problems.hpp"

namespace pdb200 {

inline void throw_status(int st, const pd_engine* e) {
    if (st == PD_OK) return;
    const std::string m = pd_last_error(e);
    switch (st) {
        case PD_NON_POSITIVE_JACOBIAN: throw NonPositiveJacobian(m);
        case PD_MIXED_TERM_UNSUPPORTED: throw MixedTermUnsupported(m);
        case PD_STABILITY_VIOLATION: throw StabilityViolation(m);
        case PD_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(m);
        case PD_SHAPE_MISMATCH: throw ShapeMismatch(m);
        case PD_MACRO_INSTABILITY: throw MacroInstability(m);
        case PD_MACRO_PATCH_ERROR: throw MacroPatchError(m);
        case PD_VALIDATION_ERROR: throw ValidationError(m);
        case PD_UNSUPPORTED: throw Unsupported(m);
        default: throw DeviceError(m);
    }
}

namespace gaptooth {

enum class SidePolicy { DirichletFromProblem, Periodic };

struct CoarseGrid {
    double a = 0, b = 1, c = 0, d = 1;
    int Nxi = 1, Neta = 1;
    double dxi() const { return (b - a) / Nxi; }
    double deta() const { return (d - c) / Neta; }
    double xi(int i) const { return a + dxi() * i; }
    double eta(int j) const { return c + deta() * j; }
};

struct CoarseField {
    CoarseGrid grid;
    bool periodic = false;
    Field2D U;
    bool periodic_xi() const { return periodic; }
    double& at(int i, int j) { return U(i, j); }
    double at(int i, int j) const { return U(i, j); }
};

class GapToothEngine {
public:
    GapToothEngine(const problems::ProblemSpec& problem, const cpi::SchemeConfig& cfg, int host_threads = 0)
        : problem_(problem), cfg_(cfg) {
        cfg_.validate(problem.b - problem.a, problem.d - problem.c);
        if (!problem.periodic_xi && (!problem.bcW || !problem.bcE))
            throw ValidationError("problem lacks W/E boundary functions");
        if (!problem.bcS || !problem.bcN) throw ValidationError("problem lacks S/N boundary functions");
        grid_ = CoarseGrid{problem.a, problem.b, problem.c, problem.d, cfg.N_xi, cfg.N_eta};
        tables_ = build_tables(problem_, cfg_, host_threads);
        check_stability(tables_, cfg_);
        // linear_cache  gaptooth.cpp:213-224
        const bool linear_eligible =
            problem.coeffs_time_independent && problem.source_zero && problem.coeffs_xi_independent;
        switch (cfg.linear_cache) {
            case cpi::SchemeConfig::LinearCache::Off: use_fast_ = false; break;
            case cpi::SchemeConfig::LinearCache::Auto: use_fast_ = linear_eligible; break;
            case cpi::SchemeConfig::LinearCache::On:
                if (!linear_eligible)
                    throw ValidationError(
                        "linear_cache=on requires time-independent coefficients, a zero source and "
                        "xi-independent coefficients");
                use_fast_ = true;
                break;
        }
        pd_engine* e = nullptr;
        throw_status(pd_engine_create(&tables_.desc, &e), nullptr);
        eng_.reset(e);
    }

    CoarseField initial_field() const {
        CoarseField F{grid_, problem_.periodic_xi, Field2D(grid_.Nxi + 1, grid_.Neta + 1)};
        for (int i = 0; i <= grid_.Nxi; ++i)
            for (int j = 0; j <= grid_.Neta; ++j) F.U(i, j) = problem_.initial(grid_.xi(i), grid_.eta(j));
        if (problem_.periodic_xi)
            for (int j = 0; j <= grid_.Neta; ++j) F.U(grid_.Nxi, j) = F.U(0, j);
        return F;
    }

    // refresh_boundary  gaptooth.cpp:296-310
    void refresh_boundary(CoarseField& F, double t) const {
        const int N1 = grid_.Nxi, N2 = grid_.Neta;
        for (int i = 0; i <= N1; ++i) {
            F.U(i, 0) = problem_.bcS(grid_.xi(i), t);
            F.U(i, N2) = problem_.bcN(grid_.xi(i), t);
        }
        if (problem_.periodic_xi) {
            for (int j = 0; j <= N2; ++j) F.U(N1, j) = F.U(0, j);
        } else {
            for (int j = 0; j <= N2; ++j) {
                F.U(0, j) = problem_.bcW(grid_.eta(j), t);
                F.U(N1, j) = problem_.bcE(grid_.eta(j), t);
            }
        }
    }

    // One gap-tooth step t -> t+tau (gaptooth.cpp:396-418): the linear-response
    // 9-point stencil when linear_cache enabled it (row weights built lazily on
    // the device, as build_row_weights does on first use), else step_direct.
    CoarseField step(const CoarseField& F, double t) const {
        if (!use_fast_) return step_direct(F, t);
        select_step(true);
        return device_step(F, t);
    }

    CoarseField step_direct(const CoarseField& F, double t) const {
        select_step(false);
        return device_step(F, t);
    }

    bool uses_linear_cache() const { return use_fast_; }
    // make the device engine's step the one GapToothEngine::step would take
    void select_step(bool linear) const {
        if (linear && !weights_ready_) {
            std::vector<double> w(9 * static_cast<size_t>(grid_.Neta + 1));
            throw_status(pd_linear_weights(eng_.get(), w.data()), eng_.get());
            throw_status(pd_engine_set_linear(eng_.get(), w.data()), eng_.get());
            weights_ready_ = true;
        }
        throw_status(pd_engine_set_step_kind(eng_.get(), linear ? PD_STEP_LINEAR : PD_STEP_DIRECT), eng_.get());
    }
    void select_default_step() const { select_step(use_fast_); }

    // time-dependent coefficients or a general source: the per-micro-step
    // sampling of PatchIntegrator::integrate (microsim.cpp:537-542, 265-281)
    // happens here on the host and the device runs the sweeps on the samples
    bool sampled() const {
        return !problem_.coeffs_time_independent || (!problem_.source_zero && !problem_.source_separable);
    }
    // [subs][nt][sets][6][N] coefficient and [subs][nt][sets][N] source samples
    // for the substeps starting at t, t + tau, ...
    void sample_tables(double t, int subs, std::vector<double>& c, std::vector<double>& g) const {
        const size_t N = static_cast<size_t>(cfg_.nx + 1) * (cfg_.ny + 1), S = tables_.desc.ncoeff_sets;
        const size_t per_c = cfg_.nt * S * PD_NCOEF * N, per_g = cfg_.nt * S * N;
        const bool gen = !problem_.source_zero && !problem_.source_separable;
        c.assign(subs * per_c, 0.0);
        g.assign(gen ? subs * per_g : 0, 0.0);
        for (int m = 0; m < subs; ++m)
            sample_substep(problem_, cfg_, tables_, t + m * cfg_.tau, c.data() + m * per_c,
                           gen ? g.data() + m * per_g : nullptr);
    }

private:
    CoarseField device_step(const CoarseField& F, double t) const {
        CoarseField out{grid_, F.periodic, Field2D(F.U.n1(), F.U.n2())};
        const std::vector<double> bnd = perimeter(t + cfg_.tau);
        if (sampled()) {
            std::vector<double> c, g;
            sample_tables(t, 1, c, g);
            throw_status(pd_gaptooth_step_sampled(eng_.get(), F.U.data(), out.U.data(), t, bnd.data(), c.data(),
                                                  g.empty() ? nullptr : g.data()),
                         eng_.get());
            return out;
        }
        const std::vector<double> src = source_factors(t, 0);
        throw_status(pd_gaptooth_step(eng_.get(), F.U.data(), out.U.data(), t, bnd.data(),
                                      src.empty() ? nullptr : src.data()),
                     eng_.get());
        return out;
    }

public:
    const CoarseGrid& grid() const { return grid_; }
    const cpi::SchemeConfig& config() const { return cfg_; }
    const problems::ProblemSpec& problem() const { return problem_; }
    pd_engine* device() const { return eng_.get(); }
    int kernel_family() const { return pd_engine_mode(eng_.get()); }

    // refresh values at t in the pd_perimeter layout
    std::vector<double> perimeter(double t) const {
        const int N1 = grid_.Nxi, N2 = grid_.Neta;
        std::vector<double> b(pd_perimeter_len(N1, N2), 0.0);
        for (int i = 0; i <= N1; ++i) {
            b[i] = problem_.bcS(grid_.xi(i), t);
            b[N1 + 1 + i] = problem_.bcN(grid_.xi(i), t);
        }
        if (!problem_.periodic_xi)
            for (int j = 0; j <= N2; ++j) {
                b[2 * (N1 + 1) + j] = problem_.bcW(grid_.eta(j), t);
                b[2 * (N1 + 1) + N2 + 1 + j] = problem_.bcE(grid_.eta(j), t);
            }
        return b;
    }

    // separable source factors time(t')/l for k+1 substeps starting at t (microsim.cpp:272-277)
    std::vector<double> source_factors(double t, int k) const {
        if (problem_.source_zero) return {};
        const double mdt = cfg_.tau / cfg_.nt;
        std::vector<double> f(static_cast<size_t>(k + 1) * cfg_.nt);
        for (int m = 0; m <= k; ++m)
            for (int s = 0; s < cfg_.nt; ++s)
                f[static_cast<size_t>(m) * cfg_.nt + s] =
                    problem_.source_time(cfg_.solver == cpi::SchemeConfig::Solver::ADI ? (t + m * cfg_.tau) + (s + 0.5) * mdt
                                                                                       : (t + m * cfg_.tau) + s * mdt) /
                    problem_.physical.l;
        return f;
    }

private:
    struct EngineDeleter {
        void operator()(pd_engine* e) const { pd_engine_destroy(e); }
    };
    problems::ProblemSpec problem_;
    cpi::SchemeConfig cfg_;
    CoarseGrid grid_;
    EngineTables tables_;
    std::unique_ptr<pd_engine, EngineDeleter> eng_;
    bool use_fast_ = false;
    mutable bool weights_ready_ = false;
};

} // namespace gaptooth

namespace cpi {

// projective_step  cpi.cpp:58-77: k+1 fused substeps + extrapolation + refresh
inline gaptooth::CoarseField projective_step(const gaptooth::GapToothEngine& engine, const gaptooth::CoarseField& U,
                                             double t) {
    const SchemeConfig& cfg = engine.config();
    std::vector<double> bnd;
    for (int m = 0; m <= cfg.k; ++m) {
        const std::vector<double> b = engine.perimeter((t + m * cfg.tau) + cfg.tau);
        bnd.insert(bnd.end(), b.begin(), b.end());
    }
    const std::vector<double> last = engine.perimeter(t + cfg.dt());
    bnd.insert(bnd.end(), last.begin(), last.end());
    const std::vector<double> src = engine.source_factors(t, cfg.k);
    gaptooth::CoarseField out{U.grid, U.periodic, Field2D(U.U.n1(), U.U.n2())};
    engine.select_default_step(); // cpi.cpp:65 calls engine.step
    if (engine.sampled()) {
        std::vector<double> c, g;
        engine.sample_tables(t, cfg.k + 1, c, g);
        throw_status(pd_projective_step_sampled(engine.device(), U.U.data(), out.U.data(), t, bnd.data(), c.data(),
                                                g.empty() ? nullptr : g.data()),
                     engine.device());
        return out;
    }
    throw_status(pd_projective_step(engine.device(), U.U.data(), out.U.data(), t, bnd.data(),
                                    src.empty() ? nullptr : src.data()),
                 engine.device());
    return out;
}

struct RunOptions {
    std::vector<double> snapshot_times;
    std::vector<std::pair<int, int>> probe_nodes;
    int progress_every = 0;
    std::function<void(int, double, double)> progress;
};
struct Snapshot {
    double t = 0.0;
    std::vector<double> U;
};
struct ProbeSeries {
    int i = 0, j = 0;
    std::vector<double> values;
};
struct RunResult {
    std::vector<double> times;
    std::vector<double> step_max_pct_err;
    double max_pct_err = 0.0;
    std::vector<Snapshot> snapshots;
    std::vector<ProbeSeries> probes;
    gaptooth::CoarseField final_field;
};

// max_percent_error  cpi.cpp:79-94
inline double max_percent_error(const gaptooth::GapToothEngine& engine, const gaptooth::CoarseField& U, double t) {
    const auto& p = engine.problem();
    if (!p.has_exact()) return 0.0;
    const auto& g = engine.grid();
    const int i_lo = U.periodic_xi() ? 0 : 1;
    double worst = 0.0;
    for (int i = i_lo; i <= g.Nxi - 1; ++i)
        for (int j = 1; j <= g.Neta - 1; ++j) {
            const double ex = p.exact(g.xi(i), g.eta(j), t);
            if (std::abs(ex) < 1e-12) continue;
            worst = std::max(worst, std::abs(U.at(i, j) - ex) / std::abs(ex) * 100.0);
        }
    return worst;
}

// cpi::run  cpi.cpp:134-216.  Without diagnostics requested, the whole macro
// loop stays on the device (pd_run: one launch sequence, blow-up guard on the
// device); with probes/snapshots/exact errors it runs in segments between the
// steps that need the field on the host.
inline RunResult run_sampled(const gaptooth::GapToothEngine& engine, const RunOptions& opts);

inline RunResult run(const gaptooth::GapToothEngine& engine, const RunOptions& opts = {}) {
    if (engine.sampled()) return run_sampled(engine, opts);
    const SchemeConfig& cfg = engine.config();
    const double dt = cfg.dt();
    gaptooth::CoarseField U = engine.initial_field();
    engine.refresh_boundary(U, 0.0);
    RunResult res;
    std::vector<int> snap;
    for (double ts : opts.snapshot_times) snap.push_back(std::clamp(static_cast<int>(std::lround(ts / dt)), 0, cfg.Nt));
    auto maybe_snapshot = [&](int n, double t) {
        for (int& s : snap)
            if (s == n) {
                res.snapshots.push_back(Snapshot{t, U.U.raw()});
                s = -1;
                break;
            }
    };
    for (auto [pi, pj] : opts.probe_nodes) res.probes.push_back(ProbeSeries{pi, pj, {}});
    maybe_snapshot(0, 0.0);
    // the exact-error metric runs on the device (pd_run_exact); probes, snapshots
    // and progress callbacks need the field on the host after every step
    const bool per_step = !opts.probe_nodes.empty() || !snap.empty() || opts.progress_every > 0;
    const bool has_exact = engine.problem().has_exact();
    const auto& g = engine.grid();
    const size_t NF = static_cast<size_t>(g.Nxi + 1) * (g.Neta + 1);
    const int i_lo = U.periodic_xi() ? 0 : 1;
    const int chunk = per_step ? 1 : cfg.Nt;
    // one blow-up scale for the whole run (cpi.cpp:142-144), whatever the segmentation
    double scale0 = 0.0;
    for (double v : U.U.raw()) scale0 = std::max(scale0, std::abs(v));
    const int k = cfg.k;
    const size_t L = pd_perimeter_len(cfg.N_xi, cfg.N_eta);
    for (int n = 0; n < cfg.Nt; n += chunk) {
        const int m = std::min(chunk, cfg.Nt - n);
        std::vector<double> bnd, src;
        for (int q = 0; q < m; ++q) {
            const double t = (n + q) * dt;
            for (int s = 0; s <= k; ++s) {
                const auto b = engine.perimeter((t + s * cfg.tau) + cfg.tau);
                bnd.insert(bnd.end(), b.begin(), b.end());
            }
            const auto b = engine.perimeter(t + dt);
            bnd.insert(bnd.end(), b.begin(), b.end());
            const auto f = engine.source_factors(t, k);
            src.insert(src.end(), f.begin(), f.end());
        }
        (void)L;
        // exact solution on the patch nodes at the end of every step of the chunk,
        // sampled as max_percent_error does (cpi.cpp:79-94)
        std::vector<double> exact, err;
        if (has_exact) {
            exact.assign(NF * static_cast<size_t>(m), 0.0);
            err.assign(static_cast<size_t>(m), 0.0);
            for (int q = 0; q < m; ++q) {
                const double t1 = (n + q + 1) * dt;
                double* ex = exact.data() + NF * static_cast<size_t>(q);
                for (int i = i_lo; i <= g.Nxi - 1; ++i)
                    for (int j = 1; j <= g.Neta - 1; ++j)
                        ex[static_cast<size_t>(i) * (g.Neta + 1) + j] = engine.problem().exact(g.xi(i), g.eta(j), t1);
            }
        }
        pd_run_stats st{};
        engine.select_default_step(); // projective_step -> engine.step  cpi.cpp:65
        throw_status(pd_engine_set_run_guard(engine.device(), std::max(scale0, 1e-12), n), engine.device());
        const int rc = pd_run_exact(engine.device(), U.U.data(), m, n * dt, bnd.data(),
                                    src.empty() ? nullptr : src.data(), has_exact ? exact.data() : nullptr,
                                    has_exact ? err.data() : nullptr, &st);
        if (rc == PD_MACRO_INSTABILITY) {
            std::ostringstream os;
            os << pd_last_error(engine.device());
            throw MacroInstability(os.str());
        }
        throw_status(rc, engine.device());
        for (int q = 0; q < m; ++q) res.times.push_back((n + q + 1) * dt);
        const double t1 = (n + m) * dt;
        for (auto& ps : res.probes) ps.values.push_back(U.at(ps.i, ps.j));
        for (double e : err) { // device max_percent_error of every step of the chunk
            res.step_max_pct_err.push_back(e);
            res.max_pct_err = std::max(res.max_pct_err, e);
        }
        maybe_snapshot(n + m, t1);
        if (opts.progress_every > 0 && opts.progress && (n + m) % opts.progress_every == 0)
            opts.progress(n + m, t1, res.max_pct_err);
    }
    throw_status(pd_engine_set_run_guard(engine.device(), 0.0, 0), engine.device());
    res.final_field = std::move(U);
    return res;
}

// cpi::run for time-dependent coefficients / general sources: the reference's
// loop (cpi.cpp:134-216) with each projective step on the device over host
// samples; guard, probes, snapshots and the exact-error metric on the host
inline RunResult run_sampled(const gaptooth::GapToothEngine& engine, const RunOptions& opts) {
    const SchemeConfig& cfg = engine.config();
    const double dt = cfg.dt();
    gaptooth::CoarseField U = engine.initial_field();
    engine.refresh_boundary(U, 0.0);
    double scale0 = 0.0;
    for (double v : U.U.raw()) scale0 = std::max(scale0, std::abs(v));
    const double blowup = 10.0 * std::max(scale0, 1e-12);
    RunResult res;
    std::vector<int> snap;
    for (double ts : opts.snapshot_times) snap.push_back(std::clamp(static_cast<int>(std::lround(ts / dt)), 0, cfg.Nt));
    auto maybe_snapshot = [&](int n, double t) {
        for (int& s : snap)
            if (s == n) {
                res.snapshots.push_back(Snapshot{t, U.U.raw()});
                s = -1;
                break;
            }
    };
    for (auto [pi, pj] : opts.probe_nodes) res.probes.push_back(ProbeSeries{pi, pj, {}});
    maybe_snapshot(0, 0.0);
    for (int n = 0; n < cfg.Nt; ++n) {
        U = projective_step(engine, U, n * dt);
        const double t1 = (n + 1) * dt;
        res.times.push_back(t1);
        double umax = 0.0;
        bool finite = true;
        for (double v : U.U.raw()) {
            if (!std::isfinite(v)) {
                finite = false;
                break;
            }
            umax = std::max(umax, std::abs(v));
        }
        if (!finite || umax > blowup) {
            std::ostringstream os;
            os << "coarse field " << (finite ? "exceeded 10x the initial magnitude" : "became non-finite")
               << " at macro step " << n + 1 << " (t=" << t1 << "); the projective step size is likely beyond the stable range";
            throw MacroInstability(os.str());
        }
        for (auto& ps : res.probes) ps.values.push_back(U.at(ps.i, ps.j));
        if (engine.problem().has_exact()) {
            const double e = max_percent_error(engine, U, t1);
            res.step_max_pct_err.push_back(e);
            res.max_pct_err = std::max(res.max_pct_err, e);
        }
        maybe_snapshot(n + 1, t1);
        if (opts.progress_every > 0 && opts.progress && (n + 1) % opts.progress_every == 0)
            opts.progress(n + 1, t1, res.max_pct_err);
    }
    res.final_field = std::move(U);
    return res;
}

} // namespace cpi
} // namespace pdb200
