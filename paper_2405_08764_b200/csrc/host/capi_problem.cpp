// C-ABI of the host problem builder (pd_problem_*, include/patchdyn_b200.h).
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "problems.hpp"

namespace pdb200 {
void set_global_error(const std::string& m); // capi_engine
}

struct pd_problem {
    pd_problem_desc desc{};
    pdb200::problems::ProblemSpec spec;
    pdb200::cpi::SchemeConfig cfg;
    pdb200::EngineTables tables;
};

namespace {

int fail(const pdb200::Error& e) {
    pdb200::set_global_error(e.what());
    return e.status;
}

// refresh_boundary values at t as a perimeter (gaptooth.cpp:296-310)
void perimeter(const pd_problem& P, double t, double* out) {
    const auto& s = P.spec;
    const int N1 = P.cfg.N_xi, N2 = P.cfg.N_eta;
    const double Dxi = (s.b - s.a) / N1, Deta = (s.d - s.c) / N2;
    double* S = out;
    double* N = out + (N1 + 1);
    double* W = out + 2 * (N1 + 1);
    double* E = W + (N2 + 1);
    for (int i = 0; i <= N1; ++i) {
        const double xi = s.a + Dxi * i;
        S[i] = s.bcS(xi, t);
        N[i] = s.bcN(xi, t);
    }
    for (int j = 0; j <= N2; ++j) {
        const double eta = s.c + Deta * j;
        W[j] = s.periodic_xi ? 0.0 : s.bcW(eta, t);
        E[j] = s.periodic_xi ? 0.0 : s.bcE(eta, t);
    }
}

} // namespace

extern "C" {

pd_status pd_problem_create(const pd_problem_desc* desc, pd_problem** out) {
    try {
        if (!desc || !out) throw pdb200::ValidationError("null argument");
        auto P = std::make_unique<pd_problem>();
        P->desc = *desc;
        pd_problem_desc& r = P->desc;
        P->spec = pdb200::problems::from_desc(r);
        const auto& s = P->spec;
        if (r.h_frac > 0.0) { // patch width as a fraction of the macro spacing
            r.h_xi = r.h_frac * ((s.b - s.a) / r.N_xi);
            r.h_eta = r.h_frac * ((s.d - s.c) / r.N_eta);
        }
        pdb200::cpi::SchemeConfig cfg = pdb200::cpi::scheme_from_desc(r);
        if (r.dt_rule != PD_DT_GIVEN && !(cfg.tau > 0)) cfg.tau = 1.0; // placeholder until resolved
        if (r.dt_over_tau > 0 && !(cfg.T > 0)) cfg.T = 1.0;
        const bool devgen = r.coeff_gen == PD_COEFF_DEVICE;
        P->tables = pdb200::build_tables(s, cfg, r.threads, !devgen);
        if (devgen) { // no host tables; one reduction-only generator pass for the pins/guards
            pd_engine_desc& ed = P->tables.desc;
            ed.coeff_generator = &P->desc;
            double st[5];
            const pd_status gst = pd_coeffs_generate(&ed, nullptr, nullptr, st);
            if (gst != PD_OK) throw pdb200::Error(gst, pd_last_error(nullptr));
            P->tables.max_abs_ac = st[0];
            P->tables.max_a_plus_c = st[1];
            P->tables.max_abs_b = st[2];
            if (st[2] > 0.0 && ed.bc_type == PD_BC_ROBIN)
                throw pdb200::MixedTermUnsupported("mixed-derivative term with Robin patch conditions is not defined");
        }
        // micro dt pins
        const double dmin = std::min(r.h_xi / r.nx, r.h_eta / r.ny);
        if (r.dt_rule == PD_DT_DIFFUSION) {
            r.tau = r.nt * (0.2 * dmin * dmin / r.eps);
        } else if (r.dt_rule == PD_DT_METRIC) {
            r.tau = r.nt * (0.2 * dmin * dmin / P->tables.max_a_plus_c);
        }
        if (r.dt_over_tau > 0) r.T = r.Nt * (r.dt_over_tau * r.tau);
        r.dt_rule = PD_DT_GIVEN;
        r.h_frac = 0.0;
        r.dt_over_tau = 0.0;
        cfg = pdb200::cpi::scheme_from_desc(r);
        cfg.validate(s.b - s.a, s.d - s.c);
        pdb200::check_stability(P->tables, cfg);
        P->tables.desc.tau = cfg.tau;
        P->tables.desc.dt_macro = cfg.dt();
        P->cfg = cfg;
        *out = P.release();
        return PD_OK;
    } catch (const pdb200::Error& e) {
        return static_cast<pd_status>(fail(e));
    } catch (const std::exception& e) {
        pdb200::set_global_error(e.what());
        return PD_VALIDATION_ERROR;
    }
}

void pd_problem_destroy(pd_problem* p) { delete p; }

pd_status pd_problem_resolved(const pd_problem* p, pd_problem_desc* out) {
    if (!p || !out) return PD_VALIDATION_ERROR;
    *out = p->desc;
    return PD_OK;
}

pd_status pd_problem_engine_desc(const pd_problem* p, pd_engine_desc* out) {
    if (!p || !out) return PD_VALIDATION_ERROR;
    *out = p->tables.desc;
    return PD_OK;
}

pd_status pd_problem_initial_field(const pd_problem* p, double* U) {
    // GapToothEngine::initial_field  gaptooth.cpp:284-294
    const auto& s = p->spec;
    const int N1 = p->cfg.N_xi, N2 = p->cfg.N_eta;
    const double Dxi = (s.b - s.a) / N1, Deta = (s.d - s.c) / N2;
    for (int i = 0; i <= N1; ++i)
        for (int j = 0; j <= N2; ++j) U[static_cast<size_t>(i) * (N2 + 1) + j] = s.initial(s.a + Dxi * i, s.c + Deta * j);
    if (s.periodic_xi)
        for (int j = 0; j <= N2; ++j) U[static_cast<size_t>(N1) * (N2 + 1) + j] = U[j];
    return PD_OK;
}

pd_status pd_problem_boundary(const pd_problem* p, double t, double* out) {
    try {
        perimeter(*p, t, out);
        return PD_OK;
    } catch (const pdb200::Error& e) {
        return static_cast<pd_status>(fail(e));
    }
}

pd_status pd_problem_boundary_table(const pd_problem* p, double t0, int32_t nsteps, double* out) {
    const int k = p->cfg.k;
    const size_t L = pd_perimeter_len(p->cfg.N_xi, p->cfg.N_eta);
    const double dt = p->cfg.dt(), tau = p->cfg.tau;
    for (int n = 0; n < nsteps; ++n) {
        const double t = t0 + n * dt; // cpi.cpp:176
        double* o = out + static_cast<size_t>(n) * (k + 2) * L;
        for (int m = 0; m <= k; ++m) perimeter(*p, (t + m * tau) + tau, o + static_cast<size_t>(m) * L);
        perimeter(*p, t + dt, o + static_cast<size_t>(k + 1) * L);
    }
    return PD_OK;
}

pd_status pd_problem_source_time(const pd_problem* p, double t0, int32_t nsteps, double* out) {
    const auto& s = p->spec;
    if (s.source_zero || !s.source_time) return PD_UNSUPPORTED;
    const int k = p->cfg.k, nt = p->cfg.nt;
    const double dt = p->cfg.dt(), tau = p->cfg.tau, mdt = tau / nt, l = s.physical.l;
    const bool adi = p->cfg.solver == pdb200::cpi::SchemeConfig::Solver::ADI;
    for (int n = 0; n < nsteps; ++n) {
        const double t = t0 + n * dt;
        for (int m = 0; m <= k; ++m) {
            const double tm = t + m * tau;
            for (int q = 0; q < nt; ++q) // coefficient/source time of micro step q  microsim.cpp:536-537
                out[(static_cast<size_t>(n) * (k + 1) + m) * nt + q] =
                    s.source_time(adi ? tm + (q + 0.5) * mdt : tm + q * mdt) / l;
        }
    }
    return PD_OK;
}

pd_status pd_problem_exact(const pd_problem* p, double t, double* U) {
    const auto& s = p->spec;
    if (!s.has_exact()) return PD_UNSUPPORTED;
    const int N1 = p->cfg.N_xi, N2 = p->cfg.N_eta;
    const double Dxi = (s.b - s.a) / N1, Deta = (s.d - s.c) / N2;
    for (int i = 0; i <= N1; ++i)
        for (int j = 0; j <= N2; ++j)
            U[static_cast<size_t>(i) * (N2 + 1) + j] = s.exact(s.a + Dxi * i, s.c + Deta * j, t);
    return PD_OK;
}

pd_status pd_problem_sample_substep(const pd_problem* p, double t0, double* coeff_steps, double* source_steps) {
    try {
        if (!p || (!coeff_steps && !source_steps)) throw pdb200::ValidationError("null argument");
        if (source_steps && (p->spec.source_zero || p->spec.source_separable))
            throw pdb200::Unsupported("the problem has no general source to sample");
        pdb200::sample_substep(p->spec, p->cfg, p->tables, t0, coeff_steps, source_steps, p->desc.threads);
        return PD_OK;
    } catch (const pdb200::Error& e) {
        return static_cast<pd_status>(fail(e));
    }
}

pd_status pd_problem_stability(const pd_problem* p, double* max_a_plus_c, double* ref_number) {
    const double dmin = std::min(p->cfg.h_xi / p->cfg.nx, p->cfg.h_eta / p->cfg.ny);
    if (max_a_plus_c) *max_a_plus_c = p->tables.max_a_plus_c;
    if (ref_number) *ref_number = p->tables.max_abs_ac * (p->cfg.tau / p->cfg.nt) / (dmin * dmin);
    return PD_OK;
}

} // extern "C"
