// TEST HARNESS for the reference-side binding (integration/gaptooth_b200_binding.hpp):
// builds the BASELINE problems with the reference's own ProblemSpec API
// (oracle/ref_problems.hpp, test infrastructure) and the reference's own
// GapToothEngine, then runs either the reference's code (ours = 0) or the
// binding over the B200 C-ABI (ours = 1) through one extern "C" surface, so
// tests/test_gpu_binding.py can compare them bit for bit.
#include <cstring>
#include <memory>
#include <string>

#include "gaptooth_b200_binding.hpp"
#include "ref_problems.hpp"

using namespace patchdyn;

namespace {
thread_local std::string g_err;
struct H {
    refshim::Built built;
    std::unique_ptr<gaptooth::GapToothEngine> ref;
    std::unique_ptr<b200::DeviceGapTooth> dev;
};
int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}
gaptooth::CoarseField field(const H& h, const double* U) {
    gaptooth::CoarseField F = h.ref->initial_field();
    std::memcpy(F.U.data(), U, F.U.size() * sizeof(double));
    return F;
}
} // namespace

extern "C" {
const char* rbh_last_error() { return g_err.c_str(); }

int rbh_create(const pd_problem_desc* d, int mode, void** out) {
    try {
        auto h = std::make_unique<H>();
        h->built = refshim::build(*d);
        h->ref = std::make_unique<gaptooth::GapToothEngine>(h->built.spec, h->built.cfg);
        h->dev = std::make_unique<b200::DeviceGapTooth>(*h->ref, mode);
        *out = h.release();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void rbh_destroy(void* p) { delete static_cast<H*>(p); }

int rbh_mode(void* p) { return static_cast<H*>(p)->dev->mode(); }

int rbh_initial_field(void* p, double* U) {
    auto* h = static_cast<H*>(p);
    gaptooth::CoarseField F = h->ref->initial_field();
    h->ref->refresh_boundary(F, 0.0);
    std::memcpy(U, F.U.data(), F.U.size() * sizeof(double));
    return 0;
}

int rbh_step_direct(void* p, const double* Uin, double* Uout, double t, int ours) {
    try {
        auto* h = static_cast<H*>(p);
        const gaptooth::CoarseField F = field(*h, Uin);
        const gaptooth::CoarseField R = ours ? h->dev->step_direct(F, t) : h->ref->step_direct(F, t);
        std::memcpy(Uout, R.U.data(), R.U.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int rbh_projective_step(void* p, const double* Uin, double* Uout, double t, int ours) {
    try {
        auto* h = static_cast<H*>(p);
        const gaptooth::CoarseField F = field(*h, Uin);
        const gaptooth::CoarseField R = ours ? h->dev->projective_step(F, t) : cpi::projective_step(*h->ref, F, t);
        std::memcpy(Uout, R.U.data(), R.U.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int rbh_run(void* p, double* Ufinal, double* max_pct_err, int ours) {
    try {
        auto* h = static_cast<H*>(p);
        const cpi::RunResult r = ours ? h->dev->run() : cpi::run(*h->ref);
        std::memcpy(Ufinal, r.final_field.U.data(), r.final_field.U.size() * sizeof(double));
        *max_pct_err = r.max_pct_err;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
} // extern "C"
