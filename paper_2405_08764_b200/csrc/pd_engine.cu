// C-ABI implementation of the B200 gap-tooth engine (include/patchdyn_b200.h).
//
// Host orchestration only: validation (same error types as the reference),
// table upload, kernel selection and launch, device-resident macro loop.
// The kernels live in kernels_exact.cuh (reference-order EXACT mode),
// kernels_fast.cuh (register-blocked FAST mode) and kernels_misc.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "coeffgen.hpp"
#include "kernels_adi.cuh"
#include "kernels_adi_fast.cuh"
#include "kernels_exact.cuh"
#include "kernels_exact_tile.cuh"
#include "kernels_fast.cuh"
#include "kernels_fast_big.cuh"
#include "kernels_misc.cuh"
#include "patchdyn_b200.h"

using namespace pdb200::dev;

namespace pdb200 {
namespace {
thread_local std::string g_global_error;
}
void set_global_error(const std::string& m) { g_global_error = m; }
} // namespace pdb200

namespace {

struct Status {
    pd_status code;
    std::string msg;
};

#define CUDA_TRY(expr)                                                                           \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess)                                                                   \
            throw Status{PD_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)};     \
    } while (0)

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        if (count <= n && p) return;
        free();
        if (count == 0) return;
        CUDA_TRY(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { free(); }
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is per function and process-wide:
// engines of different sizes share it, so it only ever grows (an engine created
// later with a smaller need must not lower it under a live larger one).
std::mutex g_attr_mutex;
void raise_dyn_smem(const void* func, size_t bytes) {
    if (bytes <= 48 * 1024) return;
    std::lock_guard<std::mutex> lock(g_attr_mutex);
    cudaFuncAttributes a{};
    CUDA_TRY(cudaFuncGetAttributes(&a, func));
    if ((size_t)a.maxDynamicSharedSizeBytes >= bytes) return;
    CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

} // namespace

constexpr size_t kLinearBlockSmemMax = 220 * 1024; // dynamic shared memory of k_linear_run_block

struct pd_engine {
    pd_engine_desc d{};
    Params prm{};
    int mode = PD_MODE_EXACT;
    FastPlan fast{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::vector<int32_t> pij, nbr, cset;
    DevBuf<int32_t> d_pij, d_nbr, d_cset, d_kinds, d_fail, d_cset_items;
    DevBuf<double> d_coeffs, d_src, d_weights, d_U, d_chain, d_bnd, d_srct, d_tmp, d_tmp2, d_rw;
    DevBuf<double> d_roww;              // linear-response row weights [Neta+1][9]
    DevBuf<double> d_lag;               // Params::lagtab: lagq then lagp, [2][33][3]
    DevBuf<double> d_adi_fac;           // ADI static line factors [sets][2][L][L][kAdiFac] (k_adi_factor)
    DevBuf<double> d_adi_fast;          // FAST ADI folded tables (adi_fast_layout, k_adi_fast_fold)
    DevBuf<double> d_exact;             // pd_run_exact: exact-solution table [nsteps][NF] + errors [nsteps]
    double coeffgen_ms = 0.0;           // on-device table generation time at create (0: host tables)
    int step_kind = PD_STEP_DIRECT;     // what one gap-tooth step means (micro-solve or linear response)
    bool subset = false;                // the patch list covers only part of the interior
    int adi_carveout = -1;              // k_fast_adi<false> shared-memory carve-out (percent), -1: default
    double guard_scale = 0.0;           // > 0: blow-up scale of a segmented run (pd_engine_set_run_guard)
    int32_t step_offset = 0;            // macro steps before this segment, for the instability message
    // sampled path (time-dependent coefficients / general sources): device
    // tables [k+1][nt][sets][6][N] / [k+1][nt][sets][N] of the current call, and
    // the substep launch_step is running (set by the step drivers)
    DevBuf<double> d_samp;
    const double* samp_coef = nullptr;
    const double* samp_src = nullptr;
    int sub_m = 0;
    DevBuf<unsigned long long> d_slot, d_spread;
    DevBuf<unsigned int> d_counter;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::string err;
    int64_t launches = 0;
    size_t NF = 0, perim = 0;
    size_t device_bytes = 0;

    ~pd_engine() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }

    void check_launch() {
        ++launches;
        CUDA_TRY(cudaGetLastError());
    }

    // ---- one gap-tooth substep F -> out (patch nodes) -------------------
    void launch_step(const double* F, double* out, int out_mode, const double* srct, const int* fail) {
        const bool sampled = samp_coef || samp_src;
        if (prm.source == PD_SOURCE_GENERAL && !samp_src)
            throw Status{PD_UNSUPPORTED, "general (non-separable) source: use the sampled step entries "
                                         "(pd_gaptooth_step_sampled / pd_projective_step_sampled)"};
        if (sampled) { // per-micro-step tables: the EXACT family reads them from HBM each step
            if (step_kind == PD_STEP_LINEAR || prm.solver == PD_SOLVER_ADI)
                throw Status{PD_UNSUPPORTED, "sampled coefficient/source tables: explicit micro-solver, direct step only"};
            const size_t per_sub_c = (size_t)prm.nt * prm.nsets * PD_NCOEF * prm.N;
            const size_t per_sub_s = (size_t)prm.nt * prm.nsets * prm.N;
            k_gaptooth_exact<<<prm.P, exact_threads(prm), exact_smem_bytes(prm), stream>>>(
                prm, F, out, out_mode, d_pij.p, d_cset.p, d_coeffs.p, d_src.p, srct, fail, nullptr, nullptr,
                d_adi_fac.p, samp_coef ? samp_coef + per_sub_c * sub_m : nullptr,
                samp_src ? samp_src + per_sub_s * sub_m : nullptr);
            check_launch();
            return;
        }
        if (step_kind == PD_STEP_LINEAR) {
            k_linear_step<<<(prm.P + 127) / 128, 128, 0, stream>>>(prm, F, out, out_mode, d_pij.p, d_roww.p, fail);
        } else if (mode == PD_MODE_FAST && fast.adi) {
            auto* kern = adi_fast_staged(prm) ? k_fast_adi<true> : k_fast_adi<false>;
            if (adi_carveout >= 0) {
                std::lock_guard<std::mutex> lock(g_attr_mutex);
                CUDA_TRY(cudaFuncSetAttribute(k_fast_adi<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                              adi_carveout));
            }
            kern<<<(prm.P + kFastAdiWarps - 1) / kFastAdiWarps, 32 * kFastAdiWarps, fast_adi_smem_bytes(prm), stream>>>(
                prm, F, out, out_mode, d_nbr.p, d_cset.p, d_adi_fast.p, srct, fail);
        } else if (mode == PD_MODE_FAST && fast.big) {
            launch_big(fast, prm, F, out, out_mode, d_nbr.p, d_weights.p, fail, stream);
        } else if (mode == PD_MODE_FAST) {
            launch_fast(fast, prm, F, out, out_mode, d_nbr.p, d_weights.p, fail, stream, srct);
        } else if (const int tile = exact_tile_plan(prm); tile >= 0) {
            // register-blocked EXACT step (kernels_exact_tile.cuh): same arithmetic, bit-identical
            launch_exact_tile(tile, prm, F, out, out_mode, d_pij.p, d_cset.p, d_coeffs.p, fail, stream, d_src.p, srct);
        } else {
            k_gaptooth_exact<<<prm.P, exact_threads(prm), exact_smem_bytes(prm), stream>>>(
                prm, F, out, out_mode, d_pij.p, d_cset.p, d_coeffs.p, d_src.p, srct, fail, nullptr, nullptr,
                d_adi_fac.p);
        }
        check_launch();
    }
    void launch_refresh(double* out, const double* F, const double* bnd, const int* fail) {
        const int n = 2 * (prm.Nxi + 1) + 2 * (prm.Neta + 1);
        k_refresh<<<(n + 255) / 256, 256, 0, stream>>>(prm, out, F, bnd, fail);
        check_launch();
    }

    // gap-tooth step (step_direct, gaptooth.cpp:360-375)
    // A patch subset (one slab of a decomposed run) leaves other patch nodes
    // untouched by the kernels: copy them through so out = in outside the
    // subset (CoarseField out = F, gaptooth.cpp:361).
    void copy_through(const double* in, double* out) {
        if (subset && in != out) CUDA_TRY(cudaMemcpyAsync(out, in, NF * 8, cudaMemcpyDeviceToDevice, stream));
    }
    void gaptooth_step_dev(const double* in, double* out, const double* bnd, const double* srct, const int* fail) {
        copy_through(in, out);
        sub_m = 0;
        launch_step(in, out, OUT_FIELD, srct, fail);
        launch_refresh(out, in, bnd, fail);
    }

    // projective step (cpi.cpp:58-77).  bnd: [k+2][perim] or null; srct [k+1][nt] or null.
    void projective_dev(const double* in, double* out, const double* bnd, const double* srct, const int* fail) {
        const int k = prm.k;
        copy_through(in, out);
        if (k == 0) {
            sub_m = 0;
            launch_step(in, out, OUT_PROJECTIVE, srct, fail);
            launch_refresh(out, in, bnd ? bnd + perim : nullptr, fail);
            return;
        }
        d_chain.alloc(NF * (size_t)(k + 1));
        const double* prev = in;
        for (int m = 0; m <= k; ++m) {
            double* nxt = d_chain.p + NF * m;
            copy_through(prev, nxt);
            sub_m = m;
            launch_step(prev, nxt, OUT_FIELD, srct ? srct + (size_t)prm.nt * m : nullptr, fail);
            launch_refresh(nxt, prev, bnd ? bnd + perim * m : nullptr, fail);
            prev = nxt;
        }
        const double* Uk = k == 0 ? in : d_chain.p + NF * (k - 1);
        const double* Uk1 = d_chain.p + NF * k;
        const double horizon = XSUB_host(prm.dt_macro, k * prm.tau);
        k_extrapolate<<<(prm.P + 255) / 256, 256, 0, stream>>>(prm, out, Uk, Uk1, d_pij.p, horizon, fail);
        check_launch();
        launch_refresh(out, in, bnd ? bnd + perim * (k + 1) : nullptr, fail);
    }
    static double XSUB_host(double a, double b) { return a - b; }
};

namespace {

pd_status fail_engine(pd_engine* e, const Status& s) {
    if (e) e->err = s.msg;
    pdb200::set_global_error(s.msg);
    return s.code;
}

void validate_desc(const pd_engine_desc* d) {
    auto bad = [](const std::string& m) { throw Status{PD_VALIDATION_ERROR, m}; };
    if (!d) bad("null descriptor");
    if (d->Nxi < 2 || d->Neta < 2) bad("coarse grid needs at least 2 intervals per direction");
    if (d->nx < 2 || d->ny < 2) bad("micro grid needs nx, ny >= 2");
    if (d->nt < 1) bad("micro grid needs nt >= 1");
    if (!(d->h_xi > 0 && d->h_eta > 0 && d->tau > 0)) bad("micro grid needs positive h_xi, h_eta, tau");
    if (d->k < 0) bad("k must be non-negative");
    if (!(d->dt_macro > 0)) bad("macro step must be positive");
    if (!d->coeffs && !d->coeff_generator) bad("coefficient table missing");
    if (d->ncoeff_sets < 1) bad("no coefficient sets");
    if (d->quadrature == PD_QUAD_SIMPSON && (d->nx % 2 || d->ny % 2))
        throw Status{PD_VALIDATION_ERROR, "Simpson restriction needs an even micro resolution"};
    if (d->bc_type == PD_BC_ROBIN && d->robin_w1 == 0.0 && d->robin_w2 == 0.0)
        bad("robin patch conditions need nonzero weights");
    if (d->source_kind == PD_SOURCE_SEPARABLE && !d->source_spatial && !d->coeff_generator)
        bad("separable source needs a spatial table");
    if (d->solver != PD_SOLVER_EXPLICIT && d->solver != PD_SOLVER_ADI) bad("unknown micro-solver");
    if (d->upwind_order < PD_UPWIND_TWO || d->upwind_order > PD_UPWIND_FOUR) bad("upwind order must be two, three or four");
    // the reference sizes its banded line matrix once per ADI step for the xi
    // lines (microsim.cpp:400, 431-432) and reuses it for the eta lines: only
    // square micro grids are well defined with the wide upwind stencils
    if (d->solver == PD_SOLVER_ADI && d->upwind_order != PD_UPWIND_TWO && d->nx != d->ny)
        throw Status{PD_UNSUPPORTED, "ADI with three/four-point upwinding needs nx == ny (the reference's banded "
                                     "line matrix is sized for the xi lines only)"};
}

Params make_params(const pd_engine_desc& d, int P) {
    Params p{};
    p.a = d.a;
    p.b = d.b;
    p.c = d.c;
    p.d = d.d;
    p.Dxi = (d.b - d.a) / d.Nxi;
    p.Deta = (d.d - d.c) / d.Neta;
    p.Nxi = d.Nxi;
    p.Neta = d.Neta;
    p.NF2 = d.Neta + 1;
    p.periodic = d.periodic_xi ? 1 : 0;
    p.nx = d.nx;
    p.ny = d.ny;
    p.n1 = d.nx + 1;
    p.n2 = d.ny + 1;
    p.N = p.n1 * p.n2;
    p.L = std::max(p.n1, p.n2);
    p.nt = d.nt;
    p.k = d.k;
    p.tau = d.tau;
    p.dt_macro = d.dt_macro;
    p.h_xi = d.h_xi;
    p.h_eta = d.h_eta;
    p.mdxi = d.h_xi / d.nx;
    p.mdeta = d.h_eta / d.ny;
    p.mdt = d.tau / d.nt;
    p.bc_type = d.bc_type;
    p.w1 = d.robin_w1;
    p.w2 = d.robin_w2;
    p.quad = d.quadrature;
    p.P = P;
    p.nsets = d.ncoeff_sets;
    p.source = d.source_kind;
    // FAST-mode constants: degree-2 Lagrange basis on {-D,0,D} (gaptooth.cpp:17-29)
    p.i2Dxi = 1.0 / (2.0 * p.Dxi);
    p.i2Deta = 1.0 / (2.0 * p.Deta);
    p.iDxi2 = 1.0 / (p.Dxi * p.Dxi);
    p.iDeta2 = 1.0 / (p.Deta * p.Deta);
    p.i4DD = 1.0 / (4.0 * p.Dxi * p.Deta);
    p.c24x = d.h_xi * d.h_xi / 24.0;
    p.c24y = d.h_eta * d.h_eta / 24.0;
    auto lag = [](double X, double D, double* o) {
        o[0] = 0.5 * X * (X - D) / (D * D);
        o[1] = 1.0 - X * X / (D * D);
        o[2] = 0.5 * X * (X + D) / (D * D);
    };
    auto dlag = [](double X, double D, double* o) {
        o[0] = (X - 0.5 * D) / (D * D);
        o[1] = -2.0 * X / (D * D);
        o[2] = (X + 0.5 * D) / (D * D);
    };
    lag(0.5 * d.h_xi, p.Dxi, p.vlag[0]);
    lag(-0.5 * d.h_xi, p.Dxi, p.vlag[1]);
    lag(0.5 * d.h_eta, p.Deta, p.vlag[2]);
    lag(-0.5 * d.h_eta, p.Deta, p.vlag[3]);
    p.pinned = d.bc_type == PD_BC_DIRICHLET || (d.bc_type == PD_BC_ROBIN && std::fabs(d.robin_w2) < 1e-300);
    for (int e = 0; e < 4; ++e) {
        const double sign = (e == PD_EDGE_E || e == PD_EDGE_N) ? 1.0 : -1.0;
        const double delta = (e == PD_EDGE_E || e == PD_EDGE_W) ? p.mdxi : p.mdeta;
        p.cedge[e] = (d.bc_type == PD_BC_ROBIN && !p.pinned) ? -sign * 2.0 * delta * d.robin_w1 / d.robin_w2 : 0.0;
    }
    dlag(0.5 * d.h_xi, p.Dxi, p.dlag[0]);
    dlag(-0.5 * d.h_xi, p.Dxi, p.dlag[1]);
    dlag(0.5 * d.h_eta, p.Deta, p.dlag[2]);
    dlag(-0.5 * d.h_eta, p.Deta, p.dlag[3]);
    for (int j = 0; j < p.n2 && j < 33; ++j) lag(-0.5 * d.h_eta + p.mdeta * j, p.Deta, p.lagq[j]);
    for (int i = 0; i < p.n1 && i < 33; ++i) lag(-0.5 * d.h_xi + p.mdxi * i, p.Dxi, p.lagp[i]);
    p.gsc[PD_EDGE_E] = 2.0 * p.mdxi;
    p.gsc[PD_EDGE_W] = -2.0 * p.mdxi;
    p.gsc[PD_EDGE_N] = 2.0 * p.mdeta;
    p.gsc[PD_EDGE_S] = -2.0 * p.mdeta;
    p.solver = d.solver;
    p.upwind_order = d.upwind_order;
    p.upwind_r = d.upwind_r;
    return p;
}

template <class F>
pd_status guarded(pd_engine* e, F&& fn) {
    try {
        fn();
        return PD_OK;
    } catch (const Status& s) {
        return fail_engine(e, s);
    } catch (const pdb200::Error& x) { // host-side error types carry their status
        return fail_engine(e, Status{static_cast<pd_status>(x.status), x.what()});
    } catch (const std::exception& x) {
        return fail_engine(e, Status{PD_VALIDATION_ERROR, x.what()});
    }
}

void upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
}
void download(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
}

} // namespace

extern "C" {

int32_t pd_abi_version(void) { return PD_ABI_VERSION; }

const char* pd_status_name(int32_t s) {
    switch (s) {
        case PD_OK: return "ok";
        case PD_NON_POSITIVE_JACOBIAN: return "NonPositiveJacobian";
        case PD_DERIVATIVE_MISMATCH: return "DerivativeMismatch";
        case PD_MIXED_TERM_UNSUPPORTED: return "MixedTermUnsupported";
        case PD_STABILITY_VIOLATION: return "StabilityViolation";
        case PD_INSUFFICIENT_STENCIL: return "InsufficientStencil";
        case PD_INDEX_OUT_OF_RANGE: return "IndexOutOfRange";
        case PD_SHAPE_MISMATCH: return "ShapeMismatch";
        case PD_INVALID_STRETCH: return "InvalidStretch";
        case PD_DOMAIN_ERROR: return "DomainError";
        case PD_MACRO_INSTABILITY: return "MacroInstability";
        case PD_MACRO_PATCH_ERROR: return "MacroPatchError";
        case PD_VALIDATION_ERROR: return "ValidationError";
        case PD_CUDA_ERROR: return "CudaError";
        case PD_UNSUPPORTED: return "Unsupported";
        default: return "Unknown";
    }
}

const char* pd_last_error(const pd_engine* e) { return e ? e->err.c_str() : pdb200::g_global_error.c_str(); }

size_t pd_perimeter_len(int32_t Nxi, int32_t Neta) { return 2 * (size_t)(Nxi + 1) + 2 * (size_t)(Neta + 1); }

pd_status pd_engine_create(const pd_engine_desc* desc, pd_engine** out) {
    if (!out) return PD_VALIDATION_ERROR;
    *out = nullptr;
    auto e = std::make_unique<pd_engine>();
    const pd_status st = guarded(e.get(), [&] {
        validate_desc(desc);
        const pd_engine_desc& d = *desc;
        e->d = d;
        // bit-exact index tables (host/index_tables.cpp; gaptooth.cpp:74-104, 251-280)
        const int P = pd_patch_count(&d);
        if (P < 1) throw Status{PD_VALIDATION_ERROR, "empty patch table"};
        e->pij.resize(2 * (size_t)P);
        e->nbr.resize(9 * (size_t)P);
        {
            const pd_status ist = pd_build_index_tables(&d, e->pij.data(), e->nbr.data());
            if (ist != PD_OK) throw Status{ist, pd_last_error(nullptr)};
        }
        if (d.coeff_set) {
            e->cset.assign(d.coeff_set, d.coeff_set + P);
            for (int v : e->cset)
                if (v < 0 || v >= d.ncoeff_sets) throw Status{PD_SHAPE_MISMATCH, "coefficient set index out of range"};
        } else if (d.ncoeff_sets < P) {
            throw Status{PD_SHAPE_MISMATCH, "fewer coefficient sets than patches and no coeff_set map"};
        }
        e->prm = make_params(d, P);
        Params& p = e->prm;
        // mixed term present?  explicit stability guard (microsim.cpp:253-262)
        const size_t Ncoef = (size_t)d.ncoeff_sets * PD_NCOEF * p.N;
        double max_ac = 0.0;
        bool mixed = false;
        CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->own_stream = true;
        CUDA_TRY(cudaEventCreate(&e->ev0));
        CUDA_TRY(cudaEventCreate(&e->ev1));
        const bool generate = !d.coeffs && d.coeff_generator;
        if (generate) { // on-device mesh/metric generation (pd_coeffgen.cu)
            const std::vector<int32_t> centres = pdb200::coeffgen_set_centres(d, e->pij.data(), P);
            e->d_coeffs.alloc(Ncoef);
            if (d.source_kind == PD_SOURCE_SEPARABLE) e->d_src.alloc((size_t)d.ncoeff_sets * p.N);
            const pdb200::CoeffGenStats gs =
                pdb200::coeffgen_run(*d.coeff_generator, d, centres.data(), e->d_coeffs.p, e->d_src.p, e->stream);
            max_ac = gs.max_abs_ac;
            mixed = gs.max_abs_b > 0.0;
            e->coeffgen_ms = gs.device_ms;
        } else {
            for (int s = 0; s < d.ncoeff_sets; ++s) {
                const double* c = d.coeffs + (size_t)s * PD_NCOEF * p.N;
                for (int k = 0; k < p.N; ++k) {
                    max_ac = std::max({max_ac, std::fabs(c[PD_COEF_A * p.N + k]), std::fabs(c[PD_COEF_C * p.N + k])});
                    if (c[PD_COEF_B * p.N + k] != 0.0) mixed = true;
                }
            }
        }
        e->d.coeffs = nullptr; // host tables are not referenced after create
        e->d.source_spatial = nullptr;
        e->d.coeff_generator = nullptr;
        p.mixed = mixed ? 1 : 0;
        if (mixed && d.solver == PD_SOLVER_ADI)
            throw Status{PD_MIXED_TERM_UNSUPPORTED, "mixed-derivative term with the ADI micro-solver is not defined"};
        if (mixed && d.bc_type == PD_BC_ROBIN)
            throw Status{PD_MIXED_TERM_UNSUPPORTED, "mixed-derivative term with Robin patch conditions is not defined"};
        const double dmin = std::min(p.mdxi, p.mdeta);
        const double number = max_ac * p.mdt / (dmin * dmin);
        if (d.solver == PD_SOLVER_EXPLICIT && number > 0.5 + 1e-12) { // the guard is the explicit scheme's
            std::ostringstream m;
            m << "explicit micro scheme diffusive stability number " << number << " exceeds 0.5";
            throw Status{PD_STABILITY_VIOLATION, m.str()};
        }
        e->NF = (size_t)(d.Nxi + 1) * (d.Neta + 1);
        e->subset = P < (d.Nxi - (d.periodic_xi ? 0 : 1)) * (d.Neta - 1);
        e->perim = pd_perimeter_len(d.Nxi, d.Neta);
        // device
        e->d_pij.alloc(e->pij.size());
        e->d_nbr.alloc(e->nbr.size());
        upload(e->d_pij.p, e->pij.data(), e->pij.size() * 4, e->stream);
        upload(e->d_nbr.p, e->nbr.data(), e->nbr.size() * 4, e->stream);
        if (!e->cset.empty()) {
            e->d_cset.alloc(e->cset.size());
            upload(e->d_cset.p, e->cset.data(), e->cset.size() * 4, e->stream);
        }
        if (!generate) {
            e->d_coeffs.alloc(Ncoef);
            upload(e->d_coeffs.p, d.coeffs, Ncoef * 8, e->stream);
            if (d.source_kind == PD_SOURCE_SEPARABLE) {
                e->d_src.alloc((size_t)d.ncoeff_sets * p.N);
                upload(e->d_src.p, d.source_spatial, (size_t)d.ncoeff_sets * p.N * 8, e->stream);
            }
        }
        e->d_lag.alloc(2 * 33 * 3);
        upload(e->d_lag.p, &p.lagq[0][0], 33 * 3 * 8, e->stream);
        upload(e->d_lag.p + 99, &p.lagp[0][0], 33 * 3 * 8, e->stream);
        p.lagtab = e->d_lag.p;
        e->d_U.alloc(2 * e->NF);
        e->d_fail.alloc(4);
        e->device_bytes = Ncoef * 8 + e->pij.size() * 4 + e->nbr.size() * 4 + 2 * e->NF * 8;
        // ADI: the line matrices are static; factor them once (bit-identical replay)
        static const bool adi_cache = [] {
            const char* v = std::getenv("PD_ADI_FACTOR_CACHE");
            return !(v && v[0] == '0');
        }();
        if (d.solver == PD_SOLVER_ADI && adi_cache) {
            const size_t nf = (size_t)d.ncoeff_sets * adi_factor_doubles(p);
            e->d_adi_fac.alloc(nf);
            CUDA_TRY(cudaMemsetAsync(e->d_adi_fac.p, 0, nf * 8, e->stream));
            const int threads = 128, total = d.ncoeff_sets * 2 * p.L;
            k_adi_factor<<<(total + threads - 1) / threads, threads, 0, e->stream>>>(p, e->d_coeffs.p, d.ncoeff_sets,
                                                                                       e->d_adi_fac.p);
            e->check_launch();
            e->device_bytes += nf * 8;
        }
        // kernel family
        e->mode = PD_MODE_EXACT;
        raise_dyn_smem((const void*)k_gaptooth_exact, exact_smem_bytes(p));
        raise_dyn_smem((const void*)k_integrate_exact, exact_smem_bytes(p));
        // FAST ADI (kernels_adi_fast.cuh) up to 32 nodes per side: with the compact per-node
        // tables it measured 1.5-2.3x faster than the EXACT ADI kernel at 11^2 and 3.0x at 21^2
        // (profiles/r01_adi.jsonl); larger patches stay on EXACT (bit-identical)
        if (d.mode == PD_MODE_FAST && d.solver == PD_SOLVER_ADI && p.L <= 32) {
            const size_t nf = (size_t)d.ncoeff_sets * adi_fast_doubles(p);
            e->d_adi_fast.alloc(nf);
            CUDA_TRY(cudaMemsetAsync(e->d_adi_fast.p, 0, nf * 8, e->stream));
            const int threads = 64, total = d.ncoeff_sets * 2 * p.L;
            k_adi_fast_fold<<<(total + threads - 1) / threads, threads, 0, e->stream>>>(p, e->d_coeffs.p, e->d_src.p,
                                                                                         d.ncoeff_sets, e->d_adi_fast.p);
            e->check_launch();
            raise_dyn_smem(adi_fast_staged(p) ? (const void*)k_fast_adi<true> : (const void*)k_fast_adi<false>,
                           fast_adi_smem_bytes(p));
            if (!adi_fast_staged(p)) {
                // the unstaged kernel reads its tables through L1: carve out only the shared
                // memory of the blocks that can be resident (at most four: its register
                // limit) and leave the rest to L1 (21^2: 1.53 -> 1.27 ms per macro step)
                const size_t per_block = fast_adi_smem_bytes(p) + 1024, smem_max = 233472;
                const size_t blocks = std::max<size_t>(1, std::min<size_t>(4, smem_max / per_block));
                // (the carve-out is a process-wide function attribute too: each engine
                // applies its own value right before its launches, launch_step)
                e->adi_carveout = (int)std::min<size_t>(100, (blocks * per_block * 100 + smem_max - 1) / smem_max);
            }
            e->device_bytes += nf * 8;
            e->fast.adi = 1;
            e->mode = PD_MODE_FAST;
        }
        if (d.mode == PD_MODE_FAST && d.solver == PD_SOLVER_EXPLICIT) { // the plans decide on sources
            if (plan_big(p, e->fast)) {
                const size_t wcount = fast_weights_count(e->fast, p);
                e->d_weights.alloc(wcount);
                fold_big(e->fast, p, e->d_coeffs.p, e->d_cset.p, e->d_weights.p, e->stream);
                e->check_launch();
                e->device_bytes += wcount * 8;
                e->mode = PD_MODE_FAST;
            } else if (plan_fast(p, e->fast)) {
                const size_t wcount = fast_weights_count(e->fast, p);
                e->d_weights.alloc(wcount);
                fold_weights(e->fast, p, e->d_coeffs.p, e->d_cset.p, e->d_weights.p, e->stream, e->d_src.p);
                e->check_launch();
                e->device_bytes += wcount * 8;
                e->mode = PD_MODE_FAST;
            }
        }
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
    if (st != PD_OK) return st;
    *out = e.release();
    return PD_OK;
}

void pd_engine_destroy(pd_engine* e) { delete e; }

int32_t pd_engine_mode(const pd_engine* e) { return e ? e->mode : -1; }
int32_t pd_engine_exact_tile(const pd_engine* e) { return e ? (exact_tile_plan(e->prm) >= 0 ? 1 : 0) : -1; }
int32_t pd_engine_mixed(const pd_engine* e) { return e ? e->prm.mixed : -1; }
int64_t pd_engine_launch_count(const pd_engine* e) { return e ? e->launches : -1; }

pd_status pd_engine_tables(const pd_engine* e, int32_t* patch_ij, int32_t* neighbours) {
    if (!e) return PD_VALIDATION_ERROR;
    if (patch_ij) std::memcpy(patch_ij, e->pij.data(), e->pij.size() * 4);
    if (neighbours) std::memcpy(neighbours, e->nbr.data(), e->nbr.size() * 4);
    return PD_OK;
}

size_t pd_engine_device_bytes(const pd_engine* e) { return e ? e->device_bytes : 0; }

pd_status pd_engine_set_stream(pd_engine* e, void* s) {
    if (!e) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        if (e->own_stream && e->stream) CUDA_TRY(cudaStreamDestroy(e->stream));
        if (s) {
            e->stream = static_cast<cudaStream_t>(s);
            e->own_stream = false;
        } else {
            CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
            e->own_stream = true;
        }
    });
}

pd_status pd_gaptooth_step(pd_engine* e, const double* U_in, double* U_out, double t, const double* bnd,
                           const double* src_time) {
    if (!e || !U_in || !U_out) return PD_VALIDATION_ERROR;
    (void)t;
    return guarded(e, [&] {
        const size_t NF = e->NF;
        upload(e->d_U.p, U_in, NF * 8, e->stream);
        const double* dbnd = nullptr;
        if (bnd) {
            e->d_bnd.alloc(e->perim);
            upload(e->d_bnd.p, bnd, e->perim * 8, e->stream);
            dbnd = e->d_bnd.p;
        }
        const double* dsrc = nullptr;
        if (src_time && e->prm.source) {
            e->d_srct.alloc(e->prm.nt);
            upload(e->d_srct.p, src_time, e->prm.nt * 8, e->stream);
            dsrc = e->d_srct.p;
        }
        CUDA_TRY(cudaMemsetAsync(e->d_fail.p, 0, 8, e->stream));
        e->gaptooth_step_dev(e->d_U.p, e->d_U.p + NF, dbnd, dsrc, nullptr);
        download(U_out, e->d_U.p + NF, NF * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}

namespace {
// gap-tooth (substeps = 1) or projective (substeps = k+1) step over per-micro-step
// sampled tables (microsim.cpp:537-542, 278-280), host buffers
pd_status sampled_step(pd_engine* e, const double* U_in, double* U_out, const double* bnd,
                       const double* coeff_steps, const double* source_steps, bool projective) {
    if (!e || !U_in || !U_out || (!coeff_steps && !source_steps)) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        struct Reset {
            pd_engine* e;
            ~Reset() { e->samp_coef = e->samp_src = nullptr; }
        } reset{e};
        const size_t NF = e->NF;
        const size_t subs = projective ? (size_t)e->prm.k + 1 : 1;
        const size_t nc = coeff_steps ? subs * e->prm.nt * e->prm.nsets * PD_NCOEF * e->prm.N : 0;
        const size_t ns = source_steps ? subs * e->prm.nt * e->prm.nsets * e->prm.N : 0;
        e->d_samp.alloc(nc + ns);
        if (nc) upload(e->d_samp.p, coeff_steps, nc * 8, e->stream);
        if (ns) upload(e->d_samp.p + nc, source_steps, ns * 8, e->stream);
        e->samp_coef = nc ? e->d_samp.p : nullptr;
        e->samp_src = ns ? e->d_samp.p + nc : nullptr;
        upload(e->d_U.p, U_in, NF * 8, e->stream);
        const double* dbnd = nullptr;
        if (bnd) {
            const size_t n = e->perim * (projective ? (size_t)e->prm.k + 2 : 1);
            e->d_bnd.alloc(n);
            upload(e->d_bnd.p, bnd, n * 8, e->stream);
            dbnd = e->d_bnd.p;
        }
        CUDA_TRY(cudaMemsetAsync(e->d_fail.p, 0, 8, e->stream));
        if (projective)
            e->projective_dev(e->d_U.p, e->d_U.p + NF, dbnd, nullptr, nullptr);
        else
            e->gaptooth_step_dev(e->d_U.p, e->d_U.p + NF, dbnd, nullptr, nullptr);
        download(U_out, e->d_U.p + NF, NF * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}
} // namespace

pd_status pd_gaptooth_step_sampled(pd_engine* e, const double* U_in, double* U_out, double t, const double* bnd,
                                   const double* coeff_steps, const double* source_steps) {
    (void)t;
    return sampled_step(e, U_in, U_out, bnd, coeff_steps, source_steps, false);
}

pd_status pd_projective_step_sampled(pd_engine* e, const double* U_in, double* U_out, double t, const double* bnd,
                                     const double* coeff_steps, const double* source_steps) {
    (void)t;
    return sampled_step(e, U_in, U_out, bnd, coeff_steps, source_steps, true);
}

pd_status pd_projective_step_device(pd_engine* e, const double* in, double* out, double t, const double* bnd,
                                    const double* src_time) {
    if (!e || !in || !out) return PD_VALIDATION_ERROR;
    (void)t;
    return guarded(e, [&] { e->projective_dev(in, out, bnd, e->prm.source ? src_time : nullptr, nullptr); });
}

pd_status pd_projective_step(pd_engine* e, const double* U_in, double* U_out, double t, const double* bnd,
                             const double* src_time) {
    if (!e || !U_in || !U_out) return PD_VALIDATION_ERROR;
    (void)t;
    return guarded(e, [&] {
        const size_t NF = e->NF;
        upload(e->d_U.p, U_in, NF * 8, e->stream);
        const double* dbnd = nullptr;
        if (bnd) {
            e->d_bnd.alloc(e->perim * (e->prm.k + 2));
            upload(e->d_bnd.p, bnd, e->perim * (e->prm.k + 2) * 8, e->stream);
            dbnd = e->d_bnd.p;
        }
        const double* dsrc = nullptr;
        if (src_time && e->prm.source) {
            e->d_srct.alloc((size_t)e->prm.nt * (e->prm.k + 1));
            upload(e->d_srct.p, src_time, (size_t)e->prm.nt * (e->prm.k + 1) * 8, e->stream);
            dsrc = e->d_srct.p;
        }
        e->projective_dev(e->d_U.p, e->d_U.p + NF, dbnd, dsrc, nullptr);
        download(U_out, e->d_U.p + NF, NF * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}

namespace {
// exact/err (device, optional): the per-step exact-error metric after every
// step — inside the single-launch run (k_fast_run) when that runs, else one
// k_exact_err launch per step; no host round trip either way
pd_status run_device_impl(pd_engine* e, double* U, double* scratch, int32_t nsteps, double t0, const double* bnd,
                          const double* src_time, const double* exact, double* err, pd_run_stats* stats) {
    if (!e || !U || !scratch || nsteps < 0 || (exact != nullptr) != (err != nullptr)) return PD_VALIDATION_ERROR;
    (void)t0;
    pd_status result = PD_OK;
    const pd_status st = guarded(e, [&] {
        const size_t NF = e->NF;
        // blow-up threshold from the initial field  cpi.cpp:142-144
        e->d_slot.alloc((size_t)nsteps + 1);
        e->d_counter.alloc((size_t)nsteps + 1);
        CUDA_TRY(cudaMemsetAsync(e->d_slot.p, 0, ((size_t)nsteps + 1) * 8, e->stream));
        CUDA_TRY(cudaMemsetAsync(e->d_counter.p, 0, ((size_t)nsteps + 1) * 4, e->stream));
        CUDA_TRY(cudaMemsetAsync(e->d_fail.p, 0, 16, e->stream));
        const int gblocks = (int)std::min<size_t>(1184, (NF + 255) / 256);
        double scale0 = e->guard_scale;
        if (!(scale0 > 0.0)) {
            // initial scale: flags go to the scratch pair d_fail[2..3], never to the run's flag
            k_guard<<<gblocks, 256, 0, e->stream>>>(U, NF, e->d_slot.p + nsteps, e->d_counter.p + nsteps,
                                                    e->d_fail.p + 2, e->d_fail.p + 3, 0, INFINITY);
            e->check_launch();
            unsigned long long s0 = 0;
            download(&s0, e->d_slot.p + nsteps, 8, e->stream);
            CUDA_TRY(cudaStreamSynchronize(e->stream));
            std::memcpy(&scale0, &s0, 8);
        }
        const double blowup = 10.0 * std::max(scale0, 1e-12);
        const size_t pk = e->perim * (e->prm.k + 2);
        const size_t sk = (size_t)e->prm.nt * (e->prm.k + 1);
        const int64_t l0 = e->launches;
        // linear-response steps on a field that fits in shared memory: the whole
        // loop is one single-CTA kernel (k_linear_run_block), same results
        // fields (2 or 3) + the row weights [Neta+1][9] staged next to them
        const size_t block_smem = ((e->prm.k == 0 ? 2 : 3) * NF + (size_t)(e->prm.Neta + 1) * 9) * 8;
        const bool block_run =
            !exact && e->step_kind == PD_STEP_LINEAR && nsteps > 0 && block_smem <= kLinearBlockSmemMax;
        // direct FAST steps (k = 0, full field): the whole run is one cooperative
        // launch (k_fast_run) when the plan's kernel can be made co-resident
        static const bool fused_enabled = [] {
            const char* v = std::getenv("PD_FUSED_RUN");
            return !(v && v[0] == '0');
        }();
        const bool fused_ok = !block_run && fused_enabled && nsteps > 0 && e->step_kind == PD_STEP_DIRECT &&
                              e->mode == PD_MODE_FAST && !e->fast.big && !e->fast.adi && e->prm.k == 0 && !e->subset;
        if (fused_ok) {
            e->d_spread.alloc((size_t)nsteps * kGuardSpread);
            CUDA_TRY(cudaMemsetAsync(e->d_spread.p, 0, (size_t)nsteps * kGuardSpread * 8, e->stream));
        }
        if (exact && nsteps > 0) CUDA_TRY(cudaMemsetAsync(err, 0, (size_t)nsteps * 8, e->stream));
        bool fused = false;
        CUDA_TRY(cudaEventRecord(e->ev0, e->stream));
        if (fused_ok) {
            fused = launch_fast_run(e->fast, e->prm, U, scratch, e->d_nbr.p, e->d_weights.p,
                                    bnd ? bnd + e->perim : nullptr, pk, (src_time && e->prm.source) ? src_time : nullptr,
                                    sk, nsteps, blowup, e->d_slot.p, e->d_spread.p, e->d_fail.p, e->stream, exact, err);
            if (fused) e->check_launch();
        }
        if (fused) {
        } else if (block_run) {
            raise_dyn_smem((const void*)k_linear_run_block, block_smem);
            // one thread per patch up to 1024 (every warp executes the per-step
            // reductions: idle warps would only cost issue slots on the one SM)
            const int nperim = 2 * (e->prm.Nxi + 1) + 2 * (e->prm.Neta + 1);
            const int lin_threads = std::min(1024, std::max(64, (std::max((int)e->prm.P, nperim) + 31) / 32 * 32));
            k_linear_run_block<<<1, lin_threads, block_smem, e->stream>>>(e->prm, U, e->d_pij.p, e->d_roww.p, bnd, e->perim,
                                                                    nsteps, blowup, e->d_slot.p, e->d_fail.p,
                                                                    e->subset ? 0 : 1);
            e->check_launch();
        } else {
            double* cur = U;
            double* nxt = scratch;
            // k = 0 on a full field: the boundary refresh and the guard share one launch
            // (k_refresh_guard; PD_FUSED_GUARD=0 keeps k_refresh + k_guard, for A/B runs)
            static const bool fuse_guard = [] {
                const char* v = std::getenv("PD_FUSED_GUARD");
                return !(v && v[0] == '0');
            }();
            const bool rg = fuse_guard && e->prm.k == 0 && !e->subset && !e->samp_coef && !e->samp_src;
            for (int n = 0; n < nsteps; ++n) {
                const double* bn = bnd ? bnd + pk * n : nullptr;
                const double* sn = (src_time && e->prm.source) ? src_time + sk * n : nullptr;
                if (rg) {
                    e->sub_m = 0;
                    e->launch_step(cur, nxt, OUT_PROJECTIVE, sn, e->d_fail.p);
                    k_refresh_guard<<<gblocks, 256, 0, e->stream>>>(e->prm, nxt, cur, bn ? bn + e->perim : nullptr,
                                                                    e->d_slot.p, e->d_counter.p, e->d_fail.p,
                                                                    e->d_fail.p + 1, n, blowup);
                } else {
                    e->projective_dev(cur, nxt, bn, sn, e->d_fail.p);
                    k_guard<<<gblocks, 256, 0, e->stream>>>(nxt, NF, e->d_slot.p, e->d_counter.p, e->d_fail.p,
                                                            e->d_fail.p + 1, n, blowup);
                }
                e->check_launch();
                if (exact) {
                    k_exact_err<<<gblocks, 256, 0, e->stream>>>(e->prm, nxt, exact + NF * n,
                                                                reinterpret_cast<unsigned long long*>(err),
                                                                e->d_fail.p, n);
                    e->check_launch();
                }
                std::swap(cur, nxt);
            }
        }
        CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
        int fail[2] = {0, 0};
        download(fail, e->d_fail.p, 8, e->stream);
        std::vector<unsigned long long> slots(nsteps > 0 ? nsteps : 1);
        if (nsteps > 0) download(slots.data(), e->d_slot.p, 8 * (size_t)nsteps, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
        // the field after the last executed step lives in buffer (done % 2 == 1 ? scratch : U)
        const int done = fail[0] ? fail[0] : nsteps;
        // the single-launch run measures a step before its (one step late) guard
        // decision: no error for the failing step or after it, as cpi::run
        if (exact && fail[0] && fail[0] <= nsteps)
            CUDA_TRY(cudaMemsetAsync(err + (fail[0] - 1), 0, (size_t)(nsteps - fail[0] + 1) * 8, e->stream));
        if (!block_run && done % 2 == 1)
            CUDA_TRY(cudaMemcpyAsync(U, scratch, NF * 8, cudaMemcpyDeviceToDevice, e->stream));
        CUDA_TRY(cudaStreamSynchronize(e->stream));
        pd_run_stats s{};
        s.steps_done = fail[0] ? fail[0] - 1 : nsteps;
        s.failed_step = fail[0];
        s.failed_nonfinite = fail[1];
        s.blowup_threshold = blowup;
        s.device_ms = ms;
        s.kernel_launches = e->launches - l0;
        if (done > 0) {
            double um;
            std::memcpy(&um, &slots[done - 1], 8);
            s.umax_last = um;
        }
        if (stats) *stats = s;
        if (fail[0]) {
            std::ostringstream m;
            m << "coarse field " << (fail[1] ? "became non-finite" : "exceeded 10x the initial magnitude")
              << " at macro step " << fail[0] + e->step_offset << " (t=" << (fail[0] + e->step_offset) * e->prm.dt_macro
              << "); the projective step size is likely beyond the stable range";
            e->err = m.str();
            result = PD_MACRO_INSTABILITY;
        }
    });
    return st != PD_OK ? st : result;
}
} // namespace

pd_status pd_run_device(pd_engine* e, double* U, double* scratch, int32_t nsteps, double t0, const double* bnd,
                        const double* src_time, pd_run_stats* stats) {
    return run_device_impl(e, U, scratch, nsteps, t0, bnd, src_time, nullptr, nullptr, stats);
}

pd_status pd_run_device_exact(pd_engine* e, double* U, double* scratch, int32_t nsteps, double t0,
                              const double* bnd, const double* src_time, const double* exact, double* err,
                              pd_run_stats* stats) {
    if (!exact || !err) return PD_VALIDATION_ERROR;
    return run_device_impl(e, U, scratch, nsteps, t0, bnd, src_time, exact, err, stats);
}

pd_status pd_run(pd_engine* e, double* U_host, int32_t nsteps, double t0, const double* bnd, const double* src_time,
                 pd_run_stats* stats) {
    return pd_run_exact(e, U_host, nsteps, t0, bnd, src_time, nullptr, nullptr, stats);
}

pd_status pd_run_exact(pd_engine* e, double* U_host, int32_t nsteps, double t0, const double* bnd,
                       const double* src_time, const double* exact, double* err_out, pd_run_stats* stats) {
    if (!e || !U_host || nsteps < 0 || (exact != nullptr) != (err_out != nullptr)) return PD_VALIDATION_ERROR;
    pd_status result = PD_OK;
    const pd_status st = guarded(e, [&] {
        const size_t NF = e->NF;
        upload(e->d_U.p, U_host, NF * 8, e->stream);
        const double* dbnd = nullptr;
        if (bnd) {
            const size_t n = e->perim * (e->prm.k + 2) * (size_t)nsteps;
            e->d_bnd.alloc(n);
            upload(e->d_bnd.p, bnd, n * 8, e->stream);
            dbnd = e->d_bnd.p;
        }
        const double* dsrc = nullptr;
        if (src_time && e->prm.source) {
            const size_t n = (size_t)e->prm.nt * (e->prm.k + 1) * nsteps;
            e->d_srct.alloc(n);
            upload(e->d_srct.p, src_time, n * 8, e->stream);
            dsrc = e->d_srct.p;
        }
        double* dex = nullptr;
        double* derr = nullptr;
        if (exact && nsteps > 0) {
            e->d_exact.alloc(NF * (size_t)nsteps + (size_t)nsteps);
            dex = e->d_exact.p;
            derr = dex + NF * (size_t)nsteps;
            upload(dex, exact, NF * (size_t)nsteps * 8, e->stream);
        }
        result = run_device_impl(e, e->d_U.p, e->d_U.p + NF, nsteps, t0, dbnd, dsrc, dex, derr, stats);
        if (result != PD_OK && result != PD_MACRO_INSTABILITY) throw Status{result, e->err};
        download(U_host, e->d_U.p, NF * 8, e->stream);
        if (derr) download(err_out, derr, (size_t)nsteps * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
    return st != PD_OK ? st : result;
}

pd_status pd_integrate_batch(pd_engine* e, const double* u0, const int32_t* edge_kind, const double* ev,
                             const double* es, const double* robin_w, double t0, const double* src_time, double* uT) {
    if (!e || !u0 || !edge_kind || !uT) return PD_VALIDATION_ERROR;
    (void)t0;
    return guarded(e, [&] {
        const Params& p = e->prm;
        for (int k = 0; k < 4; ++k)
            if (edge_kind[k] < 0 || edge_kind[k] > 2) throw Status{PD_VALIDATION_ERROR, "bad edge kind"};
        if (p.mixed)
            for (int k = 0; k < 4; ++k)
                if (edge_kind[k] == PD_EDGE_ROBIN)
                    throw Status{PD_MIXED_TERM_UNSUPPORTED, "mixed-derivative term with Robin edges is not defined"};
        const size_t nu = (size_t)p.P * p.N, ne = (size_t)p.P * 4 * p.L;
        e->d_tmp.alloc(2 * nu + 2 * ne);
        double* du0 = e->d_tmp.p;
        double* duT = du0 + nu;
        double* dev_ = duT + nu;
        double* des = dev_ + ne;
        upload(du0, u0, nu * 8, e->stream);
        std::vector<double> zeros;
        if (!ev || !es) zeros.assign(ne, 0.0);
        upload(dev_, ev ? ev : zeros.data(), ne * 8, e->stream);
        upload(des, es ? es : zeros.data(), ne * 8, e->stream);
        e->d_kinds.alloc(4);
        upload(e->d_kinds.p, edge_kind, 16, e->stream);
        double rw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (robin_w) std::memcpy(rw, robin_w, sizeof rw);
        e->d_rw.alloc(8);
        upload(e->d_rw.p, rw, 64, e->stream);
        const double* dsrc = nullptr;
        if (src_time && p.source) {
            e->d_srct.alloc(p.nt);
            upload(e->d_srct.p, src_time, (size_t)p.nt * 8, e->stream);
            dsrc = e->d_srct.p;
        }
        k_integrate_exact<<<p.P, exact_threads(p), exact_smem_bytes(p), e->stream>>>(
            p, du0, dev_, des, e->d_kinds.p, e->d_rw.p, e->d_cset.p, e->d_coeffs.p, e->d_src.p, dsrc, duT);
        e->check_launch();
        download(uT, duT, nu * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}

pd_status pd_lift_batch(pd_engine* e, int32_t n, const double* vals, const double* centers, double* u0, double* es,
                        double* ev) {
    if (!e || n < 1 || !vals || !centers) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        const Params& p = e->prm;
        const size_t nu = (size_t)n * p.N, ne = (size_t)n * 4 * p.L;
        e->d_tmp2.alloc(9 * (size_t)n + 2 * (size_t)n + nu + 2 * ne);
        double* dv = e->d_tmp2.p;
        double* dc = dv + 9 * (size_t)n;
        double* du = dc + 2 * (size_t)n;
        double* ds = du + nu;
        double* dval = ds + ne;
        CUDA_TRY(cudaMemsetAsync(ds, 0, 2 * ne * 8, e->stream));
        upload(dv, vals, 9 * (size_t)n * 8, e->stream);
        upload(dc, centers, 2 * (size_t)n * 8, e->stream);
        k_lift_exact<<<n, kExactThreads, 0, e->stream>>>(p, dv, dc, du, ds, dval);
        e->check_launch();
        if (u0) download(u0, du, nu * 8, e->stream);
        if (es) download(es, ds, ne * 8, e->stream);
        if (ev) download(ev, dval, ne * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}

pd_status pd_restrict_batch(pd_engine* e, int32_t n, const double* u, double* avg) {
    if (!e || n < 1 || !u || !avg) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        const Params& p = e->prm;
        const size_t nu = (size_t)n * p.N;
        e->d_tmp2.alloc(nu + n);
        upload(e->d_tmp2.p, u, nu * 8, e->stream);
        k_restrict_exact<<<n, kExactThreads, p.n1 * 8, e->stream>>>(p, e->d_tmp2.p, e->d_tmp2.p + nu);
        e->check_launch();
        download(avg, e->d_tmp2.p + nu, (size_t)n * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}

// ---- linear-response path (GapToothEngine::step, gaptooth.cpp:377-418) ------
pd_status pd_evolve_batch(pd_engine* e, int32_t n, const int32_t* patch_index, const double* stencils,
                          double t, double* out) {
    if (!e || n < 1 || !patch_index || !stencils || !out) return PD_VALIDATION_ERROR;
    for (int32_t m = 0; m < n; ++m)
        if (patch_index[m] < 0 || patch_index[m] >= e->prm.P) {
            e->err = "pd_evolve_batch: patch index " + std::to_string(patch_index[m]) + " outside [0," +
                     std::to_string(e->prm.P) + ")";
            return PD_INDEX_OUT_OF_RANGE;
        }
    if (e->d.source_kind != PD_SOURCE_ZERO) {
        e->err = "pd_evolve_batch: needs a zero source";
        return PD_UNSUPPORTED;
    }
    (void)t; // zero source: evolve_patch does not depend on t
    return guarded(e, [&] {
        const Params& p = e->prm;
        e->d_tmp2.alloc((size_t)10 * n);
        e->d_cset_items.alloc((size_t)n);
        upload(e->d_tmp2.p, stencils, (size_t)9 * n * 8, e->stream);
        upload(e->d_cset_items.p, patch_index, (size_t)n * 4, e->stream);
        double* res = e->d_tmp2.p + (size_t)9 * n;
        k_gaptooth_exact<<<n, kExactThreads, exact_smem_bytes(p), e->stream>>>(
            p, nullptr, res, OUT_PATCH, e->d_pij.p, e->d_cset.p, e->d_coeffs.p, nullptr, nullptr, nullptr,
            e->d_tmp2.p, e->d_cset_items.p, e->d_adi_fac.p);
        e->check_launch();
        download(out, res, (size_t)n * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}

pd_status pd_linear_weights(pd_engine* e, double* row_w) {
    if (!e || !row_w) return PD_VALIDATION_ERROR;
    const pd_engine_desc& d = e->d;
    const int Neta = d.Neta, i0 = d.periodic_xi ? 0 : 1;
    // eligibility as GapToothEngine's ctor (gaptooth.cpp:213-224): time-independent
    // coefficients (always, tables), zero source, one coefficient set per eta-row
    std::vector<int32_t> rowp(Neta + 1, -1), rowset(Neta + 1, -1);
    bool xi_indep = true;
    for (int32_t q = 0; q < e->prm.P; ++q) {
        const int i = e->pij[2 * q], j = e->pij[2 * q + 1];
        const int set = e->cset.empty() ? q : e->cset[q];
        if (rowset[j] < 0) rowset[j] = set;
        else if (rowset[j] != set) xi_indep = false;
        if (i == i0 && rowp[j] < 0) rowp[j] = q;
    }
    if (d.source_kind != PD_SOURCE_ZERO || !xi_indep) {
        e->err = "linear_cache=on requires time-independent coefficients, a zero source and "
                 "xi-independent coefficients";
        return PD_VALIDATION_ERROR;
    }
    std::vector<int32_t> items;
    std::vector<double> st;
    for (int j = 1; j <= Neta - 1; ++j) {
        if (rowp[j] < 0) {
            e->err = "pd_linear_weights: row " + std::to_string(j) + " has no patch at i = " + std::to_string(i0);
            return PD_VALIDATION_ERROR;
        }
        for (int k = 0; k < 9; ++k) {
            items.push_back(rowp[j]);
            for (int q = 0; q < 9; ++q) st.push_back(q == k ? 1.0 : 0.0);
        }
    }
    std::vector<double> res(items.size());
    const pd_status s = pd_evolve_batch(e, (int32_t)items.size(), items.data(), st.data(), 0.0, res.data());
    if (s != PD_OK) return s;
    std::fill(row_w, row_w + (size_t)9 * (Neta + 1), 0.0);
    for (int j = 1; j <= Neta - 1; ++j)
        for (int k = 0; k < 9; ++k) row_w[(size_t)9 * j + k] = res[(size_t)9 * (j - 1) + k];
    return PD_OK;
}

pd_status pd_engine_set_linear(pd_engine* e, const double* row_w) {
    if (!e) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        if (!row_w) {
            e->d_roww.free();
            e->step_kind = PD_STEP_DIRECT;
            return;
        }
        const size_t n = (size_t)9 * (e->d.Neta + 1);
        e->d_roww.alloc(n);
        upload(e->d_roww.p, row_w, n * 8, e->stream);
        CUDA_TRY(cudaStreamSynchronize(e->stream));
    });
}

pd_status pd_engine_set_step_kind(pd_engine* e, int32_t kind) {
    if (!e || (kind != PD_STEP_DIRECT && kind != PD_STEP_LINEAR)) return PD_VALIDATION_ERROR;
    if (kind == PD_STEP_LINEAR && !e->d_roww.p) {
        e->err = "pd_engine_set_step_kind: no linear-response weights (pd_engine_set_linear)";
        return PD_VALIDATION_ERROR;
    }
    e->step_kind = kind;
    return PD_OK;
}

int32_t pd_engine_step_kind(const pd_engine* e) { return e ? e->step_kind : -1; }

pd_status pd_engine_set_run_guard(pd_engine* e, double scale0, int32_t step_offset) {
    if (!e || step_offset < 0 || std::isnan(scale0)) return PD_VALIDATION_ERROR;
    e->guard_scale = scale0 > 0.0 ? scale0 : 0.0;
    e->step_offset = step_offset;
    return PD_OK;
}

} // extern "C"

// ---------------------------------------------------------------------------
// Decomposed run: fused peer-memory halo exchange
// ---------------------------------------------------------------------------
namespace {
// cuStreamWaitValue32 through the runtime's driver entry point (the library
// does not link libcuda; the symbol resolves on the GPU host's driver)
using WaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32 wait_value32() {
    static WaitValue32 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return (WaitValue32) nullptr;
        }
        return reinterpret_cast<WaitValue32>(f);
    }();
    return fn;
}

// The halo link of one call lives in the engine's Params for that call only.
struct HaloScope {
    Params& p;
    HaloScope(Params& prm, const pd_halo_out& h) : p(prm) {
        p.halo_n = h.nlinks;
        for (int l = 0; l < 2; ++l) {
            p.halo_col[l] = l < h.nlinks ? h.column[l] : -1;
            p.halo_dst[l] = l < h.nlinks ? h.dst[l] : nullptr;
            p.halo_flag[l] = l < h.nlinks ? h.flag[l] : nullptr;
        }
    }
    ~HaloScope() {
        p.halo_n = 0;
        p.halo_col[0] = p.halo_col[1] = -1;
        p.halo_dst[0] = p.halo_dst[1] = nullptr;
        p.halo_flag[0] = p.halo_flag[1] = nullptr;
    }
};

template <class F>
pd_status guarded_free(F&& fn) {
    try {
        fn();
        return PD_OK;
    } catch (const Status& s) {
        pdb200::set_global_error(s.msg);
        return s.code;
    }
}
} // namespace

extern "C" {

pd_status pd_projective_step_halo(pd_engine* e, const double* in, double* out, double t, const double* bnd,
                                  const double* src_time, const pd_halo_out* h) {
    (void)t;
    if (!e || !in || !out || !h || in == out || h->nlinks < 0 || h->nlinks > 2) return PD_VALIDATION_ERROR;
    for (int l = 0; l < h->nlinks; ++l)
        if (!h->dst[l] || !h->flag[l] || h->column[l] < 0 || h->column[l] > e->prm.Nxi) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        if (e->prm.k != 0)
            throw Status{PD_UNSUPPORTED, "halo-exchanging projective step: k = 0 only (one exchange per step)"};
        if (e->step_kind == PD_STEP_DIRECT && e->prm.source == PD_SOURCE_GENERAL)
            throw Status{PD_UNSUPPORTED, "halo-exchanging projective step: no general source"};
        HaloScope scope(e->prm, *h);
        // no copy-through: U_out's own columns come from the step kernel, its halo
        // columns from the neighbours' kernels, its boundary from the refresh
        e->sub_m = 0;
        e->launch_step(in, out, OUT_PROJECTIVE, e->prm.source ? src_time : nullptr, nullptr);
        e->launch_refresh(out, in, bnd ? bnd + e->perim : nullptr, nullptr);
    });
}

namespace {
pd_status check_halo(const pd_engine* e, const pd_halo_out* h) {
    if (!h || h->nlinks < 0 || h->nlinks > 2) return PD_VALIDATION_ERROR;
    for (int l = 0; l < h->nlinks; ++l)
        if (!h->dst[l] || !h->flag[l] || h->column[l] < 0 || h->column[l] > e->prm.Nxi) return PD_VALIDATION_ERROR;
    return PD_OK;
}
} // namespace

pd_status pd_gaptooth_substep_halo(pd_engine* e, const double* in, double* out, int32_t m, const double* bnd,
                                   const double* src_time, const pd_halo_out* h) {
    if (!e || !in || !out || in == out || m < 0 || check_halo(e, h) != PD_OK) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        if (m > e->prm.k) throw Status{PD_VALIDATION_ERROR, "substep index beyond k"};
        if (e->step_kind == PD_STEP_DIRECT && e->prm.source == PD_SOURCE_GENERAL)
            throw Status{PD_UNSUPPORTED, "halo-exchanging substep: no general source"};
        HaloScope scope(e->prm, *h);
        e->sub_m = m; // (the sampled-table offset; plain tables ignore it)
        e->launch_step(in, out, OUT_FIELD, e->prm.source ? src_time : nullptr, nullptr);
        e->launch_refresh(out, in, bnd, nullptr);
    });
}

pd_status pd_extrapolate_halo(pd_engine* e, const double* in, const double* Uk, const double* Uk1, double* out,
                              const double* bnd, const pd_halo_out* h) {
    if (!e || !in || !Uk || !Uk1 || !out || out == in || check_halo(e, h) != PD_OK) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        if (e->prm.k < 1) throw Status{PD_VALIDATION_ERROR, "extrapolation entry is for k >= 1"};
        HaloScope scope(e->prm, *h);
        const double horizon = e->prm.dt_macro - e->prm.k * e->prm.tau; // cpi.cpp:67-74
        k_extrapolate<<<(e->prm.P + 255) / 256, 256, 0, e->stream>>>(e->prm, out, Uk, Uk1, e->d_pij.p, horizon,
                                                                   nullptr);
        e->check_launch();
        e->launch_refresh(out, in, bnd, nullptr);
    });
}

pd_status pd_stream_wait_flag(pd_engine* e, const uint32_t* flag, uint32_t value) {
    if (!e || !flag) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        const WaitValue32 fn = wait_value32();
        if (!fn) throw Status{PD_CUDA_ERROR, "cuStreamWaitValue32 is not available from the driver"};
        int dev = 0, flush = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        CUDA_TRY(cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, dev));
        const unsigned flags = CU_STREAM_WAIT_VALUE_GEQ | (flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0u);
        const CUresult r = fn(reinterpret_cast<CUstream>(e->stream), reinterpret_cast<CUdeviceptr>(flag), value, flags);
        if (r != CUDA_SUCCESS)
            throw Status{PD_CUDA_ERROR, "cuStreamWaitValue32 failed (CUresult " + std::to_string((int)r) + ")"};
    });
}

pd_status pd_ipc_alloc(size_t bytes, void** dptr, unsigned char handle[64]) {
    if (!dptr || !handle || !bytes) return PD_VALIDATION_ERROR;
    return guarded_free([&] {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
        void* p = nullptr;
        CUDA_TRY(cudaMalloc(&p, bytes));
        CUDA_TRY(cudaMemset(p, 0, bytes));
        cudaIpcMemHandle_t h{};
        const cudaError_t err = cudaIpcGetMemHandle(&h, p);
        if (err != cudaSuccess) {
            cudaFree(p);
            throw Status{PD_CUDA_ERROR, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(err)};
        }
        std::memcpy(handle, &h, 64);
        *dptr = p;
    });
}

pd_status pd_ipc_open(const unsigned char handle[64], void** dptr) {
    if (!dptr || !handle) return PD_VALIDATION_ERROR;
    return guarded_free([&] {
        cudaIpcMemHandle_t h{};
        std::memcpy(&h, handle, 64);
        CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

pd_status pd_ipc_close(void* dptr) {
    if (!dptr) return PD_VALIDATION_ERROR;
    return guarded_free([&] { CUDA_TRY(cudaIpcCloseMemHandle(dptr)); });
}

pd_status pd_device_free(void* dptr) {
    if (!dptr) return PD_VALIDATION_ERROR;
    return guarded_free([&] { CUDA_TRY(cudaFree(dptr)); });
}

} // extern "C"

// ---------------------------------------------------------------------------
// Measurement hooks
// ---------------------------------------------------------------------------
namespace {
// 8 independent DFMA chains per thread, register resident; the result is
// stored only if it is impossible (keeps the chains alive without traffic).
// Block 0 / thread 0 also records clock64 and %globaltimer around its loop so
// the host can report the SM clock the chip sustained under this FP64 load.
__device__ inline unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void k_fp64_peak(double* sink, long long* clk, int iters, double a, double b) {
    const bool rec = blockIdx.x == 0 && threadIdx.x == 0;
    long long c0 = 0;
    unsigned long long g0 = 0;
    if (rec) {
        c0 = clock64();
        g0 = globaltimer_ns();
    }
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
    double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) sink[blockIdx.x] = s;
    if (rec) {
        clk[0] = clock64() - c0;
        clk[1] = (long long)(globaltimer_ns() - g0);
    }
}
} // namespace

extern "C" {

int32_t pd_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

pd_status pd_bench_step_kernel(pd_engine* e, const double* in_dev, double* out_dev, int32_t reps, double* ms) {
    if (!e || !in_dev || !out_dev || reps < 1 || !ms) return PD_VALIDATION_ERROR;
    return guarded(e, [&] {
        const int mode = e->prm.k == 0 ? OUT_PROJECTIVE : OUT_FIELD;
        e->launch_step(in_dev, out_dev, mode, nullptr, nullptr); // warm
        CUDA_TRY(cudaEventRecord(e->ev0, e->stream));
        for (int r = 0; r < reps; ++r) e->launch_step(in_dev, out_dev, mode, nullptr, nullptr);
        CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
        CUDA_TRY(cudaEventSynchronize(e->ev1));
        float t = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&t, e->ev0, e->ev1));
        *ms = (double)t / reps;
    });
}

pd_status pd_bench_fp64_peak(double ms_target, double* tflops, double* ghz) {
    try {
        int dev = 0, sms = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int threads = 512, blocks = sms * 4;
        DevBuf<double> sink;
        sink.alloc(blocks);
        DevBuf<long long> clk;
        clk.alloc(2);
        cudaEvent_t a, b;
        CUDA_TRY(cudaEventCreate(&a));
        CUDA_TRY(cudaEventCreate(&b));
        int iters = 256;
        float t = 0.f;
        for (int round = 0; round < 12; ++round) {
            CUDA_TRY(cudaEventRecord(a));
            k_fp64_peak<<<blocks, threads>>>(sink.p, clk.p, iters, 0.9999999999, 1e-12);
            CUDA_TRY(cudaEventRecord(b));
            CUDA_TRY(cudaEventSynchronize(b));
            CUDA_TRY(cudaEventElapsedTime(&t, a, b));
            if (t >= ms_target) break;
            iters = (int)std::min<double>(iters * std::max(2.0, ms_target / std::max(t, 1e-3f)), 1 << 26);
        }
        const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
        if (tflops) *tflops = flops / (t * 1e-3) / 1e12;
        long long hc[2] = {0, 1};
        CUDA_TRY(cudaMemcpy(hc, clk.p, sizeof hc, cudaMemcpyDeviceToHost));
        if (ghz) *ghz = hc[1] > 0 ? (double)hc[0] / (double)hc[1] : 0.0;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return PD_OK;
    } catch (const Status& s) {
        pdb200::set_global_error(s.msg);
        return s.code;
    }
}

} // extern "C"
