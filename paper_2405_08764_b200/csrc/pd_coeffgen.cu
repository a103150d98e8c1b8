// On-device mesh/metric generation.
//
// The host builder samples transform_coefficients (geometry.cpp:93-125) at
// every micro node through std::function closures, exactly as
// PatchIntegrator::sample_coeffs does (microsim.cpp:204-263), and ships a
// [sets][6][n1][n2] table to the device.  For the framework's built-in
// analytic problems this file computes the same table on the GPU, one thread
// per micro node: the mapping (forward map, inverse metrics, second
// derivatives), the physical coefficients, Eq. 8 of the paper in the
// evaluation order of geometry.cpp:93-125 (explicitly rounded, no FMA
// contraction, like the host's -ffp-contract=off build) and the solver form of
// microsim.cpp:245-249.  The only difference from the host table is the
// transcendental library (CUDA's sin/cos/tanh/exp against glibc's): entries
// agree to a few ulp (tests/test_gpu.py::test_coeffgen_*).
//
// Two uses: pd_problem_create with coeff_gen = PD_COEFF_DEVICE skips the host
// sampling (reduction-only pass for the dt pin and the stability guard), and
// pd_engine_create generates its coefficient table in place when the
// descriptor carries a generator instead of a host table (no host table, no
// host-to-device copy).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "coeffgen.hpp"
#include "pd_device.cuh"

namespace pdb200 {
namespace {

struct GenParams {
    int problem;
    int variable;     // REF_CDR_VAR: D = 1 + x, c0 = 8
    double lambda;    // REF_CDR stretching (0 = identity map)
    double beta, tb;  // CDR_TANH: beta, tanh(beta) (host-rounded, as the closure captures it)
    double eps, omega, vel, amp;
    double a, c;      // domain origin
    double Dxi, Deta; // macro spacings (b-a)/Nxi, (d-c)/Neta
    double mdxi, mdeta;
    int nx, ny, n1, n2;
    double l;
    int want_src;
};

struct Met {
    double x_xi, x_eta, y_xi, y_eta;
};
struct Sec {
    double x_xixi, x_xieta, x_etaeta, y_xixi, y_xieta, y_etaeta;
};

constexpr double kPi = 3.14159265358979323846; // M_PI

// ---- mappings (geometry.cpp:14-66 and the problem closures of problems.cpp) ----
__device__ void map_eval(const GenParams& g, double xi, double eta, double& x, double& y, Met& m, Sec& s) {
    m = {1.0, 0.0, 0.0, 1.0};
    s = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    x = xi;
    y = eta;
    switch (g.problem) {
        case PD_PROBLEM_REF_CDR:
        case PD_PROBLEM_REF_CDR_VAR:
            if (g.lambda != 0.0) { // stretched_map: x = s + lambda/pi sin(pi s)
                const double sx = sin(XMUL(kPi, xi)), sy = sin(XMUL(kPi, eta));
                const double lp = XDIV(g.lambda, kPi);
                x = XADD(xi, XMUL(lp, sx));
                y = XADD(eta, XMUL(lp, sy));
                m = {XADD(1.0, XMUL(g.lambda, cos(XMUL(kPi, xi)))), 0.0, 0.0,
                     XADD(1.0, XMUL(g.lambda, cos(XMUL(kPi, eta))))};
                const double ml = XMUL(-g.lambda, kPi);
                s = {XMUL(ml, sx), 0.0, 0.0, 0.0, 0.0, XMUL(ml, sy)};
            }
            break;
        case PD_PROBLEM_CDR_TANH: { // x = 1 - tanh(beta (1 - s)) / tanh(beta)
            const double tx = tanh(XMUL(g.beta, XSUB(1.0, xi))), ty = tanh(XMUL(g.beta, XSUB(1.0, eta)));
            x = XSUB(1.0, XDIV(tx, g.tb));
            y = XSUB(1.0, XDIV(ty, g.tb));
            auto Xp = [&](double th) { return XDIV(XMUL(g.beta, XSUB(1.0, XMUL(th, th))), g.tb); };
            auto Xpp = [&](double th) {
                return XDIV(XMUL(XMUL(XMUL(XMUL(2.0, g.beta), g.beta), th), XSUB(1.0, XMUL(th, th))), g.tb);
            };
            m = {Xp(tx), 0.0, 0.0, Xp(ty)};
            s = {Xpp(tx), 0.0, 0.0, 0.0, 0.0, Xpp(ty)};
            break;
        }
        case PD_PROBLEM_ANNULUS_NONAXI:
        case PD_PROBLEM_REF_ANNULUS: { // polar_map: (theta, r) -> (r sin, r cos)
            const double st = sin(xi), ct = cos(xi), r = eta;
            x = XMUL(r, st);
            y = XMUL(r, ct);
            m = {XMUL(r, ct), st, XMUL(-r, st), ct};
            s = {XMUL(-r, st), ct, 0.0, XMUL(-r, ct), -st, 0.0};
            break;
        }
        case PD_PROBLEM_SHEAR_CDR: { // x = xi + A sin 2pi eta, y = eta + A sin 2pi xi
            const double tp = XMUL(2.0, kPi);
            const double se = sin(XMUL(tp, eta)), sx = sin(XMUL(tp, xi));
            x = XADD(xi, XMUL(g.amp, se));
            y = XADD(eta, XMUL(g.amp, sx));
            const double tpa = XMUL(tp, g.amp);
            m = {1.0, XMUL(tpa, cos(XMUL(tp, eta))), XMUL(tpa, cos(XMUL(tp, xi))), 1.0};
            const double fpa = XMUL(XMUL(XMUL(-4.0, kPi), kPi), g.amp);
            s = {0.0, 0.0, XMUL(fpa, se), XMUL(fpa, sx), 0.0, 0.0};
            break;
        }
        default: // identity: DIFFUSION_SQUARE, STEADY
            break;
    }
}

// ---- physical coefficients at (x, y, t = 0): alpha = -Dx, beta = -Dy, gamma, nu, omega ----
__device__ void phys_eval(const GenParams& g, double x, double y, double& al, double& be, double& ga, double& nu,
                          double& om) {
    ga = nu = om = 0.0;
    double D = 1.0;
    switch (g.problem) {
        case PD_PROBLEM_DIFFUSION_SQUARE:
        case PD_PROBLEM_ANNULUS_NONAXI: D = g.eps; break;
        case PD_PROBLEM_CDR_TANH:
            D = g.eps;
            ga = nu = g.vel;
            om = g.omega;
            break;
        case PD_PROBLEM_SHEAR_CDR:
            D = g.eps;
            ga = sin(XMUL(kPi, y));
            nu = cos(XMUL(kPi, x));
            om = g.omega;
            break;
        case PD_PROBLEM_REF_CDR:
        case PD_PROBLEM_REF_CDR_VAR:
            D = g.variable ? XADD(1.0, x) : 1.0;
            ga = XMUL(10.0, x);
            nu = XMUL(10.0, y);
            break;
        default: D = 1.0; break; // REF_ANNULUS, STEADY
    }
    al = -D;
    be = -D;
}

__device__ __forceinline__ unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }

// one thread per (set, node); maxima as bit patterns of non-negative doubles
__global__ void k_gen_coeffs(GenParams g, const int* __restrict__ set_ij, int nsets, double* __restrict__ coeffs,
                             double* __restrict__ src, unsigned long long* __restrict__ maxima, int* __restrict__ bad) {
    const int N = g.n1 * g.n2;
    const size_t total = (size_t)nsets * N;
    unsigned long long m_ac = 0, m_apc = 0, m_b = 0;
    int nbad = 0;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const int s = (int)(t / N), k = (int)(t % N);
        const int i = k / g.n2, j = k % g.n2;
        // CoarseGrid::xi/eta (gaptooth.hpp:21-24); node coordinates microsim.cpp:208-209
        const double xc = XADD(g.a, XMUL(g.Dxi, (double)set_ij[2 * s]));
        const double ec = XADD(g.c, XMUL(g.Deta, (double)set_ij[2 * s + 1]));
        const double xi0 = XSUB(xc, XMUL(XMUL(0.5, g.mdxi), (double)g.nx));
        const double eta0 = XSUB(ec, XMUL(XMUL(0.5, g.mdeta), (double)g.ny));
        const double xi = XADD(xi0, XMUL((double)i, g.mdxi)), eta = XADD(eta0, XMUL((double)j, g.mdeta));
        double x, y;
        Met gm;
        Sec sd;
        map_eval(g, xi, eta, x, y, gm, sd);
        // transform_coefficients, geometry.cpp:93-125 (operation order kept)
        const double J = XSUB(XMUL(gm.x_xi, gm.y_eta), XMUL(gm.y_xi, gm.x_eta));
        if (!(J > 1e-14)) ++nbad;
        double al, be, ga, nu, om;
        phys_eval(g, x, y, al, be, ga, nu, om);
        const double gA = XADD(XMUL(XMUL(be, gm.x_eta), gm.x_eta), XMUL(XMUL(al, gm.y_eta), gm.y_eta));
        const double gB = XADD(XMUL(XMUL(al, gm.y_eta), gm.y_xi), XMUL(XMUL(be, gm.x_eta), gm.x_xi));
        const double gC = XADD(XMUL(XMUL(be, gm.x_xi), gm.x_xi), XMUL(XMUL(al, gm.y_xi), gm.y_xi));
        const double J2 = XMUL(J, J), J3 = XMUL(J2, J);
        const double cX = XADD(XSUB(XMUL(gA, sd.x_xixi), XMUL(XMUL(2.0, gB), sd.x_xieta)), XMUL(gC, sd.x_etaeta));
        const double cY = XADD(XSUB(XMUL(gA, sd.y_xixi), XMUL(XMUL(2.0, gB), sd.y_xieta)), XMUL(gC, sd.y_etaeta));
        const double ta = XDIV(gA, J2);
        const double tb = XDIV(XMUL(-2.0, gB), J2);
        const double tcc = XDIV(gC, J2);
        const double R = XDIV(XADD(XMUL(-gm.y_eta, cX), XMUL(gm.x_eta, cY)), J3);
        const double S = XDIV(XSUB(XMUL(gm.y_xi, cX), XMUL(gm.x_xi, cY)), J3);
        const double td = XADD(XSUB(XMUL(XDIV(ga, J), gm.y_eta), XMUL(XDIV(nu, J), gm.x_eta)), R);
        const double te = XADD(XADD(XMUL(XDIV(-ga, J), gm.y_xi), XMUL(XDIV(nu, J), gm.x_xi)), S);
        // solver form  microsim.cpp:245-249 (+ B = -b/l, |b| <= 1e-12 ignored as at :239)
        const double A = XDIV(-ta, g.l), C = XDIV(-tcc, g.l);
        const double B = fabs(tb) > 1e-12 ? XDIV(-tb, g.l) : 0.0;
        double* o = coeffs ? coeffs + (size_t)s * PD_NCOEF * N : nullptr;
        if (o) {
            o[PD_COEF_A * N + k] = A;
            o[PD_COEF_B * N + k] = B;
            o[PD_COEF_C * N + k] = C;
            o[PD_COEF_VX * N + k] = XDIV(td, g.l);
            o[PD_COEF_VY * N + k] = XDIV(te, g.l);
            o[PD_COEF_W * N + k] = XDIV(om, g.l);
        }
        if (src && g.want_src) { // problem1 source_spatial: (c0 x + 10 y - 1) e^{x+y}  (problems.cpp:19-75)
            const double c0 = g.variable ? 8.0 : 10.0;
            src[(size_t)s * N + k] = XMUL(XSUB(XADD(XMUL(c0, x), XMUL(10.0, y)), 1.0), exp(XADD(x, y)));
        }
        m_ac = max(m_ac, max(dbits(fabs(A)), dbits(fabs(C))));
        m_apc = max(m_apc, dbits(XADD(fabs(A), fabs(C))));
        m_b = max(m_b, dbits(fabs(B)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        m_ac = max(m_ac, __shfl_xor_sync(0xffffffffu, m_ac, o));
        m_apc = max(m_apc, __shfl_xor_sync(0xffffffffu, m_apc, o));
        m_b = max(m_b, __shfl_xor_sync(0xffffffffu, m_b, o));
        nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(maxima + 0, m_ac);
        atomicMax(maxima + 1, m_apc);
        atomicMax(maxima + 2, m_b);
        if (nbad) atomicAdd(bad, nbad);
    }
}

#define GEN_TRY(x)                                                                        \
    do {                                                                                  \
        cudaError_t err_ = (x);                                                           \
        if (err_ != cudaSuccess) throw DeviceError(std::string("CUDA: ") + cudaGetErrorString(err_)); \
    } while (0)

} // namespace

bool coeffgen_supported(int problem) {
    switch (problem) {
        case PD_PROBLEM_DIFFUSION_SQUARE:
        case PD_PROBLEM_CDR_TANH:
        case PD_PROBLEM_ANNULUS_NONAXI:
        case PD_PROBLEM_SHEAR_CDR:
        case PD_PROBLEM_REF_ANNULUS:
        case PD_PROBLEM_REF_CDR:
        case PD_PROBLEM_REF_CDR_VAR:
        case PD_PROBLEM_STEADY: return true;
        default: return false;
    }
}

std::vector<int32_t> coeffgen_set_centres(const pd_engine_desc& d, const int32_t* patch_ij, int P) {
    // the set's coefficients are sampled at the first patch (table order) that
    // uses it, as the host builder does (gaptooth.cpp:254-266: row sharing
    // samples at (i_lo, j))
    std::vector<int32_t> c(2 * (size_t)d.ncoeff_sets, -1);
    for (int p = 0; p < P; ++p) {
        const int s = d.coeff_set ? d.coeff_set[p] : p;
        if (s < 0 || s >= d.ncoeff_sets) throw ShapeMismatch("coefficient set index out of range");
        if (c[2 * (size_t)s] < 0) {
            c[2 * (size_t)s] = patch_ij[2 * (size_t)p];
            c[2 * (size_t)s + 1] = patch_ij[2 * (size_t)p + 1];
        }
    }
    for (int s = 0; s < d.ncoeff_sets; ++s)
        if (c[2 * (size_t)s] < 0) throw ShapeMismatch("coefficient set used by no patch");
    return c;
}

CoeffGenStats coeffgen_run(const pd_problem_desc& pd, const pd_engine_desc& d, const int32_t* set_ij,
                           double* coeffs_dev, double* src_dev, cudaStream_t stream) {
    if (!coeffgen_supported(pd.problem)) throw Unsupported("no device generator for this problem kind");
    if (!(d.l != 0.0)) throw ValidationError("time-derivative multiplier l must be nonzero");
    GenParams g{};
    g.problem = pd.problem;
    g.variable = pd.problem == PD_PROBLEM_REF_CDR_VAR;
    g.lambda = pd.lambda;
    if ((pd.problem == PD_PROBLEM_REF_CDR || pd.problem == PD_PROBLEM_REF_CDR_VAR) &&
        !(pd.lambda >= 0.0 && pd.lambda < 1.0))
        throw InvalidStretch("stretching parameter must lie in [0,1), got " + std::to_string(pd.lambda));
    g.beta = pd.beta;
    g.tb = std::tanh(pd.beta);
    g.eps = pd.eps;
    g.omega = pd.omega;
    g.vel = pd.vel;
    g.amp = pd.amp;
    g.a = d.a;
    g.c = d.c;
    g.Dxi = (d.b - d.a) / d.Nxi;
    g.Deta = (d.d - d.c) / d.Neta;
    g.mdxi = d.h_xi / d.nx;
    g.mdeta = d.h_eta / d.ny;
    g.nx = d.nx;
    g.ny = d.ny;
    g.n1 = d.nx + 1;
    g.n2 = d.ny + 1;
    g.l = d.l;
    g.want_src = d.source_kind == PD_SOURCE_SEPARABLE;
    const int S = d.ncoeff_sets;
    int32_t* d_set = nullptr;
    unsigned long long* d_max = nullptr;
    int* d_bad = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    CoeffGenStats st{};
    try {
        GEN_TRY(cudaMalloc(&d_set, 2 * sizeof(int32_t) * (size_t)S));
        GEN_TRY(cudaMalloc(&d_max, 3 * sizeof(unsigned long long) + sizeof(int)));
        d_bad = reinterpret_cast<int*>(d_max + 3);
        GEN_TRY(cudaMemcpyAsync(d_set, set_ij, 2 * sizeof(int32_t) * (size_t)S, cudaMemcpyHostToDevice, stream));
        GEN_TRY(cudaMemsetAsync(d_max, 0, 3 * sizeof(unsigned long long) + sizeof(int), stream));
        GEN_TRY(cudaEventCreate(&e0));
        GEN_TRY(cudaEventCreate(&e1));
        const size_t total = (size_t)S * g.n1 * g.n2;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int blocks = (int)std::min<size_t>((total + 255) / 256, (size_t)sms * 8);
        GEN_TRY(cudaEventRecord(e0, stream));
        k_gen_coeffs<<<blocks, 256, 0, stream>>>(g, d_set, S, coeffs_dev, src_dev, d_max, d_bad);
        GEN_TRY(cudaGetLastError());
        GEN_TRY(cudaEventRecord(e1, stream));
        unsigned long long hm[3];
        int hbad = 0;
        GEN_TRY(cudaMemcpyAsync(hm, d_max, sizeof hm, cudaMemcpyDeviceToHost, stream));
        GEN_TRY(cudaMemcpyAsync(&hbad, d_bad, sizeof hbad, cudaMemcpyDeviceToHost, stream));
        GEN_TRY(cudaStreamSynchronize(stream));
        float ms = 0.f;
        GEN_TRY(cudaEventElapsedTime(&ms, e0, e1));
        auto asd = [](unsigned long long b) {
            double v;
            std::memcpy(&v, &b, 8);
            return v;
        };
        st.max_abs_ac = asd(hm[0]);
        st.max_a_plus_c = asd(hm[1]);
        st.max_abs_b = asd(hm[2]);
        st.device_ms = ms;
        st.nodes = total;
        if (hbad) throw NonPositiveJacobian("non-positive Jacobian at " + std::to_string(hbad) + " micro node(s)");
    } catch (...) {
        cudaFree(d_set);
        cudaFree(d_max);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        throw;
    }
    cudaFree(d_set);
    cudaFree(d_max);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return st;
}

} // namespace pdb200

namespace pdb200 {
void set_global_error(const std::string& m); // capi_engine
}

extern "C" pd_status pd_coeffs_generate(const pd_engine_desc* desc, double* coeffs_host, double* src_host,
                                        double* stats) {
    using namespace pdb200;
    double* d_c = nullptr;
    double* d_s = nullptr;
    try {
        if (!desc || !desc->coeff_generator) throw ValidationError("descriptor has no coefficient generator");
        const int P = pd_patch_count(desc);
        if (P < 1) throw ValidationError("empty patch table");
        std::vector<int32_t> pij(2 * (size_t)P);
        const pd_status ist = pd_build_index_tables(desc, pij.data(), nullptr);
        if (ist != PD_OK) throw Error(ist, pd_last_error(nullptr));
        const std::vector<int32_t> centres = coeffgen_set_centres(*desc, pij.data(), P);
        const size_t N = (size_t)(desc->nx + 1) * (desc->ny + 1), S = (size_t)desc->ncoeff_sets;
        if (coeffs_host) GEN_TRY(cudaMalloc(&d_c, S * PD_NCOEF * N * 8));
        const bool want_src = src_host && desc->source_kind == PD_SOURCE_SEPARABLE;
        if (want_src) GEN_TRY(cudaMalloc(&d_s, S * N * 8));
        const CoeffGenStats st = coeffgen_run(*desc->coeff_generator, *desc, centres.data(), d_c, d_s, nullptr);
        if (coeffs_host) GEN_TRY(cudaMemcpy(coeffs_host, d_c, S * PD_NCOEF * N * 8, cudaMemcpyDeviceToHost));
        if (want_src) GEN_TRY(cudaMemcpy(src_host, d_s, S * N * 8, cudaMemcpyDeviceToHost));
        if (stats) {
            stats[0] = st.max_abs_ac;
            stats[1] = st.max_a_plus_c;
            stats[2] = st.max_abs_b;
            stats[3] = st.device_ms;
            stats[4] = (double)st.nodes;
        }
        cudaFree(d_c);
        cudaFree(d_s);
        return PD_OK;
    } catch (const Error& e) {
        cudaFree(d_c);
        cudaFree(d_s);
        set_global_error(e.what());
        return static_cast<pd_status>(e.status);
    }
}
