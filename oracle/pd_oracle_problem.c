/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this code.
 *
 * Input builder for the restated oracle on the BASELINE configs 4/5 family
 * (shear-cdr: x = xi + A sin 2 pi eta, y = eta + A sin 2 pi xi, CDR with
 * v = (sin pi y, cos pi x), D = eps, reaction omega, f = 0), so that the CPU
 * baseline / reference arm never needs the product library to build its
 * tables.  Restates, in the reference's evaluation order (IEEE double, built
 * with -ffp-contract=off like the reference's Release build):
 *   - the macro patch list, j outer / i inner   gaptooth.cpp:251-280
 *   - micro node coordinates                   microsim.cpp:18-24, 208-209
 *   - transform_coefficients (Eq. 8)           geometry.cpp:93-125
 *   - jacobian check                           geometry.cpp:80-91
 *   - solver form A=-a/l, C=-c/l, Vx=d/l, ...  microsim.cpp:245-249 (+ B=-b/l,
 *     |b| <= 1e-12 ignored as microsim.cpp:239)
 *   - the seeded initial field: std::mt19937_64 (Matsumoto & Nishimura 2000,
 *     the C++11 <random> parameters) drawn i-major as (x >> 11) * 2^-53, then
 *     Jacobi sweeps from a copy with the boundary fixed
 *   - the Appendix-A pins: h = h_frac * Delta, dt = 0.2 min(delta)^2 /
 *     max(|A| + |C|), tau = nt * dt, T = Nt * (Dt/tau) * tau.
 * Pinned bit-exactly against the product's host tables and the reference's own
 * sampling (oracle/_ref ref_sample_coeffs_desc) by tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "patchdyn_b200.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

int pdo_get_threads(void);

/* ---- std::mt19937_64 ------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t s[MT_N];
    int i;
} mt64_t;

static void mt64_seed(mt64_t* g, uint64_t seed) {
    g->s[0] = seed;
    for (int k = 1; k < MT_N; ++k)
        g->s[k] = 6364136223846793005ull * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
    g->i = MT_N;
}

static uint64_t mt64_next(mt64_t* g) {
    static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
    const uint64_t up = 0xFFFFFFFF80000000ull, lo = 0x7FFFFFFFull;
    if (g->i >= MT_N) {
        for (int k = 0; k < MT_N; ++k) {
            const uint64_t x = (g->s[k] & up) | (g->s[(k + 1) % MT_N] & lo);
            g->s[k] = g->s[(k + MT_M) % MT_N] ^ (x >> 1) ^ mag[x & 1ull];
        }
        g->i = 0;
    }
    uint64_t x = g->s[g->i++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

/* seeded U[0,1) macro field + Jacobi smoothing (configs 4/5) */
void pdo_seeded_field(int Nxi, int Neta, uint64_t seed, int sweeps, double* U) {
    const size_t n2 = (size_t)Neta + 1, nf = ((size_t)Nxi + 1) * n2;
    mt64_t g;
    mt64_seed(&g, seed);
    for (size_t q = 0; q < nf; ++q) U[q] = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
    double* V = (double*)malloc(sizeof(double) * nf);
    for (int s = 0; s < sweeps; ++s) {
        memcpy(V, U, sizeof(double) * nf);
        for (int i = 1; i < Nxi; ++i)
            for (int j = 1; j < Neta; ++j)
                U[i * n2 + j] = 0.25 * (V[(i - 1) * n2 + j] + V[(i + 1) * n2 + j] + V[i * n2 + j - 1] +
                                        V[i * n2 + j + 1]);
    }
    free(V);
}

/* transform_coefficients (geometry.cpp:93-125) for the shear map and the CDR
 * physical coefficients (alpha = beta = -eps, gamma = sin pi y, nu = cos pi x,
 * omega), solver form with l = 1.  out[6] = A, B, C, Vx, Vy, W.  Returns 0, or
 * -1 on a non-positive Jacobian (geometry.cpp:80-91). */
static int shear_node(double amp, double eps, double om, double xi, double eta, double out[6]) {
    const double x_xi = 1.0, x_eta = 2.0 * M_PI * amp * cos(2.0 * M_PI * eta);
    const double y_xi = 2.0 * M_PI * amp * cos(2.0 * M_PI * xi), y_eta = 1.0;
    const double J = x_xi * y_eta - y_xi * x_eta;
    if (!(J > 1e-14)) return -1;
    const double x_xixi = 0.0, x_xieta = 0.0, x_etaeta = -4.0 * M_PI * M_PI * amp * sin(2.0 * M_PI * eta);
    const double y_xixi = -4.0 * M_PI * M_PI * amp * sin(2.0 * M_PI * xi), y_xieta = 0.0, y_etaeta = 0.0;
    const double x = xi + amp * sin(2.0 * M_PI * eta), y = eta + amp * sin(2.0 * M_PI * xi);
    const double al = -eps, be = -eps;
    const double ga = sin(M_PI * y), nu = cos(M_PI * x);
    const double gA = be * x_eta * x_eta + al * y_eta * y_eta;
    const double gB = al * y_eta * y_xi + be * x_eta * x_xi;
    const double gC = be * x_xi * x_xi + al * y_xi * y_xi;
    const double J2 = J * J, J3 = J2 * J;
    const double cX = gA * x_xixi - 2.0 * gB * x_xieta + gC * x_etaeta;
    const double cY = gA * y_xixi - 2.0 * gB * y_xieta + gC * y_etaeta;
    const double a = gA / J2, b = -2.0 * gB / J2, c = gC / J2;
    const double R = (-y_eta * cX + x_eta * cY) / J3;
    const double S = (y_xi * cX - x_xi * cY) / J3;
    const double d = ga / J * y_eta - nu / J * x_eta + R;
    const double e = -ga / J * y_xi + nu / J * x_xi + S;
    const double l = 1.0;
    out[PD_COEF_A] = -a / l;
    out[PD_COEF_B] = fabs(b) > 1e-12 ? -b / l : 0.0;
    out[PD_COEF_C] = -c / l;
    out[PD_COEF_VX] = d / l;
    out[PD_COEF_VY] = e / l;
    out[PD_COEF_W] = om / l;
    return 0;
}

/* Resolve the pins of a shear-cdr problem description and build its tables.
 * d: in = the config (h_frac, dt_rule METRIC, dt_over_tau ...), out = resolved
 * h_xi, h_eta, tau, T (dt_rule GIVEN, h_frac = dt_over_tau = 0), as
 * pd_problem_create resolves them.  U0: (N_xi+1)(N_eta+1); patch_ij: [P][2];
 * coeffs: [P][6][n1][n2] (one set per patch: the coefficients depend on xi).
 * Returns a pd_status. */
int pdo_shear_problem(pd_problem_desc* d, double* U0, int32_t* patch_ij, double* coeffs) {
    if (d->problem != PD_PROBLEM_SHEAR_CDR) return PD_UNSUPPORTED;
    const double a = 0.0, b = 1.0, c = 0.0, dd = 1.0;
    if (d->h_frac > 0.0) {
        d->h_xi = d->h_frac * ((b - a) / d->N_xi);
        d->h_eta = d->h_frac * ((dd - c) / d->N_eta);
    }
    const int n1 = d->nx + 1, n2 = d->ny + 1;
    const size_t N = (size_t)n1 * n2;
    int P = 0;
    for (int j = 1; j <= d->N_eta - 1; ++j)
        for (int i = 1; i <= d->N_xi - 1; ++i) {
            patch_ij[2 * P] = i;
            patch_ij[2 * P + 1] = j;
            ++P;
        }
    const double Dxi = (b - a) / d->N_xi, Deta = (dd - c) / d->N_eta;
    const double mdxi = d->h_xi / d->nx, mdeta = d->h_eta / d->ny;
    double m_apc = 0.0;
    int bad = 0;
#pragma omp parallel for num_threads(pdo_get_threads()) schedule(dynamic, 4) reduction(max : m_apc)
    for (int s = 0; s < P; ++s) {
        const double xc = a + Dxi * patch_ij[2 * s], ec = c + Deta * patch_ij[2 * s + 1];
        const double xi0 = xc - 0.5 * mdxi * d->nx, eta0 = ec - 0.5 * mdeta * d->ny;
        double* o = coeffs + (size_t)s * PD_NCOEF * N;
        for (int i = 0; i < n1; ++i)
            for (int j = 0; j < n2; ++j) {
                double w[6];
                if (shear_node(d->amp, d->eps, d->omega, xi0 + i * mdxi, eta0 + j * mdeta, w)) {
                    bad = 1;
                    continue;
                }
                const size_t k = (size_t)i * n2 + j;
                for (int q = 0; q < 6; ++q) o[q * N + k] = w[q];
                const double apc = fabs(w[PD_COEF_A]) + fabs(w[PD_COEF_C]);
                if (apc > m_apc) m_apc = apc;
            }
    }
    if (bad) return PD_NON_POSITIVE_JACOBIAN;
    const double dmin = fmin(d->h_xi / d->nx, d->h_eta / d->ny);
    if (d->dt_rule == PD_DT_METRIC) d->tau = d->nt * (0.2 * dmin * dmin / m_apc);
    if (d->dt_over_tau > 0) d->T = d->Nt * (d->dt_over_tau * d->tau);
    d->dt_rule = PD_DT_GIVEN;
    d->h_frac = 0.0;
    d->dt_over_tau = 0.0;
    pdo_seeded_field(d->N_xi, d->N_eta, d->seed, d->jacobi_sweeps, U0);
    return PD_OK;
}
