// EXACT-mode ADI micro-solver: PatchIntegrator::adi_sweep (microsim.cpp:334-507)
// with its upwind convection stencils (microsim.cpp:56-119) and line solvers
// (solve_tridiagonal / BandedMatrix::solve, linalg.cpp:8-61), in the
// reference's evaluation order with explicitly rounded IEEE operations.
//
// One CTA per patch (the fused step and the batched integrate entry).  Per
// micro step: explicit right-hand side of the xi half-step on every node in
// parallel, one thread per xi-line for the implicit solve, then the same for
// eta.  The reference's default solver (scheme_config.hpp:19-20) and the one
// behind its Tables 1-3 (config.cpp:148-154).
#pragma once

#include "pd_device.cuh"

namespace pdb200::dev {

// Offsets/weights of the upwind derivative at a node; weights carry 1/delta
// (make_upwind, microsim.cpp:65-104).
struct UpwindW {
    int off[4];
    double w[4];
    int n;
};

__device__ inline UpwindW make_upwind_x(int order, double r, double delta, int vel_sign) {
    UpwindW s{};
    const double s1 = vel_sign >= 0 ? 1.0 : -1.0;
    if (order == PD_UPWIND_TWO) {
        s.n = 2;
        s.off[0] = 0;
        s.off[1] = vel_sign >= 0 ? -1 : 1;
        s.w[0] = XDIV(s1, delta);
        s.w[1] = XDIV(-s1, delta);
    } else if (order == PD_UPWIND_THREE) {
        s.n = 3;
        s.off[0] = 0;
        s.off[1] = vel_sign >= 0 ? -1 : 1;
        s.off[2] = vel_sign >= 0 ? -2 : 2;
        s.w[0] = XDIV(XMUL(3.0, s1), XMUL(2.0, delta));
        s.w[1] = XDIV(XMUL(-4.0, s1), XMUL(2.0, delta));
        s.w[2] = XDIV(s1, XMUL(2.0, delta));
    } else { // four
        s.n = 4;
        if (vel_sign >= 0) {
            s.off[0] = 1;
            s.w[0] = XSUB(XDIV(1.0, XMUL(2.0, delta)), XDIV(r, XMUL(3.0, delta)));
            s.off[1] = -1;
            s.w[1] = XSUB(XDIV(-1.0, XMUL(2.0, delta)), XDIV(r, delta));
            s.off[2] = -2;
            s.w[2] = XDIV(r, XMUL(3.0, delta));
            s.off[3] = 0;
            s.w[3] = XDIV(r, delta);
        } else {
            s.off[0] = 1;
            s.w[0] = XADD(XDIV(1.0, XMUL(2.0, delta)), XDIV(r, delta));
            s.off[1] = -1;
            s.w[1] = XADD(XDIV(-1.0, XMUL(2.0, delta)), XDIV(r, XMUL(3.0, delta)));
            s.off[2] = 2;
            s.w[2] = XDIV(-r, XMUL(3.0, delta));
            s.off[3] = 0;
            s.w[3] = XDIV(-r, delta);
        }
    }
    return s;
}

// wider stencils drop to two-point where the window leaves [0, imax]
// (upwind_with_fallback, microsim.cpp:107-119)
__device__ inline UpwindW upwind_fb_x(int order, double r, double delta, int vel_sign, int i, int imax) {
    if (order != PD_UPWIND_TWO) {
        const UpwindW s = make_upwind_x(order, r, delta, vel_sign);
        bool ok = true;
        for (int k = 0; k < s.n; ++k) {
            const int idx = i + s.off[k];
            if (idx < 0 || idx > imax) ok = false;
        }
        if (ok) return s;
    }
    return make_upwind_x(PD_UPWIND_TWO, r, delta, vel_sign);
}

// explicit operator of the direction not being swept, reaction carried half
// (cross_term, microsim.cpp:357-395).  f(k): tile value at flat node k;
// gb(k): ghost offset b at [edge * L + position]; coef [6][N].  Templated on
// the accessors so the FAST fold can probe it with unit vectors.
template <class FA, class GA>
__device__ inline double cross_term_t(const Params& p, FA f, const EdgeSh* E, GA gb, const double* coef, int i, int j,
                                      bool eta_dir) {
    const int nx = p.nx, ny = p.ny, n2 = p.n2, L = p.L, N = p.N, k = i * n2 + j;
    if (eta_dir) {
        const EdgeSh &gS = E[PD_EDGE_S], &gN = E[PD_EDGE_N];
        const double glo = ghost_x(gS, f(i * n2 + 1), f(i * n2), gb(PD_EDGE_S * L + i));
        const double ghi = ghost_x(gN, f(i * n2 + ny - 1), f(i * n2 + ny), gb(PD_EDGE_N * L + i));
        const double um = j > 0 ? f(k - 1) : glo;
        const double up = j < ny ? f(k + 1) : ghi;
        const double uc = f(k);
        const double uyy = XDIV(XADD(XSUB(um, XMUL(2.0, uc)), up), XMUL(p.mdeta, p.mdeta));
        const double v = coef[PD_COEF_VY * N + k];
        const UpwindW sw = upwind_fb_x(p.upwind_order, p.upwind_r, p.mdeta, v >= 0 ? 1 : -1, j, ny);
        double du = 0.0;
        for (int m = 0; m < sw.n; ++m) {
            const int jj = j + sw.off[m];
            const double val = jj < 0 ? glo : (jj > ny ? ghi : f(i * n2 + jj));
            du = XADD(du, XMUL(sw.w[m], val));
        }
        return XSUB(XSUB(XMUL(coef[PD_COEF_C * N + k], uyy), XMUL(v, du)),
                    XMUL(XMUL(0.5, coef[PD_COEF_W * N + k]), uc));
    }
    const EdgeSh &gW = E[PD_EDGE_W], &gE = E[PD_EDGE_E];
    const double glo = ghost_x(gW, f(n2 + j), f(j), gb(PD_EDGE_W * L + j));
    const double ghi = ghost_x(gE, f((nx - 1) * n2 + j), f(nx * n2 + j), gb(PD_EDGE_E * L + j));
    const double um = i > 0 ? f(k - n2) : glo;
    const double up = i < nx ? f(k + n2) : ghi;
    const double uc = f(k);
    const double uxx = XDIV(XADD(XSUB(um, XMUL(2.0, uc)), up), XMUL(p.mdxi, p.mdxi));
    const double v = coef[PD_COEF_VX * N + k];
    const UpwindW sw = upwind_fb_x(p.upwind_order, p.upwind_r, p.mdxi, v >= 0 ? 1 : -1, i, nx);
    double du = 0.0;
    for (int m = 0; m < sw.n; ++m) {
        const int ii = i + sw.off[m];
        const double val = ii < 0 ? glo : (ii > nx ? ghi : f(ii * n2 + j));
        du = XADD(du, XMUL(sw.w[m], val));
    }
    return XSUB(XSUB(XMUL(coef[PD_COEF_A * N + k], uxx), XMUL(v, du)), XMUL(XMUL(0.5, coef[PD_COEF_W * N + k]), uc));
}

__device__ inline double cross_term_x(const Params& p, const double* f, const EdgeSh* E, const double* gb,
                                      const double* coef, int i, int j, bool eta_dir) {
    return cross_term_t(p, [f](int k) { return f[k]; }, E, [gb](int k) { return gb[k]; }, coef, i, j, eta_dir);
}

// node_pinned  microsim.cpp:285-288
__device__ inline bool node_pinned_x(const EdgeSh* E, int i, int j, int nx, int ny) {
    return (i == 0 && E[PD_EDGE_W].pinned) || (i == nx && E[PD_EDGE_E].pinned) || (j == 0 && E[PD_EDGE_S].pinned) ||
           (j == ny && E[PD_EDGE_N].pinned);
}

// Thomas algorithm  linalg.cpp:8-25 (rhs overwritten with the solution)
__device__ inline void solve_tridiagonal_x(const double* lo, const double* di, const double* up, double* rhs,
                                           double* wk, int n) {
    double m = di[0];
    wk[0] = XDIV(up[0], m);
    rhs[0] = XDIV(rhs[0], m);
    for (int k = 1; k < n; ++k) {
        m = XSUB(di[k], XMUL(lo[k], wk[k - 1]));
        wk[k] = XDIV(up[k], m);
        rhs[k] = XDIV(XSUB(rhs[k], XMUL(lo[k], rhs[k - 1])), m);
    }
    for (int k = n - 1; k-- > 0;) rhs[k] = XSUB(rhs[k], XMUL(wk[k], rhs[k + 1]));
}

// BandedMatrix(n, 2, 2)::solve without pivoting  linalg.cpp:43-61; band[r*5 + (c-r) + 2]
__device__ inline void solve_banded_x(double* band, double* rhs, int n) {
    constexpr int kl = 2, ku = 2;
    auto B = [&](int r, int off) -> double& { return band[r * 5 + off + 2]; };
    for (int k = 0; k < n - 1; ++k) {
        const double piv = B(k, 0);
        const int last = min(k + kl, n - 1);
        for (int r = k + 1; r <= last; ++r) {
            const double f = XDIV(B(r, k - r), piv);
            if (f == 0.0) continue;
            for (int c = k + 1; c <= min(k + ku, n - 1); ++c) B(r, c - r) = XSUB(B(r, c - r), XMUL(f, B(k, c - k)));
            rhs[r] = XSUB(rhs[r], XMUL(f, rhs[k]));
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        double s = rhs[r];
        for (int c = r + 1; c <= min(r + ku, n - 1); ++c) s = XSUB(s, XMUL(B(r, c - r), rhs[c]));
        rhs[r] = XDIV(s, B(r, 0));
    }
}

// (I - half*L_swept) out = rhs_field, one thread per line (implicit_sweep,
// microsim.cpp:402-491).  lsc: per-line scratch [L][6*L].
__device__ inline void implicit_sweep_x(const Params& p, const double* rhsf, double* out, const EdgeSh* E,
                                        const double* gb, const double* val, const double* slope,
                                        const double* coef, double* lsc, bool xi_dir) {
    const int nx = p.nx, ny = p.ny, n2 = p.n2, L = p.L, N = p.N;
    const double half = XMUL(0.5, p.mdt);
    const int nline = xi_dir ? ny : nx;
    const int n = xi_dir ? nx + 1 : ny + 1;
    const double dd = xi_dir ? p.mdxi : p.mdeta;
    const int elo = xi_dir ? PD_EDGE_W : PD_EDGE_S, ehi = xi_dir ? PD_EDGE_E : PD_EDGE_N;
    const int slo = xi_dir ? PD_EDGE_S : PD_EDGE_W, shi = xi_dir ? PD_EDGE_N : PD_EDGE_E;
    const bool banded = p.upwind_order != PD_UPWIND_TWO;
    for (int line = threadIdx.x; line <= nline; line += blockDim.x) {
        auto put = [&](int k, double v) {
            if (xi_dir) out[k * n2 + line] = v;
            else out[line * n2 + k] = v;
        };
        if ((line == 0 && E[slo].pinned) || (line == nline && E[shi].pinned)) {
            const int e = line == 0 ? slo : shi;
            for (int k = 0; k < n; ++k) put(k, pinned_value_x(E[e], val + e * L, slope + e * L, k));
            continue;
        }
        double* sc = lsc + (size_t)line * 6 * L;
        double *lo = sc, *di = sc + L, *up = sc + 2 * L, *rhs = sc + 3 * L, *wk = sc + 4 * L; // tridiagonal
        double* band = sc;                                                                      // banded: 5n
        double* brhs = sc + 5 * L;
        if (banded)
            for (int q = 0; q < 5 * n; ++q) band[q] = 0.0; // BandedMatrix::clear
        for (int k = 0; k < n; ++k) {
            const bool pin_lo = k == 0 && E[elo].pinned, pin_hi = k == n - 1 && E[ehi].pinned;
            if (pin_lo || pin_hi) {
                const int e = pin_lo ? elo : ehi;
                const double pv = pinned_value_x(E[e], val + e * L, slope + e * L, line);
                if (banded) {
                    band[k * 5 + 2] = 1.0;
                    brhs[k] = pv;
                } else {
                    di[k] = 1.0;
                    lo[k] = 0.0;
                    up[k] = 0.0;
                    rhs[k] = pv;
                }
                continue;
            }
            const int i = xi_dir ? k : line, j = xi_dir ? line : k, q = i * n2 + j;
            const double A = xi_dir ? coef[PD_COEF_A * N + q] : coef[PD_COEF_C * N + q];
            const double V = xi_dir ? coef[PD_COEF_VX * N + q] : coef[PD_COEF_VY * N + q];
            const double s = XDIV(XMUL(half, A), XMUL(dd, dd));
            double diag = XADD(XADD(1.0, XMUL(2.0, s)), XMUL(XMUL(half, 0.5), coef[PD_COEF_W * N + q]));
            double sub = -s, sup = -s;
            double lo2 = 0.0, hi2 = 0.0;
            double rr = rhsf[q];
            const UpwindW sw = upwind_fb_x(p.upwind_order, p.upwind_r, dd, V >= 0 ? 1 : -1, k, n - 1);
            for (int m = 0; m < sw.n; ++m) {
                const double wgt = XMUL(XMUL(half, V), sw.w[m]);
                switch (sw.off[m]) {
                    case 0: diag = XADD(diag, wgt); break;
                    case -1: sub = XADD(sub, wgt); break;
                    case 1: sup = XADD(sup, wgt); break;
                    case -2: lo2 = XADD(lo2, wgt); break;
                    default: hi2 = XADD(hi2, wgt); break;
                }
            }
            if (k == 0) { // sub multiplies the low ghost
                const EdgeSh& g = E[elo];
                rr = XSUB(rr, XMUL(sub, gb[elo * L + line]));
                diag = XADD(diag, XMUL(sub, g.cEdge));
                sup = XADD(sup, XMUL(sub, g.cIn));
                sub = 0.0;
            } else if (k == n - 1) {
                const EdgeSh& g = E[ehi];
                rr = XSUB(rr, XMUL(sup, gb[ehi * L + line]));
                diag = XADD(diag, XMUL(sup, g.cEdge));
                sub = XADD(sub, XMUL(sup, g.cIn));
                sup = 0.0;
            }
            if (banded) {
                brhs[k] = rr;
                band[k * 5 + 2] = diag;
                if (k > 0) band[k * 5 + 1] = sub;
                if (k < n - 1) band[k * 5 + 3] = sup;
                if (lo2 != 0.0) band[k * 5 + 0] = lo2;
                if (hi2 != 0.0) band[k * 5 + 4] = hi2;
            } else {
                rhs[k] = rr;
                di[k] = diag;
                lo[k] = sub;
                up[k] = sup;
            }
        }
        if (banded) {
            solve_banded_x(band, brhs, n);
            for (int k = 0; k < n; ++k) put(k, brhs[k]);
        } else {
            solve_tridiagonal_x(lo, di, up, rhs, wk, n);
            for (int k = 0; k < n; ++k) put(k, rhs[k]);
        }
    }
}

// ---- static line factors ----------------------------------------------------
// Every value implicit_sweep computes for its line matrices depends only on the
// coefficients, the patch conditions (cIn / cEdge / pinned, never the ghost
// offsets b) and the upwind choice: the reference rebuilds and re-eliminates
// them every micro step.  k_adi_factor replays that construction and the
// matrix-only half of the elimination once per engine; the fused step then
// replays only the right-hand-side arithmetic with the stored values - the same
// IEEE operations on the same operands, so results stay bit-identical.
// Table: [set][dir (0 = xi lines, 1 = eta lines)][line < L][k < L][kAdiFac].
constexpr int kAdiFac = 8; // tri: lo, m, wk, adj | banded: f1, f2, B0, B1, B2, adj
constexpr int kAdiAdj = 7; // slot of the ghost-offset coefficient (k = 0: sub, k = n-1: sup)

__host__ __device__ inline size_t adi_factor_doubles(const Params& p) { return (size_t)2 * p.L * p.L * kAdiFac; }

// row k of line `line` after the ghost fold-in (implicit_sweep, microsim.cpp:433-470)
struct AdiRow {
    double diag, sub, sup, lo2, hi2, adj;
    int pinned;
};
__device__ inline AdiRow adi_row(const Params& p, const EdgeSh* E, const double* coef, bool xi_dir, int line,
                                 int k) {
    const int n2 = p.n2, N = p.N;
    const double half = XMUL(0.5, p.mdt);
    const int n = xi_dir ? p.nx + 1 : p.ny + 1;
    const double dd = xi_dir ? p.mdxi : p.mdeta;
    const int elo = xi_dir ? PD_EDGE_W : PD_EDGE_S, ehi = xi_dir ? PD_EDGE_E : PD_EDGE_N;
    AdiRow r{};
    if ((k == 0 && E[elo].pinned) || (k == n - 1 && E[ehi].pinned)) {
        r.pinned = 1;
        r.diag = 1.0; // di = 1, lo = up = 0 (the banded matrix: diagonal 1)
        return r;
    }
    const int i = xi_dir ? k : line, j = xi_dir ? line : k, q = i * n2 + j;
    const double A = xi_dir ? coef[PD_COEF_A * N + q] : coef[PD_COEF_C * N + q];
    const double V = xi_dir ? coef[PD_COEF_VX * N + q] : coef[PD_COEF_VY * N + q];
    const double sc = XDIV(XMUL(half, A), XMUL(dd, dd));
    double diag = XADD(XADD(1.0, XMUL(2.0, sc)), XMUL(XMUL(half, 0.5), coef[PD_COEF_W * N + q]));
    double sub = -sc, sup = -sc, lo2 = 0.0, hi2 = 0.0;
    const UpwindW sw = upwind_fb_x(p.upwind_order, p.upwind_r, dd, V >= 0 ? 1 : -1, k, n - 1);
    for (int m = 0; m < sw.n; ++m) {
        const double wgt = XMUL(XMUL(half, V), sw.w[m]);
        switch (sw.off[m]) {
            case 0: diag = XADD(diag, wgt); break;
            case -1: sub = XADD(sub, wgt); break;
            case 1: sup = XADD(sup, wgt); break;
            case -2: lo2 = XADD(lo2, wgt); break;
            default: hi2 = XADD(hi2, wgt); break;
        }
    }
    double adj = 0.0;
    if (k == 0) {
        adj = sub;
        diag = XADD(diag, XMUL(sub, E[elo].cEdge));
        sup = XADD(sup, XMUL(sub, E[elo].cIn));
        sub = 0.0;
    } else if (k == n - 1) {
        adj = sup;
        diag = XADD(diag, XMUL(sup, E[ehi].cEdge));
        sub = XADD(sub, XMUL(sup, E[ehi].cIn));
        sup = 0.0;
    }
    r.diag = diag;
    r.sub = sub;
    r.sup = sup;
    r.lo2 = lo2;
    r.hi2 = hi2;
    r.adj = adj;
    return r;
}

// One thread per (set, direction, line): rows, then the Thomas factors
// (linalg.cpp:8-25: m_k, w_k) or the pivot-free band elimination (linalg.cpp:43-61).
__global__ void k_adi_factor(Params p, const double* __restrict__ coeffs, int nsets, double* __restrict__ fac) {
    const int kind = p.bc_type == PD_BC_DIRICHLET ? PD_EDGE_DIRICHLET
                   : p.bc_type == PD_BC_ROBIN     ? PD_EDGE_ROBIN
                                                  : PD_EDGE_NEUMANN;
    EdgeSh E[4];
    make_ghost_x(E[PD_EDGE_E], kind, p.w1, p.w2, p.mdxi, +1.0, 0, nullptr, nullptr, nullptr);
    make_ghost_x(E[PD_EDGE_W], kind, p.w1, p.w2, p.mdxi, -1.0, 0, nullptr, nullptr, nullptr);
    make_ghost_x(E[PD_EDGE_N], kind, p.w1, p.w2, p.mdeta, +1.0, 0, nullptr, nullptr, nullptr);
    make_ghost_x(E[PD_EDGE_S], kind, p.w1, p.w2, p.mdeta, -1.0, 0, nullptr, nullptr, nullptr);
    const int L = p.L;
    const int total = nsets * 2 * L;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int set = t / (2 * L), dir = (t / L) % 2, line = t % L;
        const bool xi_dir = dir == 0;
        const int nline = xi_dir ? p.ny : p.nx, n = xi_dir ? p.nx + 1 : p.ny + 1;
        if (line > nline) continue;
        const double* coef = coeffs + (size_t)set * PD_NCOEF * p.N;
        double* F = fac + (((size_t)set * 2 + dir) * L + line) * L * kAdiFac;
        if (p.upwind_order == PD_UPWIND_TWO) {
            double wprev = 0.0;
            for (int k = 0; k < n; ++k) {
                const AdiRow r = adi_row(p, E, coef, xi_dir, line, k);
                const double lo = r.pinned ? 0.0 : r.sub, up = r.pinned ? 0.0 : r.sup;
                const double m = k == 0 ? r.diag : XSUB(r.diag, XMUL(lo, wprev));
                wprev = XDIV(up, m);
                F[k * kAdiFac + 0] = lo;
                F[k * kAdiFac + 1] = m;
                F[k * kAdiFac + 2] = wprev;
                F[k * kAdiFac + kAdiAdj] = r.adj;
            }
        } else {
            // band rows B(r, -2..2) held in the table's slots 2..6 during the elimination
            for (int k = 0; k < n; ++k) {
                const AdiRow r = adi_row(p, E, coef, xi_dir, line, k);
                double* b = F + k * kAdiFac;
                b[0] = b[1] = 0.0;
                b[2] = r.pinned ? 0.0 : (r.lo2 != 0.0 ? r.lo2 : 0.0);
                b[3] = (r.pinned || k == 0) ? 0.0 : r.sub;
                b[4] = r.diag;
                b[5] = (r.pinned || k == n - 1) ? 0.0 : r.sup;
                b[6] = r.pinned ? 0.0 : (r.hi2 != 0.0 ? r.hi2 : 0.0);
                b[kAdiAdj] = r.adj;
            }
            auto B = [&](int row, int off) -> double& { return F[row * kAdiFac + 4 + off]; };
            for (int k = 0; k < n - 1; ++k) {
                const double piv = B(k, 0);
                const int last = min(k + 2, n - 1);
                for (int r = k + 1; r <= last; ++r) {
                    const double f = XDIV(B(r, k - r), piv);
                    F[k * kAdiFac + (r == k + 1 ? 0 : 1)] = f; // multiplier slots f1, f2
                    if (f == 0.0) continue;
                    for (int c = k + 1; c <= min(k + 2, n - 1); ++c) B(r, c - r) = XSUB(B(r, c - r), XMUL(f, B(k, c - k)));
                }
            }
        }
    }
}

// implicit_sweep with the stored line factors (one thread per line): the
// right-hand side as the reference builds it, then the Thomas / band
// substitutions with the stored multipliers, pivots and upper band.
__device__ inline void implicit_sweep_cached(const Params& p, const double* rhsf, double* out, const EdgeSh* E,
                                             const double* gb, const double* val, const double* slope,
                                             const double* fac, double* lsc, bool xi_dir) {
    const int nx = p.nx, ny = p.ny, n2 = p.n2, L = p.L;
    const int nline = xi_dir ? ny : nx;
    const int n = xi_dir ? nx + 1 : ny + 1;
    const int elo = xi_dir ? PD_EDGE_W : PD_EDGE_S, ehi = xi_dir ? PD_EDGE_E : PD_EDGE_N;
    const int slo = xi_dir ? PD_EDGE_S : PD_EDGE_W, shi = xi_dir ? PD_EDGE_N : PD_EDGE_E;
    const bool banded = p.upwind_order != PD_UPWIND_TWO;
    for (int line = threadIdx.x; line <= nline; line += blockDim.x) {
        auto put = [&](int k, double v) {
            if (xi_dir) out[k * n2 + line] = v;
            else out[line * n2 + k] = v;
        };
        if ((line == 0 && E[slo].pinned) || (line == nline && E[shi].pinned)) {
            const int e = line == 0 ? slo : shi;
            for (int k = 0; k < n; ++k) put(k, pinned_value_x(E[e], val + e * L, slope + e * L, k));
            continue;
        }
        const double* F = fac + ((size_t)(xi_dir ? 0 : 1) * L + line) * L * kAdiFac;
        double* rhs = lsc + (size_t)line * 6 * L;
        for (int k = 0; k < n; ++k) {
            const bool pin_lo = k == 0 && E[elo].pinned, pin_hi = k == n - 1 && E[ehi].pinned;
            if (pin_lo || pin_hi) {
                const int e = pin_lo ? elo : ehi;
                rhs[k] = pinned_value_x(E[e], val + e * L, slope + e * L, line);
                continue;
            }
            const int q = xi_dir ? k * n2 + line : line * n2 + k;
            double rr = rhsf[q];
            if (k == 0) rr = XSUB(rr, XMUL(F[kAdiAdj], gb[elo * L + line]));
            else if (k == n - 1) rr = XSUB(rr, XMUL(F[k * kAdiFac + kAdiAdj], gb[ehi * L + line]));
            rhs[k] = rr;
        }
        if (banded) {
            for (int k = 0; k < n - 1; ++k) {
                const int last = min(k + 2, n - 1);
                for (int r = k + 1; r <= last; ++r) {
                    const double f = F[k * kAdiFac + (r == k + 1 ? 0 : 1)];
                    if (f == 0.0) continue;
                    rhs[r] = XSUB(rhs[r], XMUL(f, rhs[k]));
                }
            }
            for (int r = n - 1; r >= 0; --r) {
                double sacc = rhs[r];
                for (int c = r + 1; c <= min(r + 2, n - 1); ++c) sacc = XSUB(sacc, XMUL(F[r * kAdiFac + 4 + (c - r)], rhs[c]));
                rhs[r] = XDIV(sacc, F[r * kAdiFac + 4]);
            }
        } else {
            double prev = XDIV(rhs[0], F[1]);
            rhs[0] = prev;
            for (int k = 1; k < n; ++k) {
                prev = XDIV(XSUB(rhs[k], XMUL(F[k * kAdiFac + 0], prev)), F[k * kAdiFac + 1]);
                rhs[k] = prev;
            }
            for (int k = n - 1; k-- > 0;) {
                prev = XSUB(rhs[k], XMUL(F[k * kAdiFac + 2], prev));
                rhs[k] = prev;
            }
        }
        for (int k = 0; k < n; ++k) put(k, rhs[k]);
    }
}

// K Peaceman-Rachford steps on the shared tile (integrate with Scheme::ADI,
// microsim.cpp:535-548): source at t0 + (step + 1/2) dt, supplied by the host
// as src_time[step] = time(t_mid)/l.  Returns the buffer holding the result.
__device__ inline double* micro_loop_adi(const Params& p, PatchSh& s, const EdgeSh* eg, const double* coef,
                                         const double* src_sp, const double* src_time, double* rhsf,
                                         double* lsc, const double* fac = nullptr) {
    const double half = XMUL(0.5, p.mdt);
    double* u = s.u0;
    double* work = s.u1;
    for (int step = 0; step < p.nt; ++step) {
        const double ft = (src_sp && src_time) ? src_time[step] : 0.0;
        for (int pass = 0; pass < 2; ++pass) {
            const bool xi_dir = pass == 0;
            const double* f = xi_dir ? u : work;
            for (int t = threadIdx.x; t < p.N; t += blockDim.x) {
                const int i = t / p.n2, j = t % p.n2;
                const double G = (src_sp && src_time) ? XMUL(__ldg(src_sp + t), ft) : 0.0;
                rhsf[t] = node_pinned_x(eg, i, j, p.nx, p.ny)
                              ? 0.0
                              : XADD(f[t], XMUL(half, XADD(cross_term_x(p, f, eg, s.gb, coef, i, j, xi_dir), G)));
            }
            __syncthreads();
            if (fac) implicit_sweep_cached(p, rhsf, xi_dir ? work : u, eg, s.gb, s.val, s.slope, fac, lsc, xi_dir);
            else implicit_sweep_x(p, rhsf, xi_dir ? work : u, eg, s.gb, s.val, s.slope, coef, lsc, xi_dir);
            __syncthreads();
        }
    }
    return u;
}

} // namespace pdb200::dev
