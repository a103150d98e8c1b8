/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — see pd_oracle.h.  CPU restatement of
 * the reference's explicit gap-tooth path; each function cites the reference
 * lines it follows (paths relative to /root/reference/).  Compiled with
 * -ffp-contract=off so every expression rounds exactly as the reference's
 * x86-64 (SSE2, no FMA) build does.
 */
#include "pd_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 0;

/* perimeter layout of pd_perimeter_len (include/patchdyn_b200.h) */
static size_t perim_len(int Nxi, int Neta) { return 2 * (size_t)(Nxi + 1) + 2 * (size_t)(Neta + 1); }
static char g_err[512];

void pdo_set_threads(int n) { g_threads = n; }
int pdo_get_threads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}
const char* pdo_last_error(void) { return g_err; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ---- tensor Lagrange interpolant  proj/src/gaptooth.cpp:16-72 ------------ */

static void lagrange3(double X, double D, double out[3]) { /* gaptooth.cpp:17-22 */
    const double invD2 = 1.0 / (D * D);
    out[0] = 0.5 * X * (X - D) * invD2;
    out[1] = 1.0 - X * X * invD2;
    out[2] = 0.5 * X * (X + D) * invD2;
}

static void lagrange3_deriv(double X, double D, double out[3]) { /* gaptooth.cpp:24-29 */
    const double invD2 = 1.0 / (D * D);
    out[0] = (X - 0.5 * D) * invD2;
    out[1] = -2.0 * X * invD2;
    out[2] = (X + 0.5 * D) * invD2;
}

typedef struct {
    double xi_c, eta_c, dxi, deta;
    double v[3][3]; /* [p+1][q+1], p along xi  gaptooth.hpp:43-47 */
} stencil_t;

/* StencilPoly::eval / d_xi / d_eta  gaptooth.cpp:33-61; which: 0 eval, 1 d_xi, 2 d_eta */
static double poly(const stencil_t* s, double xi, double eta, int which) {
    double Lp[3], Lq[3];
    if (which == 1) lagrange3_deriv(xi - s->xi_c, s->dxi, Lp);
    else lagrange3(xi - s->xi_c, s->dxi, Lp);
    if (which == 2) lagrange3_deriv(eta - s->eta_c, s->deta, Lq);
    else lagrange3(eta - s->eta_c, s->deta, Lq);
    double acc = 0.0;
    for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) acc += Lp[p] * Lq[q] * s->v[p][q];
    return acc;
}

/* edge profiles, E,W along eta (len ny+1) and N,S along xi (len nx+1):
 * dirichlet_edge_values / neumann_edge_slopes  gaptooth.cpp:110-152 */
static void edge_profiles(const stencil_t* s, double h_xi, double h_eta, int nx, int ny, int L,
                          double* slopes, double* values) {
    const double xiE = s->xi_c + 0.5 * h_xi, xiW = s->xi_c - 0.5 * h_xi;
    const double etaN = s->eta_c + 0.5 * h_eta, etaS = s->eta_c - 0.5 * h_eta;
    for (int j = 0; j <= ny; ++j) {
        const double eta = etaS + h_eta * j / ny;
        if (slopes) {
            slopes[PD_EDGE_E * L + j] = poly(s, xiE, eta, 1);
            slopes[PD_EDGE_W * L + j] = poly(s, xiW, eta, 1);
        }
        if (values) {
            values[PD_EDGE_E * L + j] = poly(s, xiE, eta, 0);
            values[PD_EDGE_W * L + j] = poly(s, xiW, eta, 0);
        }
    }
    for (int i = 0; i <= nx; ++i) {
        const double xi = xiW + h_xi * i / nx;
        if (slopes) {
            slopes[PD_EDGE_N * L + i] = poly(s, xi, etaN, 2);
            slopes[PD_EDGE_S * L + i] = poly(s, xi, etaS, 2);
        }
        if (values) {
            values[PD_EDGE_N * L + i] = poly(s, xi, etaN, 0);
            values[PD_EDGE_S * L + i] = poly(s, xi, etaS, 0);
        }
    }
}

/* StencilPoly::center + lift  gaptooth.cpp:63-72, 154-168 */
static void lift(const stencil_t* s, double h_xi, double h_eta, int nx, int ny, double* u) {
    const double (*v)[3] = s->v;
    const double U = v[1][1];
    const double Uxi = (v[2][1] - v[0][1]) / (2.0 * s->dxi);
    const double Ueta = (v[1][2] - v[1][0]) / (2.0 * s->deta);
    const double Uxixi = (v[2][1] - 2.0 * v[1][1] + v[0][1]) / (s->dxi * s->dxi);
    const double Uetaeta = (v[1][2] - 2.0 * v[1][1] + v[1][0]) / (s->deta * s->deta);
    const double Uxieta = (v[2][2] - v[2][0] - v[0][2] + v[0][0]) / (4.0 * s->dxi * s->deta);
    const double C0 = U - h_xi * h_xi / 24.0 * Uxixi - h_eta * h_eta / 24.0 * Uetaeta;
    const double gdxi = h_xi / nx, gdeta = h_eta / ny; /* make_micro_grid  microsim.cpp:23 */
    for (int i = 0; i <= nx; ++i) {
        const double X = -0.5 * h_xi + gdxi * i;
        for (int j = 0; j <= ny; ++j) {
            const double Y = -0.5 * h_eta + gdeta * j;
            u[i * (ny + 1) + j] = C0 + X * Uxi + Y * Ueta + 0.5 * X * X * Uxixi + X * Y * Uxieta +
                                  0.5 * Y * Y * Uetaeta;
        }
    }
}

void pdo_lift(const double vals[9], double xi_c, double eta_c, double dxi, double deta,
              double h_xi, double h_eta, int nx, int ny, double* u0, double* slopes,
              double* values) {
    stencil_t s;
    s.xi_c = xi_c;
    s.eta_c = eta_c;
    s.dxi = dxi;
    s.deta = deta;
    memcpy(s.v, vals, sizeof(s.v));
    const int L = (nx > ny ? nx : ny) + 1;
    if (u0) lift(&s, h_xi, h_eta, nx, ny, u0);
    edge_profiles(&s, h_xi, h_eta, nx, ny, L, slopes, values);
}

/* restrict_average  gaptooth.cpp:170-194 */
static void quad_weights(int n, int q, double* w) {
    for (int i = 0; i <= n; ++i) {
        if (q == PD_QUAD_SIMPSON) {
            const double c = (i == 0 || i == n) ? 1.0 : (i % 2 == 1 ? 4.0 : 2.0);
            w[i] = c / (3.0 * n);
        } else {
            w[i] = (i == 0 || i == n) ? 0.5 / n : 1.0 / n;
        }
    }
}

double pdo_restrict(const double* u, int n1, int n2, int quadrature) {
    const int nx = n1 - 1, ny = n2 - 1;
    double wx[1024], wy[1024];
    quad_weights(nx, quadrature, wx);
    quad_weights(ny, quadrature, wy);
    double acc = 0.0;
    for (int i = 0; i <= nx; ++i) {
        double row = 0.0;
        for (int j = 0; j <= ny; ++j) row += wy[j] * u[i * n2 + j];
        acc += wx[i] * row;
    }
    return acc;
}

/* ---- micro-solver  proj/src/microsim.cpp:146-196, 292-332, 509-552 -------- */

typedef struct {
    int pinned;
    double cIn, cEdge;
    double* b; /* [len] */
    int kind;
    const double* value;
    const double* slope;
    double w1, w2;
} ghost_t;

/* make_ghost  microsim.cpp:152-186 (shape checks are the caller's job) */
static void make_ghost(ghost_t* g, int kind, const double* value, const double* slope, double w1,
                       double w2, double delta, double sign, int len, double* bbuf) {
    g->pinned = 0;
    g->cIn = 0.0;
    g->cEdge = 0.0;
    g->b = bbuf;
    g->kind = kind;
    g->value = value;
    g->slope = slope;
    g->w1 = w1;
    g->w2 = w2;
    if (kind == PD_EDGE_DIRICHLET) {
        g->pinned = 1;
        return;
    }
    if (kind == PD_EDGE_NEUMANN) {
        g->cIn = 1.0;
        for (int k = 0; k < len; ++k) bbuf[k] = sign * 2.0 * delta * slope[k];
        return;
    }
    if (fabs(w2) < 1e-300) { /* pure-value Robin behaves as Dirichlet */
        g->pinned = 1;
        return;
    }
    g->cIn = 1.0;
    g->cEdge = -sign * 2.0 * delta * w1 / w2;
    for (int k = 0; k < len; ++k) {
        const double q = w1 * value[k] + w2 * slope[k];
        bbuf[k] = sign * 2.0 * delta * q / w2;
    }
}

/* pinned_value  microsim.cpp:189-192 */
static double pinned_value(const ghost_t* g, int k) {
    if (g->kind == PD_EDGE_ROBIN) return g->value[k] + g->w2 / g->w1 * g->slope[k];
    return g->value[k];
}

typedef struct {
    int nx, ny;
    const double* u;
    const ghost_t *E, *W, *N, *S;
} field_t;

#define U_(f, i, j) ((f)->u[(i) * ((f)->ny + 1) + (j)])

/* value at (p,q) with p in [-1,nx+1], q in [-1,ny+1]: real node, single-edge
 * ghost (microsim.cpp:314-323 rule), or the Appendix B.4 double ghost
 * u(inner diagonal) + offset_edge1(corner) + offset_edge2(corner) with
 * offset = cEdge*u(edge node) + b. */
static double at_ext(const field_t* f, int p, int q) {
    const int nx = f->nx, ny = f->ny;
    const int pin = p >= 0 && p <= nx, qin = q >= 0 && q <= ny;
    if (pin && qin) return U_(f, p, q);
    if (qin) {
        if (p < 0) return f->W->cIn * U_(f, 1, q) + f->W->cEdge * U_(f, 0, q) + f->W->b[q];
        return f->E->cIn * U_(f, nx - 1, q) + f->E->cEdge * U_(f, nx, q) + f->E->b[q];
    }
    if (pin) {
        if (q < 0) return f->S->cIn * U_(f, p, 1) + f->S->cEdge * U_(f, p, 0) + f->S->b[p];
        return f->N->cIn * U_(f, p, ny - 1) + f->N->cEdge * U_(f, p, ny) + f->N->b[p];
    }
    const ghost_t* gx = p < 0 ? f->W : f->E;
    const ghost_t* gy = q < 0 ? f->S : f->N;
    const int ie = p < 0 ? 0 : nx, je = q < 0 ? 0 : ny;      /* corner node */
    const int ii = p < 0 ? 1 : nx - 1, jj = q < 0 ? 1 : ny - 1; /* inner diagonal */
    const double ox = gx->cEdge * U_(f, ie, je) + gx->b[je];
    const double oy = gy->cEdge * U_(f, ie, je) + gy->b[ie];
    return U_(f, ii, jj) + ox + oy;
}

/* ---- ADI micro-solver  microsim.cpp:56-138 (upwind), 334-507 (adi_sweep),
 *      linalg.cpp:8-61 (line solvers) ------------------------------------- */

typedef struct {
    int off[4];
    double w[4];
    int n;
} upw_t;

/* make_upwind  microsim.cpp:65-104 (order: PD_UPWIND_*) */
static upw_t make_upwind(int order, double r, double delta, int vel_sign) {
    upw_t s;
    memset(&s, 0, sizeof s);
    const double s1 = vel_sign >= 0 ? 1.0 : -1.0;
    if (order == PD_UPWIND_TWO) {
        s.n = 2;
        s.off[0] = 0;
        s.off[1] = vel_sign >= 0 ? -1 : 1;
        s.w[0] = s1 / delta;
        s.w[1] = -s1 / delta;
    } else if (order == PD_UPWIND_THREE) {
        s.n = 3;
        s.off[0] = 0;
        s.off[1] = vel_sign >= 0 ? -1 : 1;
        s.off[2] = vel_sign >= 0 ? -2 : 2;
        s.w[0] = 3.0 * s1 / (2 * delta);
        s.w[1] = -4.0 * s1 / (2 * delta);
        s.w[2] = s1 / (2 * delta);
    } else {
        s.n = 4;
        if (vel_sign >= 0) {
            s.off[0] = 1;  s.w[0] = 1.0 / (2 * delta) - r / (3 * delta);
            s.off[1] = -1; s.w[1] = -1.0 / (2 * delta) - r / delta;
            s.off[2] = -2; s.w[2] = r / (3 * delta);
            s.off[3] = 0;  s.w[3] = r / delta;
        } else {
            s.off[0] = 1;  s.w[0] = 1.0 / (2 * delta) + r / delta;
            s.off[1] = -1; s.w[1] = -1.0 / (2 * delta) + r / (3 * delta);
            s.off[2] = 2;  s.w[2] = -r / (3 * delta);
            s.off[3] = 0;  s.w[3] = -r / delta;
        }
    }
    return s;
}

/* upwind_with_fallback  microsim.cpp:107-119 */
static upw_t upwind_fb(int order, double r, double delta, int vel_sign, int i, int imax) {
    if (order != PD_UPWIND_TWO) {
        const upw_t s = make_upwind(order, r, delta, vel_sign);
        int ok = 1;
        for (int k = 0; k < s.n; ++k) {
            const int idx = i + s.off[k];
            if (idx < 0 || idx > imax) ok = 0;
        }
        if (ok) return s;
    }
    return make_upwind(PD_UPWIND_TWO, r, delta, vel_sign);
}

typedef struct {
    int nx, ny, N, order;
    double dxi, deta, half, r;
    const double *A, *C, *Vx, *Vy, *W;
    const ghost_t *E, *Wg, *Ng, *S;
} adi_t;

/* cross_term  microsim.cpp:357-395 */
static double cross_term(const adi_t* a, const double* f, int i, int j, int eta_dir) {
    const int nx = a->nx, ny = a->ny, n2 = ny + 1, k = i * n2 + j;
    if (eta_dir) {
        const double glo = a->S->cIn * f[i * n2 + 1] + a->S->cEdge * f[i * n2] + (a->S->b ? a->S->b[i] : 0.0);
        const double ghi = a->Ng->cIn * f[i * n2 + ny - 1] + a->Ng->cEdge * f[i * n2 + ny] + (a->Ng->b ? a->Ng->b[i] : 0.0);
        const double um = j > 0 ? f[k - 1] : glo;
        const double up = j < ny ? f[k + 1] : ghi;
        const double uc = f[k];
        const double uyy = (um - 2.0 * uc + up) / (a->deta * a->deta);
        const double v = a->Vy[k];
        const upw_t sw = upwind_fb(a->order, a->r, a->deta, v >= 0 ? 1 : -1, j, ny);
        double du = 0.0;
        for (int m = 0; m < sw.n; ++m) {
            const int jj = j + sw.off[m];
            const double val = jj < 0 ? glo : (jj > ny ? ghi : f[i * n2 + jj]);
            du += sw.w[m] * val;
        }
        return a->C[k] * uyy - v * du - 0.5 * a->W[k] * uc;
    }
    const double glo = a->Wg->cIn * f[n2 + j] + a->Wg->cEdge * f[j] + (a->Wg->b ? a->Wg->b[j] : 0.0);
    const double ghi = a->E->cIn * f[(nx - 1) * n2 + j] + a->E->cEdge * f[nx * n2 + j] + (a->E->b ? a->E->b[j] : 0.0);
    const double um = i > 0 ? f[k - n2] : glo;
    const double up = i < nx ? f[k + n2] : ghi;
    const double uc = f[k];
    const double uxx = (um - 2.0 * uc + up) / (a->dxi * a->dxi);
    const double v = a->Vx[k];
    const upw_t sw = upwind_fb(a->order, a->r, a->dxi, v >= 0 ? 1 : -1, i, nx);
    double du = 0.0;
    for (int m = 0; m < sw.n; ++m) {
        const int ii = i + sw.off[m];
        const double val = ii < 0 ? glo : (ii > nx ? ghi : f[ii * n2 + j]);
        du += sw.w[m] * val;
    }
    return a->A[k] * uxx - v * du - 0.5 * a->W[k] * uc;
}

/* solve_tridiagonal  linalg.cpp:8-25 */
static void solve_tridiagonal(const double* lo, const double* di, const double* up, double* rhs, double* wk, int n) {
    double m = di[0];
    wk[0] = up[0] / m;
    rhs[0] /= m;
    for (int k = 1; k < n; ++k) {
        m = di[k] - lo[k] * wk[k - 1];
        wk[k] = up[k] / m;
        rhs[k] = (rhs[k] - lo[k] * rhs[k - 1]) / m;
    }
    for (int k = n - 1; k-- > 0;) rhs[k] -= wk[k] * rhs[k + 1];
}

/* BandedMatrix(n,2,2)::solve  linalg.cpp:43-61; band[r*5 + (c-r) + 2] */
static void solve_banded(double* band, double* rhs, int n) {
    for (int k = 0; k < n - 1; ++k) {
        const double piv = band[k * 5 + 2];
        const int last = k + 2 < n - 1 ? k + 2 : n - 1;
        for (int r = k + 1; r <= last; ++r) {
            const double f = band[r * 5 + (k - r) + 2] / piv;
            if (f == 0.0) continue;
            const int cmax = k + 2 < n - 1 ? k + 2 : n - 1;
            for (int c = k + 1; c <= cmax; ++c) band[r * 5 + (c - r) + 2] -= f * band[k * 5 + (c - k) + 2];
            rhs[r] -= f * rhs[k];
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        double s = rhs[r];
        const int cmax = r + 2 < n - 1 ? r + 2 : n - 1;
        for (int c = r + 1; c <= cmax; ++c) s -= band[r * 5 + (c - r) + 2] * rhs[c];
        rhs[r] = s / band[r * 5 + 2];
    }
}

/* implicit_sweep  microsim.cpp:402-491: (I - half*L_swept) out = rhs_field */
static void implicit_sweep(const adi_t* a, const double* rhsf, double* out, int xi_dir, double* sc) {
    const int nx = a->nx, ny = a->ny, n2 = ny + 1;
    const int nline = xi_dir ? ny : nx, n = xi_dir ? nx + 1 : ny + 1;
    const double dd = xi_dir ? a->dxi : a->deta;
    const ghost_t* glo = xi_dir ? a->Wg : a->S;
    const ghost_t* ghi = xi_dir ? a->E : a->Ng;
    const ghost_t* slo = xi_dir ? a->S : a->Wg;
    const ghost_t* shi = xi_dir ? a->Ng : a->E;
    const int banded = a->order != PD_UPWIND_TWO;
    double *lo = sc, *di = sc + n, *up = sc + 2 * n, *rhs = sc + 3 * n, *wk = sc + 4 * n;
    double* band = sc;
    double* brhs = sc + 5 * n;
    for (int line = 0; line <= nline; ++line) {
        if ((line == 0 && slo->pinned) || (line == nline && shi->pinned)) {
            const ghost_t* e = line == 0 ? slo : shi;
            for (int k = 0; k < n; ++k) {
                if (xi_dir) out[k * n2 + line] = pinned_value(e, k);
                else out[line * n2 + k] = pinned_value(e, k);
            }
            continue;
        }
        if (banded) memset(band, 0, sizeof(double) * 5 * n);
        for (int k = 0; k < n; ++k) {
            const int pin_lo = k == 0 && glo->pinned, pin_hi = k == n - 1 && ghi->pinned;
            if (pin_lo || pin_hi) {
                const double pv = pinned_value(pin_lo ? glo : ghi, line);
                if (banded) { band[k * 5 + 2] = 1.0; brhs[k] = pv; }
                else { di[k] = 1.0; lo[k] = 0.0; up[k] = 0.0; rhs[k] = pv; }
                continue;
            }
            const int i = xi_dir ? k : line, j = xi_dir ? line : k, q = i * n2 + j;
            const double A = xi_dir ? a->A[q] : a->C[q];
            const double V = xi_dir ? a->Vx[q] : a->Vy[q];
            const double s = a->half * A / (dd * dd);
            double diag = 1.0 + 2.0 * s + a->half * 0.5 * a->W[q];
            double sub = -s, sup = -s, lo2 = 0.0, hi2 = 0.0;
            double rr = rhsf[q];
            const upw_t sw = upwind_fb(a->order, a->r, dd, V >= 0 ? 1 : -1, k, n - 1);
            for (int m = 0; m < sw.n; ++m) {
                const double wgt = a->half * V * sw.w[m];
                switch (sw.off[m]) {
                    case 0: diag += wgt; break;
                    case -1: sub += wgt; break;
                    case 1: sup += wgt; break;
                    case -2: lo2 += wgt; break;
                    default: hi2 += wgt; break;
                }
            }
            if (k == 0) {
                rr -= sub * glo->b[line];
                diag += sub * glo->cEdge;
                sup += sub * glo->cIn;
                sub = 0.0;
            } else if (k == n - 1) {
                rr -= sup * ghi->b[line];
                diag += sup * ghi->cEdge;
                sub += sup * ghi->cIn;
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
                rhs[k] = rr; di[k] = diag; lo[k] = sub; up[k] = sup;
            }
        }
        const double* res = banded ? brhs : rhs;
        if (banded) solve_banded(band, brhs, n);
        else solve_tridiagonal(lo, di, up, rhs, wk, n);
        for (int k = 0; k < n; ++k) {
            if (xi_dir) out[k * n2 + line] = res[k];
            else out[line * n2 + k] = res[k];
        }
    }
}

static int node_pinned(const adi_t* a, int i, int j) {
    return (i == 0 && a->Wg->pinned) || (i == a->nx && a->E->pinned) || (j == 0 && a->S->pinned) ||
           (j == a->ny && a->Ng->pinned);
}

/* adi_sweep  microsim.cpp:334-507 (one Peaceman-Rachford step, u in place) */
static void adi_sweep(const adi_t* a, const double* G, double* u, double* work, double* rhsf, double* sc) {
    const int nx = a->nx, ny = a->ny, n2 = ny + 1;
    for (int i = 0; i <= nx; ++i)
        for (int j = 0; j <= ny; ++j)
            rhsf[i * n2 + j] = node_pinned(a, i, j) ? 0.0 : u[i * n2 + j] + a->half * (cross_term(a, u, i, j, 1) + G[i * n2 + j]);
    implicit_sweep(a, rhsf, work, 1, sc);
    for (int i = 0; i <= nx; ++i)
        for (int j = 0; j <= ny; ++j)
            rhsf[i * n2 + j] = node_pinned(a, i, j) ? 0.0 : work[i * n2 + j] + a->half * (cross_term(a, work, i, j, 0) + G[i * n2 + j]);
    implicit_sweep(a, rhsf, u, 0, sc);
}

int pdo_integrate(const double* coef, int nx, int ny, int nt, double h_xi, double h_eta,
                  double tau, const int* kinds, const double* values, const double* slopes,
                  const double* robin_w, const double* src_spatial, const double* src_time,
                  double* u) {
    return pdo_integrate_ex(coef, nx, ny, nt, h_xi, h_eta, tau, kinds, values, slopes, robin_w, src_spatial,
                            src_time, u, PD_SOLVER_EXPLICIT, PD_UPWIND_TWO, 0.5);
}

int pdo_integrate_ex(const double* coef, int nx, int ny, int nt, double h_xi, double h_eta,
                     double tau, const int* kinds, const double* values, const double* slopes,
                     const double* robin_w, const double* src_spatial, const double* src_time,
                     double* u, int solver, int upwind_order, double upwind_r) {
    const int n1 = nx + 1, n2 = ny + 1, L = (n1 > n2 ? n1 : n2), N = n1 * n2;
    /* make_micro_grid  microsim.cpp:18-24 */
    const double dxi = h_xi / nx, deta = h_eta / ny, dt = tau / nt;
    const double *A = coef, *B = coef + N, *C = coef + 2 * N, *Vx = coef + 3 * N,
                 *Vy = coef + 4 * N, *W = coef + 5 * N;
    int mixed = 0;
    for (int k = 0; k < N; ++k)
        if (B[k] != 0.0) mixed = 1;
    double* buf = (double*)malloc(sizeof(double) * (2 * N + 4 * L));
    if (!buf) return PD_VALIDATION_ERROR;
    double* next = buf;
    double* G = buf + N;
    double* bb = buf + 2 * N;
    ghost_t gE, gW, gN, gS;
    const double w0[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const double* rw = robin_w ? robin_w : w0;
    /* GhostSet  microsim.cpp:297-300 (built once: edges are frozen over the horizon) */
    make_ghost(&gE, kinds[PD_EDGE_E], values + PD_EDGE_E * L, slopes + PD_EDGE_E * L, rw[0], rw[1], dxi, +1.0, n2, bb + 0 * L);
    make_ghost(&gW, kinds[PD_EDGE_W], values + PD_EDGE_W * L, slopes + PD_EDGE_W * L, rw[2], rw[3], dxi, -1.0, n2, bb + 1 * L);
    make_ghost(&gN, kinds[PD_EDGE_N], values + PD_EDGE_N * L, slopes + PD_EDGE_N * L, rw[4], rw[5], deta, +1.0, n1, bb + 2 * L);
    make_ghost(&gS, kinds[PD_EDGE_S], values + PD_EDGE_S * L, slopes + PD_EDGE_S * L, rw[6], rw[7], deta, -1.0, n1, bb + 3 * L);
    if (mixed && (kinds[0] == PD_EDGE_ROBIN || kinds[1] == PD_EDGE_ROBIN || kinds[2] == PD_EDGE_ROBIN ||
                  kinds[3] == PD_EDGE_ROBIN)) {
        /* our extension defines corner ghosts for Neumann/Dirichlet only */
        snprintf(g_err, sizeof g_err, "mixed-derivative term with Robin patch edges is not supported");
        free(buf);
        return PD_MIXED_TERM_UNSUPPORTED;
    }
    /* Dirichlet edges pin their nodes from the start  microsim.cpp:521-530 */
    if (kinds[PD_EDGE_W] == PD_EDGE_DIRICHLET)
        for (int j = 0; j <= ny; ++j) u[0 * n2 + j] = values[PD_EDGE_W * L + j];
    if (kinds[PD_EDGE_E] == PD_EDGE_DIRICHLET)
        for (int j = 0; j <= ny; ++j) u[nx * n2 + j] = values[PD_EDGE_E * L + j];
    if (kinds[PD_EDGE_S] == PD_EDGE_DIRICHLET)
        for (int i = 0; i <= nx; ++i) u[i * n2 + 0] = values[PD_EDGE_S * L + i];
    if (kinds[PD_EDGE_N] == PD_EDGE_DIRICHLET)
        for (int i = 0; i <= nx; ++i) u[i * n2 + ny] = values[PD_EDGE_N * L + i];

    if (solver == PD_SOLVER_ADI) {
        if (mixed) {
            snprintf(g_err, sizeof g_err, "mixed-derivative term with the ADI micro-solver is not defined");
            free(buf);
            return PD_MIXED_TERM_UNSUPPORTED;
        }
        adi_t a = {nx, ny, N, upwind_order, dxi, deta, 0.5 * dt, upwind_r, A, C, Vx, Vy, W, &gE, &gW, &gN, &gS};
        double* abuf = (double*)malloc(sizeof(double) * (2 * (size_t)N + 6 * (size_t)L));
        for (int step = 0; step < nt; ++step) {
            /* sample_source at t0 + (step + 1/2) dt  microsim.cpp:536-537 (src_time carries it) */
            if (src_spatial && src_time) {
                const double ft = src_time[step];
                for (int k = 0; k < N; ++k) G[k] = src_spatial[k] * ft;
            } else {
                for (int k = 0; k < N; ++k) G[k] = 0.0;
            }
            adi_sweep(&a, G, u, abuf, abuf + N, abuf + 2 * N);
        }
        free(abuf);
        free(buf);
        return PD_OK;
    }
    const double idx2 = 1.0 / (dxi * dxi), idy2 = 1.0 / (deta * deta);
    const double idx = 1.0 / (2.0 * dxi), idy = 1.0 / (2.0 * deta);
    const double ixy = 1.0 / (4.0 * dxi * deta); /* extension: u_xi_eta scale */
    double* cur = u;
    double* nxt = next;
    for (int step = 0; step < nt; ++step) {
        /* sample_source  microsim.cpp:265-281 (static coefficients: co0_) */
        if (src_spatial && src_time) {
            const double ft = src_time[step];
            for (int k = 0; k < N; ++k) G[k] = src_spatial[k] * ft;
        } else {
            for (int k = 0; k < N; ++k) G[k] = 0.0;
        }
        field_t f = {nx, ny, cur, &gE, &gW, &gN, &gS};
        /* explicit_sweep  microsim.cpp:292-332 */
        for (int i = 0; i <= nx; ++i) {
            for (int j = 0; j <= ny; ++j) {
                const int k = i * n2 + j;
                if ((i == 0 && gW.pinned) || (i == nx && gE.pinned) || (j == 0 && gS.pinned) ||
                    (j == ny && gN.pinned)) {
                    if (i == 0 && gW.pinned) nxt[k] = pinned_value(&gW, j);
                    else if (i == nx && gE.pinned) nxt[k] = pinned_value(&gE, j);
                    else if (j == 0 && gS.pinned) nxt[k] = pinned_value(&gS, i);
                    else nxt[k] = pinned_value(&gN, i);
                    continue;
                }
                const double uc = cur[k];
                const double uW = (i > 0) ? cur[k - n2] : gW.cIn * cur[n2 + j] + gW.cEdge * cur[j] + gW.b[j];
                const double uE = (i < nx) ? cur[k + n2]
                                           : gE.cIn * cur[(nx - 1) * n2 + j] + gE.cEdge * cur[nx * n2 + j] + gE.b[j];
                const double uS = (j > 0) ? cur[k - 1] : gS.cIn * cur[i * n2 + 1] + gS.cEdge * cur[i * n2] + gS.b[i];
                const double uN = (j < ny) ? cur[k + 1]
                                           : gN.cIn * cur[i * n2 + ny - 1] + gN.cEdge * cur[i * n2 + ny] + gN.b[i];
                const double uxx = (uW - 2.0 * uc + uE) * idx2;
                const double uyy = (uS - 2.0 * uc + uN) * idy2;
                const double ux = (uE - uW) * idx;
                const double uy = (uN - uS) * idy;
                if (!mixed) {
                    nxt[k] = uc + dt * (A[k] * uxx + C[k] * uyy - Vx[k] * ux - Vy[k] * uy - W[k] * uc + G[k]);
                } else {
                    /* extension: same term order as StencilPoly::center's Uxieta (gaptooth.cpp:70) */
                    const double uxy = (at_ext(&f, i + 1, j + 1) - at_ext(&f, i + 1, j - 1) -
                                        at_ext(&f, i - 1, j + 1) + at_ext(&f, i - 1, j - 1)) * ixy;
                    nxt[k] = uc + dt * (A[k] * uxx + B[k] * uxy + C[k] * uyy - Vx[k] * ux - Vy[k] * uy -
                                        W[k] * uc + G[k]);
                }
            }
        }
        double* tmp = cur; /* std::swap(u, next)  microsim.cpp:548 */
        cur = nxt;
        nxt = tmp;
    }
    if (cur != u) memcpy(u, cur, sizeof(double) * N);
    free(buf);
    return PD_OK;
}

/* ---- engine level  gaptooth.cpp:251-375, cpi.cpp:46-77, 134-216 ---------- */

typedef struct {
    const pd_engine_desc* d;
    int P;
    int* pij;        /* [P][2] */
    const int* cset; /* [P] or NULL */
    int n1, n2, L;
    const double* row_w; /* [Neta+1][9] linear-response weights, or NULL = direct path */
} eng_t;

static int eng_init(eng_t* e, const pd_engine_desc* d) {
    e->d = d;
    e->n1 = d->nx + 1;
    e->n2 = d->ny + 1;
    e->L = e->n1 > e->n2 ? e->n1 : e->n2;
    e->cset = d->coeff_set;
    e->row_w = NULL;
    if (d->patch_ij) {
        e->P = d->npatches;
        e->pij = (int*)malloc(sizeof(int) * 2 * e->P);
        memcpy(e->pij, d->patch_ij, sizeof(int) * 2 * e->P);
        return 0;
    }
    /* patch list order  gaptooth.cpp:251-280 */
    const int i_lo = d->periodic_xi ? 0 : 1, i_hi = d->Nxi - 1;
    e->P = (i_hi - i_lo + 1) * (d->Neta - 1);
    e->pij = (int*)malloc(sizeof(int) * 2 * e->P);
    int p = 0;
    for (int j = 1; j <= d->Neta - 1; ++j)
        for (int i = i_lo; i <= i_hi; ++i) {
            e->pij[2 * p] = i;
            e->pij[2 * p + 1] = j;
            ++p;
        }
    return 0;
}

static void eng_free(eng_t* e) { free(e->pij); }

/* refresh_boundary from a perimeter array, or keep + periodic seam  gaptooth.cpp:296-310 */
static void refresh(const pd_engine_desc* d, double* U, const double* bnd) {
    const int N1 = d->Nxi, N2 = d->Neta, n2 = N2 + 1;
    if (bnd) {
        const double *S = bnd, *Nn = bnd + (N1 + 1), *Wv = bnd + 2 * (N1 + 1), *Ev = Wv + (N2 + 1);
        for (int i = 0; i <= N1; ++i) {
            U[i * n2 + 0] = S[i];
            U[i * n2 + N2] = Nn[i];
        }
        if (!d->periodic_xi)
            for (int j = 0; j <= N2; ++j) {
                U[0 * n2 + j] = Wv[j];
                U[N1 * n2 + j] = Ev[j];
            }
    }
    if (d->periodic_xi)
        for (int j = 0; j <= N2; ++j) U[N1 * n2 + j] = U[0 * n2 + j];
}

/* one patch: build_stencil + evolve_patch  gaptooth.cpp:74-104, 312-353 */
/* vals != NULL: evolve the given 3x3 values with patch p's integrator and
 * centre instead of gathering them from F (build_row_weights, gaptooth.cpp:377-394). */
static int evolve_patch_vals(const eng_t* e, const double* vals, const double* F, int p, double t,
                             const double* src_time, double* work, double* avg) {
    const pd_engine_desc* d = e->d;
    const int i = e->pij[2 * p], j = e->pij[2 * p + 1];
    const int n1 = e->n1, n2 = e->n2, L = e->L, N = n1 * n2, NF2 = d->Neta + 1;
    if (j < 1 || j > d->Neta - 1 || (!d->periodic_xi && (i < 1 || i > d->Nxi - 1))) {
        snprintf(g_err, sizeof g_err, "patch (%d,%d): stencil centre outside interior", i, j);
        return PD_MACRO_PATCH_ERROR;
    }
    stencil_t s;
    s.dxi = (d->b - d->a) / d->Nxi; /* CoarseGrid::dxi  gaptooth.hpp:21 */
    s.deta = (d->d - d->c) / d->Neta;
    s.eta_c = d->c + s.deta * j;
    if (d->periodic_xi) {
        const int iw = ((i % d->Nxi) + d->Nxi) % d->Nxi;
        s.xi_c = d->a + s.dxi * iw;
        for (int pp = -1; pp <= 1; ++pp) {
            const int ip = ((iw + pp) % d->Nxi + d->Nxi) % d->Nxi;
            for (int q = -1; q <= 1; ++q) s.v[pp + 1][q + 1] = vals ? vals[3 * (pp + 1) + q + 1] : F[ip * NF2 + j + q];
        }
    } else {
        s.xi_c = d->a + s.dxi * i;
        for (int pp = -1; pp <= 1; ++pp)
            for (int q = -1; q <= 1; ++q)
                s.v[pp + 1][q + 1] = vals ? vals[3 * (pp + 1) + q + 1] : F[(i + pp) * NF2 + j + q];
    }
    double* u = work;
    double* slopes = work + N;
    double* values = slopes + 4 * L;
    int kinds[4];
    double rw[8];
    const int bc = d->bc_type;
    for (int k = 0; k < 4; ++k) {
        kinds[k] = bc == PD_BC_DIRICHLET ? PD_EDGE_DIRICHLET : bc == PD_BC_ROBIN ? PD_EDGE_ROBIN : PD_EDGE_NEUMANN;
        rw[2 * k] = d->robin_w1;
        rw[2 * k + 1] = d->robin_w2;
    }
    edge_profiles(&s, d->h_xi, d->h_eta, d->nx, d->ny, L, (bc != PD_BC_DIRICHLET) ? slopes : NULL,
                  (bc != PD_BC_NEUMANN) ? values : NULL);
    lift(&s, d->h_xi, d->h_eta, d->nx, d->ny, u);
    const int set = e->cset ? e->cset[p] : p;
    const double* coef = d->coeffs + (size_t)set * PD_NCOEF * N;
    const double* sp = (d->source_kind == PD_SOURCE_SEPARABLE && d->source_spatial)
                           ? d->source_spatial + (size_t)set * N : NULL;
    const int st = pdo_integrate_ex(coef, d->nx, d->ny, d->nt, d->h_xi, d->h_eta, d->tau, kinds, values,
                                    slopes, rw, sp, sp ? src_time : NULL, u, d->solver, d->upwind_order, d->upwind_r);
    if (st != PD_OK) return st;
    *avg = pdo_restrict(u, n1, n2, d->quadrature);
    (void)t;
    return PD_OK;
}

static int evolve_patch(const eng_t* e, const double* F, int p, double t, const double* src_time,
                        double* work, double* avg) {
    return evolve_patch_vals(e, NULL, F, p, t, src_time, work, avg);
}

static size_t work_len(const eng_t* e) { return (size_t)e->n1 * e->n2 + 8 * e->L; }

/* GapToothEngine::step, linear-response path  gaptooth.cpp:396-418 */
static void linear_step(const eng_t* e, const double* F, double* out, const double* bnd) {
    const pd_engine_desc* d = e->d;
    const int N1 = d->Nxi, NF2 = d->Neta + 1;
    const size_t NF = (size_t)(N1 + 1) * NF2;
    memcpy(out, F, sizeof(double) * NF);
    const int i_lo = d->periodic_xi ? 0 : 1, i_hi = N1 - 1;
    for (int j = 1; j <= d->Neta - 1; ++j) {
        const double* w = e->row_w + 9 * j;
        for (int i = i_lo; i <= i_hi; ++i) {
            double acc = 0.0;
            for (int p = -1; p <= 1; ++p) {
                int ip = i + p;
                if (d->periodic_xi) ip = ((ip % N1) + N1) % N1;
                for (int q = -1; q <= 1; ++q) acc += w[3 * (p + 1) + q + 1] * F[ip * NF2 + j + q];
            }
            out[i * NF2 + j] = acc;
        }
    }
    refresh(d, out, bnd);
}

static int step_direct(const eng_t* e, const double* F, double* out, double t, const double* bnd,
                       const double* src_time) {
    const pd_engine_desc* d = e->d;
    if (e->row_w) {
        linear_step(e, F, out, bnd);
        return PD_OK;
    }
    const size_t NF = (size_t)(d->Nxi + 1) * (d->Neta + 1);
    memcpy(out, F, sizeof(double) * NF); /* CoarseField out = F  gaptooth.cpp:361 */
    int status = PD_OK;
#pragma omp parallel num_threads(pdo_get_threads())
    {
        double* work = (double*)malloc(sizeof(double) * work_len(e));
#pragma omp for schedule(dynamic, 16)
        for (int p = 0; p < e->P; ++p) {
            double avg;
            const int st = evolve_patch(e, F, p, t, src_time, work, &avg);
            if (st != PD_OK) {
#pragma omp critical
                if (status == PD_OK) status = st;
            } else {
                out[e->pij[2 * p] * (d->Neta + 1) + e->pij[2 * p + 1]] = avg;
            }
        }
        free(work);
    }
    refresh(d, out, bnd); /* refresh_boundary(out, t+tau)  gaptooth.cpp:373 */
    return status;
}

int pdo_gaptooth_step(const pd_engine_desc* d, const double* U_in, double* U_out, double t,
                      const double* bnd, const double* src_time) {
    eng_t e;
    eng_init(&e, d);
    const int st = step_direct(&e, U_in, U_out, t, bnd, src_time);
    eng_free(&e);
    return st;
}

static int projective(const eng_t* e, const double* U, double* out, double t, const double* bnd,
                      const double* src_time) {
    const pd_engine_desc* d = e->d;
    const int k = d->k, N1 = d->Nxi, N2 = d->Neta, n2 = N2 + 1;
    const size_t NF = (size_t)(N1 + 1) * n2, perim = perim_len(N1, N2);
    double* chain = (double*)malloc(sizeof(double) * NF * (k + 2));
    memcpy(chain, U, sizeof(double) * NF);
    int st = PD_OK;
    /* chain of k+1 gap-tooth substeps  cpi.cpp:62-65 */
    for (int m = 0; m <= k && st == PD_OK; ++m)
        st = step_direct(e, chain + NF * m, chain + NF * (m + 1), t + m * d->tau,
                         bnd ? bnd + perim * m : NULL, src_time ? src_time + (size_t)d->nt * m : NULL);
    if (st == PD_OK) {
        const double* Uk = chain + NF * k;
        const double* Uk1 = chain + NF * (k + 1);
        memcpy(out, U, sizeof(double) * NF);
        const int i_lo = d->periodic_xi ? 0 : 1;
        const double horizon = d->dt_macro - k * d->tau;
        for (int i = i_lo; i <= N1 - 1; ++i)
            for (int j = 1; j <= N2 - 1; ++j) {
                /* estimate_derivative  cpi.cpp:46-56; extrapolation  cpi.cpp:68-74 */
                const double F = (Uk1[i * n2 + j] - Uk[i * n2 + j]) / d->tau;
                out[i * n2 + j] = Uk[i * n2 + j] + horizon * F;
            }
        refresh(d, out, bnd ? bnd + perim * (k + 1) : NULL); /* cpi.cpp:75 */
    }
    free(chain);
    return st;
}

int pdo_projective_step(const pd_engine_desc* d, const double* U_in, double* U_out, double t,
                        const double* bnd, const double* src_time) {
    eng_t e;
    eng_init(&e, d);
    const int st = projective(&e, U_in, U_out, t, bnd, src_time);
    eng_free(&e);
    return st;
}

/* cpi::run's macro loop with the blow-up guard  cpi.cpp:142-202.  U must hold
 * the initial field with its boundary already refreshed at t0. */
static int run_impl(const pd_engine_desc* d, const double* row_w, double* U, int nsteps, double t0,
                    const double* bnd, const double* src_time, pd_run_stats* stats);
int pdo_run(const pd_engine_desc* d, double* U, int nsteps, double t0, const double* bnd,
            const double* src_time, pd_run_stats* stats) {
    return run_impl(d, NULL, U, nsteps, t0, bnd, src_time, stats);
}
int pdo_linear_run(const pd_engine_desc* d, const double* row_w, double* U, int nsteps, double t0,
                   const double* bnd, pd_run_stats* stats) {
    return run_impl(d, row_w, U, nsteps, t0, bnd, NULL, stats);
}
static int run_impl(const pd_engine_desc* d, const double* row_w, double* U, int nsteps, double t0,
                    const double* bnd, const double* src_time, pd_run_stats* stats) {
    eng_t e;
    eng_init(&e, d);
    e.row_w = row_w;
    const size_t NF = (size_t)(d->Nxi + 1) * (d->Neta + 1), perim = perim_len(d->Nxi, d->Neta);
    double scale0 = 0.0;
    for (size_t q = 0; q < NF; ++q) scale0 = fmax(scale0, fabs(U[q]));
    const double blowup = 10.0 * fmax(scale0, 1e-12);
    double* tmp = (double*)malloc(sizeof(double) * NF);
    int st = PD_OK;
    pd_run_stats s;
    memset(&s, 0, sizeof s);
    s.blowup_threshold = blowup;
    const double tstart = now_s();
    for (int n = 0; n < nsteps; ++n) {
        const double t = t0 + n * d->dt_macro;
        st = projective(&e, U, tmp, t, bnd ? bnd + perim * (d->k + 2) * n : NULL,
                        src_time ? src_time + (size_t)d->nt * (d->k + 1) * n : NULL);
        if (st != PD_OK) break;
        memcpy(U, tmp, sizeof(double) * NF);
        double umax = 0.0;
        int finite = 1;
        for (size_t q = 0; q < NF; ++q) {
            if (!isfinite(U[q])) {
                finite = 0;
                break;
            }
            umax = fmax(umax, fabs(U[q]));
        }
        if (!finite || umax > blowup) {
            s.failed_step = n + 1;
            s.failed_nonfinite = !finite;
            snprintf(g_err, sizeof g_err, "coarse field %s at macro step %d",
                     finite ? "exceeded 10x the initial magnitude" : "became non-finite", n + 1);
            st = PD_MACRO_INSTABILITY;
            break;
        }
        s.steps_done = n + 1;
        s.umax_last = umax;
    }
    s.device_ms = 1e3 * (now_s() - tstart);
    if (stats) *stats = s;
    free(tmp);
    eng_free(&e);
    return st;
}

double pdo_patch_subset(const pd_engine_desc* d, const double* U_in, double t, int nsub,
                        const int* patch_index, double* avg_out) {
    eng_t e;
    eng_init(&e, d);
    const double t0 = now_s();
    int bad = 0;
#pragma omp parallel num_threads(pdo_get_threads())
    {
        double* work = (double*)malloc(sizeof(double) * work_len(&e));
#pragma omp for schedule(dynamic, 8)
        for (int s = 0; s < nsub; ++s) {
            if (evolve_patch(&e, U_in, patch_index[s], t, NULL, work, &avg_out[s]) != PD_OK) {
#pragma omp atomic write
                bad = 1;
            }
        }
        free(work);
    }
    const double dt = now_s() - t0;
    eng_free(&e);
    return bad ? -dt : dt;
}

/* ---- linear-response path  gaptooth.cpp:377-418 --------------------------- */

int pdo_evolve_batch(const pd_engine_desc* d, int n, const int* patch_index, const double* stencils, double t,
                     double* out) {
    eng_t e;
    eng_init(&e, d);
    int status = PD_OK;
    double* work = (double*)malloc(sizeof(double) * work_len(&e));
    for (int m = 0; m < n && status == PD_OK; ++m) {
        if (patch_index[m] < 0 || patch_index[m] >= e.P) {
            snprintf(g_err, sizeof g_err, "patch index %d outside [0,%d)", patch_index[m], e.P);
            status = PD_INDEX_OUT_OF_RANGE;
            break;
        }
        status = evolve_patch_vals(&e, stencils + 9 * (size_t)m, NULL, patch_index[m], t, NULL, work, &out[m]);
    }
    free(work);
    eng_free(&e);
    return status;
}

/* build_row_weights: the 9 unit-impulse responses of row j's integrator,
 * centred at (xi(i0), eta(j)), i0 = periodic ? 0 : 1; row_w [Neta+1][9]
 * (rows 0 and Neta left zero). */
int pdo_linear_weights(const pd_engine_desc* d, double* row_w) {
    eng_t e;
    eng_init(&e, d);
    const int i0 = d->periodic_xi ? 0 : 1;
    memset(row_w, 0, sizeof(double) * 9 * (d->Neta + 1));
    int status = PD_OK;
    double* work = (double*)malloc(sizeof(double) * work_len(&e));
    for (int j = 1; j <= d->Neta - 1 && status == PD_OK; ++j) {
        int p = -1;
        for (int q = 0; q < e.P; ++q)
            if (e.pij[2 * q] == i0 && e.pij[2 * q + 1] == j) {
                p = q;
                break;
            }
        if (p < 0) {
            snprintf(g_err, sizeof g_err, "row %d has no patch at i = %d", j, i0);
            status = PD_VALIDATION_ERROR;
            break;
        }
        for (int k = 0; k < 9 && status == PD_OK; ++k) {
            double vals[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            vals[k] = 1.0;
            status = evolve_patch_vals(&e, vals, NULL, p, 0.0, NULL, work, &row_w[9 * j + k]);
        }
    }
    free(work);
    eng_free(&e);
    return status;
}

int pdo_linear_step(const pd_engine_desc* d, const double* row_w, const double* U_in, double* U_out,
                    const double* bnd) {
    eng_t e;
    eng_init(&e, d);
    e.row_w = row_w;
    linear_step(&e, U_in, U_out, bnd);
    eng_free(&e);
    return PD_OK;
}

int pdo_linear_projective_step(const pd_engine_desc* d, const double* row_w, const double* U_in, double* U_out,
                               double t, const double* bnd) {
    eng_t e;
    eng_init(&e, d);
    e.row_w = row_w;
    const int st = projective(&e, U_in, U_out, t, bnd, NULL);
    eng_free(&e);
    return st;
}
