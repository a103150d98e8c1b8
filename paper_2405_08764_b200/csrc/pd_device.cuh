// Device-side parameters and the EXACT-mode building blocks.
//
// EXACT mode replays the reference's arithmetic in its evaluation order with
// explicitly rounded IEEE operations (__dadd_rn & co. are never contracted
// into FMA), so for b = 0 a patch evolves bit-identically to the reference's
// CPU build.  Every routine cites the reference lines it follows
// (/root/reference/proj/...).
#pragma once

#include <cstdint>

#include "patchdyn_b200.h"

namespace pdb200::dev {

#define XADD(a, b) __dadd_rn((a), (b))
#define XSUB(a, b) __dsub_rn((a), (b))
#define XMUL(a, b) __dmul_rn((a), (b))
#define XDIV(a, b) __ddiv_rn((a), (b))

// Plain-old-data engine parameters, passed by value to every kernel.
struct Params {
    double a, b, c, d;    // computational rectangle
    double Dxi, Deta;     // CoarseGrid::dxi()/deta()  gaptooth.hpp:21-22
    int Nxi, Neta, NF2;   // NF2 = Neta + 1 (Field2D row length)
    int periodic;
    int nx, ny, n1, n2, N, L, nt, k;
    double tau, dt_macro, h_xi, h_eta;
    double mdxi, mdeta, mdt; // make_micro_grid  microsim.cpp:23
    int bc_type;
    double w1, w2;
    int quad;
    int P, nsets;
    int mixed;  // any B != 0
    int source; // PD_SOURCE_*
    int solver, upwind_order; // PD_SOLVER_*, PD_UPWIND_* (ADI)
    double upwind_r;
    // FAST-mode constants, computed once on the host (no divisions on the device)
    double i2Dxi, i2Deta, iDxi2, iDeta2, i4DD; // 1/(2D), 1/D^2, 1/(4 Dxi Deta)
    double c24x, c24y;                          // h^2/24 (box-average constant of the lift)
    double dlag[4][3];   // Lagrange derivative weights at +-h/2: E, W (xi) and N, S (eta)
    double lagq[33][3];  // Lagrange value weights at the E/W edge nodes Y_j (j < n2)
    double lagp[33][3];  // Lagrange value weights at the N/S edge nodes X_i (i < n1)
    double gsc[4];       // ghost scale +-2 delta per edge (microsim.cpp:166)
    double vlag[4][3];   // Lagrange value weights at +-h/2 across each edge (E, W, N, S): edge values
    double cedge[4];     // Robin ghost coefficient cEdge = -sign 2 delta w1/w2 per edge (microsim.cpp:180)
    int pinned;          // the patch edges pin their nodes (Dirichlet, or Robin with w2 ~ 0)
    // device copy of lagq then lagp ([2][33][3]): the FAST prologues index them by
    // lane (edge node), which through the constant bank serialises per distinct
    // address; through L1 it is one request
    const double* lagtab;
    // fused peer-memory halo of a decomposed run (pd_projective_step_halo): the
    // results of the patches in column halo_col[l] also go to halo_dst[l] (the
    // neighbour's buffer), each followed by a system-scope fence and +1 on
    // *halo_flag[l]; halo_n = 0 everywhere else
    int halo_n;
    int halo_col[2];
    double* halo_dst[2];
    unsigned int* halo_flag[2];
};

// Lagrange value weights at edge node j (E/W edges, lagq) or i (N/S, lagp)
__device__ __forceinline__ double lagq_at(const Params& p, int j, int q) { return __ldg(p.lagtab + 3 * j + q); }
__device__ __forceinline__ double lagp_at(const Params& p, int i, int q) { return __ldg(p.lagtab + 99 + 3 * i + q); }

// Store v (the result at macro node `node`) into the neighbours' buffers when
// the node lies in a halo link's column, then publish it: fence.sc.sys orders
// the (NVLink / IPC) store before the counter increment the neighbour's stream
// waits on (pd_stream_wait_flag).  A uniform no-op when halo_n == 0.
__device__ __forceinline__ void halo_store(const Params& p, size_t node, double v) {
    if (!p.halo_n) return;
    const int i = (int)(node / (size_t)p.NF2);
#pragma unroll
    for (int l = 0; l < 2; ++l) {
        if (l < p.halo_n && i == p.halo_col[l]) {
            p.halo_dst[l][node] = v;
            __threadfence_system();
            atomicAdd_system(p.halo_flag[l], 1u);
        }
    }
}

// One micro edge condition in shared memory (EdgeCondition + Ghost,
// microsim.hpp:32-37, microsim.cpp:146-150).
struct EdgeSh {
    int kind, pinned;
    double cIn, cEdge, w1, w2;
};

// Shared-memory layout of one patch in the EXACT kernels.
struct PatchSh {
    double* u0;    // [N]
    double* u1;    // [N]
    double* val;   // [4][L] edge values
    double* slope; // [4][L] edge slopes
    double* gb;    // [4][L] ghost offsets b[k]
    double* row;   // [n1] restriction row sums
    EdgeSh* edge;  // [4]
    double* stencil; // [9] + xi_c, eta_c
};

__device__ inline size_t patch_smem_doubles(int N, int L, int n1) {
    return 2 * (size_t)N + 3 * 4 * (size_t)L + n1 + 11 + 4 * 6 /* EdgeSh as doubles */;
}

__device__ inline PatchSh carve(double* base, int N, int L, int n1) {
    PatchSh s;
    s.u0 = base;
    s.u1 = s.u0 + N;
    s.val = s.u1 + N;
    s.slope = s.val + 4 * L;
    s.gb = s.slope + 4 * L;
    s.row = s.gb + 4 * L;
    s.stencil = s.row + n1;
    s.edge = reinterpret_cast<EdgeSh*>(s.stencil + 11);
    return s;
}

// ---- tensor Lagrange interpolant  gaptooth.cpp:16-61 -----------------------
__device__ inline void lagrange3_x(double X, double D, double* o) {
    const double invD2 = XDIV(1.0, XMUL(D, D));
    o[0] = XMUL(XMUL(XMUL(0.5, X), XSUB(X, D)), invD2);
    o[1] = XSUB(1.0, XMUL(XMUL(X, X), invD2));
    o[2] = XMUL(XMUL(XMUL(0.5, X), XADD(X, D)), invD2);
}
__device__ inline void lagrange3_deriv_x(double X, double D, double* o) {
    const double invD2 = XDIV(1.0, XMUL(D, D));
    o[0] = XMUL(XSUB(X, XMUL(0.5, D)), invD2);
    o[1] = XMUL(XMUL(-2.0, X), invD2);
    o[2] = XMUL(XADD(X, XMUL(0.5, D)), invD2);
}
// which: 0 eval, 1 d_xi, 2 d_eta
__device__ inline double poly_x(const double* v, double xi_c, double eta_c, double Dxi, double Deta,
                                double xi, double eta, int which) {
    double Lp[3], Lq[3];
    if (which == 1) lagrange3_deriv_x(XSUB(xi, xi_c), Dxi, Lp);
    else lagrange3_x(XSUB(xi, xi_c), Dxi, Lp);
    if (which == 2) lagrange3_deriv_x(XSUB(eta, eta_c), Deta, Lq);
    else lagrange3_x(XSUB(eta, eta_c), Deta, Lq);
    double acc = 0.0;
    for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) acc = XADD(acc, XMUL(XMUL(Lp[p], Lq[q]), v[3 * p + q]));
    return acc;
}

// Edge profiles (slopes and/or values), one element per thread iteration:
// dirichlet_edge_values / neumann_edge_slopes  gaptooth.cpp:110-152.
// (tid, nth): this thread's index and the thread count of the group sharing the patch
__device__ inline void edge_profiles_t(const double* v, double xi_c, double eta_c, double Dxi, double Deta,
                                       double h_xi, double h_eta, int nx, int ny, int L, bool want_slope,
                                       bool want_value, double* slope, double* val, int tid, int nth) {
    const double xiE = XADD(xi_c, XMUL(0.5, h_xi)), xiW = XSUB(xi_c, XMUL(0.5, h_xi));
    const double etaN = XADD(eta_c, XMUL(0.5, h_eta)), etaS = XSUB(eta_c, XMUL(0.5, h_eta));
    const int nEW = ny + 1, total = 2 * (ny + 1) + 2 * (nx + 1);
    for (int t = tid; t < total; t += nth) {
        if (t < 2 * nEW) {
            const int j = t % nEW, e = t < nEW ? PD_EDGE_E : PD_EDGE_W;
            const double eta = XADD(etaS, XDIV(XMUL(h_eta, (double)j), (double)ny));
            const double xi = e == PD_EDGE_E ? xiE : xiW;
            if (want_slope) slope[e * L + j] = poly_x(v, xi_c, eta_c, Dxi, Deta, xi, eta, 1);
            if (want_value) val[e * L + j] = poly_x(v, xi_c, eta_c, Dxi, Deta, xi, eta, 0);
        } else {
            const int u = t - 2 * nEW, i = u % (nx + 1), e = u < nx + 1 ? PD_EDGE_N : PD_EDGE_S;
            const double xi = XADD(xiW, XDIV(XMUL(h_xi, (double)i), (double)nx));
            const double eta = e == PD_EDGE_N ? etaN : etaS;
            if (want_slope) slope[e * L + i] = poly_x(v, xi_c, eta_c, Dxi, Deta, xi, eta, 2);
            if (want_value) val[e * L + i] = poly_x(v, xi_c, eta_c, Dxi, Deta, xi, eta, 0);
        }
    }
}

__device__ inline void edge_profiles_x(const double* v, double xi_c, double eta_c, double Dxi, double Deta,
                                       double h_xi, double h_eta, int nx, int ny, int L, bool want_slope,
                                       bool want_value, double* slope, double* val) {
    edge_profiles_t(v, xi_c, eta_c, Dxi, Deta, h_xi, h_eta, nx, ny, L, want_slope, want_value, slope, val,
                    (int)threadIdx.x, (int)blockDim.x);
}

// StencilPoly::center + lift  gaptooth.cpp:63-72, 154-168
struct LiftConsts {
    double C0, Uxi, Ueta, Uxixi, Uetaeta, Uxieta, gdxi, gdeta;
};
__device__ inline LiftConsts lift_consts_x(const double* v, double Dxi, double Deta, double h_xi, double h_eta,
                                           int nx, int ny) {
    LiftConsts c;
    const double U = v[4];
    c.Uxi = XDIV(XSUB(v[7], v[1]), XMUL(2.0, Dxi));
    c.Ueta = XDIV(XSUB(v[5], v[3]), XMUL(2.0, Deta));
    c.Uxixi = XDIV(XADD(XSUB(v[7], XMUL(2.0, v[4])), v[1]), XMUL(Dxi, Dxi));
    c.Uetaeta = XDIV(XADD(XSUB(v[5], XMUL(2.0, v[4])), v[3]), XMUL(Deta, Deta));
    c.Uxieta = XDIV(XADD(XSUB(XSUB(v[8], v[6]), v[2]), v[0]), XMUL(XMUL(4.0, Dxi), Deta));
    c.C0 = XSUB(XSUB(U, XMUL(XDIV(XMUL(h_xi, h_xi), 24.0), c.Uxixi)),
                XMUL(XDIV(XMUL(h_eta, h_eta), 24.0), c.Uetaeta));
    c.gdxi = XDIV(h_xi, (double)nx);
    c.gdeta = XDIV(h_eta, (double)ny);
    return c;
}
__device__ inline double lift_node_x(const LiftConsts& c, double h_xi, double h_eta, int i, int j) {
    const double X = XADD(XMUL(-0.5, h_xi), XMUL(c.gdxi, (double)i));
    const double Y = XADD(XMUL(-0.5, h_eta), XMUL(c.gdeta, (double)j));
    double r = XADD(c.C0, XMUL(X, c.Uxi));
    r = XADD(r, XMUL(Y, c.Ueta));
    r = XADD(r, XMUL(XMUL(XMUL(0.5, X), X), c.Uxixi));
    r = XADD(r, XMUL(XMUL(X, Y), c.Uxieta));
    r = XADD(r, XMUL(XMUL(XMUL(0.5, Y), Y), c.Uetaeta));
    return r;
}
__device__ inline void lift_x(const double* v, double Dxi, double Deta, double h_xi, double h_eta, int nx,
                              int ny, double* u) {
    const LiftConsts c = lift_consts_x(v, Dxi, Deta, h_xi, h_eta, nx, ny);
    const int n2 = ny + 1, N = (nx + 1) * n2;
    for (int t = threadIdx.x; t < N; t += blockDim.x) u[t] = lift_node_x(c, h_xi, h_eta, t / n2, t % n2);
}

// make_ghost  microsim.cpp:152-186, for edge e (sign +1 on E/N, -1 on W/S).
// Scalars are computed redundantly by every thread; b[k] split across threads.
__device__ inline void make_ghost_t(EdgeSh& g, int kind, double w1, double w2, double delta, double sign,
                                    int len, const double* value, const double* slope, double* b, int tid, int nth) {
    g.kind = kind;
    g.w1 = w1;
    g.w2 = w2;
    g.pinned = 0;
    g.cIn = 0.0;
    g.cEdge = 0.0;
    if (kind == PD_EDGE_DIRICHLET) {
        g.pinned = 1;
        return;
    }
    if (kind == PD_EDGE_NEUMANN) {
        g.cIn = 1.0;
        for (int k = tid; k < len; k += nth) b[k] = XMUL(XMUL(XMUL(sign, 2.0), delta), slope[k]);
        return;
    }
    if (fabs(w2) < 1e-300) {
        g.pinned = 1;
        return;
    }
    g.cIn = 1.0;
    g.cEdge = XDIV(XMUL(XMUL(XMUL(-sign, 2.0), delta), w1), w2);
    for (int k = tid; k < len; k += nth) {
        const double q = XADD(XMUL(w1, value[k]), XMUL(w2, slope[k]));
        b[k] = XDIV(XMUL(XMUL(XMUL(sign, 2.0), delta), q), w2);
    }
}
__device__ inline void make_ghost_x(EdgeSh& g, int kind, double w1, double w2, double delta, double sign,
                                    int len, const double* value, const double* slope, double* b) {
    make_ghost_t(g, kind, w1, w2, delta, sign, len, value, slope, b, (int)threadIdx.x, (int)blockDim.x);
}

// pinned_value  microsim.cpp:189-192
__device__ inline double pinned_value_x(const EdgeSh& g, const double* value, const double* slope, int k) {
    if (g.kind == PD_EDGE_ROBIN) return XADD(value[k], XMUL(XDIV(g.w2, g.w1), slope[k]));
    return value[k];
}

// ghost value at a single edge: cIn*u(inner) + cEdge*u(edge) + b  (microsim.cpp:314-323)
__device__ inline double ghost_x(const EdgeSh& g, double u_inner, double u_edge, double b) {
    return XADD(XADD(XMUL(g.cIn, u_inner), XMUL(g.cEdge, u_edge)), b);
}

// value at (p,q) in [-1,nx+1]x[-1,ny+1] for the mixed term: real node, single
// edge ghost, or the SURVEY B.4 double ghost (see oracle/pd_oracle.c at_ext).
__device__ inline double at_ext_x(const double* u, const EdgeSh* E, const double* gb, int L, int nx, int ny,
                                  int p, int q) {
    const int n2 = ny + 1;
    const bool pin = p >= 0 && p <= nx, qin = q >= 0 && q <= ny;
    if (pin && qin) return u[p * n2 + q];
    if (qin) {
        if (p < 0) return ghost_x(E[PD_EDGE_W], u[n2 + q], u[q], gb[PD_EDGE_W * L + q]);
        return ghost_x(E[PD_EDGE_E], u[(nx - 1) * n2 + q], u[nx * n2 + q], gb[PD_EDGE_E * L + q]);
    }
    if (pin) {
        if (q < 0) return ghost_x(E[PD_EDGE_S], u[p * n2 + 1], u[p * n2], gb[PD_EDGE_S * L + p]);
        return ghost_x(E[PD_EDGE_N], u[p * n2 + ny - 1], u[p * n2 + ny], gb[PD_EDGE_N * L + p]);
    }
    const int ex = p < 0 ? PD_EDGE_W : PD_EDGE_E, ey = q < 0 ? PD_EDGE_S : PD_EDGE_N;
    const int ie = p < 0 ? 0 : nx, je = q < 0 ? 0 : ny;
    const int ii = p < 0 ? 1 : nx - 1, jj = q < 0 ? 1 : ny - 1;
    const double ue = u[ie * n2 + je];
    const double ox = XADD(XMUL(E[ex].cEdge, ue), gb[ex * L + je]);
    const double oy = XADD(XMUL(E[ey].cEdge, ue), gb[ey * L + ie]);
    return XADD(XADD(u[ii * n2 + jj], ox), oy);
}

// One explicit sweep for node (i,j): explicit_sweep body  microsim.cpp:304-331
// (+ mixed term after A*uxx, extension).  coef: [6][N] for this patch.
__device__ inline double sweep_node_x(const double* u, const EdgeSh* E, const double* val, const double* slope,
                                      const double* gb, int L, int nx, int ny, int i, int j, const double* coef,
                                      int N, double G, double idx2, double idy2, double idx, double idy,
                                      double ixy, double dt, bool mixed) {
    const int n2 = ny + 1, k = i * n2 + j;
    const EdgeSh &gE = E[PD_EDGE_E], &gW = E[PD_EDGE_W], &gN = E[PD_EDGE_N], &gS = E[PD_EDGE_S];
    if ((i == 0 && gW.pinned) || (i == nx && gE.pinned) || (j == 0 && gS.pinned) || (j == ny && gN.pinned)) {
        if (i == 0 && gW.pinned) return pinned_value_x(gW, val + PD_EDGE_W * L, slope + PD_EDGE_W * L, j);
        if (i == nx && gE.pinned) return pinned_value_x(gE, val + PD_EDGE_E * L, slope + PD_EDGE_E * L, j);
        if (j == 0 && gS.pinned) return pinned_value_x(gS, val + PD_EDGE_S * L, slope + PD_EDGE_S * L, i);
        return pinned_value_x(gN, val + PD_EDGE_N * L, slope + PD_EDGE_N * L, i);
    }
    const double uc = u[k];
    const double uW = i > 0 ? u[k - n2] : ghost_x(gW, u[n2 + j], u[j], gb[PD_EDGE_W * L + j]);
    const double uE = i < nx ? u[k + n2] : ghost_x(gE, u[(nx - 1) * n2 + j], u[nx * n2 + j], gb[PD_EDGE_E * L + j]);
    const double uS = j > 0 ? u[k - 1] : ghost_x(gS, u[i * n2 + 1], u[i * n2], gb[PD_EDGE_S * L + i]);
    const double uN = j < ny ? u[k + 1] : ghost_x(gN, u[i * n2 + ny - 1], u[i * n2 + ny], gb[PD_EDGE_N * L + i]);
    const double uxx = XMUL(XADD(XSUB(uW, XMUL(2.0, uc)), uE), idx2);
    const double uyy = XMUL(XADD(XSUB(uS, XMUL(2.0, uc)), uN), idy2);
    const double ux = XMUL(XSUB(uE, uW), idx);
    const double uy = XMUL(XSUB(uN, uS), idy);
    double s = XMUL(coef[PD_COEF_A * N + k], uxx);
    if (mixed) {
        const double nE = at_ext_x(u, E, gb, L, nx, ny, i + 1, j + 1);
        const double sE = at_ext_x(u, E, gb, L, nx, ny, i + 1, j - 1);
        const double nW = at_ext_x(u, E, gb, L, nx, ny, i - 1, j + 1);
        const double sW = at_ext_x(u, E, gb, L, nx, ny, i - 1, j - 1);
        const double uxy = XMUL(XADD(XSUB(XSUB(nE, sE), nW), sW), ixy);
        s = XADD(s, XMUL(coef[PD_COEF_B * N + k], uxy));
    }
    s = XADD(s, XMUL(coef[PD_COEF_C * N + k], uyy));
    s = XSUB(s, XMUL(coef[PD_COEF_VX * N + k], ux));
    s = XSUB(s, XMUL(coef[PD_COEF_VY * N + k], uy));
    s = XSUB(s, XMUL(coef[PD_COEF_W * N + k], uc));
    s = XADD(s, G);
    return XADD(uc, XMUL(dt, s));
}

// restrict_average weights  gaptooth.cpp:172-185
__device__ inline double quad_w(int i, int n, int quad) {
    if (quad == PD_QUAD_SIMPSON) {
        const double c = (i == 0 || i == n) ? 1.0 : (i % 2 == 1 ? 4.0 : 2.0);
        return XDIV(c, XMUL(3.0, (double)n));
    }
    return (i == 0 || i == n) ? XDIV(0.5, (double)n) : XDIV(1.0, (double)n);
}

// restrict_average in the reference order (row sums then accumulation,
// gaptooth.cpp:187-193).  Returns the average on thread 0 (others: garbage).
__device__ inline double restrict_x(const double* u, int nx, int ny, int quad, double* row) {
    const int n2 = ny + 1;
    for (int i = threadIdx.x; i <= nx; i += blockDim.x) {
        double r = 0.0;
        for (int j = 0; j <= ny; ++j) r = XADD(r, XMUL(quad_w(j, ny, quad), u[i * n2 + j]));
        row[i] = r;
    }
    __syncthreads();
    double acc = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i <= nx; ++i) acc = XADD(acc, XMUL(quad_w(i, nx, quad), row[i]));
    return acc;
}

// ---- 1D bulk copy (TMA, cp.async.bulk) into shared memory + mbarrier ------
__device__ __forceinline__ unsigned smem_u32(const void* ptr) {
    return static_cast<unsigned>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one lane: expect `bytes` (multiple of 16, 16-byte aligned ends) on the barrier and start the copy
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

} // namespace pdb200::dev
