// EXACT-mode fused gap-tooth step on the register-blocked tile mapping.
//
// Same arithmetic as k_gaptooth_exact (kernels_exact.cuh): every operation an
// explicitly rounded IEEE add / mul / div in the reference's evaluation order,
// never contracted into FMA, so a patch evolves bit-identically to the
// reference's CPU build (microsim.cpp:292-332, 509-552; gaptooth.cpp:110-194).
// What changes is where the data lives: the mapping of kernels_fast.cuh.  A
// patch of N1 x N2 micro nodes is split into BI x BJ node blocks, one block per
// lane (LP lanes per patch, G = 32/LP patches per warp, one warp per CTA); the
// lane keeps its nodes' state and their six solver-form coefficients in
// REGISTERS for all K micro-steps, and neighbour values cross lanes through
// constant-delta warp shuffles.  The shared-memory kernel it replaces re-read
// the coefficient tables from global memory and the state from shared memory at
// every micro-step, with one CTA barrier per step.
//
// Scope: the explicit micro-solver with zero or separable source and any patch
// condition (Neumann / Robin ghosts; pinned Dirichlet or degenerate-Robin edges and
// the source each run their own copy of the step loop; both together do not), on
// the exact-fit tiles 7x7, 8x8, 9x9, 11x11, 16x16 (one warp per unit) and 32x32
// (one four-warp CTA per patch, k_exact_big), with or without the mixed term.
// Everything else stays on k_gaptooth_exact (exact_tile_plan).
#pragma once

#include <cstdlib>
#include <type_traits>

#include "pd_device.cuh"
#include "kernels_exact.cuh"

namespace pdb200::dev {

// resident warps per SM the mixed-term instantiations are compiled for (8: 216 registers,
// no spills, config 4 9.01 ms per step; 10: 168 registers with 18 local accesses per
// micro-step, 9.61 ms)
#ifndef PD_XT_MIXED_BLOCKS
#define PD_XT_MIXED_BLOCKS 8
#endif

// the same for the 5-point tiles (12: 168 registers; 8: 218 registers, config 2 27.9 -> 30.0 us per launch)
#ifndef PD_XT_PLAIN_BLOCKS
#define PD_XT_PLAIN_BLOCKS 12
#endif

// micro-steps per loop trip: 2 lets ptxas overlap a step's tail with the next one's halo exchange
// (config 4 9.01 -> 8.85 ms, config 2 28.3 -> 28.0 us per launch)
#ifndef PD_XT_UNROLL
#define PD_XT_UNROLL 2
#endif
constexpr int kXtUnroll = PD_XT_UNROLL;

template <int N1_, int N2_, int BI_, int BJ_, bool MIXED_>
struct XTileCfg {
    static constexpr int N1 = N1_, N2 = N2_, BI = BI_, BJ = BJ_;
    static constexpr bool MIXED = MIXED_;
    static constexpr int LI = N1 / BI, LJ = N2 / BJ, LP = LI * LJ, G = 32 / LP;
    static constexpr int N = N1 * N2, L = N1 > N2 ? N1 : N2;
    // resident one-warp CTAs per SM the kernel is compiled for (register budget 65536 / (32 MINB))
    static constexpr int MINB = (MIXED || BI * BJ > 9) ? PD_XT_MIXED_BLOCKS : PD_XT_PLAIN_BLOCKS;
    static_assert(N1 % BI == 0 && N2 % BJ == 0, "block must tile the patch");
    static_assert(LP <= 32, "patch must fit a warp");
    // a lane on the W edge must not also be on the E edge (its inner node would
    // be a ghost): at least two block columns; along eta one block column is fine
    // when the block itself holds the inner nodes
    static_assert(LI >= 2 && (LJ >= 2 || BJ >= 3), "edge lanes need real inner nodes");
};

// ghost value of an unpinned edge: cIn u(inner) + cEdge u(edge) + b with
// cIn = 1 (make_ghost, microsim.cpp:160-183; explicit_sweep :314-323).
// 1.0 * x is x for every double, so that product is not issued.
__device__ __forceinline__ double ghost_t(double cEdge, double u_inner, double u_edge, double b) {
    return XADD(XADD(u_inner, XMUL(cEdge, u_edge)), b);
}

// a where (role & MASK) == WANT, else b: a selp by construction (written as a
// conditional, the compiler turned these lane-role selections into divergent
// branches with a warp reconvergence each — 15 % of the step loop's samples)
enum { ROLE_W = 1, ROLE_E = 2, ROLE_S = 4, ROLE_N = 8 };
template <int MASK, int WANT>
__device__ __forceinline__ double pick(int role, double a, double b) {
    double r;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %3, %4;\n\tsetp.eq.s32 p, t, %5;\n\t"
        "selp.f64 %0, %1, %2, p;\n\t}"
        : "=d"(r)
        : "d"(a), "d"(b), "r"(role), "n"(MASK), "n"(WANT));
    return r;
}

// One explicit sweep of a lane's BI x BJ block, halo entries of E already
// filled from the neighbouring lanes: ghost values on the patch edges, then
// the reference's update of every own node (explicit_sweep, microsim.cpp:304-331,
// + the mixed term after A*uxx).  Shared by the one-warp tiles and the 32x32 CTA tile.
template <int BI, int BJ, bool MIXED, bool MERGE_ETA, bool PIN, bool SRC = false, int NS = 0>
__device__ __forceinline__ void xt_sweep(double (&E)[BI + 2][BJ + 2], const double (&co)[PD_NCOEF][BI][BJ], int role,
                                         double cEx, double cEs, double cEn, double cEy, const double* gbx,
                                         const double* gbs, const double* gbn, const double* gby, double idx2,
                                         double idy2, double idx, double idy, double ixy, double dt,
                                         const double* spn = nullptr, double ft = 0.0) {
    constexpr int B0 = MIXED ? -1 : 0, B1 = MIXED ? BJ : BJ - 1; // rows / columns whose halo is needed
    constexpr int A0 = MIXED ? -1 : 0, A1 = MIXED ? BI : BI - 1;
    // Patch edges: replace what the shuffles brought by the ghost values
    // (explicit_sweep, microsim.cpp:314-323; at_ext_x for the mixed term's
    // diagonal neighbours).  Every formula reads own nodes or halo entries
    // that are real nodes for this lane, never an entry written here.
    // S / N ghosts of the columns a in [A0, A1] inside the patch (the halo
    // columns a = -1 / BI only where they are not past the W / E edge)
#pragma unroll
    for (int a = A0; a <= A1; ++a) {
        constexpr int W_ = ROLE_W, E_ = ROLE_E, S_ = ROLE_S, N_ = ROLE_N;
        double gsv, gnv;
        if constexpr (MERGE_ETA) {
            const double inner = pick<N_, N_>(role, E[a + 1][BJ - 1], E[a + 1][2]);
            const double edge = pick<N_, N_>(role, E[a + 1][BJ], E[a + 1][1]);
            gsv = gnv = ghost_t(cEy, inner, edge, gby[a + 1]);
        } else {
            gsv = ghost_t(cEs, E[a + 1][2], E[a + 1][1], gbs[a + 1]);
            gnv = ghost_t(cEn, E[a + 1][BJ - 1], E[a + 1][BJ], gbn[a + 1]);
        }
        if (a == -1) {
            E[a + 1][0] = pick<S_ | W_, S_>(role, gsv, E[a + 1][0]);
            E[a + 1][BJ + 1] = pick<N_ | W_, N_>(role, gnv, E[a + 1][BJ + 1]);
        } else if (a == BI) {
            E[a + 1][0] = pick<S_ | E_, S_>(role, gsv, E[a + 1][0]);
            E[a + 1][BJ + 1] = pick<N_ | E_, N_>(role, gnv, E[a + 1][BJ + 1]);
        } else {
            E[a + 1][0] = pick<S_, S_>(role, gsv, E[a + 1][0]);
            E[a + 1][BJ + 1] = pick<N_, N_>(role, gnv, E[a + 1][BJ + 1]);
        }
    }
    // W / E ghosts of the rows b in [B0, B1] inside the patch (one xi role per lane)
#pragma unroll
    for (int b = B0; b <= B1; ++b) {
        constexpr int W_ = ROLE_W, E_ = ROLE_E, S_ = ROLE_S, N_ = ROLE_N;
        const double inner = pick<E_, E_>(role, E[BI - 1][b + 1], E[2][b + 1]);
        const double edge = pick<E_, E_>(role, E[BI][b + 1], E[1][b + 1]);
        const double gv = ghost_t(cEx, inner, edge, gbx[b + 1]);
        if (b == -1) {
            E[0][b + 1] = pick<W_ | S_, W_>(role, gv, E[0][b + 1]);
            E[BI + 1][b + 1] = pick<E_ | S_, E_>(role, gv, E[BI + 1][b + 1]);
        } else if (b == BJ) {
            E[0][b + 1] = pick<W_ | N_, W_>(role, gv, E[0][b + 1]);
            E[BI + 1][b + 1] = pick<E_ | N_, E_>(role, gv, E[BI + 1][b + 1]);
        } else {
            E[0][b + 1] = pick<W_, W_>(role, gv, E[0][b + 1]);
            E[BI + 1][b + 1] = pick<E_, E_>(role, gv, E[BI + 1][b + 1]);
        }
    }
    if constexpr (MIXED) {
        // patch corners: the double ghost u(ii, jj) + ox + oy (at_ext_x),
        // computed by every lane, kept by the corner lanes
        constexpr int W_ = ROLE_W, E_ = ROLE_E, S_ = ROLE_S, N_ = ROLE_N;
        if constexpr (MERGE_ETA) { // at most one corner per lane: one computation
            const double ue = pick<N_, N_>(role, pick<E_, E_>(role, E[BI][BJ], E[1][BJ]),
                                           pick<E_, E_>(role, E[BI][1], E[1][1]));
            const double ui = pick<N_, N_>(role, pick<E_, E_>(role, E[BI - 1][BJ - 1], E[2][BJ - 1]),
                                           pick<E_, E_>(role, E[BI - 1][2], E[2][2]));
            const double bxc = pick<N_, N_>(role, gbx[BJ], gbx[1]);
            const double byc = pick<E_, E_>(role, gby[BI], gby[1]);
            const double ox = XADD(XMUL(cEx, ue), bxc);
            const double oy = XADD(XMUL(cEy, ue), byc);
            const double cv = XADD(XADD(ui, ox), oy);
            E[BI + 1][0] = pick<S_ | E_, S_ | E_>(role, cv, E[BI + 1][0]);
            E[0][0] = pick<S_ | W_, S_ | W_>(role, cv, E[0][0]);
            E[BI + 1][BJ + 1] = pick<N_ | E_, N_ | E_>(role, cv, E[BI + 1][BJ + 1]);
            E[0][BJ + 1] = pick<N_ | W_, N_ | W_>(role, cv, E[0][BJ + 1]);
        } else {
            {
                const double ue = pick<E_, E_>(role, E[BI][1], E[1][1]);
                const double ox = XADD(XMUL(cEx, ue), gbx[1]);
                const double by = pick<E_, E_>(role, gbs[BI], gbs[1]);
                const double ui = pick<E_, E_>(role, E[BI - 1][2], E[2][2]);
                const double oy = XADD(XMUL(cEs, ue), by);
                const double cv = XADD(XADD(ui, ox), oy);
                E[BI + 1][0] = pick<S_ | E_, S_ | E_>(role, cv, E[BI + 1][0]);
                E[0][0] = pick<S_ | W_, S_ | W_>(role, cv, E[0][0]);
            }
            {
                const double ue = pick<E_, E_>(role, E[BI][BJ], E[1][BJ]);
                const double ox = XADD(XMUL(cEx, ue), gbx[BJ]);
                const double by = pick<E_, E_>(role, gbn[BI], gbn[1]);
                const double ui = pick<E_, E_>(role, E[BI - 1][BJ - 1], E[2][BJ - 1]);
                const double oy = XADD(XMUL(cEn, ue), by);
                const double cv = XADD(XADD(ui, ox), oy);
                E[BI + 1][BJ + 1] = pick<N_ | E_, N_ | E_>(role, cv, E[BI + 1][BJ + 1]);
                E[0][BJ + 1] = pick<N_ | W_, N_ | W_>(role, cv, E[0][BJ + 1]);
            }
        }
    }
    double nu[BI][BJ];
#pragma unroll
    for (int ii = 0; ii < BI; ++ii)
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
            const double uc = E[ii + 1][jj + 1];
            const double uW = E[ii][jj + 1], uE = E[ii + 2][jj + 1];
            const double uS = E[ii + 1][jj], uN = E[ii + 1][jj + 2];
            const double uc2 = XMUL(2.0, uc);
            const double uxx = XMUL(XADD(XSUB(uW, uc2), uE), idx2);
            const double uyy = XMUL(XADD(XSUB(uS, uc2), uN), idy2);
            const double ux = XMUL(XSUB(uE, uW), idx);
            const double uy = XMUL(XSUB(uN, uS), idy);
            double s = XMUL(co[PD_COEF_A][ii][jj], uxx);
            if constexpr (MIXED) {
                const double nE = E[ii + 2][jj + 2], sE = E[ii + 2][jj], nW = E[ii][jj + 2], sW = E[ii][jj];
                const double uxy = XMUL(XADD(XSUB(XSUB(nE, sE), nW), sW), ixy);
                s = XADD(s, XMUL(co[PD_COEF_B][ii][jj], uxy));
            }
            s = XADD(s, XMUL(co[PD_COEF_C][ii][jj], uyy));
            s = XSUB(s, XMUL(co[PD_COEF_VX][ii][jj], ux));
            s = XSUB(s, XMUL(co[PD_COEF_VY][ii][jj], uy));
            s = XSUB(s, XMUL(co[PD_COEF_W][ii][jj], uc));
            // + G (microsim.cpp:329): zero, or the separable source spatial(node) * time(t)/l of
            // sample_source (microsim.cpp:272-277); spn = this lane's block in the staged table
            double G = 0.0;
            if constexpr (SRC) G = XMUL(spn[ii * NS + jj], ft);
            s = XADD(s, G);
            nu[ii][jj] = XADD(uc, XMUL(dt, s));
        }
    if constexpr (PIN) {
        // pinned edges (Dirichlet, or Robin with w2 ~ 0): the edge nodes take their pinned value,
        // first match in W, E, S, N order (explicit_sweep, microsim.cpp:306-311); the rows gb*
        // hold pinned values instead of ghost offsets then.  Applied in reverse so W wins.
        constexpr int W_ = ROLE_W, E_ = ROLE_E, S_ = ROLE_S, N_ = ROLE_N;
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) {
                if (jj == BJ - 1) nu[ii][jj] = pick<N_, N_>(role, gbn[ii + 1], nu[ii][jj]);
                if (jj == 0) nu[ii][jj] = pick<S_, S_>(role, gbs[ii + 1], nu[ii][jj]);
                if (ii == BI - 1) nu[ii][jj] = pick<E_, E_>(role, gbx[jj + 1], nu[ii][jj]);
                if (ii == 0) nu[ii][jj] = pick<W_, W_>(role, gbx[jj + 1], nu[ii][jj]);
            }
    }
#pragma unroll
    for (int ii = 0; ii < BI; ++ii)
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) E[ii + 1][jj + 1] = nu[ii][jj];
}

// Dirichlet edges pin their nodes from the start (integrate, microsim.cpp:521-530: W, E, S, N in
// turn, the later edge winning at corners); val rows are the padded pinned-value rows.
template <int BI, int BJ>
__device__ __forceinline__ void xt_pin_initial(double (&E)[BI + 2][BJ + 2], int role, const double* gbx,
                                               const double* gbs, const double* gbn) {
    constexpr int W_ = ROLE_W, E_ = ROLE_E, S_ = ROLE_S, N_ = ROLE_N;
#pragma unroll
    for (int ii = 0; ii < BI; ++ii)
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
            double u = E[ii + 1][jj + 1];
            if (ii == 0) u = pick<W_, W_>(role, gbx[jj + 1], u);
            if (ii == BI - 1) u = pick<E_, E_>(role, gbx[jj + 1], u);
            if (jj == 0) u = pick<S_, S_>(role, gbs[ii + 1], u);
            if (jj == BJ - 1) u = pick<N_, N_>(role, gbn[ii + 1], u);
            E[ii + 1][jj + 1] = u;
        }
}

// Edge kind of the patch conditions (evolve_patch, gaptooth.cpp:312-353) and the pinned node
// values of one edge (pinned_value, microsim.cpp:189-192) into its padded row.
__device__ __forceinline__ int xt_edge_kind(const Params& p) {
    return p.bc_type == PD_BC_DIRICHLET ? PD_EDGE_DIRICHLET : p.bc_type == PD_BC_ROBIN ? PD_EDGE_ROBIN : PD_EDGE_NEUMANN;
}
__device__ __forceinline__ void xt_pinned_row(const EdgeSh& g, const double* value, const double* slope, double* row,
                                              int len, int tid, int nth) {
    for (int k = tid; k < len; k += nth) row[k] = pinned_value_x(g, value, slope, k);
}

template <class Cfg>
__global__ void __launch_bounds__(32, Cfg::MINB)
k_exact_tile(Params p, const double* __restrict__ F, double* __restrict__ out, int out_mode,
             const int* __restrict__ pij, const int* __restrict__ cset, const double* __restrict__ coeffs,
             const int* __restrict__ fail_flag, int nunits, const double* __restrict__ src_sp,
             const double* __restrict__ src_time) {
    constexpr int BI = Cfg::BI, BJ = Cfg::BJ, LI = Cfg::LI, LJ = Cfg::LJ, LP = Cfg::LP, G = Cfg::G;
    constexpr int N1 = Cfg::N1, N2 = Cfg::N2, N = Cfg::N, L = Cfg::L;
    constexpr int nx = N1 - 1, ny = N2 - 1;
    constexpr bool MIXED = Cfg::MIXED;
    __shared__ double s_st[G][9];
    __shared__ double s_slope[G][4][L], s_val[G][4][L];
    // ghost offsets b[k] per edge, one pad entry at each end: the step loop reads rows / columns
    // j0 - 1 .. j0 + BJ with immediate offsets (the out-of-range ends are never selected)
    __shared__ double s_gb[G][4][L + 2];
    __shared__ double s_u[G][N];
    __shared__ double s_row[G][N1];
    if (fail_flag && *fail_flag) return;
    const int unit = blockIdx.x;
    if (unit >= nunits) return;
    const int lane = threadIdx.x;
    const int g = lane / LP, r = lane % LP;
    const int gs = g < G ? g : 0;
    const int patch = unit * G + g;
    const bool valid = g < G && patch < p.P;
    const int bi = r % LI, bj = r / LI;
    const int i0 = bi * BI, j0 = bj * BJ;
    const bool isW = bi == 0, isE = bi == LI - 1, isS = bj == 0, isN = bj == LJ - 1;
    int role = (isW ? ROLE_W : 0) | (isE ? ROLE_E : 0) | (isS ? ROLE_S : 0) | (isN ? ROLE_N : 0);
    asm volatile("mov.b32 %0, %0;" : "+r"(role)); // one live register, not re-derived from the lane id per use

    // ---- build_stencil (gaptooth.cpp:74-104) ----------------------------------
    int pi = 0, pj = 0, ic = 0;
    if (valid) {
        pi = pij[2 * patch];
        pj = pij[2 * patch + 1];
        ic = pi;
        if (p.periodic) ic = ((pi % p.Nxi) + p.Nxi) % p.Nxi;
        for (int t = r; t < 9; t += LP) {
            const int dp = t / 3 - 1, dq = t % 3 - 1;
            const int ip = p.periodic ? ((ic + dp) % p.Nxi + p.Nxi) % p.Nxi : pi + dp;
            s_st[gs][t] = F[(size_t)ip * p.NF2 + pj + dq];
        }
    }
    __syncwarp();
    const double* v = s_st[gs];
    const double xi_c = XADD(p.a, XMUL(p.Dxi, (double)ic));
    const double eta_c = XADD(p.c, XMUL(p.Deta, (double)pj));

    // ---- edge profiles and ghost offsets (gaptooth.cpp:110-152, microsim.cpp:152-186)
    const int kind = xt_edge_kind(p);
    if (valid) {
        edge_profiles_t(v, xi_c, eta_c, p.Dxi, p.Deta, p.h_xi, p.h_eta, nx, ny, L, kind != PD_EDGE_DIRICHLET,
                        kind != PD_EDGE_NEUMANN, &s_slope[gs][0][0], &s_val[gs][0][0], r, LP);
    }
    __syncwarp();
    double cedge[4] = {0.0, 0.0, 0.0, 0.0}; // E, W, N, S
    bool pinned = false;
    if (valid) {
        EdgeSh eg;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdxi, +1.0, N2, s_val[gs][PD_EDGE_E], s_slope[gs][PD_EDGE_E],
                     &s_gb[gs][PD_EDGE_E][1], r, LP);
        cedge[PD_EDGE_E] = eg.cEdge;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdxi, -1.0, N2, s_val[gs][PD_EDGE_W], s_slope[gs][PD_EDGE_W],
                     &s_gb[gs][PD_EDGE_W][1], r, LP);
        cedge[PD_EDGE_W] = eg.cEdge;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdeta, +1.0, N1, s_val[gs][PD_EDGE_N], s_slope[gs][PD_EDGE_N],
                     &s_gb[gs][PD_EDGE_N][1], r, LP);
        cedge[PD_EDGE_N] = eg.cEdge;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdeta, -1.0, N1, s_val[gs][PD_EDGE_S], s_slope[gs][PD_EDGE_S],
                     &s_gb[gs][PD_EDGE_S][1], r, LP);
        cedge[PD_EDGE_S] = eg.cEdge;
        pinned = eg.pinned != 0; // all four edges share the kind: pinned together
        if (pinned) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                xt_pinned_row(eg, s_val[gs][e], s_slope[gs][e], &s_gb[gs][e][1], e < 2 ? N2 : N1, r, LP);
        }
    }
    pinned = __any_sync(0xffffffffu, pinned); // warp-uniform (lanes past the last patch follow)
    __syncwarp();
    // This lane's ghost data, by role: a lane is on at most one xi edge (LI >= 2);
    // on both eta edges only when LJ == 1, where S and N are kept apart.
    // gbx[b + 1]: offset of the lane's xi edge at row j0 + b, b in [-1, BJ];
    // gbs / gbn[a + 1]: offsets of the S / N edge at column i0 + a, a in [-1, BI]
    // (read from shared memory in the step loop: registers go to the coefficients).
    const int ex = isE ? PD_EDGE_E : PD_EDGE_W;
    const double cEx = isE ? cedge[PD_EDGE_E] : cedge[PD_EDGE_W], cEs = cedge[PD_EDGE_S], cEn = cedge[PD_EDGE_N];
    const double* gbx = &s_gb[gs][ex][j0];
    const double* gbs = &s_gb[gs][PD_EDGE_S][i0];
    const double* gbn = &s_gb[gs][PD_EDGE_N][i0];
    // LJ >= 2: a lane is on at most one eta edge too, and S / N share one ghost computation
    constexpr bool MERGE_ETA = LJ >= 2;
    const double cEy = isN ? cEn : cEs;
    const double* gby = isN ? gbn : gbs;

    // ---- coefficients of this lane's nodes into registers --------------------
    double co[PD_NCOEF][BI][BJ];
    {
        const int set = valid ? (cset ? cset[patch] : patch) : 0;
        const double* cf = coeffs + (size_t)set * PD_NCOEF * N;
#pragma unroll
        for (int c = 0; c < PD_NCOEF; ++c) {
            if (!MIXED && c == PD_COEF_B) continue;
#pragma unroll
            for (int ii = 0; ii < BI; ++ii) {
                const double* row = cf + (size_t)c * N + (i0 + ii) * N2 + j0;
                if constexpr (BJ % 2 == 0 && N2 % 2 == 0) { // 16-byte aligned pairs
#pragma unroll
                    for (int jj = 0; jj < BJ; jj += 2) {
                        const double2 t = valid ? __ldg(reinterpret_cast<const double2*>(row + jj)) : make_double2(0.0, 0.0);
                        co[c][ii][jj] = t.x;
                        co[c][ii][jj + 1] = t.y;
                    }
                } else {
#pragma unroll
                    for (int jj = 0; jj < BJ; ++jj) co[c][ii][jj] = valid ? __ldg(row + jj) : 0.0;
                }
            }
        }
    }

    // separable source (microsim.cpp:272-277): this lane's spatial factors wait in the
    // restriction tile (free until the sweeps are over), each lane reading only what it wrote
    const bool has_src = src_sp && src_time; // without time factors g = 0, as k_gaptooth_exact
    const double* spn = &s_u[gs][i0 * N2 + j0];
    if (has_src && valid) {
        const double* sp = src_sp + (size_t)(cset ? cset[patch] : patch) * N;
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) s_u[gs][(i0 + ii) * N2 + j0 + jj] = __ldg(sp + (i0 + ii) * N2 + j0 + jj);
    }

    // ---- StencilPoly::center + lift (gaptooth.cpp:63-72, 154-168) ------------
    // E[a + 1][b + 1] = value at block-relative (a, b), a in [-1, BI], b in [-1, BJ]
    double E[BI + 2][BJ + 2];
    {
        const LiftConsts lc = lift_consts_x(v, p.Dxi, p.Deta, p.h_xi, p.h_eta, nx, ny);
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) E[ii + 1][jj + 1] = lift_node_x(lc, p.h_xi, p.h_eta, i0 + ii, j0 + jj);
    }
    if (kind == PD_EDGE_DIRICHLET) xt_pin_initial<BI, BJ>(E, role, gbx, gbs, gbn);

    // ---- K explicit sweeps (microsim.cpp:292-332, 535-550) -------------------
    const double idx2 = XDIV(1.0, XMUL(p.mdxi, p.mdxi)), idy2 = XDIV(1.0, XMUL(p.mdeta, p.mdeta));
    const double idx = XDIV(1.0, XMUL(2.0, p.mdxi)), idy = XDIV(1.0, XMUL(2.0, p.mdeta));
    const double ixy = XDIV(1.0, XMUL(XMUL(4.0, p.mdxi), p.mdeta));
    const double dt = p.mdt;
    constexpr int B0 = MIXED ? -1 : 0, B1 = MIXED ? BJ : BJ - 1; // rows / columns whose halo is needed
    constexpr int A0 = MIXED ? -1 : 0, A1 = MIXED ? BI : BI - 1;
    // (two copies of the loop, with and without the pinned-edge selection: a flag tested
    // inside the one loop cost the unpinned config-4 step 6 %)
    auto sweeps = [&](auto pin, auto src) {
#pragma unroll(kXtUnroll)
        for (int step = 0; step < p.nt; ++step) {
            double ft = 0.0;
            if constexpr (decltype(src)::value) ft = __ldg(src_time + step);
            // eta halos from lane +-LI, then xi halos (and, for the mixed term, the
            // corners: the neighbour's eta halo) from lane +-1
#pragma unroll
            for (int ii = 0; ii < BI; ++ii) {
                E[ii + 1][BJ + 1] = __shfl_down_sync(0xffffffffu, E[ii + 1][1], LI);
                E[ii + 1][0] = __shfl_up_sync(0xffffffffu, E[ii + 1][BJ], LI);
            }
#pragma unroll
            for (int b = B0; b <= B1; ++b) {
                E[BI + 1][b + 1] = __shfl_down_sync(0xffffffffu, E[1][b + 1], 1);
                E[0][b + 1] = __shfl_up_sync(0xffffffffu, E[BI][b + 1], 1);
            }
            xt_sweep<BI, BJ, MIXED, MERGE_ETA, decltype(pin)::value, decltype(src)::value, N2>(
                E, co, role, cEx, cEs, cEn, cEy, gbx, gbs, gbn, gby, idx2, idy2, idx, idy, ixy, dt, spn, ft);
        }
    };
    // (pinned edges with a source stay on k_gaptooth_exact: exact_tile_plan)
    if (has_src) sweeps(std::false_type{}, std::true_type{});
    else if (pinned) sweeps(std::true_type{}, std::false_type{});
    else sweeps(std::false_type{}, std::false_type{});
    __syncwarp();

    // ---- restrict_average in the reference order (gaptooth.cpp:170-194) ------
    if (g < G) { // (lanes past the last patch of the warp hold nothing)
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) s_u[gs][(i0 + ii) * N2 + j0 + jj] = E[ii + 1][jj + 1];
    }
    __syncwarp();
    if (valid) {
        for (int i = r; i <= nx; i += LP) {
            double rs = 0.0;
            for (int j = 0; j <= ny; ++j) rs = XADD(rs, XMUL(quad_w(j, ny, p.quad), s_u[gs][i * N2 + j]));
            s_row[gs][i] = rs;
        }
    }
    __syncwarp();
    if (valid && r == 0) {
        double avg = 0.0;
        for (int i = 0; i <= nx; ++i) avg = XADD(avg, XMUL(quad_w(i, nx, p.quad), s_row[gs][i]));
        const size_t node = (size_t)pi * p.NF2 + pj;
        if (out_mode == OUT_FIELD) {
            out[node] = avg;
            halo_store(p, node, avg);
        } else if (out_mode == OUT_PROJECTIVE) {
            const double U = F[node];
            const double Fd = XDIV(XSUB(avg, U), p.tau); // estimate_derivative  cpi.cpp:54
            const double w = XADD(U, XMUL(p.dt_macro, Fd)); // cpi.cpp:74 with k = 0
            out[node] = w;
            halo_store(p, node, w);
        } else {
            out[patch] = avg;
        }
    }
}


// ---- 32x32 patches: one CTA of four warps per patch ----------------------------
// The same 2x4 node blocks (16 lanes along xi, two lane rows per warp, warp w
// holds micro rows 8w .. 8w+7).  xi neighbours and the lane rows of one warp
// exchange by shuffles as above; the rows that face another warp are published
// to shared memory (double-buffered by step parity, one CTA barrier per
// micro-step) and read back by the neighbouring warp.  Arithmetic, ghost rules
// and the pro/epilogue are those of k_exact_tile / k_gaptooth_exact.
constexpr int kXBigWarps = 4;
template <bool MIXED>
__global__ void __launch_bounds__(32 * kXBigWarps, MIXED ? 2 : 3)
k_exact_big(Params p, const double* __restrict__ F, double* __restrict__ out, int out_mode,
            const int* __restrict__ pij, const int* __restrict__ cset, const double* __restrict__ coeffs,
            const int* __restrict__ fail_flag, const double* __restrict__ src_sp,
            const double* __restrict__ src_time) {
    constexpr int BI = 2, BJ = 4, LI = 16, N1 = 32, N2 = 32, N = N1 * N2, L = 32, NT = 32 * kXBigWarps;
    constexpr int nx = N1 - 1, ny = N2 - 1;
    __shared__ double s_st[9];
    __shared__ double s_slope[4][L], s_val[4][L];
    __shared__ double s_gb[4][L + 2];
    __shared__ double s_u[N];
    __shared__ double s_row[N1];
    // rows facing another warp: [parity][warp][0: lowest row (lane row 0, jj = 0) | 1: highest row][column + 1]
    __shared__ double s_ex[2][kXBigWarps][2][N1 + 2];
    if (fail_flag && *fail_flag) return;
    const int patch = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bi = lane & (LI - 1), bjl = lane >> 4, bj = warp * 2 + bjl;
    const int i0 = bi * BI, j0 = bj * BJ;
    const bool isW = bi == 0, isE = bi == LI - 1, isS = bj == 0, isN = bj == 2 * kXBigWarps - 1;
    int role = (isW ? ROLE_W : 0) | (isE ? ROLE_E : 0) | (isS ? ROLE_S : 0) | (isN ? ROLE_N : 0);
    asm volatile("mov.b32 %0, %0;" : "+r"(role));
    int upper = bjl; // this lane's row block is the warp's upper one: its N side faces the next warp
    asm volatile("mov.b32 %0, %0;" : "+r"(upper));

    // ---- build_stencil (gaptooth.cpp:74-104) ----------------------------------
    const int pi = pij[2 * patch], pj = pij[2 * patch + 1];
    int ic = pi;
    if (p.periodic) ic = ((pi % p.Nxi) + p.Nxi) % p.Nxi;
    if (tid < 9) {
        const int dp = tid / 3 - 1, dq = tid % 3 - 1;
        const int ip = p.periodic ? ((ic + dp) % p.Nxi + p.Nxi) % p.Nxi : pi + dp;
        s_st[tid] = F[(size_t)ip * p.NF2 + pj + dq];
    }
    __syncthreads();
    const double* v = s_st;
    const double xi_c = XADD(p.a, XMUL(p.Dxi, (double)ic));
    const double eta_c = XADD(p.c, XMUL(p.Deta, (double)pj));

    // ---- edge profiles and ghost offsets (gaptooth.cpp:110-152, microsim.cpp:152-186)
    const int kind = xt_edge_kind(p);
    edge_profiles_t(v, xi_c, eta_c, p.Dxi, p.Deta, p.h_xi, p.h_eta, nx, ny, L, kind != PD_EDGE_DIRICHLET,
                    kind != PD_EDGE_NEUMANN, &s_slope[0][0], &s_val[0][0], tid, NT);
    __syncthreads();
    double cedge[4];
    bool pinned;
    {
        EdgeSh eg;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdxi, +1.0, N2, s_val[PD_EDGE_E], s_slope[PD_EDGE_E], &s_gb[PD_EDGE_E][1],
                     tid, NT);
        cedge[PD_EDGE_E] = eg.cEdge;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdxi, -1.0, N2, s_val[PD_EDGE_W], s_slope[PD_EDGE_W], &s_gb[PD_EDGE_W][1],
                     tid, NT);
        cedge[PD_EDGE_W] = eg.cEdge;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdeta, +1.0, N1, s_val[PD_EDGE_N], s_slope[PD_EDGE_N], &s_gb[PD_EDGE_N][1],
                     tid, NT);
        cedge[PD_EDGE_N] = eg.cEdge;
        make_ghost_t(eg, kind, p.w1, p.w2, p.mdeta, -1.0, N1, s_val[PD_EDGE_S], s_slope[PD_EDGE_S], &s_gb[PD_EDGE_S][1],
                     tid, NT);
        cedge[PD_EDGE_S] = eg.cEdge;
        pinned = eg.pinned != 0;
        if (pinned) {
#pragma unroll
            for (int e = 0; e < 4; ++e) xt_pinned_row(eg, s_val[e], s_slope[e], &s_gb[e][1], L, tid, NT);
        }
    }
    __syncthreads();
    const double cEx = isE ? cedge[PD_EDGE_E] : cedge[PD_EDGE_W], cEs = cedge[PD_EDGE_S], cEn = cedge[PD_EDGE_N];
    const double cEy = isN ? cEn : cEs;
    const double* gbx = &s_gb[isE ? PD_EDGE_E : PD_EDGE_W][j0];
    const double* gbs = &s_gb[PD_EDGE_S][i0];
    const double* gbn = &s_gb[PD_EDGE_N][i0];
    const double* gby = isN ? gbn : gbs;

    // ---- coefficients of this lane's nodes into registers --------------------
    double co[PD_NCOEF][BI][BJ];
    {
        const int set = cset ? cset[patch] : patch;
        const double* cf = coeffs + (size_t)set * PD_NCOEF * N;
#pragma unroll
        for (int c = 0; c < PD_NCOEF; ++c) {
            if (!MIXED && c == PD_COEF_B) continue;
#pragma unroll
            for (int ii = 0; ii < BI; ++ii) {
                const double* row = cf + (size_t)c * N + (i0 + ii) * N2 + j0;
#pragma unroll
                for (int jj = 0; jj < BJ; jj += 2) {
                    const double2 t = __ldg(reinterpret_cast<const double2*>(row + jj));
                    co[c][ii][jj] = t.x;
                    co[c][ii][jj + 1] = t.y;
                }
            }
        }
    }

    const bool has_src = src_sp && src_time; // separable source, staged as in k_exact_tile
    const double* spn = &s_u[i0 * N2 + j0];
    if (has_src) {
        const double* sp = src_sp + (size_t)(cset ? cset[patch] : patch) * N;
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) s_u[(i0 + ii) * N2 + j0 + jj] = __ldg(sp + (i0 + ii) * N2 + j0 + jj);
    }

    // ---- StencilPoly::center + lift (gaptooth.cpp:63-72, 154-168) ------------
    double E[BI + 2][BJ + 2];
    {
        const LiftConsts lc = lift_consts_x(v, p.Dxi, p.Deta, p.h_xi, p.h_eta, nx, ny);
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) E[ii + 1][jj + 1] = lift_node_x(lc, p.h_xi, p.h_eta, i0 + ii, j0 + jj);
    }
    if (kind == PD_EDGE_DIRICHLET) xt_pin_initial<BI, BJ>(E, role, gbx, gbs, gbn);

    // ---- K explicit sweeps (microsim.cpp:292-332, 535-550) -------------------
    const double idx2 = XDIV(1.0, XMUL(p.mdxi, p.mdxi)), idy2 = XDIV(1.0, XMUL(p.mdeta, p.mdeta));
    const double idx = XDIV(1.0, XMUL(2.0, p.mdxi)), idy = XDIV(1.0, XMUL(2.0, p.mdeta));
    const double ixy = XDIV(1.0, XMUL(XMUL(4.0, p.mdxi), p.mdeta));
    const double dt = p.mdt;
    constexpr int B0 = MIXED ? -1 : 0, B1 = MIXED ? BJ : BJ - 1;
    // the neighbouring warp's facing row: the next warp's lowest row for an upper
    // lane row, the previous warp's highest row for a lower one (clamped at the
    // patch's S / N ends, where the ghost values replace what is read)
    const int nbw = bjl ? (warp + 1 < kXBigWarps ? warp + 1 : warp) : (warp > 0 ? warp - 1 : 0);
    auto sweeps = [&](auto pin, auto src) {
#pragma unroll(kXtUnroll)
        for (int step = 0; step < p.nt; ++step) {
            const int par = step & 1;
            double ft = 0.0;
            if constexpr (decltype(src)::value) ft = __ldg(src_time + step);
            // publish the row that faces the other warp: row jj = BJ-1 of an upper lane row, jj = 0 of a lower one
            double* mine = &s_ex[par][warp][bjl][i0 + 1];
    #pragma unroll
            for (int ii = 0; ii < BI; ++ii) mine[ii] = pick<1, 1>(upper, E[ii + 1][BJ], E[ii + 1][1]);
            __syncthreads();
            const double* theirs = &s_ex[par][nbw][bjl ^ 1][i0 + 1];
    #pragma unroll
            for (int ii = 0; ii < BI; ++ii) {
                const double x = theirs[ii];
                const double sn = __shfl_down_sync(0xffffffffu, E[ii + 1][1], LI);  // lower lane row: its N halo
                const double ss = __shfl_up_sync(0xffffffffu, E[ii + 1][BJ], LI);   // upper lane row: its S halo
                E[ii + 1][BJ + 1] = pick<1, 1>(upper, x, sn);
                E[ii + 1][0] = pick<1, 1>(upper, ss, x);
            }
    #pragma unroll
            for (int b = B0; b <= B1; ++b) {
                E[BI + 1][b + 1] = __shfl_down_sync(0xffffffffu, E[1][b + 1], 1);
                E[0][b + 1] = __shfl_up_sync(0xffffffffu, E[BI][b + 1], 1);
            }
            xt_sweep<BI, BJ, MIXED, true, decltype(pin)::value, decltype(src)::value, N2>(
                E, co, role, cEx, cEs, cEn, cEy, gbx, gbs, gbn, gby, idx2, idy2, idx, idy, ixy, dt, spn, ft);
        }
    };
    if (has_src) sweeps(std::false_type{}, std::true_type{});
    else if (pinned) sweeps(std::true_type{}, std::false_type{});
    else sweeps(std::false_type{}, std::false_type{});
    __syncthreads();

    // ---- restrict_average in the reference order (gaptooth.cpp:170-194) ------
#pragma unroll
    for (int ii = 0; ii < BI; ++ii)
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) s_u[(i0 + ii) * N2 + j0 + jj] = E[ii + 1][jj + 1];
    __syncthreads();
    for (int i = tid; i <= nx; i += NT) {
        double rs = 0.0;
        for (int j = 0; j <= ny; ++j) rs = XADD(rs, XMUL(quad_w(j, ny, p.quad), s_u[i * N2 + j]));
        s_row[i] = rs;
    }
    __syncthreads();
    if (tid == 0) {
        double avg = 0.0;
        for (int i = 0; i <= nx; ++i) avg = XADD(avg, XMUL(quad_w(i, nx, p.quad), s_row[i]));
        const size_t node = (size_t)pi * p.NF2 + pj;
        if (out_mode == OUT_FIELD) {
            out[node] = avg;
            halo_store(p, node, avg);
        } else if (out_mode == OUT_PROJECTIVE) {
            const double U = F[node];
            const double Fd = XDIV(XSUB(avg, U), p.tau); // estimate_derivative  cpi.cpp:54
            const double w = XADD(U, XMUL(p.dt_macro, Fd)); // cpi.cpp:74 with k = 0
            out[node] = w;
            halo_store(p, node, w);
        } else {
            out[patch] = avg;
        }
    }
}

// ---- dispatch -----------------------------------------------------------------
using XT7 = XTileCfg<7, 7, 1, 7, false>;
using XT7M = XTileCfg<7, 7, 1, 7, true>;
using XT8 = XTileCfg<8, 8, 2, 4, false>;
using XT8M = XTileCfg<8, 8, 2, 4, true>;
using XT9 = XTileCfg<9, 9, 3, 3, false>;
using XT9M = XTileCfg<9, 9, 3, 3, true>;
using XT16 = XTileCfg<16, 16, 2, 4, false>;
using XT16M = XTileCfg<16, 16, 2, 4, true>;
// 11x11 nodes: the reference's default micro grid (nx = ny = 10, scheme_config.hpp:17); one eta
// column per lane, two patches per warp
using XT11 = XTileCfg<11, 11, 1, 11, false>;
using XT11M = XTileCfg<11, 11, 1, 11, true>;
#define PD_XTILE_CONFIGS(X) \
    X(0, XT7) X(1, XT7M) X(2, XT8) X(3, XT8M) X(4, XT9) X(5, XT9M) X(6, XT16) X(7, XT16M) X(10, XT11) X(11, XT11M)

// Tile id of the register-blocked EXACT step for these parameters, or -1: the
// shared-memory kernel (k_gaptooth_exact) carries everything else — ADI,
// general (sampled) sources, other patch shapes.
// PD_EXACT_TILE=0 forces -1 (A/B runs and the equality test of the two kernels).
inline int exact_tile_plan(const Params& p) {
    static const bool off = [] {
        const char* e = std::getenv("PD_EXACT_TILE");
        return e && e[0] == '0';
    }();
    if (off) return -1;
    if (p.solver != PD_SOLVER_EXPLICIT) return -1;
    if (p.source != PD_SOURCE_ZERO && p.source != PD_SOURCE_SEPARABLE) return -1;
    const bool pins = p.bc_type == PD_BC_DIRICHLET || (p.bc_type == PD_BC_ROBIN && fabs(p.w2) < 1e-300);
    if (p.source == PD_SOURCE_SEPARABLE && pins) return -1; // pinned edges with a source: shared-memory kernel
    int id = -1;
    if (p.n1 == 32 && p.n2 == 32) id = p.mixed ? 9 : 8; // the four-warp CTA tile (k_exact_big)
#define PD_XMATCH(ID, CFG) \
    if (p.n1 == CFG::N1 && p.n2 == CFG::N2 && (p.mixed != 0) == CFG::MIXED) id = ID;
    PD_XTILE_CONFIGS(PD_XMATCH)
#undef PD_XMATCH
    return id;
}

inline void launch_exact_tile(int id, const Params& p, const double* F, double* out, int out_mode, const int* pij,
                              const int* cset, const double* coeffs, const int* fail, cudaStream_t s,
                              const double* src_sp, const double* src_time) {
    if (p.source != PD_SOURCE_SEPARABLE) src_sp = nullptr;
#define PD_XLAUNCH(ID, CFG)                                                                              \
    if (id == ID) {                                                                                      \
        const int nunits = (p.P + CFG::G - 1) / CFG::G;                                                  \
        k_exact_tile<CFG><<<nunits, 32, 0, s>>>(p, F, out, out_mode, pij, cset, coeffs, fail, nunits, src_sp,  \
                                                src_time);                                              \
    }
    PD_XTILE_CONFIGS(PD_XLAUNCH)
#undef PD_XLAUNCH
    if (id == 8)
        k_exact_big<false><<<p.P, 32 * kXBigWarps, 0, s>>>(p, F, out, out_mode, pij, cset, coeffs, fail, src_sp, src_time);
    if (id == 9)
        k_exact_big<true><<<p.P, 32 * kXBigWarps, 0, s>>>(p, F, out, out_mode, pij, cset, coeffs, fail, src_sp, src_time);
}

} // namespace pdb200::dev
