// FAST-mode fused gap-tooth kernel: register-blocked FP64 stencil.
//
// Mapping.  A patch of N1 x N2 micro nodes is split into
// BI x BJ node blocks, one block per lane: LI = N1/BI lanes along xi, LJ =
// N2/BJ along eta, LP = LI*LJ lanes per patch, G = 32/LP patches per warp.
// Each lane keeps its nodes' state u and its nodes' folded stencil weights in
// REGISTERS for all K micro-steps; neighbours cross lanes only through warp
// shuffles (no shared memory or barriers in the hot loop).  The micro update
// is the reference's explicit FTCS (microsim.cpp:313-329) with the
// coefficients folded into per-node weights:
//   u' = wC u + wE uE + wW uW + wN uN + wS uS + wD ((uNE+uSW)-(uNW+uSE)) + c
// where c carries the frozen Neumann ghost offsets (microsim.cpp:146-167,
// SURVEY B.4 corners) folded onto the patch-boundary ring once per macro step.
//
// Per macro step and patch: 3x3 gather through the neighbour table
// (gaptooth.cpp:74-104), centre derivatives + quadratic lift
// (gaptooth.cpp:63-72,154-168), edge slopes (gaptooth.cpp:132-152) as
// shared-Lagrange dot products, K fused micro-steps, trapezoid restriction
// (gaptooth.cpp:170-194) by a lane reduction, and the k = 0 projective
// extrapolation (cpi.cpp:67-74) in the epilogue.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "pd_device.cuh"
#include "kernels_misc.cuh"


namespace pdb200::dev {

struct FastPlan {
    int id = -1; // instantiation index
    int LP = 0, G = 0, S = 0, nunits = 0;
    int mixed = 0;
    int big = 0; // 32x32 patches: kernels_fast_big.cuh (one CTA of 4 warps per patch)
    int adi = 0; // ADI micro-solver: kernels_adi_fast.cuh (one warp per patch)
};

template <int N1_, int N2_, int BI_, int BJ_, bool MIXED_, bool PAD_ = false, bool GEN_ = false, bool SRC_ = false>
struct FastCfg {
    static constexpr int N1 = N1_, N2 = N2_, BI = BI_, BJ = BJ_;
    static constexpr bool MIXED = MIXED_;
    // GEN: Robin / Dirichlet patch conditions compiled in (the Neumann-only
    // instantiation keeps the BASELINE kernels free of their branches)
    static constexpr bool GEN = GEN_;
    // SRC: separable source g = spatial * time(t)/l (microsim.cpp:272-277); the
    // sixth weight slot (the mixed term's, unused without it) holds dt * spatial
    static constexpr bool SRC = SRC_;
    static_assert(!(MIXED_ && SRC_), "the source variant is compiled for the 5-point operator only");
    // PAD: the patch (p.n1 x p.n2, runtime) is smaller than the N1 x N2 tile;
    // the extra "phantom" nodes carry zero weights and stay out of the restriction
    static constexpr bool PAD = PAD_;
    static constexpr int LI = N1 / BI, LJ = N2 / BJ, LP = LI * LJ, G = 32 / LP;
    static constexpr int NPL = BI * BJ;          // nodes per lane
    static constexpr int NW = (MIXED || SRC) ? 6 : 5; // weights per node: C,E,W,N,S,(D | source)
    static constexpr int NWL = NW * NPL;         // weight doubles per lane
    static constexpr int S = (NWL + 1) / 2;      // 16-byte slots per lane
    static constexpr int L = N1 > N2 ? N1 : N2;
    static_assert(N1 % BI == 0 && N2 % BJ == 0, "block must tile the patch");
    static_assert(LP <= 32, "patch must fit a warp");
};
enum { WC = 0, WE = 1, WW = 2, WN = 3, WS = 4, WD = 5 };
constexpr int kFastWarps = 1; // one warp per CTA: warps retire and are replaced independently

// ---- fold: solver-form coefficients -> lane-interleaved weight table -------
// Table layout: unit u (one warp = G patches) owns S*32 double2 slots; slot s
// of lane l is at ((u*S + s)*32 + l); lane-local weight index f = k*NPL + ii*BJ + jj.
template <class Cfg>
__global__ void k_fold(Params p, const double* __restrict__ coeffs, const int* __restrict__ cset,
                       double* __restrict__ W, int nunits, const double* __restrict__ src_sp) {
    const size_t total = (size_t)nunits * 32 * (2 * Cfg::S);
    const double idx2 = 1.0 / (p.mdxi * p.mdxi), idy2 = 1.0 / (p.mdeta * p.mdeta);
    const double idx = 1.0 / (2.0 * p.mdxi), idy = 1.0 / (2.0 * p.mdeta);
    const double ixy = 1.0 / (4.0 * p.mdxi * p.mdeta);
    const double dt = p.mdt;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const int half = (int)(t & 1);
        const size_t q = t >> 1;
        const int lane = (int)(q % 32);
        const size_t us = q / 32;
        const int s = (int)(us % Cfg::S);
        const size_t unit = us / Cfg::S;
        const int f = 2 * s + half;
        double val = 0.0;
        const int g = lane / Cfg::LP, r = lane % Cfg::LP;
        const long patch = (long)unit * Cfg::G + g;
        if (g < Cfg::G && patch < p.P && f < Cfg::NWL) {
            const int kind = f / Cfg::NPL, node = f % Cfg::NPL;
            const int ii = node / Cfg::BJ, jj = node % Cfg::BJ;
            const int bi = r % Cfg::LI, bj = r / Cfg::LI;
            const int i = bi * Cfg::BI + ii, j = bj * Cfg::BJ + jj;
            const int n1 = Cfg::PAD ? p.n1 : Cfg::N1, n2 = Cfg::PAD ? p.n2 : Cfg::N2;
            if (Cfg::PAD && (i >= n1 || j >= n2)) { // phantom node of a padded tile
                W[((unit * Cfg::S + s) * 32 + lane) * 2 + half] = 0.0;
                continue;
            }
            const int set = cset ? cset[patch] : (int)patch;
            const double* c = coeffs + (size_t)set * PD_NCOEF * p.N;
            const int k = i * p.n2 + j;
            const double A = c[PD_COEF_A * p.N + k], B = c[PD_COEF_B * p.N + k], C = c[PD_COEF_C * p.N + k];
            const double Vx = c[PD_COEF_VX * p.N + k], Vy = c[PD_COEF_VY * p.N + k], Wr = c[PD_COEF_W * p.N + k];
            const double ax = A * idx2, vx = Vx * idx, cy = C * idy2, vy = Vy * idy;
            const double wE = dt * (ax - vx), wW = dt * (ax + vx), wN = dt * (cy - vy), wS = dt * (cy + vy);
            // Neumann reflection u_ghost = u_inner + g (microsim.cpp:314-323): the
            // inward weight absorbs the outward one; the outward slot keeps the
            // original weight for the per-patch ghost constant (zeroed in k_fast).
            const bool Wb = i == 0, Eb = i == n1 - 1, Sb = j == 0, Nb = j == n2 - 1;
            if (Cfg::GEN && p.pinned && (Wb || Eb || Sb || Nb)) {
                val = 0.0; // pinned edge node: u' = its pinned value, set as the node constant
            } else {
                switch (kind) {
                    case WE: val = Wb ? wE + wW : wE; break;
                    case WW: val = Eb ? wW + wE : wW; break;
                    case WN: val = Sb ? wN + wS : wN; break;
                    case WS: val = Nb ? wS + wN : wS; break;
                    case WD: val = Cfg::SRC ? dt * src_sp[(size_t)set * p.N + k] : dt * (B * ixy); break;
                    default: { // Robin ghosts also carry cEdge * u(edge) (microsim.cpp:178-183)
                        double wc = 1.0 - dt * (2.0 * ax + 2.0 * cy + Wr);
                        if (Wb) wc += wW * p.cedge[PD_EDGE_W];
                        if (Eb) wc += wE * p.cedge[PD_EDGE_E];
                        if (Sb) wc += wS * p.cedge[PD_EDGE_S];
                        if (Nb) wc += wN * p.cedge[PD_EDGE_N];
                        val = wc;
                        break;
                    }
                }
            }
        }
        W[((unit * Cfg::S + s) * 32 + lane) * 2 + half] = val;
    }
}

// restrict_average weight of node k of n+1 (gaptooth.cpp:172-185): trapezoid
// 1/n (1/2n at the ends) or Simpson (1, 4, 2, ..., 4, 1)/(3n)
template <int n>
__device__ __forceinline__ double quad_weight(int k, int quad) {
    constexpr double tr = 1.0 / n, te = 0.5 / n;
    constexpr double s1 = 1.0 / (3.0 * n), s2 = 2.0 / (3.0 * n), s4 = 4.0 / (3.0 * n);
    const bool end = k == 0 || k == n;
    if (quad == PD_QUAD_SIMPSON) return end ? s1 : ((k & 1) ? s4 : s2);
    return end ? te : tr;
}

// a0*b0 + a1*b1 + a2*b2 with a fixed rounding (two fma, left to right)
__device__ __forceinline__ double dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
    return __fma_rn(a2, b2, __fma_rn(a1, b1, __dmul_rn(a0, b0)));
}

__device__ __forceinline__ double quad_weight_rt(int k, int n, int quad) {
    const bool end = k == 0 || k == n;
    if (quad == PD_QUAD_SIMPSON) return (end ? 1.0 : ((k & 1) ? 4.0 : 2.0)) / (3.0 * n);
    return (end ? 0.5 : 1.0) / n;
}

// Per-edge-node constant of the boundary fold-in: Robin ghost offset
// b = sign 2 delta (w1 value + w2 slope) / w2 (make_ghost, microsim.cpp:176-183)
// or, on a pinned edge, the pinned value (pinned_value, microsim.cpp:189-192).
__device__ __forceinline__ double edge_constant(const Params& p, int e, double value, double slope) {
    if (p.bc_type == PD_BC_DIRICHLET) return value;
    if (p.pinned) return __fma_rn(__ddiv_rn(p.w2, p.w1), slope, value); // Robin with w2 ~ 0 behaves as Dirichlet
    return __dmul_rn(p.gsc[e], __ddiv_rn(__fma_rn(p.w2, slope, __dmul_rn(p.w1, value)), p.w2));
}

// ---- mixed-term ring offsets ------------------------------------------------
// For a boundary-ring node the reflected node values cancel in
// (uNE + uSW) - (uNW + uSE) (u_ghost = u_inner + off, corner
// ghosts carry both edges' offsets); what remains is a signed difference of
// the node's own edge offsets plus, at the two ends of the edge, the
// neighbouring edges' offsets.  Ring entry t: E (j = t), W, N (i), S order.
__device__ __forceinline__ int e_of_ring(int N1, int N2, int t, int& e, int& k) {
    const bool xi_edge = t < 2 * N2;
    const int L = xi_edge ? N2 : N1, u = xi_edge ? t : t - 2 * N2;
    const bool first = u < L;
    k = first ? u : u - L;
    e = xi_edge ? (first ? PD_EDGE_E : PD_EDGE_W) : (first ? PD_EDGE_N : PD_EDGE_S);
    return e;
}
__device__ __forceinline__ double ring_offset(int N1, int N2, const double* gE, const double* gW, const double* gN,
                                              const double* gS, int t) {
    const bool xi_edge = t < 2 * N2;
    const int L = xi_edge ? N2 : N1, M = xi_edge ? N1 : N2, u = xi_edge ? t : t - 2 * N2;
    const bool first = u < L; // E or N: +, W or S: -
    const int k = first ? u : u - L;
    const double* ge = xi_edge ? (first ? gE : gW) : (first ? gN : gS);
    const double* gh = xi_edge ? gN : gE; // edge crossing the k = L-1 end
    const double* gl = xi_edge ? gS : gW; // edge crossing the k = 0 end
    const int a = first ? M - 1 : 1, b = first ? M - 2 : 0;
    const double d = ge[k + 1 < L ? k + 1 : L - 1] - ge[k > 0 ? k - 1 : 0];
    double o = first ? d : -d;
    if (k == L - 1) o += gh[a] - gh[b];
    if (k == 0) o += gl[b] - gl[a];
    return o;
}

// ---- per-patch body: lift, boundary fold-in, K micro-steps, restriction --
// Everything after the weights (w, registers) and the 3x3 stencil (v) are in
// hand; shared by the one-shot and the persistent kernels.
// Returns |value written| on the lane that writes a patch result (0 elsewhere):
// the fused run's blow-up guard reduces it.
template <class Cfg>
__device__ __forceinline__ double patch_body(const Params& p, double (&w)[2 * Cfg::S], const double (&v)[9], int lane,
                                           bool valid, int patch, double (*sg)[8][Cfg::L], double* sred,
                                           const int* __restrict__ nbr, double* __restrict__ out, int out_mode,
                                           const double* __restrict__ srct) {
    constexpr int BI = Cfg::BI, BJ = Cfg::BJ, LI = Cfg::LI, LP = Cfg::LP, G = Cfg::G, NPL = Cfg::NPL;
    constexpr int N1 = Cfg::N1, N2 = Cfg::N2;
    constexpr bool MIXED = Cfg::MIXED;
    const int n1 = Cfg::PAD ? p.n1 : N1, n2 = Cfg::PAD ? p.n2 : N2; // the patch's real extent
    const int g = lane / LP, r = lane % LP;
    const int bi = r % LI, bj = r / LI;
    const int gs = g < G ? g : 0;
#define WT(k, ii, jj) w[(k) * NPL + (ii) * BJ + (jj)]
    // centre derivatives (StencilPoly::center, gaptooth.cpp:63-72); reciprocals
    // come precomputed from the host (no device divisions)
    // (explicit fma / rounded ops outside the step loop: the same rounding
    // whether this body is inlined into k_fast or into the loop of k_fast_run)
    const double Uxi = __dmul_rn(__dsub_rn(v[7], v[1]), p.i2Dxi);
    const double Ueta = __dmul_rn(__dsub_rn(v[5], v[3]), p.i2Deta);
    const double hUxx = 0.5 * __dmul_rn(__dadd_rn(__fma_rn(-2.0, v[4], v[7]), v[1]), p.iDxi2);
    const double hUyy = 0.5 * __dmul_rn(__dadd_rn(__fma_rn(-2.0, v[4], v[5]), v[3]), p.iDeta2);
    const double Uxy = __dmul_rn(__dadd_rn(__dsub_rn(__dsub_rn(v[8], v[6]), v[2]), v[0]), p.i4DD);
    const double C0 = __fma_rn(-p.c24y, 2.0 * hUyy, __fma_rn(-p.c24x, 2.0 * hUxx, v[4]));

    // ---- ghost offsets g = +-2 delta * slope along the four edges ---------
    // slope_E(j) = sum_q Lq(Y_j)[q] * sum_p Lp'(+h/2)[p] v[p][q] (tensor Lagrange,
    // gaptooth.cpp:43-61, weights from the host).  Lanes of a patch share the
    // 2*N1 + 2*N2 entries; then, for the mixed term, the boundary-ring offsets
    // Doff (the reflected node values cancel in (uNE+uSW)-(uNW+uSE); what
    // remains is a signed sum of ghost offsets, SURVEY B.4 corners).
    for (int t = r; g < G && t < 2 * n2 + 2 * n1; t += LP) {
        if (t < 2 * n2) {
            const int e = t < n2 ? PD_EDGE_E : PD_EDGE_W, j = t < n2 ? t : t - n2;
            const double* d = p.dlag[e];
            const double G0 = dot3(d[0], v[0], d[1], v[3], d[2], v[6]);
            const double G1 = dot3(d[0], v[1], d[1], v[4], d[2], v[7]);
            const double G2 = dot3(d[0], v[2], d[1], v[5], d[2], v[8]);
            const double sl = dot3(lagq_at(p, j, 0), G0, lagq_at(p, j, 1), G1, lagq_at(p, j, 2), G2);
            if (!Cfg::GEN || p.bc_type == PD_BC_NEUMANN) {
                sg[gs][e][j] = __dmul_rn(p.gsc[e], sl);
            } else { // Robin / Dirichlet need the edge value too (dirichlet_edge_values, gaptooth.cpp:110-130)
                const double* w = p.vlag[e];
                const double V0 = dot3(w[0], v[0], w[1], v[3], w[2], v[6]);
                const double V1 = dot3(w[0], v[1], w[1], v[4], w[2], v[7]);
                const double V2 = dot3(w[0], v[2], w[1], v[5], w[2], v[8]);
                sg[gs][e][j] = edge_constant(p, e, dot3(lagq_at(p, j, 0), V0, lagq_at(p, j, 1), V1, lagq_at(p, j, 2), V2), sl);
            }
        } else {
            const int u = t - 2 * n2;
            const int e = u < n1 ? PD_EDGE_N : PD_EDGE_S, i = u < n1 ? u : u - n1;
            const double* d = p.dlag[e];
            const double H0 = dot3(d[0], v[0], d[1], v[1], d[2], v[2]);
            const double H1 = dot3(d[0], v[3], d[1], v[4], d[2], v[5]);
            const double H2 = dot3(d[0], v[6], d[1], v[7], d[2], v[8]);
            const double sl = dot3(lagp_at(p, i, 0), H0, lagp_at(p, i, 1), H1, lagp_at(p, i, 2), H2);
            if (!Cfg::GEN || p.bc_type == PD_BC_NEUMANN) {
                sg[gs][e][i] = __dmul_rn(p.gsc[e], sl);
            } else {
                const double* w = p.vlag[e];
                const double V0 = dot3(w[0], v[0], w[1], v[1], w[2], v[2]);
                const double V1 = dot3(w[0], v[3], w[1], v[4], w[2], v[5]);
                const double V2 = dot3(w[0], v[6], w[1], v[7], w[2], v[8]);
                sg[gs][e][i] = edge_constant(p, e, dot3(lagp_at(p, i, 0), V0, lagp_at(p, i, 1), V1, lagp_at(p, i, 2), V2), sl);
            }
        }
    }
    __syncwarp();
    const double* gE = sg[gs][PD_EDGE_E];
    const double* gW = sg[gs][PD_EDGE_W];
    const double* gN = sg[gs][PD_EDGE_N];
    const double* gS = sg[gs][PD_EDGE_S];
    if constexpr (MIXED) {
        if (Cfg::GEN && p.pinned) {
            // pinned ring nodes do not update; the interior reads real nodes only
        } else if constexpr (LP == 32) { // one patch per warp: closed form (measured faster at 16x16)
            for (int t = r; t < 2 * n2 + 2 * n1; t += LP) {
                int e, k;
                sg[gs][4 + e_of_ring(n1, n2, t, e, k)][k] = ring_offset(n1, n2, gE, gW, gN, gS, t);
            }
        } else { // several patches per warp: generic corner rule (measured faster at 8x8)
            auto off = [&](int pp, int qq) {
                const int qc = qq < 0 ? 0 : (qq > n2 - 1 ? n2 - 1 : qq);
                const int pc = pp < 0 ? 0 : (pp > n1 - 1 ? n1 - 1 : pp);
                double o = 0.0;
                if (pp < 0) o += gW[qc];
                if (pp > n1 - 1) o += gE[qc];
                if (qq < 0) o += gS[pc];
                if (qq > n2 - 1) o += gN[pc];
                return o;
            };
            for (int t = r; g < G && t < 2 * n2 + 2 * n1; t += LP) {
                int e, k;
                e_of_ring(n1, n2, t, e, k);
                const int i = e == PD_EDGE_E ? n1 - 1 : e == PD_EDGE_W ? 0 : k;
                const int j = e == PD_EDGE_N ? n2 - 1 : e == PD_EDGE_S ? 0 : k;
                sg[gs][4 + e][k] = (off(i + 1, j + 1) + off(i - 1, j - 1)) - (off(i - 1, j + 1) + off(i + 1, j - 1));
            }
        }
        __syncwarp();
    }

    // ---- lift + boundary fold-in ------------------------------------------
    // Static reflections (wE += wW on the W edge, ...) are folded into the
    // table by k_fold; the outward slot still holds the original weight, used
    // here once for the per-patch constant and then zeroed.
    double u[BI][BJ], c[BI][BJ];
#pragma unroll
    for (int ii = 0; ii < BI; ++ii) {
        const int i = bi * BI + ii;
        const double X = __fma_rn(p.mdxi, (double)i, -0.5 * p.h_xi);
        const double Ai = __fma_rn(X, __fma_rn(X, hUxx, Uxi), C0), Bi = __fma_rn(X, Uxy, Ueta);
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
            const int j = bj * BJ + jj;
            const double Y = __fma_rn(p.mdeta, (double)j, -0.5 * p.h_eta);
            u[ii][jj] = __fma_rn(Y, __fma_rn(Y, hUyy, Bi), Ai); // quadratic lift (gaptooth.cpp:154-168)
            if (Cfg::PAD && (i >= n1 || j >= n2)) { // phantom node: zero weights, zero state
                u[ii][jj] = 0.0;
                c[ii][jj] = 0.0;
                continue;
            }
            // only block-edge nodes can be patch-edge nodes of an exact-fit tile:
            // written so the compiler drops the impossible cases at compile time
            const bool Wb = ii == 0 && bi == 0;
            const bool Eb = Cfg::PAD ? i == n1 - 1 : (ii == BI - 1 && bi == LI - 1);
            const bool Sb = jj == 0 && bj == 0;
            const bool Nb = Cfg::PAD ? j == n2 - 1 : (jj == BJ - 1 && bj == Cfg::LJ - 1);
            double cc = 0.0;
            if (Cfg::GEN && p.pinned) {
                // pinned edge nodes keep their value (all their weights are zero): the
                // sweep's priority W, E, S, N for the value (microsim.cpp:306-311); a
                // Dirichlet edge also pins the initial field, in W, E, S, N order with
                // the later edge winning at corners (microsim.cpp:521-530)
                if (Wb) cc = gW[j];
                else if (Eb) cc = gE[j];
                else if (Sb) cc = gS[i];
                else if (Nb) cc = gN[i];
                if (p.bc_type == PD_BC_DIRICHLET) {
                    if (Wb) u[ii][jj] = gW[j];
                    if (Eb) u[ii][jj] = gE[j];
                    if (Sb) u[ii][jj] = gS[i];
                    if (Nb) u[ii][jj] = gN[i];
                }
                c[ii][jj] = cc;
                continue;
            }
            // single-edge reflections u_ghost = u_inner + cEdge u_edge + b (microsim.cpp:314-323)
            if (Wb) { cc = fma(WT(WW, ii, jj), gW[j], cc); WT(WW, ii, jj) = 0.0; }
            if (Eb) { cc = fma(WT(WE, ii, jj), gE[j], cc); WT(WE, ii, jj) = 0.0; }
            if (Sb) { cc = fma(WT(WS, ii, jj), gS[i], cc); WT(WS, ii, jj) = 0.0; }
            if (Nb) { cc = fma(WT(WN, ii, jj), gN[i], cc); WT(WN, ii, jj) = 0.0; }
            if constexpr (MIXED) {
                if (Wb || Eb || Sb || Nb) {
                    const double* dd = sg[gs][4 + (Wb ? PD_EDGE_W : Eb ? PD_EDGE_E : Sb ? PD_EDGE_S : PD_EDGE_N)];
                    cc = fma(WT(WD, ii, jj), dd[(Wb || Eb) ? j : i], cc);
                    WT(WD, ii, jj) = 0.0;
                }
            }
            c[ii][jj] = cc;
        }
    }

    // ---- K fused micro-steps, state and weights in registers --------------
    // Neighbour blocks are at lane +-1 (xi) and lane +-LI (eta).  The exchange
    // uses constant-delta shuffles (SHFL.DOWN/UP with an immediate), which
    // overlap with DFMA issue on B200, unlike SHFL.IDX with a register lane
    // (measured: scripts/ubench/ubench2.cu).  A lane on a
    // patch edge receives some other finite value for the missing side; the
    // boundary fold-in above has zeroed every weight that would read it.
    auto micro_step = [&](int step) {
        double hN[BI], hS[BI];
#pragma unroll
        for (int ii = 0; ii < BI; ++ii) {
            hN[ii] = __shfl_down_sync(0xffffffffu, u[ii][0], LI);
            hS[ii] = __shfl_up_sync(0xffffffffu, u[ii][BJ - 1], LI);
        }
        double cE[BJ + 2], cW[BJ + 2];
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
            cE[jj + 1] = __shfl_down_sync(0xffffffffu, u[0][jj], 1);
            cW[jj + 1] = __shfl_up_sync(0xffffffffu, u[BI - 1][jj], 1);
        }
        cE[0] = cE[BJ + 1] = cW[0] = cW[BJ + 1] = 0.0; // corners are not exchanged (difference form)
        // value at block-relative (a, b), a in [-1,BI], b in [-1,BJ]
        auto at = [&](int a, int b) -> double {
            if (a == BI) return cE[b + 1];
            if (a == -1) return cW[b + 1];
            if (b == BJ) return hN[a];
            if (b == -1) return hS[a];
            return u[a][b];
        };
        // Term-major order: the NPL accumulation chains of this lane advance
        // together, so consecutive DFMAs are independent (8-way ILP per warp)
        // and the terms that use shuffled values come last.
        double nu[BI][BJ];
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(WC, ii, jj), u[ii][jj], c[ii][jj]);
        if constexpr (MIXED) {
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(WN, ii, jj), at(ii, jj + 1), nu[ii][jj]);
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(WS, ii, jj), at(ii, jj - 1), nu[ii][jj]);
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(WE, ii, jj), at(ii + 1, jj), nu[ii][jj]);
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(WW, ii, jj), at(ii - 1, jj), nu[ii][jj]);
        } else {
            // 5-point tiles: the neighbour-term order of the fastest single-launch run
            // measured (candidates from the control-word stall sums of
            // scripts/lab/stallsearch.py, then timed): 9x9 W, S, E, N; 7x7 N, E, S, W
            auto ord = [](int q) constexpr {
#ifdef PD_LAB_O0 // scripts/lab/stallsearch.py override
                constexpr int ol[4] = {PD_LAB_O0, PD_LAB_O1, PD_LAB_O2, PD_LAB_O3};
                return ol[q];
#else
                constexpr int o9[4] = {WW, WS, WE, WN}, o7[4] = {WN, WE, WS, WW}, o0[4] = {WN, WS, WE, WW};
                return N1 == 9 ? o9[q] : N1 == 7 ? o7[q] : o0[q];
#endif
            };
            auto term = [&](int k) {
                const int da = k == WE ? 1 : k == WW ? -1 : 0, db = k == WN ? 1 : k == WS ? -1 : 0;
#pragma unroll
                for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                    for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(k, ii, jj), at(ii + da, jj + db), nu[ii][jj]);
            };
#pragma unroll
            for (int q = 0; q < 4; ++q) term(ord(q));
        }
        if constexpr (MIXED) {
            // difference form: e(i,j) = u(i+1,j) - u(i-1,j) once per node, then
            // D(i,j) = e(i,j+1) - e(i,j-1); e crosses lanes only at the block's
            // eta ends.  3 DP per node instead of 4 (8 per update in total).
            double e[BI][BJ];
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) e[ii][jj] = at(ii + 1, jj) - at(ii - 1, jj);
            double eN[BI], eS[BI];
#pragma unroll
            for (int ii = 0; ii < BI; ++ii) {
                eN[ii] = __shfl_down_sync(0xffffffffu, e[ii][0], LI);
                eS[ii] = __shfl_up_sync(0xffffffffu, e[ii][BJ - 1], LI);
            }
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) {
                    const double up = jj + 1 < BJ ? e[ii][jj + 1] : eN[ii];
                    const double dn = jj > 0 ? e[ii][jj - 1] : eS[ii];
                    nu[ii][jj] = fma(WT(WD, ii, jj), up - dn, nu[ii][jj]);
                }
        }
        if constexpr (Cfg::SRC) { // + dt * spatial * time(t0 + step dt)/l  (microsim.cpp:272-277, 329)
            const double ft = srct ? __ldg(srct + step) : 0.0; // no factors given: g = 0, as EXACT
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(WD, ii, jj), ft, nu[ii][jj]);
        }
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) u[ii][jj] = nu[ii][jj];
    };
    if constexpr (!MIXED) {
        // 5-point tiles (configs 1-3, latency-bound single-launch runs): two micro-steps
        // per loop trip let ptxas overlap one step's tail with the next one's shuffles
        // (configs 1-3 5-7 % faster); the 9-point 16x16 loop is throughput-bound and
        // slower unrolled (+1 %), so it keeps one step per trip
#pragma unroll 2
        for (int step = 0; step < p.nt; ++step) micro_step(step);
    } else {
        for (int step = 0; step < p.nt; ++step) micro_step(step);
    }

    // ---- trapezoid / Simpson restriction (gaptooth.cpp:170-194) -------------
    double part = 0.0;
    // Simpson needs even nx, ny (odd node counts): compiled only for those shapes
    constexpr bool kSimpsonShape = (N1 - 1) % 2 == 0 && (N2 - 1) % 2 == 0;
    if constexpr (Cfg::PAD) { // real extent at run time, phantom nodes weigh nothing
#pragma unroll
        for (int ii = 0; ii < BI; ++ii) {
            const int i = bi * BI + ii;
            double row = 0.0;
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) {
                const int j = bj * BJ + jj;
                row = __fma_rn(j < n2 ? quad_weight_rt(j, n2 - 1, p.quad) : 0.0, u[ii][jj], row);
            }
            part = __fma_rn(i < n1 ? quad_weight_rt(i, n1 - 1, p.quad) : 0.0, row, part);
        }
    } else if (kSimpsonShape && p.quad == PD_QUAD_SIMPSON) {
#pragma unroll
        for (int ii = 0; ii < BI; ++ii) {
            double row = 0.0;
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) row = __fma_rn(quad_weight<N2 - 1>(bj * BJ + jj, PD_QUAD_SIMPSON), u[ii][jj], row);
            part = __fma_rn(quad_weight<N1 - 1>(bi * BI + ii, PD_QUAD_SIMPSON), row, part);
        }
    } else {
        const double ox = 1.0 / (N1 - 1), oy = 1.0 / (N2 - 1);
#pragma unroll
        for (int ii = 0; ii < BI; ++ii) {
            double row = 0.0;
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) {
                const bool edge = (jj == 0 && bj == 0) || (jj == BJ - 1 && bj == Cfg::LJ - 1);
                row = __fma_rn(edge ? 0.5 * oy : oy, u[ii][jj], row);
            }
            const bool edge = (ii == 0 && bi == 0) || (ii == BI - 1 && bi == LI - 1);
            part = __fma_rn(edge ? 0.5 * ox : ox, row, part);
        }
    }
    double avg = 0.0;
    if constexpr (LP == 32) { // one patch per warp: butterfly reduction
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        avg = part;
    } else { // several patches per warp: lane r == 0 of each sums its LP partials
        sred[lane] = part;
        __syncwarp();
        if (r == 0)
#pragma unroll
            for (int q = 0; q < LP; ++q) avg += sred[g * LP + q];
    }
    double written = 0.0;
    if (valid && r == 0) {
        const size_t node = (size_t)__ldg(nbr + 9 * patch + 4);
        if (out_mode == 0) {
            out[node] = written = avg;
        } else if (out_mode == 1 || out_mode == 3) {
            const double U = v[4];
            written = __fma_rn(p.dt_macro, __ddiv_rn(__dsub_rn(avg, U), p.tau), U); // cpi.cpp:54, 74 (k = 0)
            out[node] = written;
            // 3: fused run, the column-0 patch also writes the periodic seam U(Nxi,j) = U(0,j)
            if (out_mode == 3 && p.periodic && node < (size_t)p.NF2) out[(size_t)p.Nxi * p.NF2 + node] = written;
        } else {
            out[patch] = written = avg;
        }
        if (out_mode <= 1) halo_store(p, node, written); // decomposed run: fused peer-memory halo
    }
    return fabs(written);
#undef WT
}

// ---- the fused step, one warp-unit per launch slot -----------------------
template <class Cfg>
__global__ void __launch_bounds__(32 * kFastWarps)
k_fast(Params p, const double* __restrict__ F, double* __restrict__ out, int out_mode, const int* __restrict__ nbr,
       const double* __restrict__ Wt, int nunits, const int* __restrict__ fail_flag, const double* __restrict__ srct) {
    constexpr int G = Cfg::G, LP = Cfg::LP, L = Cfg::L;
    __shared__ double s_g[kFastWarps][G][8][L]; // ghost offsets + mixed-term ring offsets per edge
    __shared__ double s_red[kFastWarps][32];
    if (fail_flag && *fail_flag) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int unit = blockIdx.x * kFastWarps + warp;
    if (unit >= nunits) return; // warp-uniform
    const int g = lane / LP;
    const int patch = unit * G + g;
    const bool valid = g < G && patch < p.P;
    // The stencil gather is a dependent pair (index, then value): issue the
    // index loads first so they are not queued behind the weight tile.
    int idx[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) idx[q] = valid ? __ldg(nbr + 9 * patch + q) : 0;
    double w[2 * Cfg::S];
    {
        const double2* wp = reinterpret_cast<const double2*>(Wt) + (size_t)unit * Cfg::S * 32 + lane;
#pragma unroll
        for (int s = 0; s < Cfg::S; ++s) {
            // tiles that leave lanes idle (G LP < 32: 7x7, 9x9, 11x11) skip those lanes' all-zero
            // slots: whole 32-byte sectors of the streamed table (11x11: 0.56 -> 0.38 GB per launch)
            double2 t = make_double2(0.0, 0.0);
            if (G * LP == 32 || g < G) t = __ldg(wp + s * 32);
            w[2 * s] = t.x;
            w[2 * s + 1] = t.y;
        }
    }
    double v[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = valid ? __ldg(F + idx[q]) : 0.0;
    patch_body<Cfg>(p, w, v, lane, valid, patch, s_g[warp], s_red[warp], nbr, out, out_mode, srct);
}

// ---- the whole projective run in one cooperative launch (k = 0) -----------
// Device-resident cpi::run (cpi.cpp:175-202) for the FAST tiles:
// per macro step every warp runs the fused step of its units (stride over the
// grid; projective epilogue, the column-0 patches also write the periodic seam),
// the grid refreshes the boundary from the perimeter table (refresh_boundary,
// gaptooth.cpp:296-310), max |U| of every written node is reduced with spread
// atomics, and ONE grid barrier per step replaces the three launches (step,
// refresh, guard) of the multi-launch loop; after it every thread reads the
// same maximum and takes the same guard decision.  Arithmetic identical to
// k_fast + k_refresh + k_guard.  F is re-read with L2 loads (__ldcg): it was
// written by other CTAs during this launch.
constexpr int kGuardSpread = 32;
// Four warps per CTA: the grid barrier's arrival count is per CTA (one atomic
// per CTA), so fewer, larger CTAs make it cheaper; 3 CTAs/SM = 12 warps.
constexpr int kRunWarps = 4;

// 12 warps/SM (168 registers) for the plain 5-point tiles (configs 1-3; spill-
// free or a few bytes outside the step loop); the mixed / padded / source
// variants carry more state and keep 8 warps/SM rather than spill.
// blow-up guard (cpi.cpp:187-202) on the spread maxima of one step: max over
// the warp's 32 slots, recorded in slot[step]; true when the run stops.
__device__ __forceinline__ bool guard_trips(unsigned long long v, int step, int gw, int lane, double blowup,
                                            unsigned long long* slot, int* fail) {
    v = warp_max_u64(v);
    if (gw == 0 && lane == 0) slot[step] = v;
    const bool nonfinite = v >= 0x7FF0000000000000ull;
    if (nonfinite || __longlong_as_double((long long)v) > blowup) {
        if (gw == 0 && lane == 0) {
            fail[1] = nonfinite ? 1 : 0;
            fail[0] = step + 1;
        }
        return true;
    }
    return false;
}

template <class Cfg>
constexpr int run_min_blocks() { return (Cfg::MIXED || Cfg::PAD || Cfg::SRC || Cfg::NPL > 9) ? 8 : 12; }

template <class Cfg>
__global__ void __launch_bounds__(32 * kRunWarps, run_min_blocks<Cfg>() / kRunWarps)
k_fast_run(Params p, double* __restrict__ UA, double* __restrict__ UB, const int* __restrict__ nbr,
           const double* __restrict__ Wt, int nunits, const double* __restrict__ bnd, size_t bnd_stride,
           const double* __restrict__ srct, size_t srct_stride, int nsteps, double blowup,
           unsigned long long* __restrict__ slot, unsigned long long* __restrict__ spread, int* __restrict__ fail,
           const double* __restrict__ exact, unsigned long long* __restrict__ err) {
    constexpr int G = Cfg::G, LP = Cfg::LP, L = Cfg::L;
    __shared__ double s_g[kRunWarps][G][8][L];
    __shared__ double s_red[kRunWarps][32];
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * kRunWarps + warp, nw = gridDim.x * kRunWarps;
    const int nperim = 2 * (p.Nxi + 1) + 2 * (p.Neta + 1);
    unsigned long long pend = 0; // this lane's spread slot of the previous step
    for (int n = 0; n < nsteps; ++n) {
        const double* F = (n & 1) ? UB : UA;
        double* out = (n & 1) ? UA : UB;
        unsigned long long m = 0;
        for (int unit = gw; unit < nunits; unit += nw) {
            // lane-dependent setup re-derived per unit: keeps the compiler from
            // hoisting the per-lane constants of patch_body out of the step loop
            // (live across the K-step loop they cost ~50 registers = occupancy)
            int lane;
            asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
            const int g = lane / LP;
            const int patch = unit * G + g;
            const bool valid = g < G && patch < p.P;
            int idx[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) idx[q] = valid ? __ldg(nbr + 9 * patch + q) : 0;
            double w[2 * Cfg::S];
            {
                const double2* wp = reinterpret_cast<const double2*>(Wt) + (size_t)unit * Cfg::S * 32 + lane;
#pragma unroll
                for (int s = 0; s < Cfg::S; ++s) {
                    const double2 t = __ldg(wp + s * 32);
                    w[2 * s] = t.x;
                    w[2 * s + 1] = t.y;
                }
            }
            double v[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) v[q] = valid ? __ldcg(F + idx[q]) : 0.0;
            const double wv = patch_body<Cfg>(p, w, v, lane, valid, patch, s_g[warp], s_red[warp], nbr, out, 3,
                                              srct ? srct + srct_stride * n : nullptr);
            m = max(m, (unsigned long long)__double_as_longlong(wv));
        }
        const double* bn = bnd ? bnd + bnd_stride * n : nullptr;
        for (int t = gw * 32 + lane; t < nperim; t += nw * 32)
            m = max(m, (unsigned long long)__double_as_longlong(refresh_one(p, out, F, bn, t, true)));
        m = warp_max_u64(m);
        if (lane == 0) atomicMax(spread + (size_t)n * kGuardSpread + gw % kGuardSpread, m);
        // the guard decision of step n-1 is taken here, one step late: its maximum
        // was loaded right after the previous barrier, so the L2 round trip hid
        // behind this step's body.  Step n wrote the other buffer, so a trip still
        // leaves the field after step n-1 (and its statistics) exactly as cpi::run
        // reports them; every thread decides alike (same maximum).
        if (n > 0 && guard_trips(pend, n - 1, gw, lane, blowup, slot, fail)) return;
        grid.sync();
        pend = __ldcg(spread + (size_t)n * kGuardSpread + lane);
        if (exact) { // cpi::run's max_percent_error of step n (k_exact_err's arithmetic) over the patch nodes
            const double* ex = exact + (size_t)n * (p.Nxi + 1) * p.NF2;
            unsigned long long em = 0;
            for (int q = gw * 32 + lane; q < p.P; q += nw * 32) {
                const int node = __ldg(nbr + 9 * q + 4);
                const double e = ex[node];
                if (fabs(e) < 1e-12) continue;
                const double pct = __dmul_rn(__ddiv_rn(fabs(__dsub_rn(__ldcg(out + node), e)), fabs(e)), 100.0);
                em = max(em, (unsigned long long)__double_as_longlong(pct));
            }
            em = warp_max_u64(em);
            if (lane == 0 && em) atomicMax(err + n, em);
        }
    }
    if (nsteps > 0) guard_trips(pend, nsteps - 1, gw, lane, blowup, slot, fail);
}

// ---- instantiations --------------------------------------------------------
// tiles: 7x7 (1x7 blocks, four patches per warp), 8x8 (2x4, four), 9x9 (3x3,
// three), 11x11 (1x11, two), 16x16 (2x4, one); each with/without the mixed term, exact-fit or
// padded (PAD), Neumann-only or with Robin/Dirichlet compiled in (GEN)
#define PD_FAST_TILE(NAME, N, BI, BJ)                                                          \
    using NAME = FastCfg<N, N, BI, BJ, false>;                                                 \
    using NAME##M = FastCfg<N, N, BI, BJ, true>;                                               \
    using NAME##P = FastCfg<N, N, BI, BJ, false, true>;                                        \
    using NAME##MP = FastCfg<N, N, BI, BJ, true, true>;                                        \
    using NAME##G = FastCfg<N, N, BI, BJ, false, false, true>;                                 \
    using NAME##MG = FastCfg<N, N, BI, BJ, true, false, true>;                                 \
    using NAME##PG = FastCfg<N, N, BI, BJ, false, true, true>;                                 \
    using NAME##MPG = FastCfg<N, N, BI, BJ, true, true, true>;
PD_FAST_TILE(FC7, 7, 1, 7)
PD_FAST_TILE(FC8, 8, 2, 4)
PD_FAST_TILE(FC9, 9, 3, 3)
PD_FAST_TILE(FC11, 11, 1, 11) // the reference's default micro grid (nx = ny = 10, scheme_config.hpp:17)
PD_FAST_TILE(FC16, 16, 2, 4)
#undef PD_FAST_TILE
// separable-source variants (5-point operator): exact / padded x Neumann / general
#define PD_FAST_SRC_TILE(NAME, N, BI, BJ)                                           \
    using NAME##S = FastCfg<N, N, BI, BJ, false, false, false, true>;               \
    using NAME##SP = FastCfg<N, N, BI, BJ, false, true, false, true>;               \
    using NAME##SG = FastCfg<N, N, BI, BJ, false, false, true, true>;               \
    using NAME##SPG = FastCfg<N, N, BI, BJ, false, true, true, true>;
PD_FAST_SRC_TILE(FC7, 7, 1, 7)
PD_FAST_SRC_TILE(FC8, 8, 2, 4)
PD_FAST_SRC_TILE(FC9, 9, 3, 3)
PD_FAST_SRC_TILE(FC11, 11, 1, 11)
PD_FAST_SRC_TILE(FC16, 16, 2, 4)
#undef PD_FAST_SRC_TILE

#define PD_FAST_TILE_IDS(X, B, NAME) \
    X(B + 0, NAME) X(B + 1, NAME##M) X(B + 2, NAME##P) X(B + 3, NAME##MP) X(B + 4, NAME##G) X(B + 5, NAME##MG) \
        X(B + 6, NAME##PG) X(B + 7, NAME##MPG)
#define PD_FAST_SRC_IDS(X, B, NAME) X(B + 0, NAME##S) X(B + 1, NAME##SP) X(B + 2, NAME##SG) X(B + 3, NAME##SPG)
#define PD_FAST_CONFIGS(X)                                                                                         \
    PD_FAST_TILE_IDS(X, 0, FC7) PD_FAST_TILE_IDS(X, 8, FC8) PD_FAST_TILE_IDS(X, 16, FC9) PD_FAST_TILE_IDS(X, 48, FC11) \
        PD_FAST_TILE_IDS(X, 24, FC16) PD_FAST_SRC_IDS(X, 32, FC7) PD_FAST_SRC_IDS(X, 36, FC8) PD_FAST_SRC_IDS(X, 40, FC9) \
        PD_FAST_SRC_IDS(X, 56, FC11) PD_FAST_SRC_IDS(X, 44, FC16)

inline bool plan_fast(const Params& p, FastPlan& plan) {
    // Neumann (every BASELINE config), Robin and Dirichlet patch conditions are
    // folded into the weights / node constants, both quadratures into the
    // restriction (Simpson exists only for odd node counts); sources stay EXACT
    const bool src = p.source == PD_SOURCE_SEPARABLE;
    if (p.source != PD_SOURCE_ZERO && !(src && !p.mixed)) return false; // sources: 5-point variant only
    if (p.quad == PD_QUAD_SIMPSON && ((p.n1 - 1) % 2 || (p.n2 - 1) % 2)) return false;
    int id = -1;
    // an exact-fit tile first (compile-time extents), else the smallest padded tile
    // (the 11x11 tile only as an exact fit: its padded variants index their 11-node
    // columns at run time; PD_FAST_TILE11=0 sends 11x11 to the padded 16x16 tile, for A/B runs)
    static const bool no11 = [] {
        const char* e = std::getenv("PD_FAST_TILE11");
        return e && e[0] == '0';
    }();
    const bool gen = p.bc_type != PD_BC_NEUMANN;
#define PD_MATCH(ID, CFG)                                                                                       \
    if (id < 0 && !CFG::PAD && CFG::GEN == gen && CFG::SRC == src && p.n1 == CFG::N1 && p.n2 == CFG::N2 &&        \
        (p.mixed != 0) == CFG::MIXED && !(no11 && CFG::N1 == 11))                                                   \
        id = ID;
    PD_FAST_CONFIGS(PD_MATCH)
#undef PD_MATCH
#define PD_MATCH_PAD(ID, CFG)                                                                                   \
    if (id < 0 && CFG::PAD && CFG::N1 != 11 && CFG::GEN == gen && CFG::SRC == src && p.n1 <= CFG::N1 &&           \
        p.n2 <= CFG::N2 && (p.mixed != 0) == CFG::MIXED)                                                            \
        id = ID;
    PD_FAST_CONFIGS(PD_MATCH_PAD)
#undef PD_MATCH_PAD
    if (id < 0) return false;
    plan.id = id;
    plan.mixed = p.mixed;
#define PD_FILL(ID, CFG)                               \
    if (id == ID) {                                    \
        plan.LP = CFG::LP;                             \
        plan.G = CFG::G;                               \
        plan.S = CFG::S;                               \
        plan.nunits = (p.P + CFG::G - 1) / CFG::G;     \
    }
    PD_FAST_CONFIGS(PD_FILL)
#undef PD_FILL
    return true;
}

inline size_t fast_weights_count(const FastPlan& plan, const Params&) {
    return (size_t)plan.nunits * plan.S * 64;
}

inline void fold_weights(const FastPlan& plan, const Params& p, const double* coeffs, const int* cset, double* W,
                         cudaStream_t s, const double* src_sp) {
    const size_t total = fast_weights_count(plan, p);
    const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
#define PD_FOLD(ID, CFG) \
    if (plan.id == ID) k_fold<CFG><<<blocks, 256, 0, s>>>(p, coeffs, cset, W, plan.nunits, src_sp);
    PD_FAST_CONFIGS(PD_FOLD)
#undef PD_FOLD
}

inline void launch_fast(const FastPlan& plan, const Params& p, const double* F, double* out, int out_mode,
                        const int* nbr, const double* W, const int* fail, cudaStream_t s, const double* srct) {
    const int blocks = (plan.nunits + kFastWarps - 1) / kFastWarps;
#define PD_LAUNCH(ID, CFG) \
    if (plan.id == ID)     \
        k_fast<CFG><<<blocks, 32 * kFastWarps, 0, s>>>(p, F, out, out_mode, nbr, W, plan.nunits, fail, srct);
    PD_FAST_CONFIGS(PD_LAUNCH)
#undef PD_LAUNCH
}

// Cooperative whole-run launch (at most one block per co-resident slot);
// returns false (nothing launched) when the units exceed run_waves() per
// co-resident warp.  The run kernel carries more live state than k_fast (about
// 220 registers instead of 168: 8-9 instead of 12 warps/SM), so it is used
// where per-step launch latency dominates (configs 1-3, small sweep points),
// not where the step is throughput-bound.
// The run kernel's warps stride over the units.  Measured (config-5 shapes,
// 20-step runs): with at most two units per co-resident warp the single launch
// wins at every K (8x8, 2^13 patches: 22.7 -> 14.1 us per step at K = 10,
// 102.3 -> 99.7 at K = 200); with more it wins only while a step is short
// (<= 2.5e7 node updates: 16x16 2^12 at K = 10 26.7 -> 20.8 us, 8x8 2^15
// 46.8 -> 42.4) and loses beyond (the run kernel's lower occupancy: 16x16 2^12
// at K = 200 165 -> 196 us).  PD_RUN_WAVES overrides for A/B runs.
inline int run_waves(const Params& p) {
    static const int forced = [] {
        const char* e = std::getenv("PD_RUN_WAVES");
        return e ? std::max(1, std::atoi(e)) : 0;
    }();
    if (forced) return forced;
    const double updates = (double)p.P * p.n1 * p.n2 * p.nt;
    return updates <= 2.5e7 ? 8 : 2;
}
inline bool launch_fast_run(const FastPlan& plan, const Params& p, double* UA, double* UB, const int* nbr,
                            const double* W, const double* bnd, size_t bnd_stride, const double* srct,
                            size_t srct_stride, int nsteps, double blowup, unsigned long long* slot,
                            unsigned long long* spread, int* fail, cudaStream_t s, const double* exact = nullptr,
                            double* err = nullptr) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int nunits = plan.nunits;
    bool launched = false;
#define PD_RUN(ID, CFG)                                                                                        \
    if (plan.id == ID) {                                                                                       \
        int per_sm = 0;                                                                                        \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fast_run<CFG>, 32 * kRunWarps, 0);            \
        const int blocks = (nunits + kRunWarps - 1) / kRunWarps;                                               \
        if (std::getenv("PD_DEBUG_RUN"))                                                                       \
            fprintf(stderr, "k_fast_run plan %d: %d blocks, %d per SM x %d SMs\n", ID, blocks, per_sm, sms);     \
        if (per_sm > 0 && blocks <= run_waves(p) * per_sm * sms) {                                              \
            Params pp = p;                                                                                     \
            void* args[] = {&pp, &UA, &UB, (void*)&nbr, (void*)&W, &nunits, (void*)&bnd, &bnd_stride,          \
                            (void*)&srct, &srct_stride, &nsteps, &blowup, &slot, &spread, &fail,               \
                            (void*)&exact, (void*)&err};                                                       \
            const int grid = std::min(blocks, per_sm * sms); /* warps stride over the units */                 \
            launched = cudaLaunchCooperativeKernel((const void*)k_fast_run<CFG>, dim3(grid),                   \
                                                   dim3(32 * kRunWarps), args, 0, s) == cudaSuccess;           \
            if (!launched) {                                                                                   \
                const cudaError_t e_ = cudaGetLastError(); /* the multi-launch loop runs instead */            \
                if (std::getenv("PD_DEBUG_RUN"))                                                               \
                    fprintf(stderr, "k_fast_run not launched: %s\n", cudaGetErrorString(e_));                  \
            }                                                                                                  \
        }                                                                                                      \
    }
    PD_FAST_CONFIGS(PD_RUN)
#undef PD_RUN
    return launched;
}

} // namespace pdb200::dev
