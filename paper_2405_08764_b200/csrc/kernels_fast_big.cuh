// FAST-mode fused gap-tooth kernel for large patches (32x32 micro nodes, the
// biggest config-5 shape): one CTA of WPP = 4 warps per patch.
//
// Same per-node algebra as kernels_fast.cuh (folded weights in registers,
// difference form of the mixed term, per-patch ghost constant), but a patch
// of 1024 nodes needs 128 lanes of 2x4 nodes: lane r = bj*LI + bi with LI = 16,
// so a warp holds block rows bj = 2w (lanes 0-15) and 2w+1 (lanes 16-31).
// Odd block rows store their block MIRRORED in eta (local jj = BJ-1 is the
// physical bottom row).  Then, for every lane, local "north" is the partner
// half of its own warp (one SHFL.BFLY 16, no selects) and local "south" is
// the neighbouring warp: each lane publishes its local row jj = 0 to shared
// memory (double-buffered by step parity, one CTA barrier per micro-step) and
// reads the partner row over columns i0-1 .. i0+2, which also yields the mixed
// term's xi-differences there without a second exchange.  Mirroring swaps the
// N/S weights and negates the mixed weight of odd block rows (k_fold_big).
#pragma once

#include "kernels_fast.cuh"

namespace pdb200::dev {

template <int N_, bool MIXED_, bool PAD_ = false, bool GEN_ = false>
struct BigCfg {
    static constexpr int N1 = N_, N2 = N_, BI = 2, BJ = 4;
    static constexpr bool MIXED = MIXED_;
    static constexpr bool GEN = GEN_; // Robin / Dirichlet patch conditions compiled in (as FastCfg)
    static constexpr bool PAD = PAD_; // patch smaller than the tile: phantom nodes (as FastCfg)
    static constexpr int LI = N1 / BI, LJ = N2 / BJ, LP = LI * LJ, WPP = LP / 32;
    static constexpr int NPL = BI * BJ, NW = MIXED ? 6 : 5, NWL = NW * NPL, S = (NWL + 1) / 2;
    static constexpr int L = N_;
    static constexpr int ROW = N1 + 4; // padded row: column i at index i + 2
    static_assert(LP % 32 == 0 && LI <= 32, "rows of blocks must not straddle warps");
};

// Weight tile of warp w of patch q at unit q*WPP + w: the FastCfg layout with
// one "unit" per warp (lane r = w*32 + lane of the patch).
template <class Cfg>
__global__ void k_fold_big(Params p, const double* __restrict__ coeffs, const int* __restrict__ cset,
                           double* __restrict__ W, int nunits) {
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
        const long patch = (long)(unit / Cfg::WPP);
        const int r = (int)(unit % Cfg::WPP) * 32 + lane;
        double val = 0.0;
        if (patch < p.P && f < Cfg::NWL) {
            const int lkind = f / Cfg::NPL, node = f % Cfg::NPL;
            const int ii = node / Cfg::BJ, jj = node % Cfg::BJ;
            const int bi = r % Cfg::LI, bj = r / Cfg::LI;
            const bool flip = bj & 1; // mirrored block row: local N/S = physical S/N
            const int i = bi * Cfg::BI + ii, j = bj * Cfg::BJ + (flip ? Cfg::BJ - 1 - jj : jj);
            const int kind = flip && lkind == WN ? WS : flip && lkind == WS ? WN : lkind;
            const int n1 = Cfg::PAD ? p.n1 : Cfg::N1, n2 = Cfg::PAD ? p.n2 : Cfg::N2;
            if (Cfg::PAD && (i >= n1 || j >= n2)) { // phantom node
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
            const bool Wb = i == 0, Eb = i == n1 - 1, Sb = j == 0, Nb = j == n2 - 1;
            if (Cfg::GEN && p.pinned && (Wb || Eb || Sb || Nb)) {
                val = 0.0; // pinned edge node (as k_fold)
            } else {
                switch (kind) { // same static reflections as k_fold
                    case WE: val = Wb ? wE + wW : wE; break;
                    case WW: val = Eb ? wW + wE : wW; break;
                    case WN: val = Sb ? wN + wS : wN; break;
                    case WS: val = Nb ? wS + wN : wS; break;
                    case WD: val = flip ? -(dt * (B * ixy)) : dt * (B * ixy); break;
                    default: {
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

template <class Cfg>
__global__ void __launch_bounds__(32 * Cfg::WPP, 3)
k_fast_big(Params p, const double* __restrict__ F, double* __restrict__ out, int out_mode,
           const int* __restrict__ nbr, const double* __restrict__ Wt, const int* __restrict__ fail_flag) {
    constexpr int BI = Cfg::BI, BJ = Cfg::BJ, LI = Cfg::LI, LJ = Cfg::LJ, NPL = Cfg::NPL, S = Cfg::S;
    constexpr int N1 = Cfg::N1, N2 = Cfg::N2, ROW = Cfg::ROW, WPP = Cfg::WPP;
    constexpr bool MIXED = Cfg::MIXED;
    const int n1 = Cfg::PAD ? p.n1 : N1, n2 = Cfg::PAD ? p.n2 : N2; // the patch's real extent
    __shared__ double s_g[8][Cfg::L];                   // ghost offsets + mixed ring offsets
    __shared__ __align__(16) double s_row[2][LJ][ROW]; // [parity][block row][padded column]: local row jj = 0
    __shared__ double s_red[WPP];
    if (fail_flag && *fail_flag) return;
    const int patch = blockIdx.x;
    const int r = threadIdx.x, lane = r & 31, warp = r >> 5;
    const int bi = r % LI, bj = r / LI;
    const int i0 = bi * BI, j0 = bj * BJ;
    const bool flip = bj & 1; // mirrored block row (local jj <-> physical j0 + BJ-1-jj)

    // ---- loads: stencil indices first, then the weight tile ----------------
    int idx[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) idx[q] = __ldg(nbr + 9 * patch + q);
    double w[2 * S];
    {
        const double2* wp = reinterpret_cast<const double2*>(Wt) + ((size_t)patch * WPP + warp) * S * 32 + lane;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const double2 t = __ldg(wp + s * 32);
            w[2 * s] = t.x;
            w[2 * s + 1] = t.y;
        }
    }
#define WT(k, ii, jj) w[(k) * NPL + (ii) * BJ + (jj)]
    double v[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = __ldg(F + idx[q]);
    // zero the row pads once (columns -2, -1, N1, N1+1 are never written)
    for (int t = r; t < 2 * LJ * 4; t += 32 * WPP) {
        const int pad = t & 3, rest = t >> 2;
        (&s_row[0][0][0])[rest * ROW + (pad < 2 ? pad : N1 + pad)] = 0.0;
    }


    // ---- centre derivatives, ghost offsets, ring offsets (as patch_body) ----
    const double Uxi = (v[7] - v[1]) * p.i2Dxi;
    const double Ueta = (v[5] - v[3]) * p.i2Deta;
    const double hUxx = 0.5 * ((v[7] - 2.0 * v[4] + v[1]) * p.iDxi2);
    const double hUyy = 0.5 * ((v[5] - 2.0 * v[4] + v[3]) * p.iDeta2);
    const double Uxy = (v[8] - v[6] - v[2] + v[0]) * p.i4DD;
    const double C0 = v[4] - p.c24x * (2.0 * hUxx) - p.c24y * (2.0 * hUyy);
    for (int t = r; t < 2 * n2 + 2 * n1; t += 32 * WPP) {
        if (t < 2 * n2) {
            const int e = t < n2 ? PD_EDGE_E : PD_EDGE_W, j = t < n2 ? t : t - n2;
            const double* d = p.dlag[e];
            const double G0 = d[0] * v[0] + d[1] * v[3] + d[2] * v[6];
            const double G1 = d[0] * v[1] + d[1] * v[4] + d[2] * v[7];
            const double G2 = d[0] * v[2] + d[1] * v[5] + d[2] * v[8];
            const double sl = lagq_at(p, j, 0) * G0 + lagq_at(p, j, 1) * G1 + lagq_at(p, j, 2) * G2;
            if (!Cfg::GEN || p.bc_type == PD_BC_NEUMANN) {
                s_g[e][j] = p.gsc[e] * sl;
            } else {
                const double* w = p.vlag[e];
                const double V0 = w[0] * v[0] + w[1] * v[3] + w[2] * v[6];
                const double V1 = w[0] * v[1] + w[1] * v[4] + w[2] * v[7];
                const double V2 = w[0] * v[2] + w[1] * v[5] + w[2] * v[8];
                s_g[e][j] = edge_constant(p, e, lagq_at(p, j, 0) * V0 + lagq_at(p, j, 1) * V1 + lagq_at(p, j, 2) * V2, sl);
            }
        } else {
            const int u = t - 2 * n2;
            const int e = u < n1 ? PD_EDGE_N : PD_EDGE_S, i = u < n1 ? u : u - n1;
            const double* d = p.dlag[e];
            const double H0 = d[0] * v[0] + d[1] * v[1] + d[2] * v[2];
            const double H1 = d[0] * v[3] + d[1] * v[4] + d[2] * v[5];
            const double H2 = d[0] * v[6] + d[1] * v[7] + d[2] * v[8];
            const double sl = lagp_at(p, i, 0) * H0 + lagp_at(p, i, 1) * H1 + lagp_at(p, i, 2) * H2;
            if (!Cfg::GEN || p.bc_type == PD_BC_NEUMANN) {
                s_g[e][i] = p.gsc[e] * sl;
            } else {
                const double* w = p.vlag[e];
                const double V0 = w[0] * v[0] + w[1] * v[1] + w[2] * v[2];
                const double V1 = w[0] * v[3] + w[1] * v[4] + w[2] * v[5];
                const double V2 = w[0] * v[6] + w[1] * v[7] + w[2] * v[8];
                s_g[e][i] = edge_constant(p, e, lagp_at(p, i, 0) * V0 + lagp_at(p, i, 1) * V1 + lagp_at(p, i, 2) * V2, sl);
            }
        }
    }
    __syncthreads();
    const double* gE = s_g[PD_EDGE_E];
    const double* gW = s_g[PD_EDGE_W];
    const double* gN = s_g[PD_EDGE_N];
    const double* gS = s_g[PD_EDGE_S];
    if constexpr (MIXED) if (!(Cfg::GEN && p.pinned)) { // pinned ring nodes do not update
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
        for (int t = r; t < 2 * n2 + 2 * n1; t += 32 * WPP) {
            int e, i, j, k;
            if (t < 2 * n2) {
                e = t < n2 ? PD_EDGE_E : PD_EDGE_W;
                k = j = t < n2 ? t : t - n2;
                i = e == PD_EDGE_E ? n1 - 1 : 0;
            } else {
                const int u = t - 2 * n2;
                e = u < n1 ? PD_EDGE_N : PD_EDGE_S;
                k = i = u < n1 ? u : u - n1;
                j = e == PD_EDGE_N ? n2 - 1 : 0;
            }
            s_g[4 + e][k] = (off(i + 1, j + 1) + off(i - 1, j - 1)) - (off(i - 1, j + 1) + off(i + 1, j - 1));
        }
        __syncthreads();
    }

    // ---- lift + boundary fold-in ------------------------------------------
    // A physical eta edge can only be a local row jj = 0 (bj = 0 unmirrored: S;
    // bj = LJ-1 mirrored: N); its outward weight sits in the local S slot.
    double u[BI][BJ], c[BI][BJ];
    const bool etaEdge = bj == 0 || bj == LJ - 1;
    const double* gEta = flip ? gN : gS;
#pragma unroll
    for (int ii = 0; ii < BI; ++ii) {
        const int i = i0 + ii;
        const double X = -0.5 * p.h_xi + p.mdxi * i;
        const double Ai = C0 + X * (Uxi + X * hUxx), Bi = Ueta + X * Uxy;
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
            const int j = flip ? j0 + BJ - 1 - jj : j0 + jj;
            const double Y = -0.5 * p.h_eta + p.mdeta * j;
            u[ii][jj] = Ai + Y * (Bi + Y * hUyy);
            if constexpr (Cfg::PAD) {
                // padded tile: the physical N edge (j = n2-1) can sit in any block row;
                // its outward neighbour is local N in an unmirrored row, local S in a
                // mirrored one (compile-time slots in each branch)
                if (i >= n1 || j >= n2) { // phantom node
                    u[ii][jj] = 0.0;
                    c[ii][jj] = 0.0;
                    continue;
                }
                const bool Wb = i == 0, Eb = i == n1 - 1, Sb = j == 0, Nb = j == n2 - 1;
                double cc = 0.0;
                if (Cfg::GEN && p.pinned) {
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
                if (Wb) { cc = fma(WT(WW, ii, jj), gW[j], cc); WT(WW, ii, jj) = 0.0; }
                if (Eb) { cc = fma(WT(WE, ii, jj), gE[j], cc); WT(WE, ii, jj) = 0.0; }
                if (Sb) { cc = fma(WT(WS, ii, jj), gS[i], cc); WT(WS, ii, jj) = 0.0; } // row 0 is never mirrored
                if (Nb) {
                    if (flip) { cc = fma(WT(WS, ii, jj), gN[i], cc); WT(WS, ii, jj) = 0.0; }
                    else { cc = fma(WT(WN, ii, jj), gN[i], cc); WT(WN, ii, jj) = 0.0; }
                }
                if constexpr (MIXED) {
                    if (Wb || Eb || Sb || Nb) {
                        const double* dd = s_g[4 + (Wb ? PD_EDGE_W : Eb ? PD_EDGE_E : Sb ? PD_EDGE_S : PD_EDGE_N)];
                        const double o = dd[(Wb || Eb) ? j : i];
                        cc = fma(WT(WD, ii, jj), flip ? -o : o, cc);
                        WT(WD, ii, jj) = 0.0;
                    }
                }
                c[ii][jj] = cc;
                continue;
            }
            const bool Wb = ii == 0 && bi == 0, Eb = ii == BI - 1 && bi == LI - 1;
            const bool Hb = jj == 0 && etaEdge; // physical S (unmirrored) or N (mirrored) edge
            double cc = 0.0;
            if (Cfg::GEN && p.pinned) { // as patch_body: sweep priority W, E, S|N; Dirichlet pins u0 in W, E, S|N order
                if (Wb) cc = gW[j];
                else if (Eb) cc = gE[j];
                else if (Hb) cc = gEta[i];
                if (p.bc_type == PD_BC_DIRICHLET) {
                    if (Wb) u[ii][jj] = gW[j];
                    if (Eb) u[ii][jj] = gE[j];
                    if (Hb) u[ii][jj] = gEta[i];
                }
                c[ii][jj] = cc;
                continue;
            }
            if (Wb) { cc = fma(WT(WW, ii, jj), gW[j], cc); WT(WW, ii, jj) = 0.0; }
            if (Eb) { cc = fma(WT(WE, ii, jj), gE[j], cc); WT(WE, ii, jj) = 0.0; }
            if (Hb) { cc = fma(WT(WS, ii, jj), gEta[i], cc); WT(WS, ii, jj) = 0.0; }
            if constexpr (MIXED) {
                if (Wb || Eb || Hb) {
                    // ring offsets are physical; the mirrored mixed weight carries a minus sign
                    const double* dd = s_g[4 + (Wb ? PD_EDGE_W : Eb ? PD_EDGE_E : flip ? PD_EDGE_N : PD_EDGE_S)];
                    const double o = dd[(Wb || Eb) ? j : i];
                    cc = fma(WT(WD, ii, jj), flip ? -o : o, cc);
                    WT(WD, ii, jj) = 0.0;
                }
            }
            c[ii][jj] = cc;
        }
    }

    // ---- K fused micro-steps ------------------------------------------------
    // local S partner row: the neighbouring warp's block row (clamped at the
    // patch edge, where the weights that would read it are zero)
    const int bjX = flip ? (bj + 1 < LJ ? bj + 1 : bj) : (bj > 0 ? bj - 1 : bj);
    double* const mine0 = &s_row[0][bj][i0 + 2];
    const double* const rx0 = &s_row[0][bjX][i0 + 2];
    // The hand-off of step s+1's row is published at the END of step s (after the
    // whole update), then one barrier; step 0's before the loop.  Measured against
    // publishing at the top of each step (same arithmetic, ptxas places the barrier
    // differently): 9-11 % faster at K = 10-200 (profiles/r02_ceiling.md).
    static_assert(BI == 2, "the row hand-off moves one 16-byte pair per lane");
    // local row jj = 0 as one 128-bit store / load per lane (bank-conflict free;
    // two 64-bit accesses at a 16-byte lane stride conflicted 2-way)
    *reinterpret_cast<double2*>(mine0) = make_double2(u[0][0], u[1][0]);
    __syncthreads();
    for (int step = 0; step < p.nt; ++step) {
        const int po = (step & 1) * LJ * ROW;
        const double2 pr = *reinterpret_cast<const double2*>(rx0 + po);
        double hS[BI], hN[BI], eS[BI], eN[BI];
        hS[0] = pr.x;
        hS[1] = pr.y;
#pragma unroll
        for (int ii = 0; ii < BI; ++ii) hN[ii] = __shfl_xor_sync(0xffffffffu, u[ii][BJ - 1], 16); // partner half
        if constexpr (MIXED) {
            // columns i0-1 and i0+2 of the partner row are the neighbouring lanes' pairs
            // (at a half-warp end the value is finite and its weight zero: patch edge)
            const double lft = __shfl_up_sync(0xffffffffu, pr.y, 1), rgt = __shfl_down_sync(0xffffffffu, pr.x, 1);
            eS[0] = pr.y - lft;
            eS[1] = rgt - pr.x;
        }
        double cE[BJ], cW[BJ];
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
            cE[jj] = __shfl_down_sync(0xffffffffu, u[0][jj], 1);
            cW[jj] = __shfl_up_sync(0xffffffffu, u[BI - 1][jj], 1);
        }
        auto at = [&](int a, int b) -> double { // block-relative, a in [-1,BI], b in [-1,BJ] (no corners)
            if (a == BI) return cE[b];
            if (a == -1) return cW[b];
            if (b == BJ) return hN[a];
            if (b == -1) return hS[a];
            return u[a][b];
        };
        double nu[BI][BJ];
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(WC, ii, jj), u[ii][jj], c[ii][jj]);
        // term order N, W, S, E: of the 24 orders x {barrier at the top, at the end}
        // this one gives ptxas's shortest loop (control-word stall sum 175 vs 235 for
        // the previous E, W, N, S with the barrier at the top; scripts/lab/stallsearch.py)
        auto term = [&](int k) {
            const int da = k == WE ? 1 : k == WW ? -1 : 0, db = k == WN ? 1 : k == WS ? -1 : 0;
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) nu[ii][jj] = fma(WT(k, ii, jj), at(ii + da, jj + db), nu[ii][jj]);
        };
        term(WN);
        term(WW);
        term(WS);
        term(WE);
        if constexpr (MIXED) {
            double e[BI][BJ];
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) e[ii][jj] = at(ii + 1, jj) - at(ii - 1, jj);
#pragma unroll
            for (int ii = 0; ii < BI; ++ii) eN[ii] = __shfl_xor_sync(0xffffffffu, e[ii][BJ - 1], 16);
#pragma unroll
            for (int ii = 0; ii < BI; ++ii)
#pragma unroll
                for (int jj = 0; jj < BJ; ++jj) {
                    const double upv = jj + 1 < BJ ? e[ii][jj + 1] : eN[ii];
                    const double dnv = jj > 0 ? e[ii][jj - 1] : eS[ii];
                    nu[ii][jj] = fma(WT(WD, ii, jj), upv - dnv, nu[ii][jj]);
                }
        }
#pragma unroll
        for (int ii = 0; ii < BI; ++ii)
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) u[ii][jj] = nu[ii][jj];
        if (step + 1 < p.nt) { // double-buffered by step parity: one barrier per micro-step
            *reinterpret_cast<double2*>(mine0 + ((step + 1) & 1) * LJ * ROW) = make_double2(u[0][0], u[1][0]);
            __syncthreads();
        }
    }
#undef WT

    // ---- trapezoid restriction: lane partials, warp reduce, CTA reduce -------
    double part = 0.0;
    if constexpr (Cfg::PAD) { // real extent at run time, phantom nodes weigh nothing
#pragma unroll
        for (int ii = 0; ii < BI; ++ii) {
            const int i = i0 + ii;
            double row = 0.0;
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) {
                const int j = flip ? j0 + BJ - 1 - jj : j0 + jj;
                row += (j < n2 ? quad_weight_rt(j, n2 - 1, p.quad) : 0.0) * u[ii][jj];
            }
            part += (i < n1 ? quad_weight_rt(i, n1 - 1, p.quad) : 0.0) * row;
        }
    } else {
        const double ox = 1.0 / (N1 - 1), oy = 1.0 / (N2 - 1);
#pragma unroll
        for (int ii = 0; ii < BI; ++ii) {
            double row = 0.0;
#pragma unroll
            for (int jj = 0; jj < BJ; ++jj) {
                const bool edge = jj == 0 && etaEdge; // physical eta edges are local rows jj = 0
                row += (edge ? 0.5 * oy : oy) * u[ii][jj];
            }
            const bool edge = (ii == 0 && bi == 0) || (ii == BI - 1 && bi == LI - 1);
            part += (edge ? 0.5 * ox : ox) * row;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_red[warp] = part;
    __syncthreads();
    if (r == 0) {
        double avg = 0.0;
#pragma unroll
        for (int q = 0; q < WPP; ++q) avg += s_red[q];
        const size_t node = (size_t)idx[4];
        if (out_mode == 0) {
            out[node] = avg;
            halo_store(p, node, avg);
        } else if (out_mode == 1) {
            const double U = v[4];
            const double w = U + p.dt_macro * ((avg - U) / p.tau); // cpi.cpp:54, 74 (k = 0)
            out[node] = w;
            halo_store(p, node, w); // decomposed run: fused peer-memory halo
        } else {
            out[patch] = avg;
        }
    }
}

using BC32 = BigCfg<32, false>;
using BC32M = BigCfg<32, true>;
using BC32P = BigCfg<32, false, true>;  // padded: any patch of 17..32 micro nodes per side
using BC32MP = BigCfg<32, true, true>;
using BC32G = BigCfg<32, false, false, true>; // with Robin / Dirichlet patch conditions
using BC32MG = BigCfg<32, true, false, true>;
using BC32PG = BigCfg<32, false, true, true>;
using BC32MPG = BigCfg<32, true, true, true>;

} // namespace pdb200::dev

namespace pdb200::dev {

inline bool plan_big(const Params& p, FastPlan& plan) {
    if (p.source != PD_SOURCE_ZERO) return false;
    // exact 32 x 32 tiles, or padded ones for patches of up to 32 nodes per side
    // that do not fit the one-warp 16 x 16 tile
    const bool exact = p.n1 == 32 && p.n2 == 32;
    const bool pad = !exact && p.n1 <= 32 && p.n2 <= 32 && (p.n1 > 16 || p.n2 > 16);
    if (!exact && !pad) return false;
    plan.big = 1;
    plan.mixed = p.mixed;
    plan.id = (p.mixed ? 101 : 100) + (pad ? 2 : 0) + (p.bc_type != PD_BC_NEUMANN ? 4 : 0);
    plan.LP = BC32::LP;
    plan.G = 1;
    plan.S = p.mixed ? BC32M::S : BC32::S;
    plan.nunits = p.P * BC32::WPP;
    return true;
}

#define PD_BIG_CONFIGS(X)                                                                                  \
    X(100, BC32) X(101, BC32M) X(102, BC32P) X(103, BC32MP) X(104, BC32G) X(105, BC32MG) X(106, BC32PG) \
        X(107, BC32MPG)

inline void fold_big(const FastPlan& plan, const Params& p, const double* coeffs, const int* cset, double* W,
                     cudaStream_t s) {
    const size_t total = (size_t)plan.nunits * plan.S * 64;
    const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
#define PD_BIG_FOLD(ID, CFG) \
    if (plan.id == ID) k_fold_big<CFG><<<blocks, 256, 0, s>>>(p, coeffs, cset, W, plan.nunits);
    PD_BIG_CONFIGS(PD_BIG_FOLD)
#undef PD_BIG_FOLD
}

inline void launch_big(const FastPlan& plan, const Params& p, const double* F, double* out, int out_mode,
                       const int* nbr, const double* W, const int* fail, cudaStream_t s) {
#define PD_BIG_LAUNCH(ID, CFG) \
    if (plan.id == ID) k_fast_big<CFG><<<p.P, 32 * CFG::WPP, 0, s>>>(p, F, out, out_mode, nbr, W, fail);
    PD_BIG_CONFIGS(PD_BIG_LAUNCH)
#undef PD_BIG_LAUNCH
}

} // namespace pdb200::dev
