// FAST-mode ADI micro-solver: the reference's Peaceman-Rachford step
// (PatchIntegrator::adi_sweep, microsim.cpp:334-507) with everything static
// folded once per engine.
//
// The explicit half of each pass (cross_term, microsim.cpp:357-395, plus the
// identity and the half-weighted source) is affine in the tile and in the
// ghost offsets b, with operator weights that never change: k_adi_fast_fold
// PROBES the EXACT restatement (cross_term_t) with unit vectors to obtain, per
// node, the weights of its five neighbours along the explicit direction
// (offsets -2..2; the ghost rule's cIn / cEdge land on in-range nodes), of the
// two ghost offsets and of the source.  The implicit half's line matrices
// (adi_row, the reference's rows after the ghost fold-in) are factored once
// with reciprocal pivots: Thomas (l, 1/m, w) for two-point upwinding, the
// pivot-free kl = ku = 2 band elimination (multipliers, 1/B0, upper band)
// otherwise (linalg.cpp:8-61).  The fused step then does, per micro step and
// pass, one 3- (5-)term dot product and one substitution per node.
//
// One warp per patch (patches up to 32x32): the tile lives in shared memory
// (two padded copies, ping-pong); the right-hand side runs with the lanes
// across nodes, then lane l solves line l of the current pass down its own
// column/row.  Within 1e-11 of the reference like the
// explicit FAST kernels (reciprocal pivots and fma instead of IEEE divisions
// in the reference's order); EXACT stays the bit-identical path.
#pragma once

#include "kernels_adi.cuh"
#include "kernels_fast.cuh"

namespace pdb200::dev {

constexpr int kFastAdiWarps = 4;

// Per-set table, [dir] = 0 (implicit xi: lines j, k = i) / 1 (implicit eta: lines i, k = j), nodes in
// line order (t = line * n + k):
//   core [2][N][KC]: the explicit half's along-direction weights and the line factors
//        two-point upwinding  KC = 6:  W(-1) W(0) W(+1) | l  1/m  w        (Thomas)
//        three/four-point     KC = 10: W(-2..+2)        | f1 f2 1/B0 B1 B2 (band LU)
//   blo/bhi [2][L]: ghost-offset weights, nonzero only on the first / last line
//   adjlo/adjhi [2][L]: the implicit rows' ghost-offset coefficient at k = 0 / n-1
//   src [2][N]: half * spatial source (separable sources only)
// Only what a node uses is stored: 48 bytes per node and pass for two-point upwinding.
struct AdiFastLayout {
    int KC;
    size_t blo, bhi, adjlo, adjhi, src, total;
};
__host__ __device__ inline AdiFastLayout adi_fast_layout(const Params& p) {
    AdiFastLayout l;
    l.KC = p.upwind_order == PD_UPWIND_TWO ? 6 : 10;
    l.blo = (size_t)2 * p.N * l.KC;
    l.bhi = l.blo + 2 * (size_t)p.L;
    l.adjlo = l.bhi + 2 * (size_t)p.L;
    l.adjhi = l.adjlo + 2 * (size_t)p.L;
    l.src = l.adjhi + 2 * (size_t)p.L;
    l.total = l.src + (p.source == PD_SOURCE_SEPARABLE ? 2 * (size_t)p.N : 0);
    return l;
}
__host__ __device__ inline size_t adi_fast_doubles(const Params& p) { return adi_fast_layout(p).total; }

// One thread per (set, direction, line); the table must be zeroed (unused weights stay 0).
__global__ void k_adi_fast_fold(Params p, const double* __restrict__ coeffs, const double* __restrict__ src_sp,
                                int nsets, double* __restrict__ tab) {
    const int kind = p.bc_type == PD_BC_DIRICHLET ? PD_EDGE_DIRICHLET
                   : p.bc_type == PD_BC_ROBIN     ? PD_EDGE_ROBIN
                                                  : PD_EDGE_NEUMANN;
    EdgeSh E[4];
    make_ghost_x(E[PD_EDGE_E], kind, p.w1, p.w2, p.mdxi, +1.0, 0, nullptr, nullptr, nullptr);
    make_ghost_x(E[PD_EDGE_W], kind, p.w1, p.w2, p.mdxi, -1.0, 0, nullptr, nullptr, nullptr);
    make_ghost_x(E[PD_EDGE_N], kind, p.w1, p.w2, p.mdeta, +1.0, 0, nullptr, nullptr, nullptr);
    make_ghost_x(E[PD_EDGE_S], kind, p.w1, p.w2, p.mdeta, -1.0, 0, nullptr, nullptr, nullptr);
    const int L = p.L, n2 = p.n2;
    const double half = XMUL(0.5, p.mdt);
    const int total = nsets * 2 * L;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int set = t / (2 * L), dir = (t / L) % 2, line = t % L;
        const bool xi_dir = dir == 0; // implicit direction of this pass
        const int nline = xi_dir ? p.ny : p.nx, n = xi_dir ? p.n1 : p.n2;
        if (line > nline) continue;
        const double* coef = coeffs + (size_t)set * PD_NCOEF * p.N;
        const double* sp = src_sp ? src_sp + (size_t)set * p.N : nullptr;
        const AdiFastLayout lay = adi_fast_layout(p);
        double* S0 = tab + (size_t)set * lay.total;                       // this set's table (zeroed)
        double* C = S0 + ((size_t)dir * p.N + (size_t)line * n) * lay.KC; // this line's core rows
        const int elo_x = xi_dir ? PD_EDGE_S : PD_EDGE_W, ehi_x = xi_dir ? PD_EDGE_N : PD_EDGE_E; // explicit dir
        const int wide = lay.KC == 10 ? 2 : 1;                            // weight offsets stored: -wide..wide
        for (int k = 0; k < n; ++k) {
            const int i = xi_dir ? k : line, j = xi_dir ? line : k, q = i * n2 + j;
            double* o = C + (size_t)k * lay.KC;
            if (!node_pinned_x(E, i, j, p.nx, p.ny)) {
                // explicit half (rhs = f + half (cross_term + G)), probed with unit vectors
                for (int off = -wide; off <= wide; ++off) {
                    const int ii = xi_dir ? i : i + off, jj = xi_dir ? j + off : j;
                    if (ii < 0 || ii > p.nx || jj < 0 || jj > p.ny) continue;
                    const int tgt = ii * n2 + jj;
                    auto fu = [tgt](int kk) { return kk == tgt ? 1.0 : 0.0; };
                    auto g0 = [](int) { return 0.0; };
                    const double ct = cross_term_t(p, fu, E, g0, coef, i, j, xi_dir);
                    o[off + wide] = XADD(off == 0 ? 1.0 : 0.0, XMUL(half, ct));
                }
                const int pos = xi_dir ? i : j;
                auto f0 = [](int) { return 0.0; };
                const int glo = elo_x * L + pos, ghi = ehi_x * L + pos;
                // a ghost is read only by the first / last line's nodes (cross_term: j == 0 / ny)
                if (line == 0)
                    S0[lay.blo + dir * L + k] = XMUL(
                        half, cross_term_t(p, f0, E, [glo](int kk) { return kk == glo ? 1.0 : 0.0; }, coef, i, j, xi_dir));
                if (line == nline)
                    S0[lay.bhi + dir * L + k] = XMUL(
                        half, cross_term_t(p, f0, E, [ghi](int kk) { return kk == ghi ? 1.0 : 0.0; }, coef, i, j, xi_dir));
                if (sp) S0[lay.src + (size_t)dir * p.N + (size_t)line * n + k] = XMUL(half, sp[q]);
            }
            if (k == 0) S0[lay.adjlo + dir * L + line] = adi_row(p, E, coef, xi_dir, line, k).adj;
            if (k == n - 1) S0[lay.adjhi + dir * L + line] = adi_row(p, E, coef, xi_dir, line, k).adj;
        }
        // implicit half: factor the line matrix with reciprocal pivots
        if (lay.KC == 6) {
            double wprev = 0.0;
            for (int k = 0; k < n; ++k) {
                const AdiRow r = adi_row(p, E, coef, xi_dir, line, k);
                const double lo = r.pinned ? 0.0 : r.sub, up = r.pinned ? 0.0 : r.sup;
                const double m = k == 0 ? r.diag : r.diag - lo * wprev;
                const double im = 1.0 / m;
                wprev = up * im;
                C[(size_t)k * 6 + 3] = lo;
                C[(size_t)k * 6 + 4] = im;
                C[(size_t)k * 6 + 5] = wprev;
            }
        } else {
            double band[33][5], mult[33][2];
            for (int k = 0; k < n; ++k) {
                const AdiRow r = adi_row(p, E, coef, xi_dir, line, k);
                band[k][0] = r.pinned ? 0.0 : r.lo2;
                band[k][1] = (r.pinned || k == 0) ? 0.0 : r.sub;
                band[k][2] = r.diag;
                band[k][3] = (r.pinned || k == n - 1) ? 0.0 : r.sup;
                band[k][4] = r.pinned ? 0.0 : r.hi2;
                mult[k][0] = mult[k][1] = 0.0;
            }
            for (int k = 0; k < n - 1; ++k) { // pivot-free elimination (linalg.cpp:43-61)
                const double piv = band[k][2];
                for (int r = k + 1; r <= min(k + 2, n - 1); ++r) {
                    const double f = band[r][2 + k - r] / piv;
                    mult[k][r - k - 1] = f;
                    for (int c = k + 1; c <= min(k + 2, n - 1); ++c) band[r][2 + c - r] -= f * band[k][2 + c - k];
                }
            }
            for (int k = 0; k < n; ++k) {
                double* c = C + (size_t)k * 10;
                c[5] = mult[k][0];
                c[6] = mult[k][1];
                c[7] = 1.0 / band[k][2];
                c[8] = k + 1 < n ? band[k][3] : 0.0;
                c[9] = k + 2 < n ? band[k][4] : 0.0;
            }
        }
    }
}

// A set's table is staged in shared memory by one bulk copy per patch (the
// serial line substitutions then read it at shared-memory latency) when it is
// at most this large and its size keeps 16-byte alignment; else read from global.
constexpr size_t kAdiStageMax = 24 * 1024;
__host__ __device__ inline bool adi_fast_staged(const Params& p) {
    const size_t t = adi_fast_doubles(p);
    return t % 2 == 0 && t * sizeof(double) <= kAdiStageMax;
}
// per-warp shared region in doubles: tiles A, Bt | gb [4][L] | red [32] | mbarrier (2) | staged table
__host__ __device__ inline size_t fast_adi_warp_doubles(const Params& p) {
    const size_t tile = (size_t)(p.n1 + 4) * (p.n2 + 4);
    const size_t base = 2 * tile + 4 * (size_t)p.L + 32 + 2;
    return base + (adi_fast_staged(p) ? adi_fast_doubles(p) : 0);
}
inline size_t fast_adi_smem_bytes(const Params& p) { return sizeof(double) * kFastAdiWarps * fast_adi_warp_doubles(p); }

// The fused step with the FAST ADI micro-solver, one warp per patch.
// STAGED (adi_fast_staged): the set's table is read from shared memory; else
// through the read-only global path (a template so neither variant reads
// through a generic pointer)
template <bool STAGED>
__global__ void __launch_bounds__(32 * kFastAdiWarps, 4)
k_fast_adi(Params p, const double* __restrict__ F, double* __restrict__ out, int out_mode, const int* __restrict__ nbr,
           const int* __restrict__ cset, const double* __restrict__ tab, const double* __restrict__ srct,
           const int* __restrict__ fail_flag) {
    extern __shared__ __align__(16) double sm[];
    if (fail_flag && *fail_flag) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int patch = blockIdx.x * kFastAdiWarps + warp;
    if (patch >= p.P) return; // warp-uniform
    const int n1 = p.n1, n2 = p.n2, nx = p.nx, ny = p.ny, L = p.L, TS = n2 + 4;
    const size_t tile = (size_t)(n1 + 4) * TS;
    double* A = sm + (size_t)warp * fast_adi_warp_doubles(p);
    double* Bt = A + tile;
    double* gb = Bt + tile;     // [4][L] ghost offsets b, or pinned values on pinned edges
    double* red = gb + 4 * L;   // [32]
    auto at = [TS](int i, int j) { return (i + 2) * TS + (j + 2); };
    // the set's static table streams into shared memory behind the gather, slopes and lift
    const int set = cset ? cset[patch] : patch;
    const AdiFastLayout lay = adi_fast_layout(p);
    double* stage = red + 32 + 2;
    const unsigned bar = smem_u32(red + 32);
    if (STAGED && lane == 0) {
        mbar_init(bar, 1);
        bulk_load(smem_u32(stage), tab + (size_t)set * lay.total, (unsigned)(lay.total * sizeof(double)), bar);
    }

    double v[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = __ldg(F + __ldg(nbr + 9 * patch + q));
    const double Uxi = __dmul_rn(__dsub_rn(v[7], v[1]), p.i2Dxi);
    const double Ueta = __dmul_rn(__dsub_rn(v[5], v[3]), p.i2Deta);
    const double hUxx = 0.5 * __dmul_rn(__dadd_rn(__fma_rn(-2.0, v[4], v[7]), v[1]), p.iDxi2);
    const double hUyy = 0.5 * __dmul_rn(__dadd_rn(__fma_rn(-2.0, v[4], v[5]), v[3]), p.iDeta2);
    const double Uxy = __dmul_rn(__dadd_rn(__dsub_rn(__dsub_rn(v[8], v[6]), v[2]), v[0]), p.i4DD);
    const double C0 = __fma_rn(-p.c24y, 2.0 * hUyy, __fma_rn(-p.c24x, 2.0 * hUxx, v[4]));

    // edge profiles -> ghost offsets / pinned values (dirichlet_edge_values, neumann_edge_slopes,
    // gaptooth.cpp:110-152; make_ghost / pinned_value, microsim.cpp:146-196)
    for (int t = lane; t < 2 * n2 + 2 * n1; t += 32) {
        int e, k;
        double sl, val;
        if (t < 2 * n2) {
            e = t < n2 ? PD_EDGE_E : PD_EDGE_W;
            k = t < n2 ? t : t - n2;
            const double* d = p.dlag[e];
            const double* w = p.vlag[e];
            sl = dot3(lagq_at(p, k, 0), dot3(d[0], v[0], d[1], v[3], d[2], v[6]), lagq_at(p, k, 1),
                      dot3(d[0], v[1], d[1], v[4], d[2], v[7]), lagq_at(p, k, 2), dot3(d[0], v[2], d[1], v[5], d[2], v[8]));
            val = dot3(lagq_at(p, k, 0), dot3(w[0], v[0], w[1], v[3], w[2], v[6]), lagq_at(p, k, 1),
                       dot3(w[0], v[1], w[1], v[4], w[2], v[7]), lagq_at(p, k, 2), dot3(w[0], v[2], w[1], v[5], w[2], v[8]));
        } else {
            const int u = t - 2 * n2;
            e = u < n1 ? PD_EDGE_N : PD_EDGE_S;
            k = u < n1 ? u : u - n1;
            const double* d = p.dlag[e];
            const double* w = p.vlag[e];
            sl = dot3(lagp_at(p, k, 0), dot3(d[0], v[0], d[1], v[1], d[2], v[2]), lagp_at(p, k, 1),
                      dot3(d[0], v[3], d[1], v[4], d[2], v[5]), lagp_at(p, k, 2), dot3(d[0], v[6], d[1], v[7], d[2], v[8]));
            val = dot3(lagp_at(p, k, 0), dot3(w[0], v[0], w[1], v[1], w[2], v[2]), lagp_at(p, k, 1),
                       dot3(w[0], v[3], w[1], v[4], w[2], v[5]), lagp_at(p, k, 2), dot3(w[0], v[6], w[1], v[7], w[2], v[8]));
        }
        gb[e * L + k] = p.bc_type == PD_BC_NEUMANN ? __dmul_rn(p.gsc[e], sl) : edge_constant(p, e, val, sl);
    }
    // zero both tiles (the pads are read with zero weights), then the quadratic lift
    for (size_t t = lane; t < 2 * tile; t += 32) A[t] = 0.0;
    __syncwarp();
    const bool dir_pin = p.bc_type == PD_BC_DIRICHLET; // Dirichlet pins the initial field (microsim.cpp:521-530)
    for (int t = lane; t < p.N; t += 32) {
        const int i = t / n2, j = t % n2;
        const double X = __fma_rn(p.mdxi, (double)i, -0.5 * p.h_xi);
        const double Y = __fma_rn(p.mdeta, (double)j, -0.5 * p.h_eta);
        double u = __fma_rn(Y, __fma_rn(Y, hUyy, __fma_rn(X, Uxy, Ueta)), __fma_rn(X, __fma_rn(X, hUxx, Uxi), C0));
        if (dir_pin) {
            if (i == 0) u = gb[PD_EDGE_W * L + j];
            if (i == nx) u = gb[PD_EDGE_E * L + j];
            if (j == 0) u = gb[PD_EDGE_S * L + i];
            if (j == ny) u = gb[PD_EDGE_N * L + i];
        }
        A[at(i, j)] = u;
    }
    __syncwarp();

    const double* S0;
    if constexpr (STAGED) {
        __syncwarp();
        mbar_wait(bar, 0);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
        S0 = stage;
    } else {
        S0 = tab + (size_t)set * lay.total;
    }
    const bool banded = lay.KC == 10;
    const bool pin = p.pinned != 0;
    const double* srcw = p.source == PD_SOURCE_SEPARABLE ? S0 + lay.src : nullptr;
    for (int step = 0; step < p.nt; ++step) {
        const double ft = srct ? __ldg(srct + step) : 0.0;
#pragma unroll 1
        for (int dir = 0; dir < 2; ++dir) {
            const bool xi_dir = dir == 0;
            const double* src = xi_dir ? A : Bt;
            double* dst = xi_dir ? Bt : A;
            const int nline = xi_dir ? ny : nx, n = xi_dir ? n1 : n2;
            const int es = xi_dir ? 1 : TS;  // explicit-direction stride in the tile
            const int is = xi_dir ? TS : 1;  // implicit-direction stride
            const int elo = xi_dir ? PD_EDGE_W : PD_EDGE_S, ehi = xi_dir ? PD_EDGE_E : PD_EDGE_N;
            const int xlo = xi_dir ? PD_EDGE_S : PD_EDGE_W, xhi = xi_dir ? PD_EDGE_N : PD_EDGE_E;
            const double* Cd = S0 + (size_t)dir * p.N * lay.KC;
            // right-hand side (explicit half) on every node, lanes across nodes
            for (int t = lane; t < (nline + 1) * n; t += 32) {
                const int line = t / n, k = t - line * n;
                const int c = xi_dir ? at(k, line) : at(line, k);
                double r;
                if (pin && (line == 0 || line == nline)) { // a pinned edge line keeps its pinned values
                    r = gb[(line == 0 ? xlo : xhi) * L + k];
                } else if (pin && (k == 0 || k == n - 1)) {
                    r = gb[(k == 0 ? elo : ehi) * L + line];
                } else {
                    const double* w = Cd + (size_t)t * lay.KC;
                    if (!banded) {
                        r = w[1] * src[c];
                        r = __fma_rn(w[0], src[c - es], r);
                        r = __fma_rn(w[2], src[c + es], r);
                    } else {
                        r = w[2] * src[c];
                        r = __fma_rn(w[1], src[c - es], r);
                        r = __fma_rn(w[3], src[c + es], r);
                        r = __fma_rn(w[0], src[c - 2 * es], r);
                        r = __fma_rn(w[4], src[c + 2 * es], r);
                    }
                    if (line == 0) r = __fma_rn(S0[lay.blo + dir * L + k], gb[xlo * L + k], r);
                    if (line == nline) r = __fma_rn(S0[lay.bhi + dir * L + k], gb[xhi * L + k], r);
                    if (srcw) r = __fma_rn(srcw[(size_t)dir * p.N + t], ft, r);
                    if (k == 0) r = __fma_rn(-S0[lay.adjlo + dir * L + line], gb[elo * L + line], r);
                    else if (k == n - 1) r = __fma_rn(-S0[lay.adjhi + dir * L + line], gb[ehi * L + line], r);
                }
                dst[c] = r;
            }
            __syncwarp();
            // implicit half: one lane per line
            for (int line = lane; line <= nline; line += 32) {
                if (pin && (line == 0 || line == nline)) continue;
                const int base = xi_dir ? at(0, line) : at(line, 0);
                const double* T = Cd + (size_t)line * n * lay.KC;
                if (!banded) { // Thomas with reciprocal pivots
                    double y = 0.0;
#pragma unroll 4
                    for (int k = 0; k < n; ++k) {
                        const double* w = T + (size_t)k * 6;
                        const int c = base + k * is;
                        y = (k == 0 ? dst[c] : __fma_rn(-w[3], y, dst[c])) * w[4];
                        dst[c] = y;
                    }
#pragma unroll 4
                    for (int k = n - 2; k >= 0; --k) {
                        const int c = base + k * is;
                        y = __fma_rn(-T[(size_t)k * 6 + 5], y, dst[c]);
                        dst[c] = y;
                    }
                } else { // pivot-free band LU (kl = ku = 2)
#pragma unroll 4
                    for (int k = 0; k < n - 1; ++k) {
                        const double* w = T + (size_t)k * 10;
                        const int c = base + k * is;
                        const double rk = dst[c];
                        dst[c + is] = __fma_rn(-w[5], rk, dst[c + is]);
                        if (k + 2 < n) dst[c + 2 * is] = __fma_rn(-w[6], rk, dst[c + 2 * is]);
                    }
                    double x1 = 0.0, x2 = 0.0;
#pragma unroll 4
                    for (int k = n - 1; k >= 0; --k) {
                        const double* w = T + (size_t)k * 10;
                        const int c = base + k * is;
                        const double x = __fma_rn(-w[9], x2, __fma_rn(-w[8], x1, dst[c])) * w[7];
                        dst[c] = x;
                        x2 = x1;
                        x1 = x;
                    }
                }
            }
            __syncwarp();
        }
    }

    // restriction (trapezoid / Simpson, gaptooth.cpp:170-194): row sums per lane, then the warp
    double part = 0.0;
    for (int i = lane; i < n1; i += 32) {
        double row = 0.0;
        for (int j = 0; j < n2; ++j) row = __fma_rn(quad_weight_rt(j, ny, p.quad), A[at(i, j)], row);
        part = __fma_rn(quad_weight_rt(i, nx, p.quad), row, part);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) {
        const size_t node = (size_t)__ldg(nbr + 9 * patch + 4);
        if (out_mode == 0) {
            out[node] = part;
            halo_store(p, node, part);
        } else if (out_mode == 1) {
            const double w = __fma_rn(p.dt_macro, __ddiv_rn(__dsub_rn(part, v[4]), p.tau), v[4]); // cpi.cpp:54, 74
            out[node] = w;
            halo_store(p, node, w);
        } else {
            out[patch] = part;
        }
    }
    (void)red;
}

} // namespace pdb200::dev
