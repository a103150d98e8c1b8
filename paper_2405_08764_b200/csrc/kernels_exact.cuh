// EXACT-mode kernels: one CTA per patch, patch tile double-buffered in shared
// memory, the reference's operation order (see pd_device.cuh).  Used for
// bit-parity runs, for shapes the FAST kernel does not specialise, and for the
// unfused unit entries (pd_integrate_batch / pd_lift_batch / pd_restrict_batch).
#pragma once

#include "pd_device.cuh"

namespace pdb200::dev {

constexpr int kExactThreads = 128;
// threads per CTA of the fused EXACT step.  The ADI solver keeps only one
// thread per micro line busy in its solves: with enough patches to fill the
// chip, smaller CTAs (more of them per SM) win — measured on B200
// (profiles/r01_adi.jsonl): 16 129 patches of 11^2 nodes 1.84 -> 0.83 ms with
// 32 threads, of 21^2 nodes 7.62 -> 6.33 ms with 64; 81 patches prefer 128.
inline int exact_threads(const Params& p) {
    // explicit: two-warp CTAs for many small patches (16 384 patches of 16^2: 3.52 -> 3.27 ms)
    if (p.solver != PD_SOLVER_ADI) return (p.P >= 8 * 148 && p.N <= 256) ? 64 : kExactThreads;
    if (p.P < 8 * 148) return kExactThreads;
    return p.L <= 16 ? 32 : 64;
}

inline size_t exact_smem_bytes(const Params& p) {
    size_t d = 2 * (size_t)p.N + 3 * 4 * (size_t)p.L + p.n1 + 11 + 4 * 6;
    if (p.solver == PD_SOLVER_ADI) d += (size_t)p.N + 6 * (size_t)p.L * p.L; // rhs field + line scratch
    return sizeof(double) * d;
}

// ADI scratch behind the PatchSh region: rhs field [N], line scratch [L][6L]
__device__ inline double* adi_scratch(double* sm, const Params& p) {
    return sm + patch_smem_doubles(p.N, p.L, p.n1);
}

// Dirichlet edges pin their nodes from the start (microsim.cpp:521-530; W, E, S, N order)
__device__ inline void pin_initial_x(double* u, const int* kinds, const double* val, int L, int nx, int ny) {
    const int n2 = ny + 1, N = (nx + 1) * n2;
    for (int t = threadIdx.x; t < N; t += blockDim.x) {
        const int i = t / n2, j = t % n2;
        double v = u[t];
        bool w = false;
        if (kinds[PD_EDGE_W] == PD_EDGE_DIRICHLET && i == 0) v = val[PD_EDGE_W * L + j], w = true;
        if (kinds[PD_EDGE_E] == PD_EDGE_DIRICHLET && i == nx) v = val[PD_EDGE_E * L + j], w = true;
        if (kinds[PD_EDGE_S] == PD_EDGE_DIRICHLET && j == 0) v = val[PD_EDGE_S * L + i], w = true;
        if (kinds[PD_EDGE_N] == PD_EDGE_DIRICHLET && j == ny) v = val[PD_EDGE_N * L + i], w = true;
        if (w) u[t] = v;
    }
}

// K explicit steps on the shared tile (PatchIntegrator::integrate loop,
// microsim.cpp:535-550).  Returns the buffer holding the result.
// Sampled variant (time-dependent coefficients / general sources,
// microsim.cpp:537-542 and 278-280): coef_steps / src_steps, when given, are
// this patch's set in per-micro-step tables [nt][sets][6][N] / [nt][sets][N]
// (stride = one step's tables); they replace coef and the source term.
__device__ inline double* micro_loop_x(const Params& p, PatchSh& s, const EdgeSh* eg, const double* coef,
                                       const double* src_sp, const double* src_time, bool mixed,
                                       const double* coef_steps = nullptr, size_t coef_stride = 0,
                                       const double* src_steps = nullptr, size_t src_stride = 0) {
    const double idx2 = XDIV(1.0, XMUL(p.mdxi, p.mdxi)), idy2 = XDIV(1.0, XMUL(p.mdeta, p.mdeta));
    const double idx = XDIV(1.0, XMUL(2.0, p.mdxi)), idy = XDIV(1.0, XMUL(2.0, p.mdeta));
    const double ixy = XDIV(1.0, XMUL(XMUL(4.0, p.mdxi), p.mdeta));
    double* cur = s.u0;
    double* nxt = s.u1;
    for (int step = 0; step < p.nt; ++step) {
        const double ft = (src_sp && src_time) ? src_time[step] : 0.0;
        const double* co = coef_steps ? coef_steps + coef_stride * step : coef;
        const double* gs = src_steps ? src_steps + src_stride * step : nullptr;
        for (int t = threadIdx.x; t < p.N; t += blockDim.x) {
            const int i = t / p.n2, j = t % p.n2;
            const double G = gs ? __ldg(gs + t) : (src_sp && src_time) ? XMUL(__ldg(src_sp + t), ft) : 0.0;
            nxt[t] = sweep_node_x(cur, eg, s.val, s.slope, s.gb, p.L, p.nx, p.ny, i, j, co, p.N, G, idx2, idy2,
                                  idx, idy, ixy, p.mdt, mixed);
        }
        __syncthreads();
        double* tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    return cur;
}

__device__ inline void setup_ghosts_x(const Params& p, PatchSh& s, EdgeSh* eg, const int* kinds, const double* rw) {
    make_ghost_x(eg[PD_EDGE_E], kinds[PD_EDGE_E], rw[0], rw[1], p.mdxi, +1.0, p.n2, s.val + PD_EDGE_E * p.L,
                 s.slope + PD_EDGE_E * p.L, s.gb + PD_EDGE_E * p.L);
    make_ghost_x(eg[PD_EDGE_W], kinds[PD_EDGE_W], rw[2], rw[3], p.mdxi, -1.0, p.n2, s.val + PD_EDGE_W * p.L,
                 s.slope + PD_EDGE_W * p.L, s.gb + PD_EDGE_W * p.L);
    make_ghost_x(eg[PD_EDGE_N], kinds[PD_EDGE_N], rw[4], rw[5], p.mdeta, +1.0, p.n1, s.val + PD_EDGE_N * p.L,
                 s.slope + PD_EDGE_N * p.L, s.gb + PD_EDGE_N * p.L);
    make_ghost_x(eg[PD_EDGE_S], kinds[PD_EDGE_S], rw[6], rw[7], p.mdeta, -1.0, p.n1, s.val + PD_EDGE_S * p.L,
                 s.slope + PD_EDGE_S * p.L, s.gb + PD_EDGE_S * p.L);
}

// Output modes of the fused step kernels.
enum { OUT_FIELD = 0, OUT_PROJECTIVE = 1, OUT_PATCH = 2 };

// Fused gap-tooth step, EXACT: build_stencil -> edge profiles -> lift ->
// integrate -> restrict_average (gaptooth.cpp:74-104, 312-353) and, for
// OUT_PROJECTIVE with k = 0, the forward-Euler extrapolation of
// cpi.cpp:67-74.  One CTA per patch.
__global__ void __launch_bounds__(kExactThreads)
k_gaptooth_exact(Params p, const double* __restrict__ F, double* __restrict__ out, int out_mode,
                 const int* __restrict__ pij, const int* __restrict__ cset, const double* __restrict__ coeffs,
                 const double* __restrict__ src_sp, const double* __restrict__ src_time,
                 const int* __restrict__ fail_flag, const double* __restrict__ stencil_in = nullptr,
                 const int* __restrict__ item_patch = nullptr, const double* __restrict__ adi_fac = nullptr,
                 const double* __restrict__ coef_steps = nullptr, const double* __restrict__ src_steps = nullptr) {
    extern __shared__ double sm[];
    if (fail_flag && *fail_flag) return;
    // item_patch != NULL: evolve_patch of given 3x3 values (stencil_in [items][9])
    // with patch item_patch[item]'s integrator and centre (build_row_weights,
    // gaptooth.cpp:377-394); the average goes to out[item].
    const int item = blockIdx.x;
    const int patch = item_patch ? item_patch[item] : item;
    PatchSh s = carve(sm, p.N, p.L, p.n1);
    const int i = pij[2 * patch], j = pij[2 * patch + 1];
    int ic = i;
    if (p.periodic) ic = ((i % p.Nxi) + p.Nxi) % p.Nxi;
    if (threadIdx.x < 9) {
        const int dp = threadIdx.x / 3 - 1, dq = threadIdx.x % 3 - 1;
        const int ip = p.periodic ? ((ic + dp) % p.Nxi + p.Nxi) % p.Nxi : i + dp;
        s.stencil[threadIdx.x] = stencil_in ? stencil_in[(size_t)9 * item + threadIdx.x]
                                            : F[(size_t)ip * p.NF2 + j + dq];
    }
    const double xi_c = XADD(p.a, XMUL(p.Dxi, (double)ic));
    const double eta_c = XADD(p.c, XMUL(p.Deta, (double)j));
    __syncthreads();
    const int kind = p.bc_type == PD_BC_DIRICHLET ? PD_EDGE_DIRICHLET
                   : p.bc_type == PD_BC_ROBIN     ? PD_EDGE_ROBIN
                                                  : PD_EDGE_NEUMANN;
    edge_profiles_x(s.stencil, xi_c, eta_c, p.Dxi, p.Deta, p.h_xi, p.h_eta, p.nx, p.ny, p.L,
                    kind != PD_EDGE_DIRICHLET, kind != PD_EDGE_NEUMANN, s.slope, s.val);
    lift_x(s.stencil, p.Dxi, p.Deta, p.h_xi, p.h_eta, p.nx, p.ny, s.u0);
    __syncthreads();
    const int kinds[4] = {kind, kind, kind, kind};
    const double rw[8] = {p.w1, p.w2, p.w1, p.w2, p.w1, p.w2, p.w1, p.w2};
    EdgeSh eg[4];
    setup_ghosts_x(p, s, eg, kinds, rw);
    pin_initial_x(s.u0, kinds, s.val, p.L, p.nx, p.ny);
    __syncthreads();
    const int set = cset ? cset[patch] : patch;
    const double* coef = coeffs + (size_t)set * PD_NCOEF * p.N;
    const double* sp = src_sp ? src_sp + (size_t)set * p.N : nullptr;
    double* res;
    if (p.solver == PD_SOLVER_ADI) {
        double* xs = adi_scratch(sm, p);
        res = micro_loop_adi(p, s, eg, coef, sp, src_time, xs, xs + p.N,
                             adi_fac ? adi_fac + (size_t)set * adi_factor_doubles(p) : nullptr);
    } else {
        const size_t cst = (size_t)p.nsets * PD_NCOEF * p.N, sst = (size_t)p.nsets * p.N;
        res = micro_loop_x(p, s, eg, coef, sp, src_time, p.mixed != 0,
                           coef_steps ? coef_steps + (size_t)set * PD_NCOEF * p.N : nullptr, cst,
                           src_steps ? src_steps + (size_t)set * p.N : nullptr, sst);
    }
    const double avg = restrict_x(res, p.nx, p.ny, p.quad, s.row);
    if (threadIdx.x == 0) {
        const size_t node = (size_t)i * p.NF2 + j;
        if (out_mode == OUT_FIELD) {
            out[node] = avg;
            halo_store(p, node, avg);
        } else if (out_mode == OUT_PROJECTIVE) {
            const double U = F[node];
            const double Fd = XDIV(XSUB(avg, U), p.tau); // estimate_derivative  cpi.cpp:54
            const double w = XADD(U, XMUL(p.dt_macro, Fd)); // cpi.cpp:74 with k = 0
            out[node] = w;
            halo_store(p, node, w); // decomposed run: fused peer-memory halo
        } else {
            out[item] = avg;
        }
    }
}

// GapToothEngine::step, linear-response path (gaptooth.cpp:396-418): every
// patch value is the 9-point macro stencil with its row's impulse-response
// weights, accumulated in the reference's order (p outer, q inner, IEEE
// add/mul, no contraction).  out_mode as k_gaptooth_exact (FIELD / PROJECTIVE).
__global__ void k_linear_step(Params p, const double* __restrict__ F, double* __restrict__ out, int out_mode,
                              const int* __restrict__ pij, const double* __restrict__ row_w,
                              const int* __restrict__ fail_flag) {
    if (fail_flag && *fail_flag) return;
    const int patch = blockIdx.x * blockDim.x + threadIdx.x;
    if (patch >= p.P) return;
    const int i = pij[2 * patch], j = pij[2 * patch + 1];
    const double* w = row_w + (size_t)9 * j;
    double acc = 0.0;
#pragma unroll
    for (int dp = -1; dp <= 1; ++dp) {
        int ip = i + dp;
        if (p.periodic) ip = ((ip % p.Nxi) + p.Nxi) % p.Nxi;
#pragma unroll
        for (int dq = -1; dq <= 1; ++dq)
            acc = XADD(acc, XMUL(w[3 * (dp + 1) + dq + 1], F[(size_t)ip * p.NF2 + j + dq]));
    }
    const size_t node = (size_t)i * p.NF2 + j;
    if (out_mode == OUT_PROJECTIVE) {
        const double U = F[node];
        acc = XADD(U, XMUL(p.dt_macro, XDIV(XSUB(acc, U), p.tau))); // cpi.cpp:54, 74 (k = 0)
    }
    out[node] = acc;
    halo_store(p, node, acc);
}

// PatchIntegrator::integrate batched (microsim.cpp:509-552): u0/edges given.
__global__ void __launch_bounds__(kExactThreads)
k_integrate_exact(Params p, const double* __restrict__ u0, const double* __restrict__ ev,
                  const double* __restrict__ es, const int* __restrict__ kinds_in, const double* __restrict__ rw_in,
                  const int* __restrict__ cset, const double* __restrict__ coeffs, const double* __restrict__ src_sp,
                  const double* __restrict__ src_time, double* __restrict__ uT) {
    extern __shared__ double sm[];
    const int patch = blockIdx.x;
    PatchSh s = carve(sm, p.N, p.L, p.n1);
    for (int t = threadIdx.x; t < p.N; t += blockDim.x) s.u0[t] = u0[(size_t)patch * p.N + t];
    for (int t = threadIdx.x; t < 4 * p.L; t += blockDim.x) {
        s.val[t] = ev[(size_t)patch * 4 * p.L + t];
        s.slope[t] = es[(size_t)patch * 4 * p.L + t];
    }
    __syncthreads();
    int kinds[4];
    double rw[8];
    for (int e = 0; e < 4; ++e) kinds[e] = kinds_in[e];
    for (int e = 0; e < 8; ++e) rw[e] = rw_in[e];
    EdgeSh eg[4];
    setup_ghosts_x(p, s, eg, kinds, rw);
    pin_initial_x(s.u0, kinds, s.val, p.L, p.nx, p.ny);
    __syncthreads();
    const int set = cset ? cset[patch] : patch;
    const double* coef = coeffs + (size_t)set * PD_NCOEF * p.N;
    const double* sp = src_sp ? src_sp + (size_t)set * p.N : nullptr;
    double* res;
    if (p.solver == PD_SOLVER_ADI) {
        double* xs = adi_scratch(sm, p);
        res = micro_loop_adi(p, s, eg, coef, sp, src_time, xs, xs + p.N);
    } else {
        res = micro_loop_x(p, s, eg, coef, sp, src_time, p.mixed != 0);
    }
    for (int t = threadIdx.x; t < p.N; t += blockDim.x) uT[(size_t)patch * p.N + t] = res[t];
}

// Lifting chain for given stencils (gaptooth.cpp:110-168).
__global__ void __launch_bounds__(kExactThreads)
k_lift_exact(Params p, const double* __restrict__ vals, const double* __restrict__ centers,
             double* __restrict__ u0, double* __restrict__ slope, double* __restrict__ value) {
    const int q = blockIdx.x;
    const double* v = vals + 9 * (size_t)q;
    const double xi_c = centers[2 * q], eta_c = centers[2 * q + 1];
    edge_profiles_x(v, xi_c, eta_c, p.Dxi, p.Deta, p.h_xi, p.h_eta, p.nx, p.ny, p.L, true, true,
                    slope + (size_t)q * 4 * p.L, value + (size_t)q * 4 * p.L);
    lift_x(v, p.Dxi, p.Deta, p.h_xi, p.h_eta, p.nx, p.ny, u0 + (size_t)q * p.N);
}

__global__ void __launch_bounds__(kExactThreads)
k_restrict_exact(Params p, const double* __restrict__ u, double* __restrict__ avg) {
    extern __shared__ double sm[];
    const double a = restrict_x(u + (size_t)blockIdx.x * p.N, p.nx, p.ny, p.quad, sm);
    if (threadIdx.x == 0) avg[blockIdx.x] = a;
}

} // namespace pdb200::dev
