/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker or the CPU baseline — never as the product path.
 *
 * CPU restatement of the reference's explicit gap-tooth hot path
 * (/root/reference/proj/src/{gaptooth,microsim,cpi}.cpp), operation for
 * operation in the reference's evaluation order (IEEE double, no FMA
 * contraction: built with -ffp-contract=off), so that for b = 0 it reproduces
 * the unmodified reference bit for bit.  Extension beyond the reference (which
 * throws MixedTermUnsupported, microsim.cpp:239-244): the mixed derivative
 * B*u_xi_eta with B = -b/l and the corner-ghost rule of SURVEY Appendix B.4.
 * Parity status: b = 0 pinned against the reference itself (oracle/_ref);
 * b != 0 pinned only by its own exactness/convergence/locality tests.
 *
 * Consumes the same pd_engine_desc tables as the B200 engine.
 */
#ifndef PD_ORACLE_H
#define PD_ORACLE_H

#include "patchdyn_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

void pdo_set_threads(int n);
int pdo_get_threads(void);
const char* pdo_last_error(void);

/* build_stencil + slopes/values + lift for one stencil (gaptooth.cpp:74-168).
 * slopes/values: [4][L] in E,W,N,S order, L = max(nx,ny)+1. */
void pdo_lift(const double vals[9], double xi_c, double eta_c, double dxi, double deta,
              double h_xi, double h_eta, int nx, int ny, double* u0, double* slopes,
              double* values);
/* restrict_average (gaptooth.cpp:170-194). */
double pdo_restrict(const double* u, int n1, int n2, int quadrature);
/* PatchIntegrator::integrate, explicit (microsim.cpp:509-552), extended with
 * the mixed term.  coef: [6][n1][n2] solver form (A,B,C,Vx,Vy,W).  kinds[4]
 * E,W,N,S; values/slopes [4][L]; robin_w [4][2].  src_spatial [n1][n2] and
 * src_time [nt] (time(t0+s*dt)/l) or NULL.  u: in = initial, out = result.
 * Returns a pd_status. */
int pdo_integrate(const double* coef, int nx, int ny, int nt, double h_xi, double h_eta,
                  double tau, const int* kinds, const double* values, const double* slopes,
                  const double* robin_w, const double* src_spatial, const double* src_time,
                  double* u);
/* Same with the micro-solver chosen: PD_SOLVER_ADI runs PatchIntegrator::adi_sweep
 * (microsim.cpp:334-507) with upwind order PD_UPWIND_* and parameter r; src_time
 * then holds time(t0 + (s+1/2) dt)/l. */
int pdo_integrate_ex(const double* coef, int nx, int ny, int nt, double h_xi, double h_eta,
                     double tau, const int* kinds, const double* values, const double* slopes,
                     const double* robin_w, const double* src_spatial, const double* src_time,
                     double* u, int solver, int upwind_order, double upwind_r);

/* Engine-level restatements over the same descriptor as pd_engine_create. */
int pdo_gaptooth_step(const pd_engine_desc* d, const double* U_in, double* U_out, double t,
                      const double* bnd, const double* src_time);
int pdo_projective_step(const pd_engine_desc* d, const double* U_in, double* U_out, double t,
                        const double* bnd, const double* src_time);
int pdo_run(const pd_engine_desc* d, double* U, int nsteps, double t0, const double* bnd,
            const double* src_time, pd_run_stats* stats);
/* Restricted patch averages after one gap-tooth substep for a subset of
 * patches (indices into the patch table) — the sampled-parity and bounded
 * CPU-baseline entry for configs too large to run whole.  Returns seconds. */
double pdo_patch_subset(const pd_engine_desc* d, const double* U_in, double t, int nsub,
                        const int* patch_index, double* avg_out);

/* Input builder for the shear-cdr family (configs 4/5) without the product
 * library (pd_oracle_problem.c): resolves d's pins in place and fills the
 * seeded initial field U0 [(N_xi+1)(N_eta+1)], the patch list [P][2] and the
 * solver-form coefficient table [P][6][nx+1][ny+1].  Returns a pd_status. */
int pdo_shear_problem(pd_problem_desc* d, double* U0, int32_t* patch_ij, double* coeffs);
void pdo_seeded_field(int Nxi, int Neta, uint64_t seed, int sweeps, double* U);

/* Linear-response path (GapToothEngine::step with linear_cache, gaptooth.cpp:377-418).
 * evolve_batch: evolve_patch for n given stencils [n][3][3] (vals[p+1][q+1]) with patch
 * patch_index[m]'s integrator and centre.  linear_weights: build_row_weights,
 * row_w [Neta+1][9].  linear_step / _projective_step / _run: the 9-point macro
 * stencil with the row weights in place of the micro-solve. */
int pdo_evolve_batch(const pd_engine_desc* d, int n, const int* patch_index, const double* stencils, double t,
                     double* out);
int pdo_linear_weights(const pd_engine_desc* d, double* row_w);
int pdo_linear_step(const pd_engine_desc* d, const double* row_w, const double* U_in, double* U_out,
                    const double* bnd);
int pdo_linear_projective_step(const pd_engine_desc* d, const double* row_w, const double* U_in, double* U_out,
                               double t, const double* bnd);
int pdo_linear_run(const pd_engine_desc* d, const double* row_w, double* U, int nsteps, double t0,
                   const double* bnd, pd_run_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
