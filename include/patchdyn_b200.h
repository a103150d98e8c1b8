/*
 * patchdyn_b200.h — C-ABI of the B200-native gap-tooth hot path.
 *
 * This is the drop-in boundary between the reference's C++ operator
 * interfaces and the sm_100a kernels.  Plain pointers and sizes only; every
 * pointer argument named *_host is host memory, *_dev is device memory.
 * Citations are /root/reference/<path>:<line>.
 *
 * Entry point                      replaces (reference)
 * -------------------------------  -------------------------------------------------
 * pd_engine_create                 GapToothEngine ctor: patch list + PatchIntegrator
 *                                  coefficient sampling  proj/src/gaptooth.cpp:200-282,
 *                                  proj/src/microsim.cpp:204-263
 * pd_gaptooth_step                 GapToothEngine::step_direct  proj/src/gaptooth.cpp:360-375
 *                                  (proj/include/patchdyn/gaptooth.hpp:100)
 * pd_projective_step               cpi::projective_step  proj/src/cpi.cpp:58-77
 *                                  (proj/include/patchdyn/cpi.hpp:19-20)
 * pd_run                           cpi::run macro loop + blow-up guard
 *                                  proj/src/cpi.cpp:175-213 (cpi.hpp:45)
 * pd_integrate_batch               PatchIntegrator::integrate, batched over patches
 *                                  proj/src/microsim.cpp:509-552 (microsim.hpp:93-94)
 * pd_lift_batch                    build_stencil + neumann_edge_slopes /
 *                                  dirichlet_edge_values + lift
 *                                  proj/src/gaptooth.cpp:74-168
 * pd_restrict_batch                restrict_average  proj/src/gaptooth.cpp:170-194
 * pd_evolve_batch                  evolve_patch on given stencils  gaptooth.cpp:312-353
 * pd_linear_weights                GapToothEngine::build_row_weights  gaptooth.cpp:377-394
 * pd_engine_set_linear /           GapToothEngine::step's linear-response path
 *   pd_engine_set_step_kind        (linear_cache, gaptooth.cpp:213-224, 396-418)
 * pd_last_error / pd_status        typed exceptions proj/include/patchdyn/errors.hpp:9-61
 *
 * Host-side problem builder (mesh/metric setup, stays on the host as in the
 * reference; proj/src/geometry.cpp:93-125, microsim.cpp:226-263):
 * pd_problem_create / pd_problem_engine_desc / pd_problem_initial_field /
 * pd_problem_boundary / pd_problem_destroy.
 *
 * Threading: an engine owns one CUDA stream and is not thread-safe, matching
 * the reference engine (gaptooth.hpp:121-122 mutable caches).
 */
#ifndef PATCHDYN_B200_H
#define PATCHDYN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PD_ABI_VERSION 5

/* Status codes map 1:1 onto the reference exception types
 * (proj/include/patchdyn/errors.hpp:9-61). */
typedef enum pd_status {
    PD_OK = 0,
    PD_NON_POSITIVE_JACOBIAN = 1,  /* NonPositiveJacobian  errors.hpp:13 */
    PD_DERIVATIVE_MISMATCH = 2,    /* DerivativeMismatch   errors.hpp:16 */
    PD_MIXED_TERM_UNSUPPORTED = 3, /* MixedTermUnsupported errors.hpp:19 */
    PD_STABILITY_VIOLATION = 4,    /* StabilityViolation   errors.hpp:22 */
    PD_INSUFFICIENT_STENCIL = 5,   /* InsufficientStencil  errors.hpp:25 */
    PD_INDEX_OUT_OF_RANGE = 6,     /* IndexOutOfRange      errors.hpp:28 */
    PD_SHAPE_MISMATCH = 7,         /* ShapeMismatch        errors.hpp:31 */
    PD_INVALID_STRETCH = 8,        /* InvalidStretch       errors.hpp:34 */
    PD_DOMAIN_ERROR = 9,           /* DomainError          errors.hpp:37 */
    PD_MACRO_INSTABILITY = 12,     /* MacroInstability     errors.hpp:46 */
    PD_MACRO_PATCH_ERROR = 13,     /* MacroPatchError      errors.hpp:50 */
    PD_VALIDATION_ERROR = 15,      /* ValidationError      errors.hpp:56 */
    PD_CUDA_ERROR = 100,           /* device failure (no reference analogue) */
    PD_UNSUPPORTED = 101           /* feature outside the device path (ADI 3/4-point upwinding on non-square
                                      patches; a general source or time-dependent tables outside the
                                      sampled entries) */
} pd_status;

/* SchemeConfig::BCType  proj/include/patchdyn/scheme_config.hpp:21-23 */
enum { PD_BC_NEUMANN = 0, PD_BC_DIRICHLET = 1, PD_BC_ROBIN = 2 };
/* microsim::EdgeKind  proj/include/patchdyn/microsim.hpp:23 */
enum { PD_EDGE_DIRICHLET = 0, PD_EDGE_NEUMANN = 1, PD_EDGE_ROBIN = 2 };
/* microsim::Edge order  microsim.hpp:26 */
enum { PD_EDGE_E = 0, PD_EDGE_W = 1, PD_EDGE_N = 2, PD_EDGE_S = 3 };
/* SchemeConfig::Quadrature  scheme_config.hpp:25-26 */
enum { PD_QUAD_TRAPEZOID = 0, PD_QUAD_SIMPSON = 1 };
/* source structure  microsim.hpp:58-64 */
enum { PD_SOURCE_ZERO = 0, PD_SOURCE_SEPARABLE = 1,
       /* general f(x, y, t) (microsim.cpp:278-280): supplied per micro step through the
        * sampled entries below; the other step entries return PD_UNSUPPORTED */
       PD_SOURCE_GENERAL = 2 };
/* Micro-solver (SchemeConfig::Solver, scheme_config.hpp:19-20; NOTE the C
 * values differ from the reference's enum order so that a zero-initialised
 * descriptor selects the explicit scheme of the BASELINE configs) and the ADI
 * path's upwind convection order (UpwindOrder, microsim.hpp). */
enum { PD_SOLVER_EXPLICIT = 0, PD_SOLVER_ADI = 1 };
enum { PD_UPWIND_TWO = 0, PD_UPWIND_THREE = 1, PD_UPWIND_FOUR = 2 };
/* Kernel family.  EXACT replays the reference's operation order (IEEE, no FMA
 * contraction) and is bit-identical to the reference for b = 0; FAST is the
 * register-blocked folded-weight kernel (FMA), within 1e-11 of it. */
enum { PD_MODE_FAST = 0, PD_MODE_EXACT = 1 };

/* Solver-form coefficient slots per micro node (microsim.hpp:101-102, plus the
 * mixed term B = -b/l that the reference rejects at microsim.cpp:239-244). */
enum { PD_COEF_A = 0, PD_COEF_B = 1, PD_COEF_C = 2, PD_COEF_VX = 3, PD_COEF_VY = 4,
       PD_COEF_W = 5, PD_NCOEF = 6 };

/* Everything the engine needs; the library copies all tables to the device
 * and the caller keeps ownership of the host buffers. */
typedef struct pd_engine_desc {
    /* CoarseGrid  gaptooth.hpp:18-25 */
    double a, b, c, d;
    int32_t Nxi, Neta;
    int32_t periodic_xi;
    /* SchemeConfig subset  scheme_config.hpp:9-37 */
    int32_t nx, ny, nt, k;
    double tau;      /* gap-tooth horizon */
    double dt_macro; /* projective step  SchemeConfig::dt() = T/Nt */
    double h_xi, h_eta;
    int32_t bc_type;
    double robin_w1, robin_w2;
    int32_t quadrature;
    /* patch table in the reference's order (gaptooth.cpp:259-280): j outer,
     * i inner.  NULL = build it in that order. */
    int32_t npatches;
    const int32_t* patch_ij; /* [npatches][2] */
    /* solver-form coefficients, [ncoeff_sets][PD_NCOEF][nx+1][ny+1], node
     * (i,j) at i*(ny+1)+j (field.hpp:20-27); coeff_set[p] selects the set of
     * patch p (row sharing, gaptooth.cpp:254-266).  NULL coeff_set = identity. */
    int32_t ncoeff_sets;
    const int32_t* coeff_set;
    const double* coeffs;
    /* separable source g = spatial(xi,eta) * time(t) / l  (microsim.cpp:272-277) */
    int32_t source_kind;
    const double* source_spatial; /* [ncoeff_sets][nx+1][ny+1] or NULL */
    double l;
    int32_t mode;
    /* micro-solver: PD_SOLVER_EXPLICIT (microsim.cpp:292-332) or PD_SOLVER_ADI
     * (Peaceman-Rachford, microsim.cpp:334-507; EXACT family, or FAST for patches up to 32x32), with the
     * ADI upwind order/parameter (UpwindSpec, microsim.hpp) */
    int32_t solver;
    int32_t upwind_order;
    double upwind_r;
    /* On-device mesh/metric generation: when coeffs == NULL and
     * this points at a built-in problem (pd_problem_desc, PD_PROBLEM_*), the
     * engine computes the coefficient table (and a separable source's spatial
     * table) on the GPU instead of copying host tables, sampling each set at
     * the first patch that uses it.  Agrees with the host table to a few ulp
     * (the transcendental library differs).  NULL otherwise. */
    const struct pd_problem_desc* coeff_generator;
} pd_engine_desc;

typedef struct pd_engine pd_engine;

/* Run statistics of pd_run (cpi::RunResult subset, cpi.hpp:28-35). */
typedef struct pd_run_stats {
    int32_t steps_done;      /* macro steps completed without tripping the guard */
    int32_t failed_step;     /* 1-based step that tripped the guard, 0 if none */
    int32_t failed_nonfinite;/* 1 if the failure was a non-finite value */
    double umax_last;        /* max |U| after the last completed step */
    double blowup_threshold; /* 10 * max(max|U0|, 1e-12)  cpi.cpp:142-144 */
    double device_ms;        /* device time of the macro loop (CUDA events) */
    int64_t kernel_launches; /* kernels launched by this call */
} pd_run_stats;

int32_t pd_abi_version(void);
const char* pd_status_name(int32_t status);
/* Last error message of the engine, or the thread's last global error when
 * engine == NULL (create failures). */
const char* pd_last_error(const pd_engine* engine);

/* Host-only (no device needed): the bit-exact index tables an engine for
 * `desc` will use — patch list [P][2] (gaptooth.cpp:251-280 order unless
 * desc->patch_ij is given) and 3x3 neighbour table [P][9] of flat macro
 * indices i*(Neta+1)+j in build_stencil order (gaptooth.cpp:74-104).  Returns
 * PD_MACRO_PATCH_ERROR for a patch whose stencil leaves the interior. */
int32_t pd_patch_count(const pd_engine_desc* desc);
pd_status pd_build_index_tables(const pd_engine_desc* desc, int32_t* patch_ij, int32_t* neighbours);

pd_status pd_engine_create(const pd_engine_desc* desc, pd_engine** out);
void pd_engine_destroy(pd_engine* engine);
/* Kernel family actually used by the engine (FAST may fall back to EXACT for
 * shapes or features the fast kernel does not cover; never to a CPU path). */
int32_t pd_engine_mode(const pd_engine* engine);
/* 1 when the engine's EXACT gap-tooth step runs on the register-blocked tile kernel
 * (k_exact_tile / k_exact_big: explicit solver, zero or separable source,
 * 7x7/8x8/9x9/11x11/16x16/32x32 patches; same bits as the shared-memory EXACT kernel, which carries every other
 * case), 0 otherwise, -1 for NULL.  Replaces nothing in the reference: diagnostics. */
int32_t pd_engine_exact_tile(const pd_engine* engine);
/* 1 when the engine's coefficient table carries the mixed term (some |b| > 1e-12,
 * the 9-point operator; microsim.cpp:239), 0 for the 5-point operator, -1 for NULL. */
int32_t pd_engine_mixed(const pd_engine* engine);
/* Kernels the engine has launched since it was created (every entry point
 * counts its own launches; pd_run_stats.kernel_launches is the per-call share). */
int64_t pd_engine_launch_count(const pd_engine* engine);
/* Bit-exact index tables built by the engine: patch_ij [P][2] and the 3x3
 * neighbour table [P][9] of flat macro indices i*(Neta+1)+j, stencil order
 * vals[p+1][q+1] with p along xi (gaptooth.cpp:74-104).  Either may be NULL. */
pd_status pd_engine_tables(const pd_engine* engine, int32_t* patch_ij, int32_t* neighbours);
size_t pd_engine_device_bytes(const pd_engine* engine);
/* Optional: run the engine on an external cudaStream_t (NULL = own stream). */
pd_status pd_engine_set_stream(pd_engine* engine, void* cuda_stream);

/* Boundary refresh arrays ("perimeter"): [S: Nxi+1][N: Nxi+1][W: Neta+1][E: Neta+1]
 * applied in refresh_boundary's order (gaptooth.cpp:296-310): S/N rows, then
 * W/E columns (or the periodic seam copy U(Nxi,j) = U(0,j)). */
size_t pd_perimeter_len(int32_t Nxi, int32_t Neta);

/* One gap-tooth step t -> t+tau over all patches (step_direct).  U_out gets a
 * copy of U_in with every patch node replaced; then the boundary is refreshed
 * from bnd (perimeter at t+tau) or, when bnd == NULL, kept from U_in (periodic
 * seam applied).  src_time: [nt] values time(t+s*dt)/l for separable sources. */
pd_status pd_gaptooth_step(pd_engine* e, const double* U_in_host, double* U_out_host, double t,
                           const double* bnd_host, const double* src_time_host);
/* One projective forward-Euler step t -> t+dt_macro (k+1 substeps fused).
 * bnd: [k+2][perimeter] = refresh values at t+(m+1)tau (m=0..k) and t+dt, or NULL. */
pd_status pd_projective_step(pd_engine* e, const double* U_in_host, double* U_out_host, double t,
                             const double* bnd_host, const double* src_time_host);
pd_status pd_projective_step_device(pd_engine* e, const double* U_in_dev, double* U_out_dev,
                                    double t, const double* bnd_dev, const double* src_time_dev);
/* nsteps projective steps from t0, device resident, with the blow-up guard of
 * cpi.cpp:187-202.  U_host is in/out.  bnd: [nsteps][k+2][perimeter] or NULL
 * (frozen).  Returns PD_MACRO_INSTABILITY when the guard trips; U_host then
 * holds the field after the failing step, stats says which step. */
pd_status pd_run(pd_engine* e, double* U_host, int32_t nsteps, double t0, const double* bnd_host,
                 const double* src_time_host, pd_run_stats* stats);
pd_status pd_run_device(pd_engine* e, double* U_dev, double* U_scratch_dev, int32_t nsteps,
                        double t0, const double* bnd_dev, const double* src_time_dev,
                        pd_run_stats* stats);
/* pd_run / pd_run_device plus cpi::run's per-step exact-error metric on the
 * device (max_percent_error, cpi.cpp:79-94 called at cpi.cpp:204-209; replaces
 * the host loop a RunResult's step_max_pct_err needs): exact: [nsteps][NF] =
 * the exact solution sampled on every macro node at t0 + (n+1) dt_macro
 * (ProblemSpec::exact(xi(i), eta(j), t), i-major like Field2D; only the patch
 * nodes are read); err_out: [nsteps] = max over the patch nodes with
 * |exact| >= 1e-12 of |U - exact| / |exact| * 100, 0 when none — bit-identical
 * to the reference's loop.  Steps after a tripped guard are left at 0. */
pd_status pd_run_exact(pd_engine* e, double* U_host, int32_t nsteps, double t0, const double* bnd_host,
                       const double* src_time_host, const double* exact_host, double* err_out_host,
                       pd_run_stats* stats);
pd_status pd_run_device_exact(pd_engine* e, double* U_dev, double* U_scratch_dev, int32_t nsteps,
                              double t0, const double* bnd_dev, const double* src_time_dev,
                              const double* exact_dev, double* err_out_dev, pd_run_stats* stats);

/* Measurement hooks (no reference analogue; used by bench.py).
 * pd_device_count: CUDA devices visible (0 on a CPU-only host).
 * pd_bench_step_kernel: average device time (CUDA events on the engine's
 *   stream) of the dominant kernel alone — the fused gap-tooth kernel of one
 *   projective substep — over `reps` back-to-back launches in_dev -> out_dev.
 * pd_bench_fp64_peak: register-resident DFMA microbenchmark on the current
 *   device: sustained FP64 TFLOP/s (FMA = 2 flops) over ~ms_target ms. */
int32_t pd_device_count(void);
pd_status pd_bench_step_kernel(pd_engine* e, const double* in_dev, double* out_dev, int32_t reps,
                               double* ms_per_launch);
pd_status pd_bench_fp64_peak(double ms_target, double* tflops, double* sm_clock_ghz);

/* Unfused micro-solver, batched (explicit or ADI per desc->solver): PatchIntegrator::integrate for every patch
 * p (coefficient set coeff_set[p]) from u0 [P][n1][n2] over nt steps at t0.
 * edge_kind[4] (E,W,N,S), edge_value/edge_slope [P][4][max(n1,n2)],
 * robin_w[4][2].  Result in uT [P][n1][n2]. */
pd_status pd_integrate_batch(pd_engine* e, const double* u0_host, const int32_t* edge_kind,
                             const double* edge_value_host, const double* edge_slope_host,
                             const double* robin_w, double t0, const double* src_time_host,
                             double* uT_host);
/* Lifting for P stencils [P][3][3] (vals[p+1][q+1]) centred at (xi_c,eta_c)
 * [P][2]: u0 [P][n1][n2] plus the four edge profiles [P][4][max(n1,n2)] in
 * E,W,N,S order (slopes for Neumann, values for Dirichlet, both for Robin:
 * values then slopes).  dxi/deta are the macro spacings. */
pd_status pd_lift_batch(pd_engine* e, int32_t nstencils, const double* vals_host,
                        const double* centers_host, double* u0_host, double* edge_slope_host,
                        double* edge_value_host);
pd_status pd_restrict_batch(pd_engine* e, int32_t nfields, const double* u_host, double* avg_host);

/* Linear-response path.  With time-independent coefficients, a zero source
 * and one integrator per eta-row the reference's GapToothEngine::step (when
 * SchemeConfig::linear_cache enables it, gaptooth.cpp:213-224) replaces the
 * micro-solve by a 9-point macro stencil whose row weights are the patch
 * responses to the 9 unit stencils (build_row_weights, gaptooth.cpp:377-394;
 * step, :396-418).
 * pd_evolve_batch: evolve_patch (gaptooth.cpp:312-353) of n given stencils
 *   [n][3][3] (vals[p+1][q+1]) with the integrator and centre of patch
 *   patch_index[m]; out[m] = the restricted average.  EXACT arithmetic (bit-
 *   identical to the reference), whatever the engine's kernel family.
 * pd_linear_weights: row_w [Neta+1][3][3] (rows 0 and Neta zero) built like
 *   build_row_weights from row j's patch (i0, j), i0 = periodic ? 0 : 1.
 *   PD_VALIDATION_ERROR (the reference's message) when ineligible.
 * pd_engine_set_linear: upload row weights (NULL drops them).
 * pd_engine_set_step_kind: PD_STEP_DIRECT (micro-solve, the default) or
 *   PD_STEP_LINEAR; every step entry point (pd_gaptooth_step,
 *   pd_projective_step[_device], pd_run[_device], pd_bench_step_kernel) then
 *   uses that step.  The linear step accumulates in the reference's order and
 *   is bit-identical to GapToothEngine::step's fast path. */
enum { PD_STEP_DIRECT = 0, PD_STEP_LINEAR = 1 };
pd_status pd_evolve_batch(pd_engine* e, int32_t n, const int32_t* patch_index, const double* stencils_host,
                          double t, double* out_host);
pd_status pd_linear_weights(pd_engine* e, double* row_w_host);
pd_status pd_engine_set_linear(pd_engine* e, const double* row_w_host);
pd_status pd_engine_set_step_kind(pd_engine* e, int32_t kind);
int32_t pd_engine_step_kind(const pd_engine* e);

/* Time-dependent coefficients and general sources (microsim.cpp:537-542,
 * 278-280) on the device.  The reference re-samples its coefficient closures at
 * every micro step (t_co = t_substep + s*dt) and evaluates a general source per
 * node; closures cannot run on the GPU, so the caller samples them (as the
 * reference does, e.g. pd_problem_sample_steps) and the device does the solve:
 *   coeff_steps  [subs][nt][ncoeff_sets][PD_NCOEF][nx+1][ny+1] solver form, or NULL
 *                (the engine's static table),
 *   source_steps [subs][nt][ncoeff_sets][nx+1][ny+1] = general(node)/l, or NULL,
 * with subs = 1 (gap-tooth step) or k+1 (projective step: substep m starts at
 * t + m*tau).  bnd as pd_gaptooth_step ([perimeter]) / pd_projective_step
 * ([k+2][perimeter]).  Explicit micro-solver; runs the EXACT kernel family
 * (bit-identical to the reference).  Host buffers. */
pd_status pd_gaptooth_step_sampled(pd_engine* e, const double* U_in, double* U_out, double t, const double* bnd,
                                   const double* coeff_steps, const double* source_steps);
pd_status pd_projective_step_sampled(pd_engine* e, const double* U_in, double* U_out, double t, const double* bnd,
                                     const double* coeff_steps, const double* source_steps);

/* Segmented cpi::run (cpi.cpp:134-216 split around probes / snapshots /
 * progress callbacks): the blow-up threshold is 10 x max(scale0, 1e-12) with
 * scale0 = max|U| of the RUN's initial field after refresh_boundary
 * (cpi.cpp:142-144), not of each segment's input.  With scale0 > 0 every later
 * pd_run* call uses it (scale0 <= 0: measure the call's own input, the
 * default); step_offset = macro steps already done, so the instability message
 * names the run's step and time ("macro step n (t=...)", cpi.cpp:196-200).
 * pd_run_stats.failed_step stays relative to the call. */
pd_status pd_engine_set_run_guard(pd_engine* e, double scale0, int32_t step_offset);

/* ---------------------------------------------------------------------------
 * Decomposed run over xi-slabs with a fused peer-memory halo exchange
 * (DESIGN.md §6).  No reference analogue: the reference's serial
 * patch loop (gaptooth.cpp:362-372) is split into contiguous slabs of patch
 * columns, one engine (a patch subset) per rank/GPU.  Each rank's macro field
 * buffers hold its own columns, the two halo columns and the boundary.
 *
 * pd_projective_step_halo: pd_projective_step_device (k = 0) whose step kernel
 *   ALSO stores every result of a patch in column halo->column[l] into
 *   halo->dst[l] (the neighbour's output buffer of this step — a peer pointer
 *   over NVLink/NVSwitch, or a CUDA IPC mapping) at the same node index, then,
 *   after a system-scope fence, adds 1 to *halo->flag[l] (the neighbour's
 *   counter for this link) — one fused kernel, no separate exchange, no NCCL.
 *   U_out is NOT pre-filled from U_in (columns the rank does not own are only
 *   ever written by their owners); the boundary is refreshed as usual.
 * pd_stream_wait_flag: the engine's stream waits (a stream memory operation
 *   in the front end: no kernel spins, no host round trip) until
 *   (int32_t)(*flag_dev - value) >= 0.  A link's counter reaches
 *   (n+1)*(Neta-1) when the neighbour's step n has stored (and finished
 *   reading) that column, so waiting for n*(Neta-1) on both links before step
 *   n orders both the halo reads and the overwrite of the neighbour's buffer.
 * pd_ipc_alloc / pd_ipc_open / pd_ipc_close / pd_device_free: device buffers
 *   shareable across the processes of a one-process-per-GPU run
 *   (cudaIpcGetMemHandle, 64-byte handles; opened with lazy peer access). */
typedef struct pd_halo_out {
    int32_t nlinks;      /* 0, 1 or 2 */
    int32_t column[2];   /* macro column i (an edge column of this slab) */
    double* dst[2];      /* neighbour's field buffer receiving this step's output */
    uint32_t* flag[2];   /* neighbour's counter for this link */
} pd_halo_out;
pd_status pd_projective_step_halo(pd_engine* e, const double* U_in_dev, double* U_out_dev, double t,
                                  const double* bnd_dev, const double* src_time_dev, const pd_halo_out* halo);
/* k > 0: the projective step as its pieces, each with the same fused halo store
 * (the neighbours' counters then advance k+2 times per projective step):
 * substep m (0..k) of step_direct into U_out (refreshed from bnd = that substep's
 * [perimeter] row, or kept from U_in), and the extrapolation U_out = U_k +
 * (dt - k tau)(U_{k+1} - U_k)/tau on the engine's patch nodes (cpi.cpp:58-77),
 * refreshed from bnd (row k+1) or kept from U_in (the step's input). */
pd_status pd_gaptooth_substep_halo(pd_engine* e, const double* U_in_dev, double* U_out_dev, int32_t m,
                                   const double* bnd_dev, const double* src_time_dev, const pd_halo_out* halo);
pd_status pd_extrapolate_halo(pd_engine* e, const double* U_in_dev, const double* U_k_dev, const double* U_k1_dev,
                              double* U_out_dev, const double* bnd_dev, const pd_halo_out* halo);
pd_status pd_stream_wait_flag(pd_engine* e, const uint32_t* flag_dev, uint32_t value);
pd_status pd_ipc_alloc(size_t bytes, void** dev_ptr, unsigned char handle_out[64]);
pd_status pd_ipc_open(const unsigned char handle[64], void** dev_ptr);
pd_status pd_ipc_close(void* dev_ptr);
pd_status pd_device_free(void* dev_ptr);

/* ---------------------------------------------------------------------------
 * Host problem builder: the B200 framework's own mesh/metric setup for the
 * BASELINE configs and the reference benchmark problems.  It samples
 * transform_coefficients (geometry.cpp:93-125) at every micro node exactly as
 * PatchIntegrator::sample_coeffs does (microsim.cpp:226-263), on the host.
 * ------------------------------------------------------------------------- */
enum {
    PD_PROBLEM_DIFFUSION_SQUARE = 1, /* config 1: identity map, D=1, sin(pi x) sin(pi y) */
    PD_PROBLEM_CDR_TANH = 2,         /* config 2: tanh-stretched CDR, exact solution */
    PD_PROBLEM_ANNULUS_NONAXI = 3,   /* config 3: polar map, non-axisymmetric IC */
    PD_PROBLEM_SHEAR_CDR = 4,        /* configs 4/5: sinusoidal non-orthogonal map */
    PD_PROBLEM_REF_ANNULUS = 10,     /* problems::problem2_annulus  problems.cpp:110-138 */
    PD_PROBLEM_REF_CDR = 11,         /* problems::problem1_constant(lambda)  problems.cpp:19-73 */
    PD_PROBLEM_REF_CDR_VAR = 13,     /* problems::problem1_variable(lambda)  problems.cpp:19-75 */
    PD_PROBLEM_STEADY = 12,          /* harmonic u = x + y (test_gaptooth.cpp:32-49) */
    PD_PROBLEM_PULSED_CDR = 14       /* time-dependent coefficients + a general (non-separable)
                                        source: D(t) = eps (1 + sin(w t)/2), v(t) = vel (cos w t, 1/2),
                                        f = sin(pi x) cos(pi y + w t), w = omega; identity map, zero Dirichlet
                                        (exercises microsim.cpp:537-542 and 278-280) */
};
enum { PD_DT_GIVEN = 0, PD_DT_DIFFUSION = 1, PD_DT_METRIC = 2 };
enum { PD_COEFF_HOST = 0, PD_COEFF_DEVICE = 1 };

typedef struct pd_problem_desc {
    int32_t problem;
    double lambda;       /* REF_CDR stretching */
    double beta;         /* CDR_TANH stretching */
    double eps;          /* diffusivity */
    double omega;        /* reaction coefficient c */
    double vel;          /* constant velocity magnitude (CDR_TANH a = b) */
    double amp;          /* SHEAR map amplitude (0.1) */
    uint64_t seed;       /* SHEAR initial noise (mt19937_64) */
    int32_t jacobi_sweeps;
    /* SchemeConfig (scheme_config.hpp:9-37) */
    int32_t N_xi, N_eta, Nt, k;
    double T, tau, h_xi, h_eta;
    int32_t nx, ny, nt;
    int32_t bc_type;
    double robin_w1, robin_w2;
    int32_t quadrature;
    int32_t mode;
    /* pin rules; resolved by pd_problem_create */
    int32_t dt_rule;     /* PD_DT_*: GIVEN uses tau; DIFFUSION 0.2 d^2/D; METRIC 0.2 min d^2 / max(|A|+|C|) */
    double h_frac;       /* > 0: h = h_frac * macro spacing per direction */
    double dt_over_tau;  /* > 0: T = Nt * dt_over_tau * tau */
    int32_t threads;     /* host threads for coefficient sampling (0 = all) */
    int32_t solver;      /* PD_SOLVER_* */
    int32_t upwind_order;/* PD_UPWIND_* (ADI) */
    double upwind_r;     /* four-point upwind parameter r (ADI) */
    int32_t coeff_gen;   /* PD_COEFF_HOST: host tables (bit-identical to the reference's sampling);
                            PD_COEFF_DEVICE: no host tables, engines generate them on the GPU */
} pd_problem_desc;

typedef struct pd_problem pd_problem;

pd_status pd_problem_create(const pd_problem_desc* desc, pd_problem** out);
void pd_problem_destroy(pd_problem* p);
/* The resolved description (tau, T, h filled in by the pin rules). */
pd_status pd_problem_resolved(const pd_problem* p, pd_problem_desc* out);
/* Engine descriptor whose table pointers stay valid while p lives. */
pd_status pd_problem_engine_desc(const pd_problem* p, pd_engine_desc* out);
/* GapToothEngine::initial_field (gaptooth.cpp:284-294): (Nxi+1)(Neta+1). */
pd_status pd_problem_initial_field(const pd_problem* p, double* U_host);
/* refresh_boundary values at time t as a perimeter array. */
pd_status pd_problem_boundary(const pd_problem* p, double t, double* perimeter_host);
/* Boundary table for pd_run: [nsteps][k+2][perimeter] from t0. */
pd_status pd_problem_boundary_table(const pd_problem* p, double t0, int32_t nsteps, double* out_host);
/* Separable-source time factors time(t)/l (microsim.cpp:272-277) for pd_run:
 * [nsteps][k+1][nt], macro step n from t0 + n*dt, substep m from
 * t_n + m*tau (cpi.cpp:65), micro step s at t_m + s*dt_micro for the
 * explicit scheme and t_m + (s+1/2)*dt_micro for ADI (microsim.cpp:536-537).
 * PD_UNSUPPORTED when the source is zero. */
pd_status pd_problem_source_time(const pd_problem* p, double t0, int32_t nsteps, double* out_host);
/* Exact solution on the macro grid at t; PD_UNSUPPORTED if none. */
pd_status pd_problem_exact(const pd_problem* p, double t, double* U_host);
/* max |A|+|C| over all sampled nodes (the dt pin's denominator) and the
 * reference's single-direction stability number (microsim.cpp:253-262). */
pd_status pd_problem_stability(const pd_problem* p, double* max_a_plus_c, double* ref_number);
/* Time-dependent coefficients / general sources: the samples of one gap-tooth
 * substep starting at t0 that PatchIntegrator::integrate takes at every micro
 * step t0 + s*dt (sample_coeffs / sample_source, microsim.cpp:537-542,
 * 265-281) for every coefficient set, laid out for pd_*_step_sampled:
 * coeff_steps [nt][sets][PD_NCOEF][nx+1][ny+1], source_steps [nt][sets][nx+1][ny+1]
 * (= general(x, y, t)/l), either NULL.  Every coefficient sample passes the
 * explicit stability guard or PD_STABILITY_VIOLATION (microsim.cpp:253-262). */
pd_status pd_problem_sample_substep(const pd_problem* p, double t0, double* coeff_steps_host,
                                    double* source_steps_host);

/* The device generator on its own (desc->coeff_generator must be set): the
 * table into coeffs_host [ncoeff_sets][PD_NCOEF][n1][n2] and the source's
 * spatial table into source_spatial_host [ncoeff_sets][n1][n2] (either may be
 * NULL); stats[5] = max(|A|,|C|), max(|A|+|C|), max|B|, generator kernel ms
 * (CUDA events), micro nodes generated.  PD_NON_POSITIVE_JACOBIAN as
 * geometry.cpp:80-91 when J <= 1e-14 at some node. */
pd_status pd_coeffs_generate(const pd_engine_desc* desc, double* coeffs_host, double* source_spatial_host,
                             double* stats);

#ifdef __cplusplus
}
#endif
#endif /* PATCHDYN_B200_H */
