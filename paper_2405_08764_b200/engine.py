"""Python binding of the C-ABI (include/patchdyn_b200.h) for tests and bench.

The product path is ``lib/libpatchdyn_b200.so`` (sm_100a kernels + C++ host
problem builder).  There is no CPU fallback: if the library is missing, or the
device is absent, every call raises.  Names follow the reference's interfaces
(GapToothEngine::step_direct, cpi::projective_step, cpi::run,
PatchIntegrator::integrate) so parity tests read like the reference's own.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import abi
from .abi import EngineDesc, ProblemDesc, RunStats, perimeter_len

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpatchdyn_b200.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lib = None


class PatchdynError(RuntimeError):
    """Raised for a non-OK pd_status; .status and .kind mirror errors.hpp types."""

    def __init__(self, status: int, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.status = status
        self.kind = kind


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise FileNotFoundError(
            f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a). "
            "There is no CPU fallback for the hot path.")
    L = C.CDLL(str(LIB_PATH))
    vp = C.c_void_p
    L.pd_abi_version.restype = C.c_int32
    L.pd_status_name.restype = C.c_char_p
    L.pd_status_name.argtypes = [C.c_int32]
    L.pd_last_error.restype = C.c_char_p
    L.pd_last_error.argtypes = [vp]
    L.pd_patch_count.argtypes = [C.POINTER(EngineDesc)]
    L.pd_patch_count.restype = C.c_int32
    L.pd_build_index_tables.argtypes = [C.POINTER(EngineDesc), _ip, _ip]
    L.pd_build_index_tables.restype = C.c_int32
    L.pd_engine_create.argtypes = [C.POINTER(EngineDesc), C.POINTER(vp)]
    L.pd_engine_destroy.argtypes = [vp]
    L.pd_engine_mode.argtypes = [vp]
    L.pd_engine_mode.restype = C.c_int32
    L.pd_engine_exact_tile.argtypes = [vp]
    L.pd_engine_exact_tile.restype = C.c_int32
    L.pd_engine_tables.argtypes = [vp, _ip, _ip]
    L.pd_engine_device_bytes.argtypes = [vp]
    L.pd_engine_device_bytes.restype = C.c_size_t
    L.pd_engine_set_stream.argtypes = [vp, vp]
    L.pd_perimeter_len.argtypes = [C.c_int32, C.c_int32]
    L.pd_perimeter_len.restype = C.c_size_t
    L.pd_gaptooth_step.argtypes = [vp, _dp, _dp, C.c_double, _dp, _dp]
    L.pd_projective_step.argtypes = [vp, _dp, _dp, C.c_double, _dp, _dp]
    L.pd_projective_step_device.argtypes = [vp, vp, vp, C.c_double, vp, vp]
    L.pd_run.argtypes = [vp, _dp, C.c_int32, C.c_double, _dp, _dp, C.POINTER(RunStats)]
    L.pd_run_device.argtypes = [vp, vp, vp, C.c_int32, C.c_double, vp, vp, C.POINTER(RunStats)]
    L.pd_run_exact.argtypes = [vp, _dp, C.c_int32, C.c_double, _dp, _dp, _dp, _dp, C.POINTER(RunStats)]
    L.pd_run_device_exact.argtypes = [vp, vp, vp, C.c_int32, C.c_double, vp, vp, vp, vp, C.POINTER(RunStats)]
    L.pd_integrate_batch.argtypes = [vp, _dp, _ip, _dp, _dp, _dp, C.c_double, _dp, _dp]
    L.pd_lift_batch.argtypes = [vp, C.c_int32, _dp, _dp, _dp, _dp, _dp]
    L.pd_restrict_batch.argtypes = [vp, C.c_int32, _dp, _dp]
    L.pd_evolve_batch.argtypes = [vp, C.c_int32, _ip, _dp, C.c_double, _dp]
    L.pd_linear_weights.argtypes = [vp, _dp]
    L.pd_engine_set_linear.argtypes = [vp, _dp]
    L.pd_engine_set_step_kind.argtypes = [vp, C.c_int32]
    L.pd_engine_step_kind.argtypes = [vp]
    L.pd_engine_step_kind.restype = C.c_int32
    L.pd_engine_set_run_guard.argtypes = [vp, C.c_double, C.c_int32]
    L.pd_gaptooth_step_sampled.argtypes = [vp, _dp, _dp, C.c_double, _dp, _dp, _dp]
    L.pd_projective_step_sampled.argtypes = [vp, _dp, _dp, C.c_double, _dp, _dp, _dp]
    L.pd_problem_sample_substep.argtypes = [vp, C.c_double, _dp, _dp]
    L.pd_engine_mixed.argtypes = [vp]
    L.pd_engine_mixed.restype = C.c_int32
    L.pd_engine_launch_count.argtypes = [vp]
    L.pd_engine_launch_count.restype = C.c_int64
    L.pd_problem_create.argtypes = [C.POINTER(ProblemDesc), C.POINTER(vp)]
    L.pd_problem_destroy.argtypes = [vp]
    L.pd_problem_resolved.argtypes = [vp, C.POINTER(ProblemDesc)]
    L.pd_problem_engine_desc.argtypes = [vp, C.POINTER(EngineDesc)]
    L.pd_problem_initial_field.argtypes = [vp, _dp]
    L.pd_problem_boundary.argtypes = [vp, C.c_double, _dp]
    L.pd_problem_boundary_table.argtypes = [vp, C.c_double, C.c_int32, _dp]
    L.pd_problem_exact.argtypes = [vp, C.c_double, _dp]
    L.pd_problem_source_time.argtypes = [vp, C.c_double, C.c_int32, _dp]
    L.pd_problem_source_time.restype = C.c_int32
    L.pd_problem_stability.argtypes = [vp, _dp, _dp]
    L.pd_device_count.restype = C.c_int32
    L.pd_bench_step_kernel.argtypes = [vp, vp, vp, C.c_int32, _dp]
    L.pd_bench_fp64_peak.argtypes = [C.c_double, _dp, _dp]
    L.pd_coeffs_generate.argtypes = [C.POINTER(EngineDesc), _dp, _dp, _dp]
    L.pd_projective_step_halo.argtypes = [vp, vp, vp, C.c_double, vp, vp, C.POINTER(abi.HaloOut)]
    L.pd_stream_wait_flag.argtypes = [vp, vp, C.c_uint32]
    L.pd_gaptooth_substep_halo.argtypes = [vp, vp, vp, C.c_int32, vp, vp, C.POINTER(abi.HaloOut)]
    L.pd_extrapolate_halo.argtypes = [vp, vp, vp, vp, vp, vp, C.POINTER(abi.HaloOut)]
    L.pd_ipc_alloc.argtypes = [C.c_size_t, C.POINTER(vp), C.c_char_p]
    L.pd_ipc_open.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.pd_ipc_close.argtypes = [vp]
    L.pd_device_free.argtypes = [vp]
    for name in ["pd_projective_step_halo", "pd_gaptooth_substep_halo", "pd_extrapolate_halo", "pd_stream_wait_flag", "pd_ipc_alloc", "pd_ipc_open", "pd_ipc_close",
                 "pd_device_free"]:
        getattr(L, name).restype = C.c_int32
    for name in ["pd_bench_step_kernel", "pd_bench_fp64_peak", "pd_engine_create", "pd_engine_tables", "pd_engine_set_stream", "pd_gaptooth_step",
                 "pd_projective_step", "pd_projective_step_device", "pd_run", "pd_run_device",
                 "pd_integrate_batch", "pd_lift_batch", "pd_restrict_batch", "pd_evolve_batch",
                 "pd_linear_weights", "pd_engine_set_linear", "pd_engine_set_step_kind", "pd_engine_set_run_guard",
                 "pd_gaptooth_step_sampled", "pd_projective_step_sampled", "pd_problem_sample_substep",
                 "pd_problem_create",
                 "pd_problem_resolved", "pd_problem_engine_desc", "pd_problem_initial_field",
                 "pd_problem_boundary", "pd_problem_boundary_table", "pd_problem_exact",
                 "pd_problem_stability", "pd_coeffs_generate"]:
        getattr(L, name).restype = C.c_int32
    _lib = L
    return L


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def _check(status: int, handle=None):
    if status != abi.PD_OK:
        L = lib()
        kind = L.pd_status_name(status).decode()
        msg = L.pd_last_error(handle).decode()
        raise PatchdynError(status, kind, msg)


class Problem:
    """Host mesh/metric setup for a pd_problem_desc (C++ side of the ABI)."""

    def __init__(self, desc: ProblemDesc):
        L = lib()
        self.h = C.c_void_p()
        _check(L.pd_problem_create(C.byref(desc), C.byref(self.h)))
        self.desc = ProblemDesc()
        _check(L.pd_problem_resolved(self.h, C.byref(self.desc)))
        self.shape = (self.desc.N_xi + 1, self.desc.N_eta + 1)

    def __del__(self):
        if getattr(self, "h", None):
            lib().pd_problem_destroy(self.h)
            self.h = None

    def engine_desc(self) -> EngineDesc:
        d = EngineDesc()
        _check(lib().pd_problem_engine_desc(self.h, C.byref(d)))
        d._owner = self  # tables live in the problem
        return d

    def initial_field(self, refresh=True):
        """GapToothEngine::initial_field; refresh=True also applies
        refresh_boundary(U, 0) as cpi::run does (cpi.cpp:138-140)."""
        U = np.empty(self.shape)
        _check(lib().pd_problem_initial_field(self.h, _d(U)))
        if refresh:
            U = apply_perimeter(U, self.boundary(0.0), bool(self.engine_desc().periodic_xi))
        return U

    def boundary(self, t):
        b = np.empty(perimeter_len(*[s - 1 for s in self.shape]))
        _check(lib().pd_problem_boundary(self.h, t, _d(b)))
        return b

    def boundary_table(self, t0, nsteps):
        k = self.desc.k
        b = np.empty((nsteps, k + 2, perimeter_len(*[s - 1 for s in self.shape])))
        _check(lib().pd_problem_boundary_table(self.h, t0, nsteps, _d(b)))
        return b

    def source_time(self, t0, nsteps):
        """[nsteps][k+1][nt] separable-source factors time(t)/l, or None (zero source)."""
        k, nt = self.desc.k, self.desc.nt
        out = np.empty((nsteps, k + 1, nt))
        st = lib().pd_problem_source_time(self.h, t0, nsteps, _d(out))
        if st == abi.PD_UNSUPPORTED:
            return None
        _check(st)
        return out

    def exact(self, t):
        U = np.empty(self.shape)
        st = lib().pd_problem_exact(self.h, t, _d(U))
        if st == abi.PD_UNSUPPORTED:
            return None
        _check(st)
        return U

    def sample_substep(self, t0, coeffs=True, source=True):
        """Per-micro-step samples of one substep from t0 (time-dependent
        coefficients / general sources, microsim.cpp:537-542, 265-281):
        (coeff_steps [nt][sets][6][n1][n2] or None, source_steps [nt][sets][n1][n2] or None)."""
        ed = self.engine_desc()
        nt, S, n1, n2 = ed.nt, ed.ncoeff_sets, ed.nx + 1, ed.ny + 1
        c = np.empty((nt, S, abi.PD_NCOEF, n1, n2)) if coeffs else None
        g = np.empty((nt, S, n1, n2)) if source else None
        _check(lib().pd_problem_sample_substep(self.h, t0, _d(c), _d(g)))
        return c, g

    def sample_projective(self, t):
        """[k+1] substeps (substep m from t + m tau) stacked for pd_projective_step_sampled."""
        k, tau = self.desc.k, self.desc.tau
        ed = self.engine_desc()
        gen = ed.source_kind == abi.PD_SOURCE_GENERAL
        parts = [self.sample_substep(t + m * tau, coeffs=True, source=gen) for m in range(k + 1)]
        c = np.concatenate([p[0] for p in parts])
        g = np.concatenate([p[1] for p in parts]) if gen else None
        return c, g

    def stability(self):
        a, r = C.c_double(), C.c_double()
        _check(lib().pd_problem_stability(self.h, C.byref(a), C.byref(r)))
        return a.value, r.value


def device_count() -> int:
    return lib().pd_device_count()


def fp64_peak(ms_target: float = 200.0):
    """Measured FP64 DFMA throughput (TFLOP/s) and the SM clock it ran at (GHz)."""
    tf, ghz = C.c_double(), C.c_double()
    _check(lib().pd_bench_fp64_peak(ms_target, C.byref(tf), C.byref(ghz)))
    return tf.value, ghz.value


def generate_coeffs(desc: EngineDesc, tables: bool = True):
    """On-device mesh/metric generation (pd_coeffs_generate; desc.coeff_generator
    set, e.g. the engine_desc of a Problem created with coeff_gen=PD_COEFF_DEVICE).
    Returns (coeffs [sets][6][n1][n2] or None, source spatial [sets][n1][n2] or
    None, stats dict)."""
    n1, n2, S = desc.nx + 1, desc.ny + 1, desc.ncoeff_sets
    co = np.empty((S, abi.PD_NCOEF, n1, n2)) if tables else None
    sp = np.empty((S, n1, n2)) if tables and desc.source_kind == abi.PD_SOURCE_SEPARABLE else None
    st = np.empty(5)
    _check(lib().pd_coeffs_generate(C.byref(desc), _d(co), _d(sp), _d(st)))
    return co, sp, {"max_abs_ac": st[0], "max_a_plus_c": st[1], "max_abs_b": st[2], "device_ms": st[3],
                    "nodes": int(st[4])}


def index_tables(desc: EngineDesc):
    """Host-only bit-exact patch list and neighbour table (pd_build_index_tables)."""
    L = lib()
    P = L.pd_patch_count(C.byref(desc))
    pij = np.empty((P, 2), dtype=np.int32)
    nbr = np.empty((P, 9), dtype=np.int32)
    _check(L.pd_build_index_tables(C.byref(desc), _i(pij), _i(nbr)))
    return pij, nbr


def apply_perimeter(U, perim, periodic):
    """refresh_boundary from a perimeter array (gaptooth.cpp:296-310), host side."""
    U = np.array(U, copy=True)
    N1, N2 = U.shape[0] - 1, U.shape[1] - 1
    S, N = perim[: N1 + 1], perim[N1 + 1: 2 * (N1 + 1)]
    W, E = perim[2 * (N1 + 1): 2 * (N1 + 1) + N2 + 1], perim[2 * (N1 + 1) + N2 + 1:]
    U[:, 0] = S
    U[:, N2] = N
    if periodic:
        U[N1, :] = U[0, :]
    else:
        U[0, :] = W
        U[N1, :] = E
    return U


class Engine:
    """pd_engine: device tables + fused kernels for one problem/scheme."""

    def __init__(self, desc: EngineDesc, mode: int | None = None):
        L = lib()
        if mode is not None:
            desc.mode = mode
        self.desc = desc
        self.h = C.c_void_p()
        _check(L.pd_engine_create(C.byref(desc), C.byref(self.h)))
        self.shape = (desc.Nxi + 1, desc.Neta + 1)
        self.P = desc.npatches if desc.patch_ij else ((desc.Nxi - (0 if desc.periodic_xi else 1)) * (desc.Neta - 1))
        self.n1, self.n2 = desc.nx + 1, desc.ny + 1
        self.L = max(self.n1, self.n2)
        self.perim = perimeter_len(desc.Nxi, desc.Neta)

    @classmethod
    def from_problem(cls, problem: Problem, mode: int | None = None) -> "Engine":
        e = cls(problem.engine_desc(), mode)
        e.problem = problem
        return e

    def __del__(self):
        if getattr(self, "h", None):
            lib().pd_engine_destroy(self.h)
            self.h = None

    @property
    def mode(self) -> int:
        return lib().pd_engine_mode(self.h)

    @property
    def exact_tile(self) -> bool:
        """EXACT steps of this engine run on the register-blocked tile kernel (k_exact_tile)."""
        return lib().pd_engine_exact_tile(self.h) == 1

    @property
    def device_bytes(self) -> int:
        return lib().pd_engine_device_bytes(self.h)

    def tables(self):
        pij = np.empty((self.P, 2), dtype=np.int32)
        nbr = np.empty((self.P, 9), dtype=np.int32)
        _check(lib().pd_engine_tables(self.h, _i(pij), _i(nbr)), self.h)
        return pij, nbr

    def step_direct(self, U, t, bnd=None, src_time=None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        b = None if bnd is None else np.ascontiguousarray(bnd, dtype=np.float64)
        s = None if src_time is None else np.ascontiguousarray(src_time, dtype=np.float64)
        _check(lib().pd_gaptooth_step(self.h, _d(U), _d(out), t, _d(b), _d(s)), self.h)
        return out

    def projective_step(self, U, t, bnd=None, src_time=None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        b = None if bnd is None else np.ascontiguousarray(bnd, dtype=np.float64)
        s = None if src_time is None else np.ascontiguousarray(src_time, dtype=np.float64)
        _check(lib().pd_projective_step(self.h, _d(U), _d(out), t, _d(b), _d(s)), self.h)
        return out

    def run(self, U0, nsteps, t0=0.0, bnd=None, src_time=None, raise_on_instability=True):
        U = np.array(U0, dtype=np.float64, copy=True, order="C")
        b = None if bnd is None else np.ascontiguousarray(bnd, dtype=np.float64)
        s = None if src_time is None else np.ascontiguousarray(src_time, dtype=np.float64)
        stats = RunStats()
        st = lib().pd_run(self.h, _d(U), nsteps, t0, _d(b), _d(s), C.byref(stats))
        if st != abi.PD_MACRO_INSTABILITY or raise_on_instability:
            _check(st, self.h)
        return U, stats

    @property
    def mixed(self) -> bool:
        """True when the table carries the mixed term (9-point operator)."""
        return lib().pd_engine_mixed(self.h) == 1

    @property
    def launch_count(self) -> int:
        return int(lib().pd_engine_launch_count(self.h))

    def step_sampled(self, U, t, coeff_steps=None, source_steps=None, bnd=None):
        """step_direct with per-micro-step sampled tables (pd_gaptooth_step_sampled)."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        c = None if coeff_steps is None else np.ascontiguousarray(coeff_steps, dtype=np.float64)
        g = None if source_steps is None else np.ascontiguousarray(source_steps, dtype=np.float64)
        b = None if bnd is None else np.ascontiguousarray(bnd, dtype=np.float64)
        _check(lib().pd_gaptooth_step_sampled(self.h, _d(U), _d(out), t, _d(b), _d(c), _d(g)), self.h)
        return out

    def projective_step_sampled(self, U, t, coeff_steps=None, source_steps=None, bnd=None):
        """cpi::projective_step with per-micro-step sampled tables ([k+1][nt]...)."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        c = None if coeff_steps is None else np.ascontiguousarray(coeff_steps, dtype=np.float64)
        g = None if source_steps is None else np.ascontiguousarray(source_steps, dtype=np.float64)
        b = None if bnd is None else np.ascontiguousarray(bnd, dtype=np.float64)
        _check(lib().pd_projective_step_sampled(self.h, _d(U), _d(out), t, _d(b), _d(c), _d(g)), self.h)
        return out

    def set_run_guard(self, scale0: float = 0.0, step_offset: int = 0):
        """Segmented cpi::run: later runs use 10 x max(scale0, 1e-12) as the
        blow-up threshold and number steps from step_offset (scale0 <= 0:
        measure each call's input, the default)."""
        _check(lib().pd_engine_set_run_guard(self.h, float(scale0), int(step_offset)), self.h)

    def run_exact(self, U0, nsteps, exact, t0=0.0, bnd=None, src_time=None, raise_on_instability=True):
        """run() plus cpi::run's per-step exact-error metric on the device
        (max_percent_error, cpi.cpp:79-94): exact [nsteps][Nxi+1][Neta+1] at the
        end of every step; returns (U, stats, err[nsteps])."""
        U = np.array(U0, dtype=np.float64, copy=True, order="C")
        b = None if bnd is None else np.ascontiguousarray(bnd, dtype=np.float64)
        s = None if src_time is None else np.ascontiguousarray(src_time, dtype=np.float64)
        ex = np.ascontiguousarray(exact, dtype=np.float64)
        if ex.shape != (nsteps,) + U.shape:
            raise ValueError(f"exact table shape {ex.shape} != {(nsteps,) + U.shape}")
        err = np.zeros(nsteps)
        stats = RunStats()
        st = lib().pd_run_exact(self.h, _d(U), nsteps, t0, _d(b), _d(s), _d(ex), _d(err), C.byref(stats))
        if st != abi.PD_MACRO_INSTABILITY or raise_on_instability:
            _check(st, self.h)
        return U, stats, err

    # ---- device-resident entries (pointers are raw device addresses) ----
    def projective_step_device(self, in_ptr: int, out_ptr: int, t: float = 0.0):
        _check(lib().pd_projective_step_device(self.h, in_ptr, out_ptr, t, None, None), self.h)

    def run_device(self, u_ptr: int, scratch_ptr: int, nsteps: int, t0: float = 0.0, raise_on_instability=True):
        stats = RunStats()
        st = lib().pd_run_device(self.h, u_ptr, scratch_ptr, nsteps, t0, None, None, C.byref(stats))
        if st != abi.PD_MACRO_INSTABILITY or raise_on_instability:
            _check(st, self.h)
        return stats

    def bench_step_kernel(self, in_ptr: int, out_ptr: int, reps: int = 5) -> float:
        ms = C.c_double()
        _check(lib().pd_bench_step_kernel(self.h, in_ptr, out_ptr, reps, C.byref(ms)), self.h)
        return ms.value

    def integrate(self, u0, kinds, values=None, slopes=None, robin_w=None, t0=0.0, src_time=None):
        u0 = np.ascontiguousarray(u0, dtype=np.float64).reshape(self.P, self.n1, self.n2)
        kinds = np.ascontiguousarray(kinds, dtype=np.int32)
        v = None if values is None else np.ascontiguousarray(values, dtype=np.float64).reshape(self.P, 4, self.L)
        s = None if slopes is None else np.ascontiguousarray(slopes, dtype=np.float64).reshape(self.P, 4, self.L)
        rw = None if robin_w is None else np.ascontiguousarray(robin_w, dtype=np.float64).reshape(8)
        st_ = None if src_time is None else np.ascontiguousarray(src_time, dtype=np.float64)
        uT = np.empty_like(u0)
        _check(lib().pd_integrate_batch(self.h, _d(u0), _i(kinds), _d(v), _d(s), _d(rw), t0, _d(st_), _d(uT)),
               self.h)
        return uT

    def lift(self, vals, centers):
        vals = np.ascontiguousarray(vals, dtype=np.float64).reshape(-1, 9)
        centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 2)
        n = len(vals)
        u0 = np.empty((n, self.n1, self.n2))
        sl = np.empty((n, 4, self.L))
        va = np.empty((n, 4, self.L))
        _check(lib().pd_lift_batch(self.h, n, _d(vals), _d(centers), _d(u0), _d(sl), _d(va)), self.h)
        return u0, sl, va

    def restrict(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1, self.n1, self.n2)
        avg = np.empty(len(u))
        _check(lib().pd_restrict_batch(self.h, len(u), _d(u), _d(avg)), self.h)
        return avg

    # ---- linear-response path (GapToothEngine::step with linear_cache) ----
    def evolve(self, patch_index, stencils, t=0.0):
        """evolve_patch (gaptooth.cpp:312-353) of given stencils [n][3][3] with
        the integrators/centres of patches patch_index[n] (EXACT arithmetic)."""
        idx = np.ascontiguousarray(patch_index, dtype=np.int32).reshape(-1)
        st = np.ascontiguousarray(stencils, dtype=np.float64).reshape(len(idx), 9)
        out = np.empty(len(idx))
        _check(lib().pd_evolve_batch(self.h, len(idx), _i(idx), _d(st), t, _d(out)), self.h)
        return out

    def linear_weights(self):
        """build_row_weights (gaptooth.cpp:377-394): [Neta+1][3][3]."""
        w = np.zeros((self.shape[1], 3, 3))
        _check(lib().pd_linear_weights(self.h, _d(w)), self.h)
        return w

    def set_linear(self, row_w=None):
        """Upload row weights (built here when None) and make every step the
        linear-response step; set_direct() switches back."""
        w = self.linear_weights() if row_w is None else np.ascontiguousarray(row_w, dtype=np.float64)
        _check(lib().pd_engine_set_linear(self.h, _d(w)), self.h)
        _check(lib().pd_engine_set_step_kind(self.h, abi.PD_STEP_LINEAR), self.h)
        return w

    def set_direct(self):
        _check(lib().pd_engine_set_step_kind(self.h, abi.PD_STEP_DIRECT), self.h)

    @property
    def step_kind(self) -> int:
        return lib().pd_engine_step_kind(self.h)
