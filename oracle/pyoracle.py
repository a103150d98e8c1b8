"""ORACLE / TEST INFRASTRUCTURE ONLY.

Python bindings for the two CPU checkers:

* ``Restated`` — oracle/build/libpd_oracle.so, the C restatement of the
  reference's explicit path (+ mixed term), built from oracle/pd_oracle.c.
* ``Reference`` — oracle/_ref/libpatchdyn_ref.so, the UNMODIFIED reference
  sources (compiled from /root/reference by oracle/Makefile) behind a C shim.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2405_08764_b200.abi import EngineDesc, ProblemDesc, RunStats, perimeter_len

HERE = Path(__file__).resolve().parent
RESTATED_SO = HERE / "build" / "libpd_oracle.so"
REF_SO = HERE / "_ref" / "libpatchdyn_ref.so"

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def build_restated() -> Path:
    """Compile the C restatement if it is missing (gcc is on every box)."""
    if not RESTATED_SO.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "restated"], check=True)
    return RESTATED_SO


class Restated:
    def __init__(self, threads: int | None = None):
        self.lib = C.CDLL(str(build_restated()))
        L = self.lib
        L.pdo_set_threads.argtypes = [C.c_int]
        L.pdo_get_threads.restype = C.c_int
        L.pdo_last_error.restype = C.c_char_p
        L.pdo_lift.argtypes = [_dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                               C.c_double, C.c_int, C.c_int, _dp, _dp, _dp]
        L.pdo_restrict.argtypes = [_dp, C.c_int, C.c_int, C.c_int]
        L.pdo_restrict.restype = C.c_double
        L.pdo_integrate.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                    _ip, _dp, _dp, _dp, _dp, _dp, _dp]
        desc_p = C.POINTER(EngineDesc)
        L.pdo_gaptooth_step.argtypes = [desc_p, _dp, _dp, C.c_double, _dp, _dp]
        L.pdo_projective_step.argtypes = [desc_p, _dp, _dp, C.c_double, _dp, _dp]
        L.pdo_run.argtypes = [desc_p, _dp, C.c_int, C.c_double, _dp, _dp, C.POINTER(RunStats)]
        L.pdo_patch_subset.argtypes = [desc_p, _dp, C.c_double, C.c_int, _ip, _dp]
        L.pdo_patch_subset.restype = C.c_double
        L.pdo_evolve_batch.argtypes = [desc_p, C.c_int, _ip, _dp, C.c_double, _dp]
        L.pdo_linear_weights.argtypes = [desc_p, _dp]
        L.pdo_linear_step.argtypes = [desc_p, _dp, _dp, _dp, _dp]
        L.pdo_linear_projective_step.argtypes = [desc_p, _dp, _dp, _dp, C.c_double, _dp]
        L.pdo_linear_run.argtypes = [desc_p, _dp, _dp, C.c_int, C.c_double, _dp, C.POINTER(RunStats)]
        L.pdo_shear_problem.argtypes = [C.POINTER(ProblemDesc), _dp, _ip, _dp]
        L.pdo_seeded_field.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _dp]
        if threads is not None:
            L.pdo_set_threads(int(threads))

    @property
    def threads(self) -> int:
        return self.lib.pdo_get_threads()

    def set_threads(self, n: int):
        self.lib.pdo_set_threads(int(n))

    def lift(self, vals, xi_c, eta_c, dxi, deta, h_xi, h_eta, nx, ny):
        L = max(nx, ny) + 1
        vals = np.ascontiguousarray(vals, dtype=np.float64).reshape(9)
        u0 = np.zeros((nx + 1, ny + 1))
        sl = np.zeros((4, L))
        va = np.zeros((4, L))
        self.lib.pdo_lift(_d(vals), xi_c, eta_c, dxi, deta, h_xi, h_eta, nx, ny, _d(u0), _d(sl), _d(va))
        return u0, sl, va

    def restrict(self, u, quadrature=0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        return self.lib.pdo_restrict(_d(u), u.shape[0], u.shape[1], quadrature)

    def integrate(self, coef, nx, ny, nt, h_xi, h_eta, tau, kinds, values, slopes, robin_w, u0,
                  src_spatial=None, src_time=None):
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        u = np.array(u0, dtype=np.float64, copy=True, order="C")
        kinds = np.ascontiguousarray(kinds, dtype=np.int32)
        values = np.ascontiguousarray(values, dtype=np.float64)
        slopes = np.ascontiguousarray(slopes, dtype=np.float64)
        robin_w = np.ascontiguousarray(robin_w, dtype=np.float64)
        sp = None if src_spatial is None else np.ascontiguousarray(src_spatial, dtype=np.float64)
        st = None if src_time is None else np.ascontiguousarray(src_time, dtype=np.float64)
        r = self.lib.pdo_integrate(_d(coef), nx, ny, nt, h_xi, h_eta, tau, _i(kinds), _d(values),
                                   _d(slopes), _d(robin_w), _d(sp), _d(st), _d(u))
        return r, u

    def gaptooth_step(self, desc: EngineDesc, U, t, bnd=None, src_time=None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        r = self.lib.pdo_gaptooth_step(C.byref(desc), _d(U), _d(out), t, _d(bnd), _d(src_time))
        return r, out

    def projective_step(self, desc: EngineDesc, U, t, bnd=None, src_time=None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        r = self.lib.pdo_projective_step(C.byref(desc), _d(U), _d(out), t, _d(bnd), _d(src_time))
        return r, out

    def run(self, desc: EngineDesc, U0, nsteps, t0=0.0, bnd=None, src_time=None):
        U = np.array(U0, dtype=np.float64, copy=True, order="C")
        stats = RunStats()
        r = self.lib.pdo_run(C.byref(desc), _d(U), nsteps, t0, _d(bnd), _d(src_time), C.byref(stats))
        return r, U, stats

    # linear-response path  gaptooth.cpp:377-418
    def evolve_batch(self, desc: EngineDesc, patch_index, stencils, t=0.0):
        idx = np.ascontiguousarray(patch_index, dtype=np.int32)
        st = np.ascontiguousarray(stencils, dtype=np.float64).reshape(len(idx), 9)
        out = np.empty(len(idx))
        r = self.lib.pdo_evolve_batch(C.byref(desc), len(idx), _i(idx), _d(st), t, _d(out))
        return r, out

    def linear_weights(self, desc: EngineDesc):
        w = np.zeros((desc.Neta + 1, 3, 3))
        r = self.lib.pdo_linear_weights(C.byref(desc), _d(w))
        return r, w

    def linear_step(self, desc: EngineDesc, row_w, U, bnd=None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        w = np.ascontiguousarray(row_w, dtype=np.float64)
        out = np.empty_like(U)
        r = self.lib.pdo_linear_step(C.byref(desc), _d(w), _d(U), _d(out), _d(bnd))
        return r, out

    def linear_projective_step(self, desc: EngineDesc, row_w, U, t, bnd=None):
        U = np.ascontiguousarray(U, dtype=np.float64)
        w = np.ascontiguousarray(row_w, dtype=np.float64)
        out = np.empty_like(U)
        r = self.lib.pdo_linear_projective_step(C.byref(desc), _d(w), _d(U), _d(out), t, _d(bnd))
        return r, out

    def linear_run(self, desc: EngineDesc, row_w, U0, nsteps, t0=0.0, bnd=None):
        U = np.array(U0, dtype=np.float64, copy=True, order="C")
        w = np.ascontiguousarray(row_w, dtype=np.float64)
        stats = RunStats()
        r = self.lib.pdo_linear_run(C.byref(desc), _d(w), _d(U), nsteps, t0, _d(bnd), C.byref(stats))
        return r, U, stats

    def shear_problem(self, pdesc: ProblemDesc, mode: int = 1):
        """Configs 4/5 built by the oracle alone (pd_oracle_problem.c): the
        resolved problem description, an engine descriptor over oracle-owned
        tables and the seeded initial field — no product library involved."""
        r = ProblemDesc.from_buffer_copy(pdesc)
        n1, n2 = r.nx + 1, r.ny + 1
        P = (r.N_xi - 1) * (r.N_eta - 1)
        U0 = np.empty((r.N_xi + 1, r.N_eta + 1))
        pij = np.empty((P, 2), dtype=np.int32)
        coeffs = np.empty((P, 6, n1, n2))
        st = self.lib.pdo_shear_problem(C.byref(r), _d(U0), _i(pij), _d(coeffs))
        if st:
            raise RuntimeError(f"oracle shear problem: status {st}")
        ed = engine_desc_from_tables(r, False, (0.0, 1.0, 0.0, 1.0), pij, coeffs, mode=mode)
        return r, ed, U0

    def patch_subset(self, desc: EngineDesc, U, t, patch_index):
        U = np.ascontiguousarray(U, dtype=np.float64)
        idx = np.ascontiguousarray(patch_index, dtype=np.int32)
        out = np.empty(len(idx))
        sec = self.lib.pdo_patch_subset(C.byref(desc), _d(U), t, len(idx), _i(idx), _d(out))
        if sec < 0:
            raise RuntimeError("oracle patch subset failed")
        return out, sec


def reference_available() -> bool:
    return REF_SO.exists()


class Reference:
    """The unmodified reference, via oracle/_ref/libpatchdyn_ref.so."""

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref, needs /root/reference)")
        self.lib = C.CDLL(str(REF_SO))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        pd = C.POINTER(ProblemDesc)
        vp = C.c_void_p
        L.ref_engine_create.argtypes = [pd, C.POINTER(vp)]
        L.ref_engine_create_lc.argtypes = [pd, C.c_int, C.POINTER(vp)]
        L.ref_step.argtypes = [vp, _dp, _dp, C.c_double]
        L.ref_engine_destroy.argtypes = [vp]
        L.ref_initial_field.argtypes = [vp, _dp]
        L.ref_refresh_boundary.argtypes = [vp, _dp, C.c_double]
        L.ref_step_direct.argtypes = [vp, _dp, _dp, C.c_double]
        L.ref_projective_step.argtypes = [vp, _dp, _dp, C.c_double]
        L.ref_run.argtypes = [vp, _dp, _dp, _dp]
        L.ref_steps.argtypes = [vp, _dp, C.c_int, C.c_int, _dp]
        L.ref_sample_coeffs.argtypes = [vp, C.c_int, _ip, _dp]
        L.ref_neighbours.argtypes = [vp, C.c_int, _ip, _ip]
        L.ref_sample_coeffs_desc.argtypes = [pd, C.c_int, _ip, _dp]
        L.ref_integrate.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.c_double, _ip, _dp, _dp, _dp, C.c_double,
                                    _dp, _dp]
        L.ref_lift.argtypes = [_dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                               C.c_double, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_restrict.argtypes = [_dp, C.c_int, C.c_int, C.c_int]
        L.ref_restrict.restype = C.c_double
        L.ref_problem_domain.argtypes = [pd, _dp, _ip]

    def error(self) -> str:
        return self.lib.ref_last_error().decode()

    def sample_coeffs(self, pdesc: ProblemDesc, patch_ij):
        """Reference transform_coefficients at PatchIntegrator node coordinates
        without constructing a GapToothEngine (works for b != 0)."""
        pij = np.ascontiguousarray(patch_ij, dtype=np.int32).reshape(-1, 2)
        out = np.empty((len(pij), 6, pdesc.nx + 1, pdesc.ny + 1))
        r = self.lib.ref_sample_coeffs_desc(C.byref(pdesc), len(pij), _i(pij), _d(out))
        if r:
            raise RuntimeError(f"reference sample_coeffs_desc: {r}: {self.error()}")
        return out

    def engine(self, pdesc: ProblemDesc, linear_cache: str = "off") -> "RefEngine":
        """linear_cache: 'off' (the BASELINE pin, B3), 'auto' (the reference's default) or 'on'."""
        return RefEngine(self, pdesc, linear_cache)

    def integrate(self, coef5, nx, ny, nt, h_xi, h_eta, tau, xi_c, eta_c, kinds, values, slopes,
                  robin_w, u0, t0=0.0, coef_table=None):
        c5 = None if coef5 is None else np.ascontiguousarray(coef5, dtype=np.float64)
        tab = None if coef_table is None else np.ascontiguousarray(coef_table, dtype=np.float64)
        kinds = np.ascontiguousarray(kinds, dtype=np.int32)
        values = np.ascontiguousarray(values, dtype=np.float64)
        slopes = np.ascontiguousarray(slopes, dtype=np.float64)
        robin_w = np.ascontiguousarray(robin_w, dtype=np.float64)
        u0 = np.ascontiguousarray(u0, dtype=np.float64)
        uT = np.empty_like(u0)
        r = self.lib.ref_integrate(_d(c5), _d(tab), nx, ny, nt, h_xi, h_eta, tau, xi_c, eta_c, _i(kinds),
                                   _d(values), _d(slopes), _d(robin_w), t0, _d(u0), _d(uT))
        return r, uT

    def lift(self, vals, xi_c, eta_c, dxi, deta, h_xi, h_eta, nx, ny):
        L = max(nx, ny) + 1
        vals = np.ascontiguousarray(vals, dtype=np.float64).reshape(9)
        u0 = np.zeros((nx + 1, ny + 1))
        sl = np.zeros((4, L))
        va = np.zeros((4, L))
        r = self.lib.ref_lift(_d(vals), xi_c, eta_c, dxi, deta, h_xi, h_eta, nx, ny, _d(u0), _d(sl), _d(va))
        return r, u0, sl, va

    def restrict(self, u, simpson=False):
        u = np.ascontiguousarray(u, dtype=np.float64)
        return self.lib.ref_restrict(_d(u), u.shape[0], u.shape[1], int(simpson))


class RefEngine:
    LINEAR_CACHE = {"auto": 0, "on": 1, "off": 2}

    def __init__(self, ref: Reference, pdesc: ProblemDesc, linear_cache: str = "off"):
        self.ref = ref
        self.L = ref.lib
        self.h = C.c_void_p()
        self.pdesc = pdesc
        r = self.L.ref_engine_create_lc(C.byref(pdesc), self.LINEAR_CACHE[linear_cache], C.byref(self.h))
        if r != 0:
            raise RuntimeError(f"reference engine: status {r}: {ref.error()}")
        self.shape = (pdesc.N_xi + 1, pdesc.N_eta + 1)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_engine_destroy(self.h)
            self.h = None

    def initial_field(self):
        U = np.empty(self.shape)
        self.L.ref_initial_field(self.h, _d(U))
        return U

    def refresh_boundary(self, U, t):
        U = np.array(U, dtype=np.float64, copy=True, order="C")
        self.L.ref_refresh_boundary(self.h, _d(U), t)
        return U

    def step_direct(self, U, t):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        r = self.L.ref_step_direct(self.h, _d(U), _d(out), t)
        if r:
            raise RuntimeError(f"reference step_direct: {r}: {self.ref.error()}")
        return out

    def step(self, U, t):
        """GapToothEngine::step: the linear-response path when the engine enabled it."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        r = self.L.ref_step(self.h, _d(U), _d(out), t)
        if r:
            raise RuntimeError(f"reference step: {r}: {self.ref.error()}")
        return out

    def projective_step(self, U, t):
        U = np.ascontiguousarray(U, dtype=np.float64)
        out = np.empty_like(U)
        r = self.L.ref_projective_step(self.h, _d(U), _d(out), t)
        if r:
            raise RuntimeError(f"reference projective_step: {r}: {self.ref.error()}")
        return out

    def run(self):
        U = np.empty(self.shape)
        err = C.c_double()
        sec = C.c_double()
        r = self.L.ref_run(self.h, _d(U), C.byref(err), C.byref(sec))
        return r, U, err.value, sec.value

    def steps(self, U, n0, nsteps):
        U = np.array(U, dtype=np.float64, copy=True, order="C")
        sec = C.c_double()
        r = self.L.ref_steps(self.h, _d(U), n0, nsteps, C.byref(sec))
        if r:
            raise RuntimeError(f"reference steps: {r}: {self.ref.error()}")
        return U, sec.value

    def sample_coeffs(self, patch_ij):
        pij = np.ascontiguousarray(patch_ij, dtype=np.int32).reshape(-1, 2)
        n1, n2 = self.pdesc.nx + 1, self.pdesc.ny + 1
        out = np.empty((len(pij), 6, n1, n2))
        r = self.L.ref_sample_coeffs(self.h, len(pij), _i(pij), _d(out))
        if r:
            raise RuntimeError(f"reference sample_coeffs: {r}: {self.ref.error()}")
        return out

    def neighbours(self, patch_ij):
        pij = np.ascontiguousarray(patch_ij, dtype=np.int32).reshape(-1, 2)
        out = np.empty((len(pij), 9), dtype=np.int32)
        r = self.L.ref_neighbours(self.h, len(pij), _i(pij), _i(out))
        if r:
            raise RuntimeError(f"reference neighbours: {r}: {self.ref.error()}")
        return out


def ref_problem_desc(desc: ProblemDesc) -> ProblemDesc:
    """Resolve a config's pins without the product library,
    as pd_problem_create does: h = h_frac * Delta over the reference's own
    domain, dt = 0.2 min(delta)^2 / eps (diffusion rule) or / max(|A| + |C|)
    over the reference's own coefficient sampling (metric rule), tau = nt dt,
    T = Nt (Dt/tau) tau.  tests/test_oracle.py pins it against the product."""
    ref = Reference()
    L = ref.lib
    r = ProblemDesc.from_buffer_copy(desc)
    dom = np.zeros(4)
    flags = np.zeros(2, dtype=np.int32)
    st = L.ref_problem_domain(C.byref(r), _d(dom), _i(flags))
    if st:
        raise RuntimeError(f"reference problem: {st}: {ref.error()}")
    a, b, c, d = (float(x) for x in dom)
    if r.h_frac > 0.0:
        r.h_xi = r.h_frac * ((b - a) / r.N_xi)
        r.h_eta = r.h_frac * ((d - c) / r.N_eta)
    if r.dt_rule != 0 and not r.tau > 0:
        r.tau = 1.0  # placeholder: node coordinates do not depend on it
    if r.dt_over_tau > 0 and not r.T > 0:
        r.T = 1.0
    dmin = min(r.h_xi / r.nx, r.h_eta / r.ny)
    if r.dt_rule == 1:  # PD_DT_DIFFUSION
        r.tau = r.nt * (0.2 * dmin * dmin / r.eps)
    elif r.dt_rule == 2:  # PD_DT_METRIC
        pij = reference_patch_order(r.N_xi, r.N_eta, bool(flags[0]))
        if flags[1]:  # one integrator per eta-row (gaptooth.cpp:254-266): its first patch
            pij = pij[pij[:, 0] == pij[0, 0]]
        m = 0.0
        for q in range(0, len(pij), 4096):
            co = ref.sample_coeffs(r, pij[q:q + 4096])
            m = max(m, float((np.abs(co[:, 0]) + np.abs(co[:, 2])).max()))
        r.tau = r.nt * (0.2 * dmin * dmin / m)
    if r.dt_over_tau > 0:
        r.T = r.Nt * (r.dt_over_tau * r.tau)
    r.dt_rule = 0
    r.h_frac = 0.0
    r.dt_over_tau = 0.0
    return r


def reference_patch_order(Nxi, Neta, periodic):
    """Patch order of the GapToothEngine ctor (gaptooth.cpp:251-280)."""
    i_lo = 0 if periodic else 1
    return np.array([(i, j) for j in range(1, Neta) for i in range(i_lo, Nxi)], dtype=np.int32)


def engine_desc_from_tables(pdesc: ProblemDesc, periodic: bool, dom, patch_ij, coeffs, coeff_set=None,
                            mode=1):
    """Assemble a pd_engine_desc around numpy tables (kept alive on the object)."""
    d = EngineDesc()
    d.a, d.b, d.c, d.d = dom
    d.Nxi, d.Neta, d.periodic_xi = pdesc.N_xi, pdesc.N_eta, int(periodic)
    d.nx, d.ny, d.nt, d.k = pdesc.nx, pdesc.ny, pdesc.nt, pdesc.k
    d.tau, d.dt_macro = pdesc.tau, pdesc.T / pdesc.Nt
    d.h_xi, d.h_eta = pdesc.h_xi, pdesc.h_eta
    d.bc_type, d.robin_w1, d.robin_w2, d.quadrature = pdesc.bc_type, pdesc.robin_w1, pdesc.robin_w2, pdesc.quadrature
    keep = {}
    keep["pij"] = np.ascontiguousarray(patch_ij, dtype=np.int32)
    keep["coeffs"] = np.ascontiguousarray(coeffs, dtype=np.float64)
    d.npatches = len(keep["pij"])
    d.patch_ij = _i(keep["pij"])
    d.ncoeff_sets = keep["coeffs"].shape[0]
    if coeff_set is not None:
        keep["cset"] = np.ascontiguousarray(coeff_set, dtype=np.int32)
        d.coeff_set = _i(keep["cset"])
    d.coeffs = _d(keep["coeffs"])
    d.source_kind = 0
    d.l = 1.0
    d.mode = mode
    d._keep = keep
    return d


__all__ = ["Restated", "Reference", "reference_available", "reference_patch_order", "ref_problem_desc",
           "engine_desc_from_tables", "perimeter_len", "build_restated"]
