"""The reference-side binding (integration/gaptooth_b200_binding.hpp), compiled
against the UNMODIFIED reference headers and objects: the reference's own
GapToothEngine hands its patch list and its own coefficient sampling to
pd_engine_create, and step_direct / projective_step / cpi::run go through the
C-ABI.  EXACT must equal the reference's own step_direct, projective_step and
cpi::run bit for bit (final field and RunResult::max_pct_err) on configs 1-3;
FAST within the north_star tolerance.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import ROOT
from helpers import rel
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Problem

SO = ROOT / "integration" / "_build" / "libref_binding.so"
_dp = C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def binding():
    if not SO.exists():
        pytest.skip("integration/_build not built (needs /root/reference at build time)")
    L = C.CDLL(str(SO))
    L.rbh_last_error.restype = C.c_char_p
    L.rbh_create.argtypes = [C.POINTER(abi.ProblemDesc), C.c_int, C.POINTER(C.c_void_p)]
    L.rbh_destroy.argtypes = [C.c_void_p]
    L.rbh_mode.argtypes = [C.c_void_p]
    L.rbh_initial_field.argtypes = [C.c_void_p, _dp]
    L.rbh_step_direct.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int]
    L.rbh_projective_step.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int]
    L.rbh_run.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
    return L


def test_binding_library_exports(binding):
    for s in ("rbh_create", "rbh_step_direct", "rbh_projective_step", "rbh_run", "rbh_destroy"):
        assert hasattr(binding, s)


class Bound:
    def __init__(self, L, desc, mode):
        self.L = L
        self.h = C.c_void_p()
        st = L.rbh_create(C.byref(desc), mode, C.byref(self.h))
        assert st == 0, L.rbh_last_error().decode()
        self.shape = (desc.N_xi + 1, desc.N_eta + 1)

    def __del__(self):
        if self.h:
            self.L.rbh_destroy(self.h)

    def initial(self):
        U = np.empty(self.shape)
        self.L.rbh_initial_field(self.h, U.ctypes.data_as(_dp))
        return U

    def _call(self, fn, U, t, ours):
        U = np.ascontiguousarray(U)
        out = np.empty_like(U)
        st = fn(self.h, U.ctypes.data_as(_dp), out.ctypes.data_as(_dp), t, ours)
        assert st == 0, self.L.rbh_last_error().decode()
        return out

    def step_direct(self, U, t, ours):
        return self._call(self.L.rbh_step_direct, U, t, ours)

    def projective_step(self, U, t, ours):
        return self._call(self.L.rbh_projective_step, U, t, ours)

    def run(self, ours):
        U = np.empty(self.shape)
        e = C.c_double()
        st = self.L.rbh_run(self.h, U.ctypes.data_as(_dp), C.byref(e), ours)
        assert st == 0, self.L.rbh_last_error().decode()
        return U, e.value


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1_diffusion", "c2_cdr_tanh", "c3_annulus"])
@pytest.mark.parametrize("mode", [abi.PD_MODE_EXACT, abi.PD_MODE_FAST], ids=["exact", "fast"])
def test_binding_equals_reference(binding, name, mode, gpu):
    d, _ = configs.load(name)
    desc = Problem(d).desc  # resolved pins
    B = Bound(binding, desc, mode)
    assert binding.rbh_mode(B.h) == mode
    U0 = B.initial()
    dt = desc.T / desc.Nt
    same = np.array_equal if mode == abi.PD_MODE_EXACT else (lambda a, b: rel(a, b) < 1e-11)
    assert same(B.step_direct(U0, 0.0, 1), B.step_direct(U0, 0.0, 0))
    U1r = B.projective_step(U0, 0.0, 0)
    assert same(B.projective_step(U0, 0.0, 1), U1r)
    assert same(B.projective_step(U1r, dt, 1), B.projective_step(U1r, dt, 0))
    Ur, er = B.run(0)
    Ug, eg = B.run(1)
    assert same(Ug, Ur)
    if mode == abi.PD_MODE_EXACT:
        assert eg == er  # RunResult::max_pct_err, computed on the device
    else:
        assert eg == pytest.approx(er, rel=1e-6, abs=1e-12)
