"""CPU tests of the C-ABI library and the host-side mesh/metric + index builders.

No kernel runs here (no GPU in the build container): the library must load,
export every symbol include/patchdyn_b200.h declares, and its host-side table
builders must reproduce the reference bit for bit.
"""
import ctypes as C
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import PatchdynError, Problem, index_tables, lib


def header_symbols():
    text = (ROOT / "include" / "patchdyn_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pd_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = lib()
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, f"declared but not exported: {missing}"
    assert L.pd_abi_version() == abi.PD_ABI_VERSION


def test_status_names_follow_reference_exception_types():
    L = lib()
    names = {abi.PD_NON_POSITIVE_JACOBIAN: "NonPositiveJacobian", abi.PD_MIXED_TERM_UNSUPPORTED: "MixedTermUnsupported",
             abi.PD_STABILITY_VIOLATION: "StabilityViolation", abi.PD_MACRO_INSTABILITY: "MacroInstability",
             abi.PD_MACRO_PATCH_ERROR: "MacroPatchError", abi.PD_VALIDATION_ERROR: "ValidationError",
             abi.PD_SHAPE_MISMATCH: "ShapeMismatch"}
    for code, name in names.items():
        assert L.pd_status_name(code).decode() == name


def test_perimeter_len():
    assert lib().pd_perimeter_len(19, 19) == abi.perimeter_len(19, 19) == 80


@pytest.mark.parametrize("name,periodic", [("c1_diffusion", False), ("c3_annulus", True),
                                           ("ref_annulus_16x10", True), ("c2_cdr_tanh", False)])
def test_index_tables_bit_exact_vs_reference(name, periodic, reference):
    from oracle.pyoracle import reference_patch_order

    d, _ = configs.load(name)
    P = Problem(d)
    ed = P.engine_desc()
    assert bool(ed.periodic_xi) == periodic
    pij, nbr = index_tables(ed)
    # patch order of the GapToothEngine ctor (gaptooth.cpp:251-280)
    assert np.array_equal(pij, reference_patch_order(d.N_xi, d.N_eta, periodic))
    # 3x3 gather of the reference's own build_stencil (gaptooth.cpp:74-104)
    R = reference.engine(P.desc)
    assert np.array_equal(nbr, R.neighbours(pij))


def test_index_tables_reject_patch_outside_interior():
    d, _ = configs.load("c1_diffusion")
    ed = Problem(d).engine_desc()
    bad = np.array([[0, 5]], dtype=np.int32)  # i = 0 is a boundary node on a non-periodic side
    ed.npatches = 1
    ed.patch_ij = bad.ctypes.data_as(C.POINTER(C.c_int32))
    with pytest.raises(PatchdynError) as e:
        index_tables(ed)
    assert e.value.status == abi.PD_MACRO_PATCH_ERROR and "outside interior" in str(e.value)


@pytest.mark.parametrize("name", ["c1_diffusion", "c2_cdr_tanh", "c3_annulus", "ref_annulus_16x10"])
def test_coefficient_tables_bit_exact_vs_reference_sampling(name, reference):
    """Host mesh/metric setup == PatchIntegrator::sample_coeffs of the reference
    (geometry.cpp:93-125, microsim.cpp:236-249), including row sharing."""
    d, _ = configs.load(name)
    P = Problem(d)
    ed = P.engine_desc()
    n1, n2 = d.nx + 1, d.ny + 1
    co = np.ctypeslib.as_array(ed.coeffs, shape=(ed.ncoeff_sets, 6, n1, n2))
    pij = np.ctypeslib.as_array(ed.patch_ij, shape=(ed.npatches, 2))
    if ed.coeff_set:  # one set per eta-row, sampled at xi(i_lo) (gaptooth.cpp:254-266)
        i_lo = 0 if ed.periodic_xi else 1
        sets = np.array([(i_lo, j) for j in range(1, d.N_eta)], dtype=np.int32)
    else:
        sets = pij
    pick = np.unique(np.linspace(0, len(sets) - 1, 40).astype(int))
    ref = reference.sample_coeffs(P.desc, sets[pick])
    assert np.array_equal(ref, co[pick])


def test_config4_coefficients_bit_exact_and_reference_rejects_mixed_term(reference):
    d, _ = configs.load("c4_shear")
    d = configs.copy_desc(d, N_xi=65, N_eta=65)
    P = Problem(d)
    ed = P.engine_desc()
    co = np.ctypeslib.as_array(ed.coeffs, shape=(ed.ncoeff_sets, 6, 16, 16))
    pij = np.ctypeslib.as_array(ed.patch_ij, shape=(ed.npatches, 2))
    pick = np.arange(0, ed.npatches, 97)
    ref = reference.sample_coeffs(P.desc, pij[pick])
    assert np.array_equal(ref, co[pick])
    assert np.abs(co[:, abi.PD_COEF_B]).max() > 1e-3  # g12 != 0
    # the unmodified reference refuses this problem (microsim.cpp:239-244)
    with pytest.raises(RuntimeError, match="status 3"):
        reference.engine(P.desc)


def test_initial_fields_bit_exact_vs_reference(reference):
    for name in ["c1_diffusion", "c2_cdr_tanh", "c3_annulus", "ref_annulus_16x10"]:
        d, _ = configs.load(name)
        P = Problem(d)
        assert np.array_equal(P.initial_field(), reference.engine(P.desc).initial_field()), name


def test_pins_resolved_as_documented():
    d, _ = configs.load("c1_diffusion")
    r = Problem(d).desc
    D = 1.0 / 19
    h = 0.2 * D
    delta = h / 6
    assert r.h_xi == pytest.approx(h, rel=1e-15) and r.h_eta == pytest.approx(h, rel=1e-15)
    assert r.tau == pytest.approx(20 * 0.2 * delta * delta, rel=1e-15)
    assert r.T == pytest.approx(200 * 5 * r.tau, rel=1e-15)
    # metric rule: 2-D 9-point symbol <= 1 and the reference's guard passes
    for name in ["c2_cdr_tanh", "c3_annulus"]:
        P = Problem(configs.load(name)[0])
        apc, ref_number = P.stability()
        dmin = min(P.desc.h_xi / P.desc.nx, P.desc.h_eta / P.desc.ny)
        assert P.desc.tau / P.desc.nt * apc / dmin ** 2 == pytest.approx(0.2, rel=1e-12)
        assert ref_number <= 0.5


def test_stability_guard_matches_reference():
    d, _ = configs.load("c1_diffusion")
    d = configs.copy_desc(d, dt_rule=abi.PD_DT_GIVEN, tau=1e-2, h_frac=0.2, dt_over_tau=5)
    with pytest.raises(PatchdynError) as e:
        Problem(d)
    assert e.value.status == abi.PD_STABILITY_VIOLATION


def test_config_parser_rejects_unknown_keys_and_sweep_shapes():
    with pytest.raises(ValueError, match="unknown key"):
        configs.parse("[problem]\nkind = steady\nbogus = 1\n")
    with pytest.raises(ValueError, match="unknown section"):
        configs.parse("[nope]\nx = 1\n")
    base, vals = configs.load("c5_sweep")
    assert vals["sweep.K"] == "10, 50, 200"
    for k in range(12, 21):
        s = configs.sweep_desc(base, k, 16, 50)
        assert (s.N_xi - 1) * (s.N_eta - 1) == 2 ** k
        assert s.nx == s.ny == 15 and s.nt == 50


def test_seeded_field_is_deterministic_and_smoothed():
    d, _ = configs.load("c4_shear")
    d = configs.copy_desc(d, N_xi=33, N_eta=33)
    U1 = Problem(d).initial_field()
    U2 = Problem(d).initial_field()
    assert np.array_equal(U1, U2)
    raw = Problem(configs.copy_desc(d, jacobi_sweeps=0)).initial_field()
    assert 0.0 <= raw.min() and raw.max() < 1.0
    assert np.array_equal(U1[0, :], raw[0, :]) and np.array_equal(U1[:, -1], raw[:, -1])  # boundary fixed
    assert U1[1:-1, 1:-1].std() < raw[1:-1, 1:-1].std()  # Jacobi sweeps smooth the interior


def test_time_dependent_boundary_table_matches_exact_solution():
    d, _ = configs.load("c2_cdr_tanh")
    P = Problem(d)
    dt = P.desc.T / P.desc.Nt
    bt = P.boundary_table(0.0, 3)
    assert bt.shape == (3, 2, abi.perimeter_len(63, 63))
    for n in range(3):
        ex = P.exact((n + 1) * dt)
        np.testing.assert_array_equal(bt[n, 1][:64], ex[:, 0])       # S row
        np.testing.assert_array_equal(bt[n, 1][64:128], ex[:, 63])   # N row
        np.testing.assert_array_equal(bt[n, 1][128:192], ex[0, :])   # W column


def test_separable_source_time_factors():
    d = configs.default_desc()
    d.problem = abi.PD_PROBLEM_REF_CDR
    d.N_xi = d.N_eta = 10
    d.Nt = 1001
    d.nx = d.ny = 10
    d.nt = 500  # explicit micro-solver: 0.2 on the reference's guard (ADI is the reference default here)
    P = Problem(d)
    st = P.source_time(0.0, 2)
    dt, tau = P.desc.T / P.desc.Nt, P.desc.tau
    assert st.shape == (2, 1, 500)
    assert st[1, 0, 250] == pytest.approx(np.exp(dt + tau / 2), rel=1e-15)
    assert Problem(configs.load("c1_diffusion")[0]).source_time(0.0, 1) is None


def test_device_coefficient_generation_fails_loudly_without_a_gpu():
    """coeff_gen = PD_COEFF_DEVICE never falls back to host sampling: on a host
    without a CUDA device the problem build reports a device error."""
    from paper_2405_08764_b200.engine import device_count

    if device_count() > 0:
        pytest.skip("a CUDA device is visible (covered by tests/test_gpu.py)")
    d = configs.copy_desc(configs.load("c1_diffusion")[0], coeff_gen=abi.PD_COEFF_DEVICE)
    with pytest.raises(PatchdynError) as ei:
        Problem(d)
    assert ei.value.status == abi.PD_CUDA_ERROR
    # the host path of the same problem is unaffected and still builds its tables
    ed = Problem(configs.copy_desc(d, coeff_gen=abi.PD_COEFF_HOST)).engine_desc()
    assert ed.coeffs and not ed.coeff_generator
