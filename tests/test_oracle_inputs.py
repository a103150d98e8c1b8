"""The oracle's own input builders (round 2), pinned.

bench.py's reference arm must not load the product library, so the oracle
builds its inputs itself: the shear-cdr tables of configs 4/5
(oracle/pd_oracle_problem.c) and the resolved pins of configs 1-3 over the
reference's own sampling (pyoracle.ref_problem_desc).  Both must equal what
the product builds bit for bit, and the shear tables must equal the
reference's own transform_coefficients sampling (geometry.cpp:93-125).
Also: the committed full-size config-4 fixture reproduces.
"""
import numpy as np
import pytest

from conftest import GOLDEN
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Problem


def product_tables(P):
    ed = P.engine_desc()
    n1, n2 = ed.nx + 1, ed.ny + 1
    pij = np.ctypeslib.as_array(ed.patch_ij, shape=(ed.npatches, 2)).copy()
    co = np.ctypeslib.as_array(ed.coeffs, shape=(ed.ncoeff_sets, 6, n1, n2)).copy()
    return ed, pij, co


SHEAR_CASES = {
    "c4-33x33": lambda: configs.copy_desc(configs.load("c4_shear")[0], N_xi=33, N_eta=33),
    "c4-65x17-8x8": lambda: configs.copy_desc(configs.load("c4_shear")[0], N_xi=65, N_eta=17, nx=7, ny=7),
    "c5-2^11-32x32": lambda: configs.sweep_desc(configs.load("c5_sweep")[0], 11, 32, 10),
}


@pytest.mark.parametrize("case", list(SHEAR_CASES))
def test_oracle_shear_tables_equal_product_tables(case, restated):
    d = SHEAR_CASES[case]()
    P = Problem(d)
    ed, pij, co = product_tables(P)
    r, oed, U0 = restated.shear_problem(d)
    assert np.array_equal(U0, P.initial_field())
    opij = np.ctypeslib.as_array(oed.patch_ij, shape=(oed.npatches, 2))
    assert np.array_equal(opij, pij)
    oco = np.ctypeslib.as_array(oed.coeffs, shape=(oed.ncoeff_sets, 6, ed.nx + 1, ed.ny + 1))
    assert ed.coeff_set is None or not ed.coeff_set  # one set per patch: the coefficients depend on xi
    assert np.array_equal(oco, co)
    pr = P.desc
    for f in ("tau", "T", "h_xi", "h_eta"):
        assert getattr(r, f) == getattr(pr, f), f
    assert (oed.tau, oed.dt_macro) == (ed.tau, ed.dt_macro)


def test_oracle_shear_tables_equal_reference_sampling(restated, reference):
    d = SHEAR_CASES["c4-33x33"]()
    r, oed, _ = restated.shear_problem(d)
    pij = np.ctypeslib.as_array(oed.patch_ij, shape=(oed.npatches, 2)).copy()
    sel = np.random.default_rng(0).choice(len(pij), 64, replace=False)
    got = np.ctypeslib.as_array(oed.coeffs, shape=(oed.ncoeff_sets, 6, r.nx + 1, r.ny + 1))[sel]
    assert np.array_equal(got, reference.sample_coeffs(r, pij[sel]))


@pytest.mark.parametrize("name", ["c1_diffusion", "c2_cdr_tanh", "c3_annulus"])
def test_reference_pin_resolution_equals_product(name, reference):
    from oracle.pyoracle import ref_problem_desc

    d, _ = configs.load(name)
    got = ref_problem_desc(d)
    want = Problem(d).desc
    for f, _ in abi.ProblemDesc._fields_:
        assert getattr(got, f) == getattr(want, f), f


def test_seeded_field_mt19937_64_known_answer(restated):
    """std::mt19937_64 default seed 5489: the 10000th draw is 9981545732273789042
    (C++11 [rand.predef]); our field draws (x >> 11) * 2^-53 from it."""
    import ctypes as C

    U = np.empty((100, 100))
    restated.lib.pdo_seeded_field(99, 99, 5489, 0, U.ctypes.data_as(C.POINTER(C.c_double)))
    x = U.ravel()[9999]
    assert x == (9981545732273789042 >> 11) * 2.0 ** -53


def test_config4_full_fixture_first_step_reproduces(restated):
    """tests/golden/c4_full.npz (made by make_golden.py on this oracle) holds the
    first projective step of the full-size config 4; recompute it here."""
    fx = np.load(GOLDEN / "c4_full.npz")
    d, _ = configs.load("c4_shear")
    r, ed, U0 = restated.shear_problem(d)
    assert U0.sum() == float(fx["U0_sum"])
    assert r.tau == float(fx["tau"]) and r.T == float(fx["T"])
    st, U1 = restated.projective_step(ed, U0, 0.0)
    assert st == 0
    assert np.array_equal(U1, fx["U1"])
