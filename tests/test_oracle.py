"""The CPU oracle, pinned.

1. The C restatement (oracle/pd_oracle.c) reproduces the UNMODIFIED reference
   (oracle/_ref, compiled from /root/reference) bit for bit, and the committed
   golden fixtures (made by the reference, tests/golden/make_golden.py).
2. The reference's own known-answer tests (proj/tests/test_microsim.cpp,
   test_gaptooth.cpp, test_cpi.cpp), restated on the oracle.
3. The mixed-term extension (the reference rejects b != 0): exactness,
   convergence, linearity and locality.
"""
import numpy as np
import pytest

from conftest import GOLDEN
from helpers import D_, N_, R_, const_coef, edges, rel
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Problem

UNIT = np.load(GOLDEN / "unit_cases.npz")
FINALS = np.load(GOLDEN / "ref_finals.npz")


def steady_desc(**over):
    d = configs.default_desc()
    d.problem = abi.PD_PROBLEM_STEADY
    d.N_xi = d.N_eta = 6
    d.Nt, d.T = 200, 1.0
    d.tau = 1e-6
    d.h_xi = d.h_eta = 1e-3
    d.nx = d.ny = 6
    d.nt = 200  # explicit micro-solver, dt/d^2 = 0.18 (the reference fixture uses ADI with nt = 2)
    for k, v in over.items():
        setattr(d, k, v)
    return d


# ---------------------------------------------------------------------------
# 1. restatement == reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", range(5))
def test_integrate_bit_exact_vs_reference(case, restated):
    p = UNIT[f"int{case}_params"]
    A, C, Vx, Vy, W = p[:5]
    nx, ny, nt = int(p[5]), int(p[6]), int(p[7])
    coef = const_coef(nx + 1, ny + 1, A, C, Vx, Vy, W)
    st, uT = restated.integrate(coef, nx, ny, nt, p[8], p[9], p[10], UNIT[f"int{case}_kinds"],
                                UNIT[f"int{case}_vals"], UNIT[f"int{case}_slopes"], UNIT[f"int{case}_robin"],
                                UNIT[f"int{case}_u0"])
    assert st == 0
    assert np.array_equal(uT, UNIT[f"int{case}_uT"])


@pytest.mark.parametrize("case", range(3))
def test_lift_and_edge_profiles_bit_exact_vs_reference(case, restated):
    nx, ny = (int(x) for x in UNIT[f"lift{case}_in"])
    u0, sl, va = restated.lift(UNIT[f"lift{case}_vals"], 0.3, 0.55, 0.1, 0.05, 0.02, 0.01, nx, ny)
    assert np.array_equal(u0, UNIT[f"lift{case}_u0"])
    assert np.array_equal(sl, UNIT[f"lift{case}_slopes"])
    assert np.array_equal(va, UNIT[f"lift{case}_values"])


def test_restriction_known_answers(restated, reference):
    # proj/tests/test_gaptooth.cpp:196-218
    n = 10
    i = np.arange(n + 1)
    ss = np.outer(np.sin(np.pi * i / n), np.sin(np.pi * i / n))
    v = restated.restrict(ss)
    assert v == reference.restrict(ss)
    assert v == pytest.approx(0.39863458189061401, rel=1e-13)
    bil = np.outer(2 * i / n - 1, 3 * i / n + 2)
    assert abs(restated.restrict(bil)) < 1e-14
    assert abs(restated.restrict(ss, abi.PD_QUAD_SIMPSON) - 4 / np.pi ** 2) < 1e-4


@pytest.mark.parametrize("name", ["c1_diffusion", "c2_cdr_tanh", "c3_annulus"])
def test_full_runs_bit_exact_vs_reference_golden(name, restated):
    """cpi::run with linear_cache=off (configs 1-3): the whole trajectory."""
    P = Problem(configs.load(name)[0])
    ed = P.engine_desc()
    U0 = P.initial_field()
    assert np.array_equal(U0, FINALS[f"{name}_U0"])
    st, U1 = restated.projective_step(ed, U0, 0.0, bnd=P.boundary_table(0.0, 1)[0])
    assert st == 0 and np.array_equal(U1, FINALS[f"{name}_U1"])
    st, UT, stats = restated.run(ed, U0, P.desc.Nt, bnd=P.boundary_table(0.0, P.desc.Nt))
    assert st == 0 and stats.steps_done == P.desc.Nt
    assert np.array_equal(UT, FINALS[f"{name}_final"])


def make_variant(name, **over):
    d, _ = configs.load(name)
    return configs.copy_desc(d, **over)


@pytest.mark.parametrize("over", [dict(k=1), dict(bc_type=abi.PD_BC_DIRICHLET), dict(bc_type=abi.PD_BC_ROBIN),
                                  dict(quadrature=abi.PD_QUAD_SIMPSON)],
                         ids=["k1", "dirichlet", "robin", "simpson"])
def test_scheme_variants_bit_exact_vs_reference(over, restated, reference):
    P = Problem(make_variant("c1_diffusion", Nt=20, **over))
    ed = P.engine_desc()
    R = reference.engine(P.desc)
    U = R.initial_field()
    bt = P.boundary_table(0.0, 3)
    for n in range(3):
        t = n * P.desc.T / P.desc.Nt
        Ur = R.projective_step(U, t)
        st, Uo = restated.projective_step(ed, U, t, bnd=bt[n])
        assert st == 0 and np.array_equal(Ur, Uo), (over, n)
        U = Ur


def test_separable_source_bit_exact_vs_reference(restated, reference):
    """problem1_constant (cdr-const) on the explicit micro-solver: separable source
    time(t)/l (microsim.cpp:272-277) and time-dependent Dirichlet data."""
    d = configs.default_desc()
    d.problem = abi.PD_PROBLEM_REF_CDR
    d.N_xi = d.N_eta = 10
    d.Nt, d.T, d.tau = 1001, 1.0, 1e-6
    d.nx = d.ny = 10
    d.nt = 500  # 2-D explicit stability: dt/d^2 = 0.2 per direction
    P = Problem(d)
    ed = P.engine_desc()
    R = reference.engine(P.desc)
    U = R.initial_field()
    bt, stt = P.boundary_table(0.0, 3), P.source_time(0.0, 3)
    for n in range(3):
        t = n * P.desc.T / P.desc.Nt
        Ur = R.projective_step(U, t)
        st, Uo = restated.projective_step(ed, U, t, bnd=bt[n], src_time=stt[n])
        assert st == 0 and np.array_equal(Ur, Uo), n
        U = Ur
    assert np.abs(U).max() < 10.0  # e^(x+y+t) stays bounded: the explicit patch solve is stable


def test_macro_instability_guard_matches_reference(restated, reference):
    """proj/tests/test_cpi.cpp:212-223: dt ~100x beyond the stable projective step."""
    d = configs.default_desc()
    d.problem = abi.PD_PROBLEM_REF_ANNULUS
    d.N_xi, d.N_eta, d.Nt, d.T, d.tau = 16, 10, 5, 1.0, 1e-6
    d.h_xi = d.h_eta = 1e-3
    d.nx = d.ny = 10
    d.nt = 400
    P = Problem(d)
    R = reference.engine(P.desc)
    st_ref, _, _, _ = R.run()
    assert st_ref == abi.PD_MACRO_INSTABILITY
    step_ref = int(reference.error().split("macro step ")[1].split()[0])
    st, U, stats = restated.run(P.engine_desc(), P.initial_field(), P.desc.Nt, bnd=P.boundary_table(0.0, P.desc.Nt))
    assert st == abi.PD_MACRO_INSTABILITY and stats.failed_step == step_ref


# ---------------------------------------------------------------------------
# 2. the reference's known answers, on the oracle
# ---------------------------------------------------------------------------
def test_zero_and_constant_states(restated):
    # test_microsim.cpp:68-101
    nx, ny = 6, 8
    coef = const_coef(nx + 1, ny + 1, 1.0, 0.5, 3.0, -2.0)
    k, v, s = edges([N_] * 4, nx + 1, ny + 1)
    _, z = restated.integrate(coef, nx, ny, 3, 0.01, 0.02, 1e-6, k, v, s, np.zeros(8), np.zeros((7, 9)))
    assert np.all(z == 0.0)
    _, c = restated.integrate(coef, nx, ny, 3, 0.01, 0.02, 1e-6, k, v, s, np.zeros(8), np.full((7, 9), 3.25))
    assert np.abs(c - 3.25).max() <= 3.25e-14


def test_linear_steady_state_under_neumann_slopes(restated):
    # test_microsim.cpp:103-129
    nx, ny, h = 8, 6, 0.1
    dxi = h / nx
    u0 = np.repeat((0.3 - 0.05 + dxi * np.arange(nx + 1))[:, None], ny + 1, axis=1)
    sl = np.zeros((4, 9))
    sl[abi.PD_EDGE_E, :7] = sl[abi.PD_EDGE_W, :7] = 1.0
    k, v, s = edges([N_] * 4, 9, 7, slopes=sl)
    _, u = restated.integrate(const_coef(9, 7, 1.0, 1.0), nx, ny, 5, h, h, 1e-4, k, v, s, np.zeros(8), u0)
    assert rel(u, u0) < 1e-13


def test_one_dimensional_degenerate_patch(restated):
    # test_microsim.cpp:240-279
    h, tau, nx, ny, nt = 0.05, 2e-5, 10, 6, 40
    dxi, dt = h / nx, tau / nt
    line = np.sin(np.pi * dxi * np.arange(nx + 1) / h)
    u0 = np.repeat(line[:, None], ny + 1, axis=1)
    k, v, s = edges([D_, D_, N_, N_], nx + 1, ny + 1)
    _, u = restated.integrate(const_coef(nx + 1, ny + 1, 1.0, 1.0, 2.0, 0.0), nx, ny, nt, h, h, tau, k, v, s,
                              np.zeros(8), u0)
    ref = line.copy()
    for _ in range(nt):
        nxt = ref.copy()
        nxt[0] = nxt[nx] = 0.0
        nxt[1:nx] = ref[1:nx] + dt * ((ref[:-2] - 2 * ref[1:-1] + ref[2:]) / dxi ** 2 - 2.0 * (ref[2:] - ref[:-2]) / (2 * dxi))
        ref = nxt
    assert np.abs(u - ref[:, None]).max() < 1e-10


def test_discrete_maximum_principle(restated):
    # test_microsim.cpp:281-321
    rng = np.random.default_rng(99)
    n = 8
    u0 = rng.uniform(-1, 2, (n + 1, n + 1))
    vals = rng.uniform(-1, 2, (4, n + 1))
    lo, hi = min(u0.min(), vals.min()), max(u0.max(), vals.max())
    k, v, s = edges([D_] * 4, n + 1, n + 1, values=vals)
    _, u = restated.integrate(const_coef(n + 1, n + 1, 1.0, 1.0), n, n, 80, 0.1, 0.1, 1e-3, k, v, s, np.zeros(8), u0)
    assert u.min() >= lo - 1e-12 and u.max() <= hi + 1e-12


def _convergence_error(restated, n, B=0.0):
    # test_microsim.cpp:323-361 (+ a mixed term when B != 0)
    h, tau = 1.0, 0.01
    nt = 2 * n * n
    x = np.arange(n + 1) / n
    X, Y = np.meshgrid(x, x, indexing="ij")
    ustar = np.sin(np.pi * X) * np.sin(np.pi * Y)
    g = 2 * np.pi ** 2 * ustar - B * np.pi ** 2 * np.cos(np.pi * X) * np.cos(np.pi * Y)
    k, v, s = edges([D_] * 4, n + 1, n + 1)
    coef = const_coef(n + 1, n + 1, 1.0, 1.0, B=B)
    _, u = restated.integrate(coef, n, n, nt, h, h, tau, k, v, s, np.zeros(8), ustar, src_spatial=g,
                              src_time=np.ones(nt))
    return np.abs(u - ustar).max()


@pytest.mark.parametrize("B", [0.0, 0.5], ids=["5-point", "mixed"])
def test_second_order_convergence(restated, B):
    r = _convergence_error(restated, 8, B) / _convergence_error(restated, 16, B)
    assert 3.2 < r < 4.8


def test_robin_limits(restated):
    # test_microsim.cpp:432-482
    h, n = 0.1, 6
    d = h / n
    u0 = 1.0 + 0.3 * (d * np.arange(n + 1))[:, None] + 0.1 * (d * np.arange(n + 1))[None, :]
    vals = np.stack([u0[n, :], u0[0, :], u0[:, n], u0[:, 0]])
    sl = np.stack([np.full(n + 1, 0.3), np.full(n + 1, 0.3), np.full(n + 1, 0.1), np.full(n + 1, 0.1)])
    coef = const_coef(n + 1, n + 1, 1.0, 1.0)
    _, ur = restated.integrate(coef, n, n, 10, h, h, 1e-4, [R_] * 4, vals, sl, np.array([2.0, 0.0] * 4), u0)
    _, ud = restated.integrate(coef, n, n, 10, h, h, 1e-4, [D_] * 4, vals, sl, np.zeros(8), u0)
    assert rel(ur, ud) < 1e-12
    _, un = restated.integrate(coef, n, n, 10, h, h, 1e-4, [R_] * 4, vals, sl, np.array([0.0, 1.0] * 4), u0)
    assert rel(un, u0) < 1e-12


def test_partition_of_unity_and_quadratic_reproduction(restated):
    # test_gaptooth.cpp:99-154
    u0, sl, va = restated.lift(np.full(9, 2.75), 0.5, 0.5, 0.125, 0.125, 1e-3, 1e-3, 6, 8)
    assert np.abs(u0 - 2.75).max() <= 2.75e-14 and np.abs(sl[:, :9]).max() < 1e-11
    assert abs(restated.restrict(u0) - 2.75) <= 2.75e-14
    quad = lambda x, y: x * x + x * y - 2 * y * y + 3 * x - y + 1
    D, xc, yc, h, nx, ny = 0.1, 0.6, 0.3, 0.08, 5, 7
    vals = np.array([[quad(xc + p * D, yc + q * D) for q in (-1, 0, 1)] for p in (-1, 0, 1)])
    _, sl, va = restated.lift(vals, xc, yc, D, D, h, h, nx, ny)
    eta = yc - h / 2 + h * np.arange(ny + 1) / ny
    xi = xc - h / 2 + h * np.arange(nx + 1) / nx
    np.testing.assert_allclose(va[abi.PD_EDGE_E, :ny + 1], quad(xc + h / 2, eta), rtol=1e-12)
    np.testing.assert_allclose(sl[abi.PD_EDGE_W, :ny + 1], 2 * (xc - h / 2) + eta + 3, rtol=1e-12)
    np.testing.assert_allclose(sl[abi.PD_EDGE_N, :nx + 1], xi - 4 * (yc + h / 2) - 1, rtol=1e-12)


def test_gaptooth_zero_steady_and_bit_exact_locality(restated):
    # test_gaptooth.cpp:220-256
    P = Problem(steady_desc())
    ed = P.engine_desc()
    U0 = P.initial_field()
    _, Z = restated.gaptooth_step(ed, np.zeros_like(U0), 0.0)
    assert np.all(Z == 0.0)
    _, U1 = restated.gaptooth_step(ed, U0, 0.0, bnd=P.boundary(P.desc.tau))
    assert np.abs(U1 - U0).max() < 1e-10
    Up = U0.copy()
    Up[3, 3] += 0.1
    _, S1 = restated.gaptooth_step(ed, Up, 0.0, bnd=P.boundary(P.desc.tau))
    near = np.zeros_like(U0, dtype=bool)
    near[2:5, 2:5] = True
    interior = np.zeros_like(near)
    interior[1:-1, 1:-1] = True
    assert np.all(S1[interior & ~near] == U1[interior & ~near])
    assert np.any(S1[near] != U1[near])


def test_projective_step_is_forward_euler_extrapolation(restated):
    # test_cpi.cpp:58-83
    P = Problem(make_variant("c1_diffusion", Nt=50))
    ed = P.engine_desc()
    U = P.initial_field()
    _, U1 = restated.gaptooth_step(ed, U, 0.0)
    _, Pn = restated.projective_step(ed, U, 0.0)
    F = (U1 - U) / P.desc.tau
    manual = U + (P.desc.T / P.desc.Nt) * F
    np.testing.assert_allclose(Pn[1:-1, 1:-1], manual[1:-1, 1:-1], rtol=1e-14, atol=0)


def test_annulus_linearity_and_zero_trajectory(restated):
    # test_cpi.cpp:128-166 (power-of-two scale: exact in floating point)
    d = configs.default_desc()
    d.problem = abi.PD_PROBLEM_REF_ANNULUS
    d.N_xi, d.N_eta, d.Nt, d.T, d.tau = 8, 5, 100, 1.0, 1e-6
    d.h_xi = d.h_eta = 1e-3
    d.nx = d.ny = 10
    d.nt = 400
    P = Problem(d)
    ed = P.engine_desc()
    U0 = P.initial_field()
    _, A, _ = restated.run(ed, U0, 20)
    _, B, _ = restated.run(ed, 2.0 * U0, 20)
    assert np.array_equal(B, 2.0 * A)
    _, C, _ = restated.run(ed, 2.5 * U0, 20)
    assert rel(C, 2.5 * A) < 1e-10
    _, Z, _ = restated.run(ed, np.zeros_like(U0), 20)
    assert np.all(Z == 0.0)


# ---------------------------------------------------------------------------
# 3. mixed-term extension
# ---------------------------------------------------------------------------
def test_mixed_term_bilinear_exactness_with_corner_ghosts(restated):
    """u = a + b x + c y + d x y with exact Neumann slopes: central differences
    and the B.4 corner double ghosts are exact, so u_t = B d uniformly."""
    nx, ny, h, nt = 8, 6, 0.1, 20
    tau = 1e-5
    a, b, c, dd = 0.3, 1.2, -0.7, 2.5
    x = -h / 2 + (h / nx) * np.arange(nx + 1)
    y = -h / 2 + (h / ny) * np.arange(ny + 1)
    u0 = a + b * x[:, None] + c * y[None, :] + dd * x[:, None] * y[None, :]
    L = max(nx, ny) + 1
    sl = np.zeros((4, L))
    sl[abi.PD_EDGE_E, :ny + 1] = b + dd * y
    sl[abi.PD_EDGE_W, :ny + 1] = b + dd * y
    sl[abi.PD_EDGE_N, :nx + 1] = c + dd * x
    sl[abi.PD_EDGE_S, :nx + 1] = c + dd * x
    B = 0.7
    coef = const_coef(nx + 1, ny + 1, 1.0, 0.8, B=B)
    _, u = restated.integrate(coef, nx, ny, nt, h, h, tau, [N_] * 4, np.zeros((4, L)), sl, np.zeros(8), u0)
    np.testing.assert_allclose(u, u0 + tau * B * dd, rtol=0, atol=1e-12)


def test_mixed_term_linearity_and_locality_on_config4(restated):
    d = make_variant("c4_shear", N_xi=17, N_eta=17)
    P = Problem(d)
    ed = P.engine_desc()
    U0 = P.initial_field()
    _, S = restated.gaptooth_step(ed, U0, 0.0)
    _, S2 = restated.gaptooth_step(ed, 2.0 * U0, 0.0)
    assert np.array_equal(S2, 2.0 * S)
    Up = U0.copy()
    Up[7, 9] += 0.25
    _, Sp = restated.gaptooth_step(ed, Up, 0.0)
    diff = Sp != S
    assert diff[6:9, 8:11].all() and diff.sum() == 9  # exactly the 3x3 patches that see node (7,9)


def test_config4_small_run_reproduces_committed_oracle_fixture(restated):
    fx = np.load(GOLDEN / "c4_small.npz")
    P = Problem(make_variant("c4_shear", N_xi=33, N_eta=33))
    U0 = P.initial_field()
    assert np.array_equal(U0, fx["U0"])
    st, UT, _ = restated.run(P.engine_desc(), U0, 100)
    assert st == 0 and np.array_equal(UT, fx["final"])


# ---------------------------------------------------------------------------
# 4. linear-response path (GapToothEngine::step with linear_cache, the
#    reference's DEFAULT for row-shared problems; gaptooth.cpp:213-224, 377-418)
# ---------------------------------------------------------------------------
LINEAR = np.load(GOLDEN / "ref_linear.npz")


@pytest.mark.parametrize("name", ["c1_diffusion", "c3_annulus"])
def test_linear_path_restated_matches_reference_golden(name, restated):
    P = Problem(configs.load(name)[0])
    ed = P.engine_desc()
    st, w = restated.linear_weights(ed)
    assert st == 0
    assert np.all(w[0] == 0) and np.all(w[-1] == 0)
    U0 = P.initial_field()
    Nt = P.desc.Nt
    st, U1 = restated.linear_projective_step(ed, w, U0, 0.0, P.boundary_table(0.0, 1)[0])
    assert st == 0 and np.array_equal(U1, LINEAR[f"{name}_U1"])
    st, UT, stats = restated.linear_run(ed, w, U0, Nt, 0.0, P.boundary_table(0.0, Nt))
    assert st == 0 and stats.steps_done == Nt
    assert np.array_equal(UT, LINEAR[f"{name}_final"])
    # the shortcut agrees with the micro-solve to ~1e-13 (fast vs direct)
    assert rel(UT, FINALS[f"{name}_final"]) < 1e-11


def test_linear_path_reproduces_shipped_table4_output(restated):
    """proj/out/table4/16x10 came from the reference's linear-response path:
    the restated path reproduces every shipped snapshot bit for bit."""
    gold = np.load(GOLDEN / "annulus_16x10.npz")
    P = Problem(configs.load("ref_annulus_16x10")[0])
    ed = P.engine_desc()
    st, w = restated.linear_weights(ed)
    assert st == 0
    U, done, Nt = P.initial_field(), 0, P.desc.Nt
    dt = P.desc.T / Nt
    for key in ["t_0.25", "t_0.50", "t_0.75", "t_1.00"]:
        target = int(round(float(key[2:]) * Nt))
        st, U, _ = restated.linear_run(ed, w, U, target - done, done * dt, P.boundary_table(done * dt, target - done))
        assert st == 0
        done = target
        assert np.array_equal(U, gold[key]), key


def test_evolve_batch_is_one_patch_of_step_direct(restated):
    """evolve_patch on the gathered stencil == the patch's value after step_direct."""
    P = Problem(configs.load("c2_cdr_tanh")[0])
    ed = P.engine_desc()
    U0 = P.initial_field()
    st, U1 = restated.gaptooth_step(ed, U0, 0.0)
    assert st == 0
    pij = np.ctypeslib.as_array(ed.patch_ij, shape=(ed.npatches, 2))
    idx = np.array([0, 17, 1000, ed.npatches - 1], dtype=np.int32)
    sten = np.stack([U0[i - 1:i + 2, j - 1:j + 2] for i, j in pij[idx]])
    st, avg = restated.evolve_batch(ed, idx, sten)
    assert st == 0
    assert np.array_equal(avg, U1[pij[idx, 0], pij[idx, 1]])


def test_linear_step_is_linear_and_local(restated):
    P = Problem(configs.load("c1_diffusion")[0])
    ed = P.engine_desc()
    _, w = restated.linear_weights(ed)
    rng = np.random.default_rng(5)
    U = rng.uniform(-1, 1, P.shape)
    _, A = restated.linear_step(ed, w, U)
    _, B = restated.linear_step(ed, w, 2.0 * U)
    assert np.array_equal(B, 2.0 * A)
    # a unit impulse at an interior node reaches exactly its 3x3 neighbourhood
    E = np.zeros(P.shape)
    E[9, 9] = 1.0
    _, R = restated.linear_step(ed, w, E)
    nz = np.argwhere(R != 0)
    assert nz.min(0).tolist() == [8, 8] and nz.max(0).tolist() == [10, 10]
    # and the response of patch (9,9) to it is row 9's centre weight
    assert R[9, 9] == w[9, 1, 1]


# ---------------------------------------------------------------------------
# 5. ADI micro-solver (the reference's default solver; Tables 1-3)
# ---------------------------------------------------------------------------
ADI = np.load(GOLDEN / "ref_adi.npz")
ADI_CASES = {
    "const_two": {},
    "const_l03_three": {"lambda_": 0.3, "upwind_order": abi.PD_UPWIND_THREE},
    "var_l03_four": {"problem": abi.PD_PROBLEM_REF_CDR_VAR, "lambda_": 0.3, "upwind_order": abi.PD_UPWIND_FOUR,
                     "upwind_r": 0.3},
    "var_dirichlet_two": {"problem": abi.PD_PROBLEM_REF_CDR_VAR, "bc_type": abi.PD_BC_DIRICHLET},
    "const_robin_three": {"bc_type": abi.PD_BC_ROBIN, "robin_w1": 2.0, "robin_w2": 1.0,
                          "upwind_order": abi.PD_UPWIND_THREE},
    "var_k1_two": {"problem": abi.PD_PROBLEM_REF_CDR_VAR, "k": 1},
    "const_nx10_ny14_two": {"ny": 14, "lambda_": 0.2},
}


@pytest.mark.parametrize("name", list(ADI_CASES))
def test_adi_restated_bit_exact_vs_reference(name, restated):
    base, _ = configs.load("ref_table1_cdr_const")
    P = Problem(configs.copy_desc(base, **ADI_CASES[name]))
    ed = P.engine_desc()
    assert ed.solver == abi.PD_SOLVER_ADI
    U0 = ADI[f"{name}_U0"]
    assert np.array_equal(P.initial_field(), U0)
    st, U, stats = restated.run(ed, U0, 40, 0.0, P.boundary_table(0.0, 40), P.source_time(0.0, 40))
    assert st == 0 and stats.steps_done == 40
    assert np.array_equal(U, ADI[f"{name}_final"])


def test_adi_restated_reproduces_shipped_table1_output(restated):
    gold = np.load(GOLDEN / "table1_cdr.npz")
    P = Problem(configs.load("ref_table1_cdr_const")[0])
    ed = P.engine_desc()
    Nt = P.desc.Nt
    dt = P.desc.T / Nt
    bnd, src = P.boundary_table(0.0, Nt), P.source_time(0.0, Nt)
    U, done = P.initial_field(), 0
    for key in sorted(gold.files):
        target = int(round(float(key[2:]) / dt))
        st, U, _ = restated.run(ed, U, target - done, done * dt, bnd[done:target], src[done:target])
        assert st == 0
        done = target
        assert np.array_equal(U, gold[key]), key


def test_adi_source_times_are_midpoints():
    """ADI samples the source at t0 + (s + 1/2) dt (microsim.cpp:536-537)."""
    base, _ = configs.load("ref_table1_cdr_const")
    Pa = Problem(base)
    Pe = Problem(configs.copy_desc(base, solver=abi.PD_SOLVER_EXPLICIT, nt=200, tau=1e-6))
    mdt = Pa.desc.tau / Pa.desc.nt
    sa = Pa.source_time(0.0, 1)[0, 0]
    assert sa[0] == np.exp(0.5 * mdt) and sa[1] == np.exp(1.5 * mdt)
    se = Pe.source_time(0.0, 1)[0, 0]
    assert se[0] == 1.0
