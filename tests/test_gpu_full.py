"""Full-size parity and run-loop edge cases on a B200 (round 2).

* config 4 at its stated size (512x512 patches of 16x16, K = 50, the whole
  100-step cpi::run, cpi.cpp:134-216) against the committed oracle fixture
  tests/golden/c4_full.npz: EXACT bit for bit, FAST within the north_star
  tolerance (1e-11 relative max-norm after the full run);
* the single-launch run (k_fast_run) on grids whose warp units outnumber the
  co-resident warps (each warp strides over several units), with and without
  the device exact-error metric, against one pd_projective_step per step;
* segmented runs (cpi::run split around probes/snapshots) keep the run's
  blow-up threshold (cpi.cpp:142-144) and step numbering;
* engines of different shared-memory needs alive at the same time.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from helpers import rel
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Engine, PatchdynError, Problem

pytestmark = pytest.mark.gpu

TOL = 1e-11  # north_star: FP64 macro fields within 1e-11 relative max-norm after the full run
FAST, EXACT = abi.PD_MODE_FAST, abi.PD_MODE_EXACT


def load(name, **over):
    d, _ = configs.load(name)
    return Problem(configs.copy_desc(d, **over))


@pytest.fixture(scope="module")
def c4():
    P = load("c4_shear")
    return P, P.initial_field(), np.load(GOLDEN / "c4_full.npz")


@pytest.mark.parametrize("mode", [FAST, EXACT], ids=["fast", "exact"])
def test_config4_full_size_full_run_vs_oracle(c4, mode, gpu):
    """BASELINE config 4 exactly as stated: 262144 patches, 100 macro steps."""
    P, U0, fx = c4
    assert U0.sum() == float(fx["U0_sum"])  # same seeded + smoothed initial field
    E = Engine.from_problem(P, mode=mode)
    assert E.mode == mode and E.P == 512 * 512
    nsteps = int(fx["nsteps"])
    assert nsteps == P.desc.Nt == 100
    U1 = E.projective_step(U0, 0.0)
    UT, st = E.run(U0, nsteps)
    assert st.steps_done == nsteps and st.failed_step == 0
    if mode == EXACT:  # the restated oracle's operation order, no contraction
        assert np.array_equal(U1, fx["U1"])
        assert np.array_equal(UT, fx["final"])
    else:
        assert rel(U1, fx["U1"]) < TOL
        assert rel(UT, fx["final"]) < TOL
    assert st.umax_last == pytest.approx(float(fx["umax_last"]), rel=1e-12)


# ---------------------------------------------------------------------------
# k_fast_run with strided warp units (the reuse of s_g / s_red
# across units, the per-warp guard maximum and the strided metric loops)
# ---------------------------------------------------------------------------
def stride_case(name):
    base, _ = configs.load("c5_sweep")
    if name == "8x8-2^13":
        return Problem(configs.sweep_desc(base, 13, 8, 10))
    if name == "16x16-2^12":
        return Problem(configs.sweep_desc(base, 12, 16, 10))
    if name == "7x7-ragged":  # 100^2 patches: 2500 four-patch units on 1776 co-resident warps
        return load("c1_diffusion", N_xi=101, N_eta=101)
    if name == "11x11-mixed":  # the exact-fit 1x11 tile, two patches per warp: 2048 units, strided
        return Problem(configs.copy_desc(configs.sweep_desc(base, 12, 16, 10), nx=10, ny=10))
    if name == "11x11-5pt":  # 45^2 patches: 1013 two-patch units (ragged), one per warp
        return load("c1_diffusion", nx=10, ny=10, N_xi=46, N_eta=46)
    raise KeyError(name)


def host_pct_error(P, U, ex):
    """cpi::max_percent_error (cpi.cpp:79-94) over the patch nodes, numpy."""
    d = P.engine_desc()
    i_lo = 0 if d.periodic_xi else 1
    e = ex[i_lo:-1, 1:-1]
    Ui = U[i_lo:-1, 1:-1]
    m = np.abs(e) >= 1e-12
    return (np.abs(Ui - e)[m] / np.abs(e)[m] * 100.0).max() if m.any() else 0.0


@pytest.mark.parametrize("case", ["8x8-2^13", "16x16-2^12", "7x7-ragged", "11x11-mixed", "11x11-5pt"])
@pytest.mark.parametrize("metric", [False, True], ids=["run", "run_exact"])
def test_fused_run_with_strided_units_equals_stepwise(case, metric, gpu):
    P = stride_case(case)
    n = 6
    U0 = P.initial_field()
    bt = P.boundary_table(0.0, n)
    E = Engine.from_problem(P, mode=FAST)
    assert E.mode == FAST
    dt = P.desc.T / P.desc.Nt
    rng = np.random.default_rng(5)
    ex = rng.uniform(0.5, 1.5, (n,) + U0.shape)
    if metric:
        Ug, st, err = E.run_exact(U0, n, ex, bnd=bt)
    else:
        Ug, st = E.run(U0, n, bnd=bt)
    assert st.kernel_launches == 1, "the single-launch run (k_fast_run) did not run"
    U = U0
    for s in range(n):
        U = E.projective_step(U, s * dt, bnd=bt[s])
        if metric:
            assert err[s] == host_pct_error(P, U, ex[s]), s
    assert np.array_equal(Ug, U)
    assert st.umax_last == np.abs(U).max()


def test_fused_run_forced_waves_subprocess(gpu):
    """PD_RUN_WAVES=8 (read once per process) forces the single launch where the
    default picks the multi-launch loop (16x16, 2^13 patches, K = 50: 8192 units,
    about seven per co-resident warp); results stay bit-identical."""
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Engine, Problem
base, _ = configs.load("c5_sweep")
P = Problem(configs.sweep_desc(base, 13, 16, 50))
E = Engine.from_problem(P)
U0 = P.initial_field()
Ug, st = E.run(U0, 4)
U = U0
for s in range(4):
    U = E.projective_step(U, s * P.desc.T / P.desc.Nt)
assert st.kernel_launches == 1, st.kernel_launches
assert np.array_equal(Ug, U)
print("ok")
""" % str(ROOT)
    env = dict(os.environ, PD_RUN_WAVES="8")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


# ---------------------------------------------------------------------------
# process-wide function attributes: an engine created later with
# a smaller (still > 48 KB) shared-memory need must not break a live larger one
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("mode", [EXACT, FAST], ids=["exact", "fast"])
def test_live_engines_with_different_shared_memory_needs(mode, gpu):
    big = load("ref_table1_cdr_const", nx=30, ny=30, mode=mode)
    small = load("ref_table1_cdr_const", nx=25, ny=25, mode=mode)
    Eb = Engine.from_problem(big, mode=mode)
    U0 = big.initial_field()
    bt = big.boundary_table(0.0, 2)
    ref, _ = Eb.run(U0, 2, bnd=bt)
    Es = Engine.from_problem(small, mode=mode)
    Us, _ = Es.run(small.initial_field(), 2, bnd=small.boundary_table(0.0, 2))
    again, _ = Eb.run(U0, 2, bnd=bt)  # launches of the larger engine still valid
    assert np.array_equal(again, ref)
    assert np.isfinite(Us).all()


# ---------------------------------------------------------------------------
# segmented runs keep the run's blow-up threshold (cpi.cpp:142-144)
# ---------------------------------------------------------------------------
def test_segmented_run_trips_at_the_runs_step(restated, gpu):
    """Config 1 with Dt/tau = 150 diverges ~4x per macro step from step ~22 on:
    never 10x in one step, so a per-segment threshold would never trip.  With
    pd_engine_set_run_guard the 1-step segments trip at the whole run's step."""
    P = load("c1_diffusion", Nt=30, dt_over_tau=150)
    U0 = P.initial_field()
    n = 30
    bt = P.boundary_table(0.0, n)
    dt = P.desc.T / P.desc.Nt
    st_o, _, so = restated.run(P.engine_desc(), U0, n, bnd=bt)
    assert st_o == abi.PD_MACRO_INSTABILITY and so.failed_step > 20
    for mode in (FAST, EXACT):
        E = Engine.from_problem(P, mode=mode)
        _, full = E.run(U0, n, bnd=bt, raise_on_instability=False)
        assert full.failed_step == so.failed_step
        scale0 = float(np.abs(U0).max())
        U, tripped = U0, 0
        for s in range(n):
            E.set_run_guard(scale0, s)
            try:
                U, st = E.run(U, 1, t0=s * dt, bnd=bt[s:s + 1])
            except PatchdynError as e:
                assert e.status == abi.PD_MACRO_INSTABILITY
                assert f"at macro step {so.failed_step} " in str(e), str(e)
                tripped = s + 1
                break
        assert tripped == so.failed_step
        # without the run-level scale every segment measures its own input: no trip
        E.set_run_guard(0.0, 0)
        U = U0
        for s in range(n):
            U, st = E.run(U, 1, t0=s * dt, bnd=bt[s:s + 1], raise_on_instability=False)
            assert st.failed_step == 0


# ---------------------------------------------------------------------------
# config 5: every (patch shape, K) combination of the sweep, whole-field runs
# against the restated oracle at 2^12 patches (the sweep's smallest size; the
# larger sizes are checked per row by bench.py --sweep: parity_rel)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("K", [10, 50, 200])
@pytest.mark.parametrize("nodes", [8, 16, 32])
def test_config5_points_full_field_vs_oracle(nodes, K, restated, gpu):
    base, _ = configs.load("c5_sweep")
    P = Problem(configs.sweep_desc(base, 12, nodes, K))
    ed = P.engine_desc()
    U0 = P.initial_field()
    n = 3
    st, Uo, _ = restated.run(ed, U0, n)
    assert st == abi.PD_OK
    F = Engine.from_problem(P, mode=FAST)
    assert F.mode == FAST
    Uf, sf = F.run(U0, n)
    assert sf.steps_done == n and rel(Uf, Uo) < TOL
    Ux, _ = Engine.from_problem(P, mode=EXACT).run(U0, n)
    assert np.array_equal(Ux, Uo)
