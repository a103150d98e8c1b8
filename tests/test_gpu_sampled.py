"""Time-dependent coefficients and general (non-separable) sources on the
device (pd_gaptooth_step_sampled / pd_projective_step_sampled): the host
samples the problem's closures at every micro step as the reference's
PatchIntegrator::integrate does (sample_coeffs / sample_source at t0 + s*dt,
microsim.cpp:537-542, 265-281) and the EXACT kernels run the sweeps on those
tables.  Checked bit for bit against the UNMODIFIED reference's own runs of
configs/pulsed_cdr.cfg (tests/golden/ref_pulsed.npz), with k = 0 and k = 1.
"""
import numpy as np
import pytest

from conftest import GOLDEN
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Engine, PatchdynError, Problem

FX = np.load(GOLDEN / "ref_pulsed.npz")


def pulsed(k):
    d, _ = configs.load("pulsed_cdr")
    return Problem(configs.copy_desc(d, k=k))


def test_pulsed_problem_tables_cpu():
    """host side (no GPU): general source kind, per-step samples really vary in time"""
    P = pulsed(0)
    assert P.engine_desc().source_kind == abi.PD_SOURCE_GENERAL
    c0, g0 = P.sample_substep(0.0)
    c1, g1 = P.sample_substep(P.desc.tau)
    assert c0.shape[0] == P.desc.nt and not np.array_equal(c0, c1) and not np.array_equal(g0, g1)
    # the t = 0 coefficient sample is the engine's static table (the reference's co0_)
    ed = P.engine_desc()
    co = np.ctypeslib.as_array(ed.coeffs, shape=(ed.ncoeff_sets, 6, ed.nx + 1, ed.ny + 1))
    assert np.array_equal(c0[0], co)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1])
@pytest.mark.parametrize("mode", [abi.PD_MODE_EXACT, abi.PD_MODE_FAST], ids=["exact", "fast"])
def test_sampled_steps_equal_reference(k, mode, gpu):
    P = pulsed(k)
    U0 = P.initial_field()
    assert np.array_equal(U0, FX[f"k{k}_U0"])
    E = Engine.from_problem(P, mode=mode)
    dt = P.desc.T / P.desc.Nt
    # step_direct (one gap-tooth substep)
    c, g = P.sample_substep(0.0)
    S1 = E.step_sampled(U0, 0.0, c, g, bnd=P.boundary(P.desc.tau))
    assert np.array_equal(S1, FX[f"k{k}_S1"])
    # cpi::projective_step x 6
    U = U0
    for n in range(6):
        t = n * dt
        c, g = P.sample_projective(t)
        U = E.projective_step_sampled(U, t, c, g, bnd=P.boundary_table(t, 1)[0])
        assert np.array_equal(U, FX[f"k{k}_U{n + 1}"]), n
    # without the sampled tables a general source has no device path (loud, no fallback)
    with pytest.raises(PatchdynError) as ei:
        E.projective_step(U0, 0.0)
    assert ei.value.status == abi.PD_UNSUPPORTED
