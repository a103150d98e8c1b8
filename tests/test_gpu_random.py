"""Seeded random cross-configurations of the device path against the restated
oracle (oracle/pd_oracle.c, pinned to the reference in test_oracle.py).

Each case draws a problem family (identity diffusion, tanh-stretched CDR with
time-dependent Dirichlet data, the periodic annulus, the sheared mesh with the
mixed term), a macro grid, a micro grid (n1 != n2 allowed, 3..32 nodes per side
-> exact-fit and padded FAST tiles, the 4-warp 32x32 tile), K, the projective k,
the patch condition and the quadrature, and runs a few macro steps through
Engine.run: EXACT must equal the oracle bit for bit, FAST must stay within the
north_star tolerance (1e-11 relative max-norm).  Combinations the reference
rejects (Robin with the mixed term, Simpson on an odd micro resolution) are
redrawn, not skipped.
"""
import numpy as np
import pytest

from helpers import rel
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Engine, Problem

pytestmark = pytest.mark.gpu

TOL = 1e-11
FAMILIES = ["c1_diffusion", "c2_cdr_tanh", "c3_annulus", "c4_shear"]
BCS = [abi.PD_BC_NEUMANN, abi.PD_BC_DIRICHLET, abi.PD_BC_ROBIN]


def draw(seed):
    rng = np.random.default_rng(1000 + seed)
    while True:
        name = FAMILIES[rng.integers(len(FAMILIES))]
        nx, ny = (int(v) for v in rng.integers(2, 32, size=2))
        if rng.random() < 0.3:
            ny = nx
        over = dict(N_xi=int(rng.integers(4, 13)), N_eta=int(rng.integers(4, 11)), nx=nx, ny=ny,
                    nt=int(rng.integers(1, 31)), k=int(rng.integers(0, 3)), Nt=int(rng.integers(3, 7)),
                    bc_type=int(BCS[rng.integers(3)]))
        if over["bc_type"] == abi.PD_BC_ROBIN:
            over.update(robin_w1=float(rng.choice([1.0, 2.0])), robin_w2=float(rng.choice([0.0, 0.5, 1.0])))
        if nx % 2 == 0 and ny % 2 == 0 and rng.random() < 0.4:
            over["quadrature"] = abi.PD_QUAD_SIMPSON
        if name == "c4_shear" and over["bc_type"] == abi.PD_BC_ROBIN:
            continue  # MixedTermUnsupported with Robin ghosts (as the reference)
        return name, over


CASES = [draw(s) for s in range(32)]


def case_id(c):
    name, o = c
    bc = {0: "neu", 1: "dir", 2: "rob"}[o["bc_type"]]
    q = "-simp" if o.get("quadrature") == abi.PD_QUAD_SIMPSON else ""
    return f"{name[:2]}-{o['N_xi']}x{o['N_eta']}-{o['nx'] + 1}x{o['ny'] + 1}-K{o['nt']}-k{o['k']}-{bc}{q}"


@pytest.mark.parametrize("case", CASES, ids=[case_id(c) for c in CASES])
def test_random_configuration_vs_oracle(case, restated, gpu):
    name, over = case
    d, _ = configs.load(name)
    P = Problem(configs.copy_desc(d, **over))
    ed = P.engine_desc()
    U0 = P.initial_field()
    n = P.desc.Nt
    bt = P.boundary_table(0.0, n)
    st, Uo, _ = restated.run(ed, U0, n, bnd=bt)
    assert st == 0 and np.isfinite(Uo).all()
    for mode in (abi.PD_MODE_EXACT, abi.PD_MODE_FAST):
        E = Engine.from_problem(P, mode=mode)
        if mode == abi.PD_MODE_FAST and max(over["nx"], over["ny"]) < 32:
            assert E.mode == abi.PD_MODE_FAST, "a FAST tile exists for every explicit patch up to 32x32"
        Ug, stats = E.run(U0, n, bnd=bt)
        assert stats.steps_done == n and stats.failed_step == 0
        if E.mode == abi.PD_MODE_EXACT:
            assert np.array_equal(Ug, Uo)
        else:
            assert rel(Ug, Uo) < TOL
