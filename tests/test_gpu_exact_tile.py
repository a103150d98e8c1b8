"""Register-blocked EXACT step (csrc/kernels_exact_tile.cuh, k_exact_tile).

The tile kernel replays the reference's arithmetic (explicit_sweep,
microsim.cpp:292-332; integrate :509-552; gaptooth.cpp:110-194) on the
lane-per-block mapping.  It must be bit-identical to

* the restated oracle (reference + mixed term) on every tile shape, with and
  without the mixed term, Neumann, (5-point) Robin and pinned (Dirichlet,
  Robin with w2 = 0) patch edges, the separable source, both quadratures,
  k = 0 and k = 1, and
* the shared-memory kernel it replaces (k_gaptooth_exact), which a child
  process runs with PD_EXACT_TILE=0 on the same cases.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2405_08764_b200 import abi, configs
from paper_2405_08764_b200.engine import Engine, Problem

pytestmark = pytest.mark.gpu
EXACT = abi.PD_MODE_EXACT

ROBIN = dict(bc_type=abi.PD_BC_ROBIN, robin_w1=2.0, robin_w2=1.0)
DIRICHLET = dict(bc_type=abi.PD_BC_DIRICHLET)
ROBIN_PINNED = dict(bc_type=abi.PD_BC_ROBIN, robin_w1=1.0, robin_w2=0.0)  # w2 = 0: behaves as Dirichlet
# name -> (config, overrides, macro steps)
CASES = {
    "7x7-5pt": ("c1_diffusion", dict(Nt=20), 5),
    "7x7-5pt-robin-k1": ("c1_diffusion", dict(Nt=20, k=1, **ROBIN), 4),
    "7x7-5pt-simpson": ("c1_diffusion", dict(Nt=20, quadrature=abi.PD_QUAD_SIMPSON), 4),
    "8x8-5pt": ("c1_diffusion", dict(nx=7, ny=7, Nt=20), 4),
    "9x9-5pt-periodic": ("c3_annulus", dict(Nt=20), 4),
    "9x9-5pt-cdr": ("c2_cdr_tanh", dict(N_xi=23, N_eta=23, Nt=20), 4),
    "16x16-5pt-robin": ("c1_diffusion", dict(nx=15, ny=15, Nt=20, **ROBIN), 3),
    "7x7-mixed": ("c4_shear", dict(nx=6, ny=6, N_xi=9, N_eta=11, nt=20, Nt=5), 4),
    "8x8-mixed": ("c4_shear", dict(nx=7, ny=7, N_xi=11, N_eta=9, nt=21, Nt=5), 4),  # odd nt: the unrolled loop's tail
    "8x8-5pt-robin": ("c1_diffusion", dict(nx=7, ny=7, Nt=20, **ROBIN), 4),
    "9x9-mixed-k1": ("c4_shear", dict(nx=8, ny=8, N_xi=10, N_eta=9, nt=20, Nt=5, k=1), 3),
    "16x16-mixed": ("c4_shear", dict(N_xi=33, N_eta=17, Nt=10), 4),
    "16x16-mixed-one-micro-step": ("c4_shear", dict(N_xi=9, N_eta=9, nt=1, tau=2e-7, Nt=50), 3),
    # pinned edges (Dirichlet; Robin with w2 = 0): edge nodes keep their pinned values
    "7x7-5pt-dirichlet": ("c1_diffusion", dict(Nt=20, **DIRICHLET), 5),
    "9x9-5pt-robin-pinned-periodic": ("c3_annulus", dict(Nt=20, **ROBIN_PINNED), 3),
    "8x8-mixed-dirichlet": ("c4_shear", dict(nx=7, ny=7, N_xi=11, N_eta=9, nt=20, Nt=5, **DIRICHLET), 4),
    "16x16-mixed-dirichlet-k1": ("c4_shear", dict(N_xi=17, N_eta=33, Nt=10, k=1, **DIRICHLET), 3),
    "11x11-5pt-dirichlet": ("c1_diffusion", dict(nx=10, ny=10, Nt=20, **DIRICHLET), 4),
    "32x32-5pt-robin-pinned": ("c1_diffusion", dict(nx=31, ny=31, Nt=20, **ROBIN_PINNED), 3),
    "32x32-mixed-dirichlet": ("c4_shear", dict(nx=31, ny=31, N_xi=9, N_eta=11, nt=21, Nt=5, **DIRICHLET), 3),
    # separable source g = spatial(x, y) time(t) / l (sample_source, microsim.cpp:272-277)
    "src-7x7": ("ref_cdr", dict(nx=6, ny=6), 3),
    "src-9x9-k1": ("ref_cdr", dict(nx=8, ny=8, k=1), 3),
    "src-11x11-robin": ("ref_cdr", dict(nx=10, ny=10, **ROBIN), 3),
    "src-16x16": ("ref_cdr", dict(nx=15, ny=15, nt=1200), 2),
    "src-32x32": ("ref_cdr", dict(nx=31, ny=31, N_xi=6, N_eta=6, nt=5000), 2),
    # 11x11 nodes: the reference's default micro grid (nx = ny = 10, scheme_config.hpp:17)
    "11x11-5pt-robin": ("c1_diffusion", dict(nx=10, ny=10, Nt=20, **ROBIN), 4),
    "11x11-5pt-cdr-simpson": ("c2_cdr_tanh", dict(nx=10, ny=10, N_xi=23, N_eta=23, Nt=20,
                                                 quadrature=abi.PD_QUAD_SIMPSON), 3),
    "11x11-mixed-k1": ("c4_shear", dict(nx=10, ny=10, N_xi=10, N_eta=12, nt=20, Nt=5, k=1), 3),
    "32x32-mixed": ("c4_shear", dict(nx=31, ny=31, N_xi=9, N_eta=11, nt=21, Nt=5), 3),
    "32x32-5pt-robin-k1": ("c1_diffusion", dict(nx=31, ny=31, Nt=20, k=1, **ROBIN), 3),
    "32x32-5pt-periodic": ("c3_annulus", dict(nx=31, ny=31, Nt=20, N_xi=16, N_eta=8), 2),
    # 17x17 nodes is not a tile: the shared-memory kernel stays in place
    "17x17-mixed-simpson": ("c4_shear", dict(nx=16, ny=16, N_xi=9, N_eta=9, nt=20, Nt=5,
                                             quadrature=abi.PD_QUAD_SIMPSON), 3),
}


def make_problem(name):
    cfg, over, n = CASES[name]
    if cfg == "ref_cdr":  # the reference's CDR problem with its separable source, explicit solver
        d = configs.default_desc()
        d.problem = abi.PD_PROBLEM_REF_CDR
        d.N_xi = d.N_eta = 10
        d.Nt, d.T, d.tau = 1001, 1.0, 1e-6
        d.nt = 500  # 2-D explicit stability: dt/d^2 = 0.2 per direction
    else:
        d, _ = configs.load(cfg)
    return Problem(configs.copy_desc(d, **over)), n


def source_time(P, n):
    return P.source_time(0.0, n) if P.engine_desc().source_kind == abi.PD_SOURCE_SEPARABLE else None


def run_case(name):
    P, n = make_problem(name)
    U0 = P.initial_field()
    bt = P.boundary_table(0.0, n)
    E = Engine.from_problem(P, mode=EXACT)
    assert E.mode == EXACT
    # the tile kernel is the one that runs (except in the PD_EXACT_TILE=0 child and on 17x17 nodes)
    assert E.exact_tile == (os.environ.get("PD_EXACT_TILE") != "0" and not name.startswith("17x17"))
    U, st = E.run(U0, n, bnd=bt, src_time=source_time(P, n))
    assert st.steps_done == n
    return P, U0, bt, n, U


@pytest.mark.parametrize("name", list(CASES))
def test_exact_tile_bit_identical_to_oracle(name, restated, gpu):
    P, U0, bt, n, U = run_case(name)
    st, Uo, _ = restated.run(P.engine_desc(), U0, n, bnd=bt, src_time=source_time(P, n))
    assert st == abi.PD_OK
    assert np.array_equal(U, Uo)


def test_exact_tile_equals_shared_memory_kernel(tmp_path, gpu):
    """PD_EXACT_TILE=0 (read once per process) keeps every EXACT step on
    k_gaptooth_exact; both kernels must produce the same bits."""
    out = tmp_path / "smem.npz"
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import test_gpu_exact_tile as t
np.savez(%r, **{k: t.run_case(k)[4] for k in t.CASES})
print("ok")
""" % (str(ROOT), str(ROOT / "tests"), str(out))
    env = dict(os.environ, PD_EXACT_TILE="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
    ref = np.load(out)
    for name in CASES:
        assert np.array_equal(run_case(name)[4], ref[name]), name
