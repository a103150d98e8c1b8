"""Generate the committed golden fixtures (run in the build container, where
/root/reference and oracle/_ref exist; the GPU box only reads the .npz files).

  python tests/golden/make_golden.py            (all fixtures)
  python tests/golden/make_golden.py linear     (ref_linear.npz only)
  python tests/golden/make_golden.py adi        (table1_cdr.npz, ref_adi.npz only)

ref_finals.npz      configs 1-3: initial field, first projective step and the
                    full-run final field computed by the UNMODIFIED reference
                    (oracle/_ref, cpi::run with linear_cache=off).
annulus_16x10.npz   the reference's shipped Table-4 outputs
                    (proj/out/table4/16x10/snapshots/*.snap, 17-digit text)
                    converted to arrays; produced by the reference's fast path.
c4_small.npz        config-4 equation on 32x32 patches, 100 macro steps, by the
                    restated oracle (reference + mixed term; the reference
                    itself rejects b != 0 — parity unpinned by the reference).
c4_sample.npz       full-size config 4: one gap-tooth substep on 1024 sampled
                    patches by the restated oracle.
c4_full.npz         full-size config 4 (512x512 patches of 16x16, K = 50): the
                    field after the first projective step and after the full
                    100-step run, by the restated oracle (OpenMP over patches,
                    bit-identical to one thread: patches are independent).
table1_cdr.npz      the reference's shipped Table-1 output (proj/out/table1/snapshots,
                    problem1_constant(0) with the ADI micro-solver) as arrays.
ref_adi.npz         ADI micro-solver variants (upwind two/three/four, Neumann/
                    Dirichlet/Robin patch conditions, k = 1, nx != ny) run by
                    the unmodified reference: 40 macro steps each.
ref_linear.npz      configs 1 and 3 with the reference's DEFAULT linear_cache=auto:
                    GapToothEngine::step takes the linear-response shortcut
                    (gaptooth.cpp:377-418); first projective step and final
                    field of the full run, by the unmodified reference.
ref_pulsed.npz      configs/pulsed_cdr.cfg (time-dependent coefficients + a general
                    source, k = 0 and k = 1): step_direct and 6 projective
                    steps by the UNMODIFIED reference (per-micro-step sampling
                    inside PatchIntegrator::integrate, microsim.cpp:537-542).
unit_cases.npz      PatchIntegrator::integrate / lift / restrict_average cases
                    run through the reference (known answers of
                    proj/tests/test_microsim.cpp and test_gaptooth.cpp).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import Reference, Restated  # noqa: E402
from paper_2405_08764_b200 import abi, configs  # noqa: E402
from paper_2405_08764_b200.engine import Problem  # noqa: E402

OUT = Path(__file__).resolve().parent
REF_OUT = Path("/root/reference/proj/out/table4/16x10")


def read_snap(p: Path):
    toks = p.read_text().split()
    assert toks[0] == "patchdyn-snapshot" and toks[1] == "1"
    t = float(toks[3])
    nxi, neta = int(toks[5]), int(toks[7])
    vals = np.array([float(x) for x in toks[8:]])
    return t, vals.reshape(nxi + 1, neta + 1)


def ref_finals(ref):
    out = {}
    for name in ["c1_diffusion", "c2_cdr_tanh", "c3_annulus"]:
        d, _ = configs.load(name)
        prob = Problem(d)
        R = ref.engine(prob.desc)
        U0 = R.initial_field()
        U1 = R.projective_step(U0, 0.0)
        st, UT, err, sec = R.run()
        assert st == 0
        out[f"{name}_U0"] = U0
        out[f"{name}_U1"] = U1
        out[f"{name}_final"] = UT
        out[f"{name}_maxpct"] = np.array(err)
        print(f"{name}: reference run {sec:.2f} s, max%err {err}")
    np.savez_compressed(OUT / "ref_finals.npz", **out)


def ref_linear(ref):
    out = {}
    for name in ["c1_diffusion", "c3_annulus"]:
        d, _ = configs.load(name)
        prob = Problem(d)
        R = ref.engine(prob.desc, linear_cache="auto")
        U0 = R.initial_field()
        out[f"{name}_U1"] = R.projective_step(U0, 0.0)
        st, UT, err, sec = R.run()
        assert st == 0
        out[f"{name}_final"] = UT
        out[f"{name}_maxpct"] = np.array(err)
        print(f"{name}: reference linear-cache run {sec:.3f} s")
    np.savez_compressed(OUT / "ref_linear.npz", **out)


ADI_CASES = {
    # name: config overrides of configs/ref_table1_cdr_const.cfg
    "const_two": {},
    "const_l03_three": {"lambda_": 0.3, "upwind_order": 1},
    "var_l03_four": {"problem": 13, "lambda_": 0.3, "upwind_order": 2, "upwind_r": 0.3},
    "var_dirichlet_two": {"problem": 13, "bc_type": 1},
    "const_robin_three": {"bc_type": 2, "robin_w1": 2.0, "robin_w2": 1.0, "upwind_order": 1},
    "var_k1_two": {"problem": 13, "k": 1},
    "const_nx10_ny14_two": {"ny": 14, "lambda_": 0.2},
}
ADI_STEPS = 40


def table1():
    arrs = {}
    for p in sorted(Path("/root/reference/proj/out/table1/snapshots").glob("t_*.snap")):
        t, U = read_snap(p)
        arrs[f"t_{t:.6f}"] = U
    np.savez_compressed(OUT / "table1_cdr.npz", **arrs)
    print("table1 snapshots:", list(arrs))


def ref_adi(ref):
    base, _ = configs.load("ref_table1_cdr_const")
    out = {}
    for name, over in ADI_CASES.items():
        prob = Problem(configs.copy_desc(base, **over))
        R = ref.engine(prob.desc)
        U0 = R.initial_field()
        U, sec = R.steps(U0, 0, ADI_STEPS)
        out[f"{name}_U0"] = U0
        out[f"{name}_final"] = U
        print(f"adi {name}: {sec * 1e3:.1f} ms")
    np.savez_compressed(OUT / "ref_adi.npz", **out)


def annulus():
    snaps = sorted(REF_OUT.glob("snapshots/t_*.snap"))
    arrs = {}
    for p in snaps:
        t, U = read_snap(p)
        arrs[f"t_{t:.2f}"] = U
    np.savez_compressed(OUT / "annulus_16x10.npz", **arrs)
    print("annulus snapshots:", list(arrs))


def c4(O):
    d, _ = configs.load("c4_shear")
    ds = configs.copy_desc(d, N_xi=33, N_eta=33)
    prob = Problem(ds)
    ed = prob.engine_desc()
    U0 = prob.initial_field()
    st, UT, stats = O.run(ed, U0, 100)
    assert st == 0
    np.savez_compressed(OUT / "c4_small.npz", U0=U0, final=UT, tau=prob.desc.tau, T=prob.desc.T)
    print("c4 small oracle run done", stats.device_ms, "ms")
    prob = Problem(d)
    ed = prob.engine_desc()
    U0 = prob.initial_field()
    rng = np.random.default_rng(2024)
    idx = np.sort(rng.choice(ed.npatches, 1024, replace=False)).astype(np.int32)
    avg, sec = O.patch_subset(ed, U0, 0.0, idx)
    pij = np.ctypeslib.as_array(ed.patch_ij, shape=(ed.npatches, 2))[idx].copy()
    np.savez_compressed(OUT / "c4_sample.npz", idx=idx, pij=pij, avg=avg, U0_sum=U0.sum(), tau=prob.desc.tau)
    print(f"c4 sample: {sec:.2f} s")


def c4_full(O):
    """BASELINE config 4 at its stated size, the whole cpi::run (cpi.cpp:134-216)."""
    import time
    d, _ = configs.load("c4_shear")
    prob = Problem(d)
    ed = prob.engine_desc()
    U0 = prob.initial_field()
    t0 = time.perf_counter()
    st, U1 = O.projective_step(ed, U0, 0.0)
    assert st == 0
    st, UT, stats = O.run(ed, U0, prob.desc.Nt)
    assert st == 0 and stats.steps_done == prob.desc.Nt, (st, stats.steps_done)
    np.savez_compressed(OUT / "c4_full.npz", U1=U1, final=UT, nsteps=prob.desc.Nt, tau=prob.desc.tau,
                        T=prob.desc.T, U0_sum=U0.sum(), umax_last=np.array(stats.umax_last))
    print(f"c4 full oracle run: {prob.desc.Nt} steps, {time.perf_counter() - t0:.1f} s, {O.threads} threads")


def ref_pulsed(ref):
    out = {}
    for k in (0, 1):
        d, _ = configs.load("pulsed_cdr")
        prob = Problem(configs.copy_desc(d, k=k))
        R = ref.engine(prob.desc)
        U0 = R.initial_field()
        dt = prob.desc.T / prob.desc.Nt
        out[f"k{k}_U0"] = U0
        out[f"k{k}_S1"] = R.step_direct(U0, 0.0)
        U = U0
        for n in range(6):
            U = R.projective_step(U, n * dt)
            out[f"k{k}_U{n + 1}"] = U
    np.savez_compressed(OUT / "ref_pulsed.npz", **out)
    print("ref_pulsed:", len(out), "arrays")


def unit_cases(ref):
    """Integrate / lift / restrict through the reference (fixtures for the GPU box)."""
    rng = np.random.default_rng(99)
    cases = {}
    # (A, C, Vx, Vy, W), (nx, ny, nt), (h_xi, h_eta, tau), kinds (E, W, N, S), robin w
    specs = [
        ((1.0, 0.5, 3.0, -2.0, 0.0), (6, 8, 3), (0.01, 0.02, 1e-6), (1, 1, 1, 1), (0,) * 8),
        ((1.0, 1.0, 2.0, 0.0, 0.0), (10, 6, 40), (0.05, 0.05, 2e-5), (0, 0, 1, 1), (0,) * 8),
        ((1.0, 1.0, 0.0, 0.0, 0.0), (8, 8, 80), (0.1, 0.1, 1e-3), (0, 0, 0, 0), (0,) * 8),
        ((1.0, 1.0, 0.0, 0.0, 0.3), (6, 6, 10), (0.1, 0.1, 1e-4), (2, 2, 2, 2), (2.0, 1.0) * 4),
        ((0.7, 1.3, -4.0, 5.0, 1.0), (9, 7, 25), (0.04, 0.03, 2e-5), (1, 0, 2, 1), (0, 0, 0, 0, 1.5, 0.5, 0, 0)),
    ]
    for c, ((A, Cc, Vx, Vy, W), (nx, ny, nt), (hx, hy, tau), kinds, rw) in enumerate(specs):
        n1, n2 = nx + 1, ny + 1
        L = max(n1, n2)
        u0 = rng.uniform(-1, 2, (n1, n2))
        vals = rng.uniform(-1, 1, (4, L))
        slopes = rng.uniform(-1, 1, (4, L))
        st, uT = ref.integrate((A, Cc, Vx, Vy, W), nx, ny, nt, hx, hy, tau, 0.5, 0.5, kinds, vals, slopes, rw, u0)
        assert st == 0, ref.error()
        cases[f"int{c}_params"] = np.array([A, Cc, Vx, Vy, W, nx, ny, nt, hx, hy, tau], dtype=np.float64)
        cases[f"int{c}_kinds"] = np.array(kinds, dtype=np.int32)
        cases[f"int{c}_robin"] = np.array(rw, dtype=np.float64)
        cases[f"int{c}_u0"], cases[f"int{c}_vals"], cases[f"int{c}_slopes"] = u0, vals, slopes
        cases[f"int{c}_uT"] = uT
    # lifting chain on random stencils
    for c, (nx, ny) in enumerate([(6, 8), (10, 10), (15, 15)]):
        vals = rng.uniform(-1, 1, 9)
        st, u0, sl, va = ref.lift(vals, 0.3, 0.55, 0.1, 0.05, 0.02, 0.01, nx, ny)
        cases[f"lift{c}_in"] = np.array([nx, ny], dtype=np.float64)
        cases[f"lift{c}_vals"], cases[f"lift{c}_u0"], cases[f"lift{c}_slopes"], cases[f"lift{c}_values"] = vals, u0, sl, va
    np.savez_compressed(OUT / "unit_cases.npz", **cases)
    print("unit cases:", len(specs), "integrate, 3 lift")


if __name__ == "__main__":
    ref = Reference()
    O = Restated()
    if sys.argv[1:] == ["linear"]:
        ref_linear(ref)
        sys.exit(0)
    if sys.argv[1:] == ["pulsed"]:
        ref_pulsed(ref)
        sys.exit(0)
    if sys.argv[1:] == ["c4full"]:
        c4_full(O)
        sys.exit(0)
    if sys.argv[1:] == ["adi"]:
        table1()
        ref_adi(ref)
        sys.exit(0)
    ref_finals(ref)
    ref_linear(ref)
    table1()
    ref_adi(ref)
    annulus()
    c4(O)
    c4_full(O)
    ref_pulsed(ref)
    unit_cases(ref)
