"""Dev check on a B200: EXACT/FAST engines vs the CPU oracle and the reference."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2405_08764_b200 import configs, abi
from paper_2405_08764_b200.engine import Problem, Engine
from oracle.pyoracle import Restated, Reference, reference_available

O = Restated()
R = Reference() if reference_available() else None

def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

for name in ['c1_diffusion', 'c2_cdr_tanh', 'c3_annulus']:
    d, _ = configs.load(name)
    P = Problem(d)
    ed = P.engine_desc()
    U0 = P.initial_field()
    Nt = P.desc.Nt
    bt = P.boundary_table(0.0, Nt)
    t = time.time(); st, Uo, sto = O.run(ed, U0, Nt, bnd=bt); to = time.time() - t
    for mode in (abi.PD_MODE_EXACT, abi.PD_MODE_FAST):
        E = Engine.from_problem(P, mode=mode)
        U1 = E.projective_step(U0, 0.0, bnd=bt[0])
        _, U1o = O.projective_step(ed, U0, 0.0, bnd=bt[0])
        Ug, stats = E.run(U0, Nt, bnd=bt)
        print(f"{name} mode={E.mode} step1 rel={rel(U1,U1o):.3e} eq={np.array_equal(U1,U1o)} run rel={rel(Ug,Uo):.3e} "
              f"eq={np.array_equal(Ug,Uo)} dev_ms={stats.device_ms:.2f} launches={stats.kernel_launches} oracle_s={to:.2f}",
              flush=True)
    if R is not None:
        RE = R.engine(P.desc)
        rr, Ur, err, sec = RE.run()
        print(f"   reference run {sec:.2f}s oracle==ref {np.array_equal(Uo, Ur)} rel {rel(Uo,Ur):.2e}", flush=True)

# config 4 shape at reduced size, then full size timing
d, _ = configs.load('c4_shear')
for N in (33, 513):
    dd = configs.copy_desc(d, N_xi=N, N_eta=N)
    t = time.time(); P = Problem(dd); tb = time.time() - t
    ed = P.engine_desc()
    U0 = P.initial_field()
    for mode in (abi.PD_MODE_EXACT, abi.PD_MODE_FAST):
        if N > 100 and mode == abi.PD_MODE_EXACT:
            continue
        t = time.time(); E = Engine.from_problem(P, mode=mode); te = time.time() - t
        U1 = E.projective_step(U0, 0.0)
        if N <= 100:
            _, U1o = O.projective_step(ed, U0, 0.0)
            print(f"c4 N={N} mode={E.mode} step1 rel={rel(U1,U1o):.3e}", flush=True)
            Ug, stats = E.run(U0, 20)
            _, Uo, _ = O.run(ed, U0, 20)
            print(f"   20 steps rel={rel(Ug,Uo):.3e} dev_ms={stats.device_ms:.2f}", flush=True)
        else:
            Ug, stats = E.run(U0, 5)
            upd = ed.npatches * 256 * 50 * 5
            print(f"c4 full mode={E.mode} build={tb:.1f}s create={te:.1f}s 5 steps {stats.device_ms:.2f} ms "
                  f"-> {upd/stats.device_ms*1e3:.3e} upd/s  ({stats.device_ms/5:.3f} ms/step)", flush=True)
            # oracle on a sample of patches for the first gap-tooth substep
            idx = np.random.default_rng(0).choice(ed.npatches, 512, replace=False).astype(np.int32)
            avg, sec = O.patch_subset(ed, U0, 0.0, idx)
            U1g = E.step_direct(U0, 0.0)
            pij = np.ctypeslib.as_array(ed.patch_ij, shape=(ed.npatches, 2))[idx]
            g = U1g[pij[:, 0], pij[:, 1]]
            print(f"   sampled substep rel={rel(g, avg):.3e} oracle {len(idx)} patches {sec:.2f}s", flush=True)
