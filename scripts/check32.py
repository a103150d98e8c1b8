"""32x32 FAST kernel: parity vs EXACT/oracle and kernel timings (dev)."""
import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2405_08764_b200 import configs, abi
from paper_2405_08764_b200.engine import Problem, Engine
from oracle.pyoracle import Restated
O = Restated()
d, _ = configs.load('c4_shear')
for K in (10, 50):
    dd = configs.sweep_desc(d, 8, 32, K, jacobi_sweeps=0)   # 256 patches of 32x32
    P = Problem(dd); ed = P.engine_desc(); U0 = P.initial_field()
    F = Engine.from_problem(P, mode=abi.PD_MODE_FAST); X = Engine.from_problem(P, mode=abi.PD_MODE_EXACT)
    a = F.projective_step(U0, 0.0); b = X.projective_step(U0, 0.0); _, o = O.projective_step(ed, U0, 0.0)
    s = np.abs(o).max()
    print(f"K={K} fast mode={F.mode} rel(fast,oracle)={np.abs(a-o).max()/s:.2e} exact==oracle {np.array_equal(b,o)}", flush=True)
    ua, _ = F.run(U0, 10); _, uo, _ = O.run(ed, U0, 10)
    print(f"   10 steps rel {np.abs(ua-uo).max()/np.abs(uo).max():.2e}", flush=True)
for lp, K in ((16, 50), (18, 10), (16, 200), (14, 200)):
    dd = configs.sweep_desc(d, lp, 32, K, jacobi_sweeps=0)
    P = Problem(dd); E = Engine.from_problem(P); U0 = P.initial_field()
    dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
    ms = E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 3)
    upd = P.engine_desc().npatches * 1024 * K
    print(f"2^{lp} 32^2 K={K}: mode={E.mode} {ms:.3f} ms {upd/ms/1e9:.3f}e12 upd/s {upd*14/ms/1e9/37.0*100:.1f}% fp64 "
          f"{P.engine_desc().npatches*(1024*48+16)/ms/1e6/6548.8*100:.1f}% hbm", flush=True)
