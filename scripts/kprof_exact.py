"""Launch the register-blocked EXACT step (k_exact_tile) a few times for ncu (dev tool).
usage: kprof_exact.py [c4|c2|big|x11|f11]  (big: 2^14 patches of 32x32, K = 50, k_exact_big; x11 / f11: 2^16 patches of
11x11, K = 50, EXACT tile / FAST exact-fit tile)"""
import sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
which = sys.argv[1] if len(sys.argv) > 1 else 'c4'
if which in ('big', 'x11', 'f11'):
    base, _ = configs.load('c5_sweep')
    d = configs.sweep_desc(base, 14, 32, 50) if which == 'big' else configs.copy_desc(configs.sweep_desc(base, 16, 16, 50), nx=10, ny=10)
else:
    d, _ = configs.load({'c4': 'c4_shear', 'c1': 'c1_diffusion', 'c3': 'c3_annulus'}.get(which, 'c2_cdr_tanh'))
P = Problem(d)
E = Engine.from_problem(P, mode=0 if which == 'f11' else 1)
U0 = P.initial_field()
dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
ms = E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 3)
print(which, 'kernel ms', ms, 'mode', E.mode)
