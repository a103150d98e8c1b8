"""Launch the register-blocked EXACT step (k_exact_tile) a few times for ncu (dev tool).
usage: kprof_exact.py [c4|c2]"""
import sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
which = sys.argv[1] if len(sys.argv) > 1 else 'c4'
d, _ = configs.load('c4_shear' if which == 'c4' else 'c2_cdr_tanh')
P = Problem(d)
E = Engine.from_problem(P, mode=1)
U0 = P.initial_field()
dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
ms = E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 3)
print(which, 'exact kernel ms', ms)
