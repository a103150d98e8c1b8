"""Launch the fused step kernel a few times for ncu (dev tool).  usage: kprof.py [c4|k200|k10]"""
import sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
d, _ = configs.load('c4_shear')
which = sys.argv[1] if len(sys.argv) > 1 else 'c4'
if which == 'k200':
    d = configs.sweep_desc(d, 16, 16, 200)
elif which == 'c4k200':
    d = configs.copy_desc(d, nt=200)
elif which == 'big':
    d = configs.sweep_desc(d, 16, 32, 200)
elif which == 'k1':
    d = configs.copy_desc(d, nt=1)
elif which == 'k10':
    d = configs.sweep_desc(d, 18, 16, 10)
P = Problem(configs.copy_desc(d, N_xi=129, N_eta=129) if which == 'c4exact' else d)
E = Engine.from_problem(P, mode=1 if which == 'c4exact' else None)
U0 = P.initial_field()
dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
ms = E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 3)
print(which, 'kernel ms', ms)
