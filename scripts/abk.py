"""Kernel-only timings for A/B of library builds (dev tool).
usage: abk.py [c4|big|c8] [K1,K2,...]   c4: config-4 shape at K=50/200; big: 32x32 nodes, 2^16 patches, K=50/200"""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
which = sys.argv[1] if len(sys.argv) > 1 else 'c4'
d, _ = configs.load('c4_shear')
out = []
Ks = tuple(int(x) for x in sys.argv[2].split(',')) if len(sys.argv) > 2 else ((10, 50) if which == 'c8' else (50, 200))
for K in Ks:
    dd = (configs.copy_desc(d, nt=K) if which == 'c4' else configs.sweep_desc(d, 16, 32, K) if which == 'big'
          else configs.sweep_desc(d, 18, 8, K))
    P = Problem(dd)
    E = Engine.from_problem(P)
    dU = torch.from_numpy(P.initial_field().ravel()).cuda(); dS = torch.empty_like(dU)
    ms = min(E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 5) for _ in range(3))
    out.append(f"K={K} {ms:.4f} ms")
print(which, ' | '.join(out), flush=True)
