"""Kernel-only timings on the config-4 shape (dev tool for A/B of library builds)."""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
d, _ = configs.load('c4_shear')
out = []
for K in (50, 200):
    P = Problem(configs.copy_desc(d, nt=K))
    E = Engine.from_problem(P)
    dU = torch.from_numpy(P.initial_field().ravel()).cuda(); dS = torch.empty_like(dU)
    ms = min(E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 5) for _ in range(3))
    out.append(f"K={K} {ms:.4f} ms")
print(' | '.join(out), flush=True)
