"""Fixed vs per-micro-step cost of the fused kernel on the config-4 shape (dev tool)."""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
d, _ = configs.load('c4_shear')
res = []
for K in (1, 2, 5, 10, 25, 50):
    P = Problem(configs.copy_desc(d, nt=K))
    E = Engine.from_problem(P)
    U0 = P.initial_field()
    dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
    ms = E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 5)
    res.append((K, ms)); print(f"K={K:3d} kernel {ms:.4f} ms", flush=True)
import numpy as np
A = np.array([[1, k] for k, _ in res]); b = np.array([m for _, m in res])
c, *_ = np.linalg.lstsq(A, b, rcond=None)
print(f"fit: fixed {c[0]:.4f} ms + {c[1]*1e3:.2f} us per micro-step")
