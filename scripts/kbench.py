"""Kernel-only timing of the fused step on config-4/5 shapes (dev tool)."""
import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
from paper_2405_08764_b200 import configs, abi
from paper_2405_08764_b200.engine import Problem, Engine, fp64_peak

p64, ghz = fp64_peak(200)
print(f"fp64 peak {p64:.2f} TF at {ghz:.3f} GHz", flush=True)
d, _ = configs.load('c4_shear')
cases = [('c4', d)]
for nodes, K, lp in [(16, 50, 18), (16, 10, 18), (16, 200, 16), (8, 50, 20), (8, 10, 20), (8, 200, 18)]:
    cases.append((f"c5 2^{lp} {nodes}^2 K={K}", configs.sweep_desc(d, lp, nodes, K)))
for name, dd in cases:
    if len(sys.argv) > 1 and sys.argv[1] not in name:
        continue
    t = time.time(); P = Problem(dd); tb = time.time() - t
    U0 = P.initial_field()
    dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
    import os
    for var in os.environ.get('VARIANTS', '0').split(','):
      os.environ['PD_FAST_VARIANT'] = var
      E = Engine.from_problem(P)
      ms = E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 5)
      name2 = name + ' v' + var
      ed = P.engine_desc()
      N = (dd.nx + 1) * (dd.ny + 1)
      upd = ed.npatches * N * dd.nt
      tf = upd * 14 / (ms * 1e-3) / 1e12
      byt = ed.npatches * (N * 48 + 16)
      print(f"{name2:28s} mode={E.mode} P={ed.npatches} build={tb:.1f}s kernel {ms:.3f} ms  {upd/ms/1e9:.3f}e12 upd/s  "
          f"{tf:.2f} TF ({tf/p64*100:.1f}% fp64)  {byt/ms/1e6:.0f} GB/s ({byt/ms/1e6/6548.8*100:.1f}% hbm)", flush=True)
      del E
    del P
