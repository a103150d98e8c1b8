#!/bin/bash
# FAST 11x11 patches (the reference's default micro grid): exact-fit 1x11 tile vs the padded 16x16 tile
cd "$(dirname "$0")/.."
python - <<'PY'
import sys, os, subprocess
code = r"""
import sys; sys.path.insert(0, '.')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
base, _ = configs.load('c5_sweep')
for lg, K in ((16, 50), (18, 10), (12, 50)):
    P = Problem(configs.copy_desc(configs.sweep_desc(base, lg, 16, K), nx=10, ny=10))
    E = Engine.from_problem(P)
    U0 = P.initial_field()
    dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
    print('11x11 mixed 2^%d K=%d mode' % (lg, K), E.mode, 'kernel ms', E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 5))
d, _ = configs.load('c1_diffusion')
P = Problem(configs.copy_desc(d, nx=10, ny=10, N_xi=129, N_eta=129))
E = Engine.from_problem(P)
U0 = P.initial_field()
dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
print('11x11 5-point 128^2 patches K=20 kernel ms', E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 5))
U, st = E.run(U0, 50)
print('run 50 steps ms/step', st.device_ms / 50, 'launches', st.kernel_launches)
"""
for v in ("1", "0"):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PD_FAST_TILE11=v), capture_output=True, text=True)
    print('PD_FAST_TILE11=' + v); print(r.stdout.strip() or r.stderr[-600:])
PY
