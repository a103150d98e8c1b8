#!/bin/bash
# EXACT-mode timings of the four BASELINE configs (bench.py --mode exact), one line each
for c in c4_shear c1_diffusion c2_cdr_tanh c3_annulus; do
  st=200; [ $c = c4_shear ] && st=5
  python bench.py --mode exact --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'ms_per_step', round(d['ms_per_step'],5), 'updates/s %.4g' % d['value'], 'kernel_ms', round(d['roofline']['kernel_ms'],5), 'frac', round(d['roofline']['frac'],4))"
done
# 32x32 patches (config-5 shape, 2^14 patches, K = 50): tile vs shared-memory kernel, one step kernel
python - <<'PY'
import sys, os, subprocess
code = r"""
import sys; sys.path.insert(0, '.')
import torch
from paper_2405_08764_b200 import configs
from paper_2405_08764_b200.engine import Problem, Engine
base, _ = configs.load('c5_sweep')
P = Problem(configs.sweep_desc(base, 14, 32, 50))
E = Engine.from_problem(P, mode=1)
U0 = P.initial_field()
dU = torch.from_numpy(U0.ravel()).cuda(); dS = torch.empty_like(dU)
print('32x32 2^14 K=50 exact_tile', E.exact_tile, 'kernel ms', E.bench_step_kernel(dU.data_ptr(), dS.data_ptr(), 3))
"""
code11 = code.replace("configs.sweep_desc(base, 14, 32, 50)", "configs.copy_desc(configs.sweep_desc(base, 16, 16, 50), nx=10, ny=10)").replace("32x32 2^14", "11x11 2^16")
for v in ("1", "0"):
    r = subprocess.run([sys.executable, "-c", code11], env=dict(os.environ, PD_EXACT_TILE=v), capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-400:])
for v in ("1", "0"):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PD_EXACT_TILE=v), capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-400:])
PY
