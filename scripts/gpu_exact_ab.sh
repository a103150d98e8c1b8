#!/bin/bash
# EXACT-mode timings of the four BASELINE configs (bench.py --mode exact), one line each
for c in c4_shear c1_diffusion c2_cdr_tanh c3_annulus; do
  st=200; [ $c = c4_shear ] && st=5
  python bench.py --mode exact --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'ms_per_step', round(d['ms_per_step'],5), 'updates/s %.4g' % d['value'], 'kernel_ms', round(d['roofline']['kernel_ms'],5), 'frac', round(d['roofline']['frac'],4))"
done
