#!/bin/bash
# Measurement session of the EXACT family (register-blocked k_exact_tile): bench lines of the four
# BASELINE configs in EXACT mode and one ncu --set full capture of the config-4 step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c4_shear c1_diffusion c2_cdr_tanh c3_annulus; do
  st=200; [ $c = c4_shear ] && st=20
  python bench.py --mode exact --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_exact_$c.json
  PD_EXACT_TILE=0 python bench.py --mode exact --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_exact_smem_$c.json
done
python scripts/kprof_exact.py c4 > gpurun_out/kprof_exact.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_exact_tile -c 1 -o gpurun_out/prof_exact_tile_c4 \
    python scripts/kprof_exact.py c4 > gpurun_out/prof_exact_tile_c4.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_exact_*.json')):
    d=json.loads(open(f).read())
    print(f.split('/')[-1], round(d['ms_per_step'],5), '%.4g'%d['value'], d['roofline']['kernel'], round(d['roofline']['frac'],4))
PY
