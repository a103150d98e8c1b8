#!/bin/bash
# Round-2 measurement session: configs 1-3 bench lines, the config-5 sweep with
# per-row parity, the launch list of the default bench and one ncu --set full
# capture of the config-4 step kernel (source-level, for the ceiling analysis).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c1_diffusion c2_cdr_tanh c3_annulus; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
timeout 2400 python bench.py --sweep --tag r02 > gpurun_out/sweep_r02.log 2>&1; cp profiles/c5_sweep_r02.jsonl gpurun_out/ 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r02.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fast -c 1 -s 1 -o gpurun_out/prof_c4_r02 \
    python scripts/kprof.py c4 > gpurun_out/prof_c4_r02.log 2>&1
