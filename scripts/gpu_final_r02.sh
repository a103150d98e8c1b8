#!/bin/bash
# Final measurement session of the round-2 build: the default bench line, the reference arm,
# configs 1-3 (FAST), the EXACT lines, and the launch list of the default bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench_line.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_reference_line.json 2> gpurun_out/final_ref.err
for c in c1_diffusion c2_cdr_tanh c3_annulus; do
  python bench.py --config $c --steps 200 --warmup 5 2>/dev/null | tail -1 > gpurun_out/final_bench_$c.json
done
scripts/gpu_exact_measure.sh > gpurun_out/final_exact.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1
tail -c 400 gpurun_out/final_bench_line.json; echo; cat gpurun_out/final_exact.log | tail -9
