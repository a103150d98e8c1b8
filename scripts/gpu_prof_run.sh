#!/bin/bash
# ncu source-level capture of the single-launch run kernel on config 2 (latency-bound configs 1-3)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/kprof_run.py c2_cdr_tanh 200 > gpurun_out/kprof_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fast_run -c 1 -o gpurun_out/prof_run_c2_r02 \
    python scripts/kprof_run.py c2_cdr_tanh 200 > gpurun_out/prof_run_c2_r02.log 2>&1
