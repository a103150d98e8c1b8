#!/bin/bash
# One GPU session: the -m gpu suite, the default bench line and the reference arm
# (outputs under gpurun_out/, merged back by gpurun).  usage: gpu_round.sh [pytest -k expr]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
K=${1:+-k "$1"}
timeout 2400 python -m pytest tests -m gpu -x -q $K > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
