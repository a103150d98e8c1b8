#!/bin/bash
# One GPU session: the -m gpu suite, smoke(), the default bench line, the
# reference arm, and the configs 1-3 lines of both arms (outputs under gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt
timeout 2700 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
for c in c1_diffusion c2_cdr_tanh c3_annulus; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 5 > gpurun_out/bench_$c.log 2>&1
  timeout 600 python bench.py --config $c --impl reference --steps 200 --warmup 5 > gpurun_out/bench_ref_$c.log 2>&1
done
