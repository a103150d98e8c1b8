#!/bin/bash
# configs 1-3 bench lines (both arms) + the reference-side binding tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_binding.py -q > gpurun_out/binding.log 2>&1; echo "rc=$?" >> gpurun_out/binding.log
for c in c1_diffusion c2_cdr_tanh c3_annulus; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 5 > gpurun_out/bench_$c.log 2>&1
  timeout 600 python bench.py --config $c --impl reference --steps 200 --warmup 5 > gpurun_out/bench_ref_$c.log 2>&1
done
