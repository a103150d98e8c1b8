#!/bin/bash
# A/B of library builds (kernel-only timings, scripts/abk.py), then the -m gpu
# suite on the first tag's build.  usage: gpu_ab.sh <c4|big|c8> tagNew tagOld [pytest -k expr]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
w=$1; a=$2; b=$3
bash scripts/ab.sh $w $a $b $a $b > gpurun_out/ab_$w.log 2>&1
cp paper_2405_08764_b200/lib/libpatchdyn_b200_$a.so paper_2405_08764_b200/lib/libpatchdyn_b200.so
timeout 1800 python -m pytest tests -m gpu -x -q ${4:+-k "$4"} > gpurun_out/test_$a.log 2>&1; echo "rc=$?" >> gpurun_out/test_$a.log
