#!/bin/bash
# A/B of the 32x32 kernel's neighbour hand-off: CTA barrier (bar) vs release/acquire flags (flg);
# then the gpu suite on the flags build, and the config-4 full-run parity numbers
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/ab.sh big bar flg bar flg > gpurun_out/ab_big.log 2>&1
cp paper_2405_08764_b200/lib/libpatchdyn_b200_flg.so paper_2405_08764_b200/lib/libpatchdyn_b200.so
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/test_flg.log 2>&1; echo "rc=$?" >> gpurun_out/test_flg.log
timeout 900 python scripts/c4_full_parity.py > gpurun_out/c4_full_parity.log 2>&1
