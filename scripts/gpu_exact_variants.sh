#!/bin/bash
# A/B library variants lib/libpatchdyn_b200_<tag>.so on the EXACT step kernels: gpu_exact_variants.sh tagA tagB ...
cd "$(dirname "$0")/.."
for t in "$@"; do
  cp paper_2405_08764_b200/lib/libpatchdyn_b200_$t.so paper_2405_08764_b200/lib/libpatchdyn_b200.so
  echo "== $t $(python scripts/kprof_exact.py c4 2>&1 | tail -1) $(python scripts/kprof_exact.py c2 2>&1 | tail -1) $(python scripts/kprof_exact.py c1 2>&1 | tail -1)"
done
