#!/bin/bash
# A/B the kernel-only timings of alternative library builds: ab.sh <c4|big> tagA tagB ...
# (build each with `make NVEXTRA=... && cp lib/libpatchdyn_b200.so lib/libpatchdyn_b200_<tag>.so`)
cd "$(dirname "$0")/.."
w=$1; shift
for t in "$@"; do
  cp paper_2405_08764_b200/lib/libpatchdyn_b200_$t.so paper_2405_08764_b200/lib/libpatchdyn_b200.so
  if [ "$w" = run ]; then echo "== $t $(python scripts/ab_run.py 2>&1 | tail -1)"; else echo "== $t $(python scripts/abk.py $w 2>&1 | tail -1)"; fi
done
