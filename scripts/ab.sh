#!/bin/bash
# A/B the kernel-only timings of alternative builds of the library: ab.sh tagA tagB ...
cd /root/repo
for t in "$@"; do
  cp paper_2405_08764_b200/lib/libpatchdyn_b200_$t.so paper_2405_08764_b200/lib/libpatchdyn_b200.so
  echo "== $t"; VARIANTS=1 python scripts/kbench.py 2>&1 | grep -E "v1"
done
