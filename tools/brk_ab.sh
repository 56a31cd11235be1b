#!/bin/bash
# A/B of a K3 build variant against the release library (same box, alternating)
V=${1:-libhetserve_b200_brk}
for T in 4096 148 1184; do
  for i in 1 2; do
    for L in libhetserve_b200 $V; do
      echo -n "T=$T $L: "; HS_LIB=$PWD/paper_2504_15303_b200/$L.so python tools/profile_kernels.py replay $T 100000 2 | head -1
    done
  done
done
