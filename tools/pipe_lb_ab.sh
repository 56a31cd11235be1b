#!/bin/bash
# A/B of the PIPE instantiation's launch bounds (release: 4 blocks/SM = 128 registers)
V=${1:-libhetserve_b200_p2}
for T in 148 512 1024; do
  for i in 1 2; do
    for L in libhetserve_b200 $V; do
      echo -n "T=$T $L: "; HS_LIB=$PWD/paper_2504_15303_b200/$L.so python tools/profile_kernels.py replay $T 100000 2 | head -1
    done
  done
done
