#!/bin/bash
# A/B of a K3 build variant against the release library on config 5 (same box, alternating)
V=${1:-libhetserve_b200_c5}
for i in 1 2; do
  for L in libhetserve_b200 $V; do
    echo -n "$L: "; HS_LIB=$PWD/paper_2504_15303_b200/$L.so python tools/profile_kernels.py config5 1024 100000 | tail -1
  done
done
