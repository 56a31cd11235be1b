#!/bin/bash
# Same-box A/B of K3 build variants: config 4 at the bench size and config 5
for i in 1 2; do
  for L in "$@"; do
    echo -n "c4 $L: "; HS_LIB=$PWD/paper_2504_15303_b200/$L.so python tools/profile_kernels.py replay 4096 100000 2 | head -1
  done
done
for i in 1 2; do
  for L in "$@"; do
    echo -n "c5 $L: "; HS_LIB=$PWD/paper_2504_15303_b200/$L.so python tools/profile_kernels.py config5 1024 100000 | tail -1
  done
done
