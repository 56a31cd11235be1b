for T in 148 592 1184 2048; do
  for v in 0 1 0 1; do
    echo -n "T=$T PIPE=$v: "; HS_REPLAY_PIPE=$v python tools/profile_kernels.py replay $T 100000 2 | head -1
  done
done
