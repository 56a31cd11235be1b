#!/bin/bash
# Round-2 measurement captures on one B200 (run through gpurun from the repo root):
#   A/B of the monotone pure-block test, ncu --set full of K3 at the bench size and
#   of the config-5 replay, written under gpurun_out/.
set -x
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export HS_REPLAY_NO_MONO=1; else unset HS_REPLAY_NO_MONO; fi
  python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-config5 > gpurun_out/ab_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('NO_MONO=$v k3', d['breakdown']['k3_replay_ms'])"
done
unset HS_REPLAY_NO_MONO
ncu --set full --import-source on --clock-control none -k regex:k_replay -c 1 -o gpurun_out/k3bench \
  python tools/profile_kernels.py replay 4096 100000 1 > gpurun_out/ncu_k3bench.log 2>&1
tail -2 gpurun_out/ncu_k3bench.log
ncu --set full --clock-control none -k regex:k_replay -c 1 -o gpurun_out/k3c5 \
  python tools/profile_kernels.py config5 1024 100000 > gpurun_out/ncu_k3c5.log 2>&1
tail -2 gpurun_out/ncu_k3c5.log
