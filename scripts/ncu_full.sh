#!/bin/bash
# ncu --set full of the hot kernels at their DART shapes (one profiled launch each).
mkdir -p gpurun_out
tag=${1:-r01}
shift
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/full_${tag} -f python scripts/ncu_targets.py "$@" > gpurun_out/ncu_full_${tag}.log 2>&1
ncu -i gpurun_out/full_${tag}.ncu-rep --page raw --csv > gpurun_out/full_${tag}_raw.csv 2>/dev/null
tail -3 gpurun_out/ncu_full_${tag}.log
