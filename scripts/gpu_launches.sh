#!/bin/bash
# Warm-cache launch lists (ncu, serialised) of one detection step at N=4 and N=80.
mkdir -p gpurun_out
tag=${1:-r02}
for n in 4 80; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    --csv --log-file gpurun_out/launches_n${n}_${tag}.csv python scripts/profile_step.py --classes $n > gpurun_out/prof_n${n}_${tag}.log 2>&1
  python scripts/summarize_launches.py gpurun_out/launches_n${n}_${tag}.csv > gpurun_out/launches_n${n}_${tag}.txt 2>&1
done
head -14 gpurun_out/launches_n4_${tag}.txt gpurun_out/launches_n80_${tag}.txt
