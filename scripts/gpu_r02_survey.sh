#!/bin/bash
# Round-2 survey: hd-80 attention NPOLY variants, warm- and cold-cache launch lists of one step.
mkdir -p gpurun_out
for v in 0 5 6 7; do DART_FA_VARIANT=$v timeout 300 python scripts/bench_attn.py >> gpurun_out/attn_variants.log 2>&1; done
for n in 4 80; do
  for cc in none all; do
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control $cc \
      --csv --log-file gpurun_out/launches_n${n}_${cc}.csv python scripts/profile_step.py --classes $n > gpurun_out/prof_n${n}_${cc}.log 2>&1
    python scripts/summarize_launches.py gpurun_out/launches_n${n}_${cc}.csv > gpurun_out/launches_n${n}_${cc}.txt 2>&1
  done
done
grep "var" gpurun_out/attn_variants.log | grep -v check
