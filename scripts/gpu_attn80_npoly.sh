#!/bin/bash
# hd-80 attention: production (NPOLY 0) vs polynomial-exponential shares 2 / 4 / 6 of 16
# (hook-free variants 3 / 4 / 5), alternating processes, two rounds.
mkdir -p gpurun_out
for r in 1 2; do for v in 0 3 4 5; do
  echo "== round $r variant $v"; DART_FA_VARIANT=$v timeout 300 python scripts/bench_attn.py 2>&1 | grep -E "FAIL|bb |rror|hd=80"
done; done > gpurun_out/attn80_npoly.log 2>&1
cat gpurun_out/attn80_npoly.log
