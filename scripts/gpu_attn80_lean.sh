#!/bin/bash
# hd-80 attention: production commit-per-tile protocol (variant 0) vs the lean protocol hook-free (variant 3)
for r in 1 2 3; do for v in 0 3; do
  echo "== round $r variant $v"; DART_FA_VARIANT=$v timeout 300 python scripts/bench_attn.py 2>&1 | grep -E "FAIL|bb |rror|hd=80"
done; done 2>&1 | tee gpurun_out/attn80_lean.log
