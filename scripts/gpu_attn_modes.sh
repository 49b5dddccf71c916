#!/bin/bash
# tcgen05 attention decomposition: full kernel (hooked twin, mode 0 via DART_FA_SOFTMAX_ONLY unset = production),
# softmax alone (1), MMA/TMA pipeline alone (2), hook-carrying twin with no mode (3 if defined)
for r in 1 2; do for m in 0 1 2; do
  echo "== DART_FA_SOFTMAX_ONLY=$m"
  DART_FA_SOFTMAX_ONLY=$m timeout 120 python scripts/bench_attn.py 2>&1 | grep -E "enc self|global|windowed"
done; done 2>&1 | tee gpurun_out/attn_modes.log
