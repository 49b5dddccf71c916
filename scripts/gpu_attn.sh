set -x
for m in 1 2; do DART_FA_SOFTMAX_ONLY=$m DART_FA_VARIANT=0 timeout 300 python scripts/bench_attn.py; done >> gpurun_out/bench_attn.log 2>&1
grep -E "enc self|bb " gpurun_out/bench_attn.log
