set -x
for v in 0 1 3 4 5; do DART_FA_VARIANT=$v timeout 300 python scripts/bench_attn.py; done > gpurun_out/bench_attn.log 2>&1
grep -E "FAIL|enc self|bb |rror" gpurun_out/bench_attn.log
