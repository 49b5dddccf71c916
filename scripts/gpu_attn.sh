set -x
DART_FA_VARIANT=10 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/attn_tests.log 2>&1; tail -3 gpurun_out/attn_tests.log
for v in 0 10 11 12 13; do DART_FA_VARIANT=$v timeout 300 python scripts/bench_attn.py; done > gpurun_out/bench_attn.log 2>&1
for m in 1 2; do DART_FA_SOFTMAX_ONLY=$m DART_FA_VARIANT=10 timeout 300 python scripts/bench_attn.py; done >> gpurun_out/bench_attn.log 2>&1
grep -E "FAIL|enc self|bb |rror" gpurun_out/bench_attn.log
