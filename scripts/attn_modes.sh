# hd-16 / hd-80 attention: full kernel vs softmax alone (stale S) vs MMA/TMA pipeline alone
python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" 2>&1 | tail -2
for m in 0 1 2; do
  echo "== DART_FA_SOFTMAX_ONLY=$m"
  DART_FA_SOFTMAX_ONLY=$m python scripts/bench_attn.py 2>&1 | grep -E "N=80|N=4|global|windowed|FAIL"
done
