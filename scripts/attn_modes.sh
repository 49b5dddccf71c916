for m in 2 3; do
  echo "== DART_FA_SOFTMAX_ONLY=$m"
  DART_FA_SOFTMAX_ONLY=$m timeout 120 python scripts/bench_attn.py 2>&1 | grep -E "N=80|global|windowed"
done
