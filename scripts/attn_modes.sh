for v in 0 4; do for m in 0 2; do
  echo "== variant $v DART_FA_SOFTMAX_ONLY=$m"
  DART_FA_VARIANT=$v DART_FA_SOFTMAX_ONLY=$m timeout 120 python scripts/bench_attn.py 2>&1 | grep -E "N=80|global|windowed"
done; done
