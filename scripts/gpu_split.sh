# split-KV decoder cross-attention: GPU suite, then bench A/B over DART_ATTN_SPLIT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do for k in 2 1 3; do
  DART_ATTN_SPLIT=$k timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('split $k', round(d['value'],2), round(d['e2e']['value'],2), round(d['value_serial'],2), 'n80', round(d['n80']['value'],2), 'launches', d['gpu_launches'])"
done; done
