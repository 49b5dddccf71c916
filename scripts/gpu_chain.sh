# row-block dependency chain fc1 -> fc2 -> LN1 -> QKV: parity (B, C, batch invariance), then bench A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_width or full_size or batch" 2>&1 | tail -3
for i in 1 2; do for c in 1 0; do
  DART_CHAIN=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('chain $c', round(d['value'],2), round(d['e2e']['value'],2), round(d['value_serial'],2), 'n80', round(d['n80']['value'],2), d['stage_ms_serial'])"
done; done
