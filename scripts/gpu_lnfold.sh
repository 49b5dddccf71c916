# Backbone LN fold: parity (fold on / off), the GPU suite, and bench A/B via DART_LN_FOLD
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_width" -s 2>&1 | grep -E "fold|passed|failed|Error" | head -20
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do for f in 1 0; do
  DART_LN_FOLD=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('fold $f', round(d['value'],2), round(d['e2e']['value'],2), round(d['value_serial'],2), 'n80', round(d['n80']['value'],2), 'launches', d['gpu_launches'])"
done; done
