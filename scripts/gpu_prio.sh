for i in 1 2; do for p in 0 1 2; do
  DART_PIPE_PRIORITY=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('prio $p', round(d['value'],2), round(d['e2e']['value'],2), 'n80', round(d['n80']['value'],2), round(d['n80']['e2e']['value'],2))"
done; done
