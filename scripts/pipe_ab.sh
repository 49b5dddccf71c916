# A/B: backbone streams in the inter-frame pipeline (DART_PIPE_BB)
for r in 1 2; do for nb in 2 3 4; do
  DART_PIPE_BB=$nb timeout 600 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bb=$nb', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_mhz'])"
done; done
DART_PIPE_BB=2 timeout 600 python bench.py --no-cpu-baseline --classes 80 --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N80 bb=2', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_mhz'])"
DART_PIPE_BB=1 timeout 600 python bench.py --no-cpu-baseline --classes 80 --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N80 bb=1', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['clocks']['sm_mhz'])"
