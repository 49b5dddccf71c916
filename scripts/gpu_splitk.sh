set -x
python -m pytest tests/test_gpu_kernels.py -x -q -k "split" 2>&1 | tail -5
python scripts/gemm_splitk.py
for sk in 0 6 2 4; do DART_SPLITK=$sk timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('SPLITK', $sk, d['value'], d['e2e']['value'], d['n80']['value'] if d.get('n80') else None, d['roofline']['frac'], d['roofline']['per_shape'])"; done
