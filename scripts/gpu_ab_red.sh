# A/B: fp32 residual epilogue as TMA reduce-add (in-tree lib) vs load-add-store (build/lib_old.so)
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for i in 1 2; do
for L in new old; do
  if [ $L = old ]; then export DART_LIB_PATH=$PWD/build/lib_old.so; else unset DART_LIB_PATH; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$L', round(d['value'],2), round(d['e2e']['value'],2), round(d['value_serial'],2), 'n80', round(d['n80']['value'],2), 'frac', round(r['frac'],3), round(r['frac_with_pdl'],3), {k: round(v['us'],1) for k,v in r['per_shape'].items()})"
done; done
