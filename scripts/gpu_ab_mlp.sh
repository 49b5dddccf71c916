timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "mlp" 2>&1 | tail -1
for i in 1 2 3; do
  echo NEW; timeout 300 python scripts/bench_mlp_ln.py
  echo OLD; DART_LIB_PATH=$PWD/build/lib_old.so timeout 300 python scripts/bench_mlp_ln.py
done
