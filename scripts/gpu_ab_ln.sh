timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "mlp or resid_ln or ln" 2>&1 | tail -1
for i in 1 2 3; do
  for L in NEW OLD; do
    if [ $L = OLD ]; then export DART_LIB_PATH=$PWD/build/lib_old.so; else unset DART_LIB_PATH; fi
    echo $L; timeout 300 python scripts/bench_resid_ln.py; timeout 300 python scripts/bench_mlp_ln.py
  done
done
