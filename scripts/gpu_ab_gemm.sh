# A/B of GEMM changes: in-tree lib (NEW) vs build/lib_old.so (OLD), alternating processes
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -1
for i in 1 2 3; do
  for L in NEW OLD; do
    if [ $L = OLD ]; then export DART_LIB_PATH=$PWD/build/lib_old.so; else unset DART_LIB_PATH; fi
    echo $L; timeout 300 python scripts/gemm_qkv_timeline.py 2>&1 | grep "=="; timeout 300 python scripts/gemm_splitk.py 2>&1 | sed 's/| split 2.*//'
  done
done
