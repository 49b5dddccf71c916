for i in 1 2; do
echo NEW; python scripts/bench_gemm.py 2>&1 | sed -n 2,6p
echo OLD; DART_LIB_PATH=$PWD/build/lib_old.so python scripts/bench_gemm.py 2>&1 | sed -n 2,6p
done
