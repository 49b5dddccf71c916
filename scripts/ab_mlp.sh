for i in 1 2; do
echo NEW; timeout 120 python scripts/bench_mlp.py 2>&1 | tail -4
echo OLD; DART_LIB_PATH=$PWD/build/lib_old.so timeout 120 python scripts/bench_mlp.py 2>&1 | tail -4
done
