# A/B of the in-tree library against build/lib_old.so (same box, interleaved)
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -1
for i in 1 2; do
echo NEW; timeout 120 python scripts/bench_gemm.py "$@" 2>&1 | tail -n +2; timeout 120 python scripts/bench_attn.py 2>&1 | grep -v check
echo OLD; DART_LIB_PATH=$PWD/build/lib_old.so timeout 120 python scripts/bench_gemm.py "$@" 2>&1 | tail -n +2; DART_LIB_PATH=$PWD/build/lib_old.so timeout 120 python scripts/bench_attn.py 2>&1 | grep -v check
done
