# A/B of the in-tree library against build/lib_old.so (same box, interleaved)
python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or rope" 2>&1 | tail -1
for i in 1 2; do
echo NEW; python scripts/bench_gemm.py ${@:-qkv} 2>&1 | tail -n +2
echo OLD; DART_LIB_PATH=$PWD/build/lib_old.so python scripts/bench_gemm.py ${@:-qkv} 2>&1 | tail -n +2
done
