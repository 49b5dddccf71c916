# A/B of the in-tree library's attention against paper_2603_11441_b200/csrc/build/lib_old.so (same box, interleaved)
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" 2>&1 | tail -1
for i in 1 2; do
echo NEW; timeout 120 python scripts/bench_attn.py 2>&1 | grep -v check
echo OLD; DART_LIB_PATH=$PWD/paper_2603_11441_b200/csrc/build/lib_old.so timeout 120 python scripts/bench_attn.py 2>&1 | grep -v check
done
