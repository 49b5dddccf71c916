DART_FA_VARIANT=${V:-4} timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" 2>&1 | tail -1
timeout 300 python scripts/ab_attn.py 0 ${V:-4} 2>&1
