DART_FA_VARIANT=${V:-4} timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" 2>&1 | tail -1
timeout 300 python scripts/ab_attn.py 0 ${V:-4} 2>&1
DART_FA_VARIANT=${V:-4} timeout 120 python scripts/trace_attn.py 16 2>&1 | sed -n 2,8p
DART_FA_VARIANT=${V:-4} timeout 120 python scripts/trace_attn.py 16 2>&1 | sed -n 36,42p
