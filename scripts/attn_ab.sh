python -m pytest tests/test_gpu_kernels.py -q -x -k "attn or attention" 2>&1 | tail -1
python scripts/ab_attn.py 0 4 5 2>&1
DART_FA_VARIANT=4 python scripts/trace_attn.py 16 2>&1 | head -22
