for p in 128,2 128,1 256,1; do DART_GEMM_PLAN=$p python scripts/bench_gemm.py attn.out fc2 "enc fc2" 2>&1 | grep -v "^GEMM"; done
