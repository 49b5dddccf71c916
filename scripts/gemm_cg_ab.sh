# A/B: CTA-pair (cg 2) vs single-CTA (cg 1) 256-wide tiles on the residual / narrow GEMMs
for r in 1 2 3; do
  for p in 256,2 256,1; do echo "plan $p"; DART_GEMM_PLAN=$p python scripts/bench_gemm.py out+res "enc q" "enc fc2" "enc out" 2>&1 | tail -n +2; done
done
