#!/bin/bash
# A/B of a GEMM environment switch: interleaved runs of scripts/gemm_epi_probe2.py / gemm_n1280.py
# with and without $1 (e.g. DART_NO_RESID_PF=1).
for r in 1 2; do
  echo "== default"; K=1280 python scripts/gemm_epi_probe2.py 2>&1 | tail -4
  echo "== $1"; env $1 K=1280 python scripts/gemm_epi_probe2.py 2>&1 | tail -4
done
echo "== n1280 default"; python scripts/gemm_n1280.py 2>&1 | grep -E "cuBLAS|bn   0"
echo "== n1280 $1"; env $1 python scripts/gemm_n1280.py 2>&1 | grep -E "cuBLAS|bn   0"
