#!/bin/bash
# Fused MLP A/B across probe builds (scripts/build_mlp_probe.sh): gpu_mlp_probe.sh name...
mkdir -p gpurun_out
L=paper_2603_11441_b200/csrc/build
for r in 1 2; do
  echo "== prod"; timeout 120 python scripts/bench_mlp_ln.py; timeout 120 python scripts/bench_mlp.py | grep -o "M=.*fused *[0-9.]* us"
  for p in "$@"; do echo "== $p"; DART_LIB_PATH=$PWD/$L/lib_mlp_$p.so timeout 120 python scripts/bench_mlp_ln.py
    DART_LIB_PATH=$PWD/$L/lib_mlp_$p.so timeout 120 python scripts/bench_mlp.py | grep -o "M=.*fused *[0-9.]* us"; done
done 2>&1 | tee gpurun_out/mlp_probe.log
