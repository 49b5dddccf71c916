#!/bin/bash
# Timing-probe builds of the fused MLP (gemm_tc.cu macros) -> csrc/build/lib_mlp_<name>.so
#   build_mlp_probe.sh name "-DMACRO=V ..." [name "-D..."]...
set -e
cd "$(dirname "$0")/../paper_2603_11441_b200/csrc"
make -j 8 > /dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
args=("$@")
for ((i = 0; i < ${#args[@]}; i += 2)); do
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr ${args[i+1]} -c gemm_tc.cu -o build/gemm_tc_${args[i]}.o &
done
wait
for ((i = 0; i < ${#args[@]}; i += 2)); do
  nvcc $ARCH -shared -cudart static -o build/lib_mlp_${args[i]}.so build/gemm_tc_${args[i]}.o build/attention.o \
    build/attention_tc.o build/rowops.o build/postprocess.o build/dart_capi.o build/nccl_shard.o -ldl
done
