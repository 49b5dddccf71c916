#!/bin/bash
# ncu --set full of the current hot kernels (one launch each) + DRAM traffic JSON + source page of the
# residual GEMM; summaries go to profiles/r02 by hand after review.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/full_r02 -f python scripts/ncu_targets.py out fc2 fc1 qkv att16 att80 att80w > gpurun_out/ncu_full_r02.log 2>&1
ncu -i gpurun_out/full_r02.ncu-rep --page raw --csv > gpurun_out/full_r02_raw.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/full_r02_raw.csv > gpurun_out/ncu_full_hot_summary_r02.txt
python scripts/traffic_json.py gpurun_out/full_r02_raw.csv gpurun_out/roofline_traffic.json fc1 attn.out qkv mlp.fc2 att16 att80 att80w > /dev/null
tail -2 gpurun_out/ncu_full_r02.log
