#!/bin/bash
# Round-2 closing measurement: GPU suite, default bench line, warm launch lists (N=4 / N=80),
# ncu --set full of the hot kernels + DRAM traffic JSON.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_r02c.log
timeout 900 python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
bash scripts/gpu_launches.sh r02c > /dev/null 2>&1
bash scripts/gpu_ncu_r02.sh > /dev/null 2>&1
cat gpurun_out/pytest_gpu_r02c.log; head -3 gpurun_out/launches_n4_r02c.txt gpurun_out/launches_n80_r02c.txt
python -c "import json; d=json.load(open('gpurun_out/bench_r02c.json')); print(d['value'], d['e2e']['value'], d['n80']['value'], d['roofline']['frac'], d['roofline_attn16']['frac'])"
