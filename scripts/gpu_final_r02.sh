#!/bin/bash
# Round-2 closing measurement: GPU suite, default bench line, warm launch lists (N=4 / N=80),
# ncu --set full of the hot kernels + DRAM traffic JSON.  TAG names the output generation.
TAG=${1:-r02d}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
bash scripts/gpu_launches.sh $TAG > /dev/null 2>&1
[ "$2" = "ncu" ] && bash scripts/gpu_ncu_r02.sh > /dev/null 2>&1
cat gpurun_out/pytest_gpu_$TAG.log; head -3 gpurun_out/launches_n4_$TAG.txt gpurun_out/launches_n80_$TAG.txt
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print(d['value'], d['e2e']['value'], d['value_serial'], d['n80']['value'], d['n80']['e2e']['value'], d['roofline']['frac'], d['roofline_attn16']['frac'], d['stage_ms_serial'], d['n80']['stage_ms_serial'], d['clocks']['sm_mhz'])"
