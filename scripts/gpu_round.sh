#!/bin/bash
# One GPU pass: gpu tests, N=4 / N=80 bench lines, N=4 launch list, ncu --set full of the hot kernels.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout 600 python bench.py --classes 80 --steps 10 --no-cpu-baseline > gpurun_out/bench_n80.json 2> gpurun_out/bench_n80.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n4.csv python scripts/profile_step.py --classes 4 > gpurun_out/prof_n4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n80.csv python scripts/profile_step.py --classes 80 > gpurun_out/prof_n80.log 2>&1
bash scripts/ncu_full.sh hot fc1 out att16 att80 att80w
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_n4.json gpurun_out/bench_n80.json
