set -x
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_kernels.py -x -q > gpurun_out/pipe_tests.log 2>&1; tail -5 gpurun_out/pipe_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout 600 python bench.py --classes 80 --steps 10 --no-cpu-baseline > gpurun_out/bench_n80.json 2> gpurun_out/bench_n80.err
cat gpurun_out/bench_n4.json gpurun_out/bench_n80.json; tail -3 gpurun_out/bench_n4.err
