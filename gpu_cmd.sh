timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench.py --no-cpu-baseline --workload cfg3 --steps 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
