timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
FSDA_B200_TRACE=1 timeout 600 python tools/time_e2e.py --reps 3 > gpurun_out/e2e.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
nproc > gpurun_out/nproc.log
