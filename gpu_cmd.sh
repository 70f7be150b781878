timeout 1200 python -m pytest tests/ -q -m gpu --timeout 900 -x > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
export FSDA_B200_EAGER=1
timeout 300 python tools/ncu_solve.py --solves 1 > gpurun_out/ncu_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_solve.py --solves 1 > gpurun_out/ncu.log 2>&1; echo ncu_rc=$? >> gpurun_out/ncu.log
