timeout 1200 python -m pytest tests/ -q -m gpu --timeout 900 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
