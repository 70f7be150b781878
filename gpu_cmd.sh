timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 1800 python tools/bench_batch.py --workload cfg4 --seq-tasks 2 > gpurun_out/batch_cfg4_full.json 2> gpurun_out/batch_cfg4_full.err
timeout 900 python tools/bench_batch.py --workload cfg2 --tasks 64 --seq-tasks 3 > gpurun_out/batch_cfg2_64.json 2> gpurun_out/batch_cfg2_64.err
