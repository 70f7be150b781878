timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_side.json 2> gpurun_out/bench_side.err
FSDA_B200_SU_INLINE=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_inline.json 2> gpurun_out/bench_inline.err
timeout 600 python bench.py --no-cpu-baseline --workload cfg3 --steps 5 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
FSDA_B200_SU_INLINE=1 timeout 600 python bench.py --no-cpu-baseline --workload cfg3 --steps 5 > gpurun_out/bench_cfg3_inline.json 2> gpurun_out/bench_cfg3_inline.err
