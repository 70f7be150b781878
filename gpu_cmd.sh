timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for v in 0 1 2 3; do
FSDA_B200_XT=$v timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2_$v.json 2> gpurun_out/bench_cfg2_$v.err
FSDA_B200_XT=$v timeout 600 python bench.py --no-cpu-baseline --workload cfg3 --steps 3 > gpurun_out/bench_cfg3_$v.json 2> gpurun_out/bench_cfg3_$v.err
done
