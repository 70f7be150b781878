FSDA_B200_PDL=7 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sa_sda.py tests/test_regression_phase.py -x -q -m gpu > gpurun_out/pytest_gpu7.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu7.log
for m in 3 7; do
FSDA_B200_PDL=$m timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2_$m.json 2> gpurun_out/bench_cfg2_$m.err
FSDA_B200_PDL=$m timeout 600 python bench.py --no-cpu-baseline --workload cfg3 --steps 3 > gpurun_out/bench_cfg3_$m.json 2> gpurun_out/bench_cfg3_$m.err
done
