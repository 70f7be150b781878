FSDA_B200_PDL=15 FSDA_B200_UNROLL=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sa_sda.py tests/test_regression_phase.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for cfgs in "7 1" "15 1" "7 2" "15 2" "15 4"; do set -- $cfgs
FSDA_B200_PDL=$1 FSDA_B200_UNROLL=$2 timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2_$1_$2.json 2> gpurun_out/bench_cfg2_$1_$2.err
FSDA_B200_PDL=$1 FSDA_B200_UNROLL=$2 timeout 600 python bench.py --no-cpu-baseline --workload cfg3 --steps 3 > gpurun_out/bench_cfg3_$1_$2.json 2> gpurun_out/bench_cfg3_$1_$2.err
done
