FSDA_B200_XT_SPLIT=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -m gpu > gpurun_out/pytest_split.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_split.log
for v in 0 1; do
if [ $v = 1 ]; then export FSDA_B200_XT_SPLIT=1; fi
timeout 600 python bench.py --no-cpu-baseline --batch-tasks 0 --concurrency 1 --steps 10 > gpurun_out/b_$v.json 2> gpurun_out/b_$v.err
timeout 600 python bench.py --no-cpu-baseline --batch-tasks 0 --concurrency 1 --workload cfg3 --steps 3 > gpurun_out/b3_$v.json 2> gpurun_out/b3_$v.err
done
