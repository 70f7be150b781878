timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for rb in 4096 8192 16384; do for v in 4 8 16; do
FSDA_B200_XT_RB=$rb FSDA_B200_XT_DPB=$v timeout 600 python bench.py --no-cpu-baseline --no-profile --steps 10 > gpurun_out/bench_cfg2_${rb}_$v.json 2> gpurun_out/bench_cfg2_${rb}_$v.err
FSDA_B200_XT_RB=$rb FSDA_B200_XT_DPB=$v timeout 600 python bench.py --no-cpu-baseline --no-profile --workload cfg3 --steps 3 > gpurun_out/bench_cfg3_${rb}_$v.json 2> gpurun_out/bench_cfg3_${rb}_$v.err
done; done
