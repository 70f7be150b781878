nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi.log
FSDA_B200_TRACE=1 timeout 900 python tools/bench_batch.py --workload cfg2 --tasks 32 --seq-tasks 2 > gpurun_out/batch_cfg2.json 2> gpurun_out/batch_cfg2.err
FSDA_B200_TRACE=1 timeout 1500 python tools/bench_batch.py --workload cfg4 --max-iter 20 --seq-tasks 1 > gpurun_out/batch_cfg4.json 2> gpurun_out/batch_cfg4.err
