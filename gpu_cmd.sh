free -g > gpurun_out/mem.log; nproc >> gpurun_out/mem.log
timeout 900 python tools/cfg5_run.py --scale 0.1 --solves 2 > gpurun_out/cfg5_s01.json 2> gpurun_out/cfg5_s01.err
timeout 2700 python tools/cfg5_run.py --solves 3 > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
