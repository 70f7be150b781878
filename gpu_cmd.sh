for m in 1 2 4; do
FSDA_B200_XT_CHUNK=$m timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2_$m.json 2> gpurun_out/bench_cfg2_$m.err
FSDA_B200_XT_CHUNK=$m timeout 600 python bench.py --no-cpu-baseline --workload cfg3 --steps 3 > gpurun_out/bench_cfg3_$m.json 2> gpurun_out/bench_cfg3_$m.err
done
