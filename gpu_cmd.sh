for lib in libfsda_b200.so libfsda_mlp8.so; do
FSDA_B200_LIB=paper_1709_04794_b200/$lib timeout 900 python tools/bench_batch.py --workload cfg2 --tasks 32 --seq-tasks 1 > gpurun_out/batch_cfg2_$lib.json 2> gpurun_out/batch_cfg2_$lib.err
FSDA_B200_LIB=paper_1709_04794_b200/$lib timeout 1500 python tools/bench_batch.py --workload cfg4 --max-iter 10 --seq-tasks 1 > gpurun_out/batch_cfg4_$lib.json 2> gpurun_out/batch_cfg4_$lib.err
done
