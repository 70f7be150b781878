for lib in libv_lb4_m4.so libv_lb5_m4.so libfsda_b200.so; do
FSDA_B200_LIB=paper_1709_04794_b200/$lib timeout 900 python tools/bench_batch.py --workload cfg2 --tasks 64 --seq-tasks 1 > gpurun_out/b2_$lib.json 2> gpurun_out/b2_$lib.err
FSDA_B200_LIB=paper_1709_04794_b200/$lib FSDA_B200_TRACE=1 timeout 1500 python tools/bench_batch.py --workload cfg4 --max-iter 20 --seq-tasks 1 > gpurun_out/b4_$lib.json 2> gpurun_out/b4_$lib.err
done
