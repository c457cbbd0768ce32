python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_dbg.txt 2>&1
tail -30 gpurun_out/bench_dbg.txt
