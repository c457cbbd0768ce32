#!/bin/bash
# One gpurun call: GPU tests, smoke, the default bench line, the ncu launch list of one step and a
# `--set full` capture of the hot kernels.  Everything lands in gpurun_out/.
#   gpurun --timeout 1800 -- bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/${TAG}_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
tail -3 $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
tail -c 600 $O/${TAG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline --e2e-steps 0 > $O/${TAG}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resblock' -c 2 -o $O/${TAG}_prof_rb -f \
    python bench.py --steps 1 --warmup 0 --no-graph --no-cpu-baseline --e2e-steps 0 > $O/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'conv_tc|bilinear|gather|pack_kernel|select_kernel|ccl_kernel|box_write' -c 10 -o $O/${TAG}_prof -f \
    python bench.py --steps 1 --warmup 0 --no-graph --no-cpu-baseline --e2e-steps 0 >> $O/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
ls -la $O; du -sh $O
