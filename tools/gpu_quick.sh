#!/bin/bash
# Quick GPU iteration: gpu tests, the bench line, optional extra command.
#   gpurun --timeout 1500 -- bash tools/gpu_quick.sh <tag> [extra shell command]
set -u
TAG=${1:-q}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
tail -15 $O/${TAG}_pytest_gpu.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
tail -3 $O/${TAG}_bench.err
python - <<PY
import json
d=json.load(open("$O/${TAG}_bench.json"))
print("value", round(d["value"]), "ms", round(d["ms_per_step"],4), "frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]))
for k,v in d["kernels"].items(): print(f'{k:24s} {v["launches_per_step"]:5.1f} {v["ms_mean"]*1000:8.1f} {v["share"]:.3f}')
PY
if [ $# -ge 2 ]; then shift; bash -c "$*"; fi
