#!/bin/bash
# GPU iteration: selected gpu tests (pytest -k expr), then bench lines for configs.
#   gpurun --timeout 1800 -- bash tools/gpu_b.sh <tag> "<pytest -k expr or ALL>" "<bench args>;<bench args>..."
set -u
TAG=$1; KEXPR=${2:-ALL}; BENCHES=${3:-}
O=gpurun_out
mkdir -p $O
if [ "$KEXPR" = "ALL" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
elif [ "$KEXPR" != "NONE" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 -k "$KEXPR" > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
fi
[ -f $O/${TAG}_pytest_gpu.log ] && tail -25 $O/${TAG}_pytest_gpu.log
IFS=';' read -ra BA <<< "$BENCHES"
i=0
for b in "${BA[@]}"; do
  [ -z "$b" ] && continue
  timeout 900 python bench.py $b > $O/${TAG}_bench$i.json 2> $O/${TAG}_bench$i.err; echo "bench [$b] rc=$?"
  tail -3 $O/${TAG}_bench$i.err
  python - <<PY
import json
try:
    d=json.loads(open("$O/${TAG}_bench$i.json").read().strip().splitlines()[-1])
    r=d.get("roofline",{}); rs=d.get("roofline_step",{})
    print("value", round(d["value"]), "ms", round(d["ms_per_step"],3), "kfrac", r.get("frac"), "stepfrac", rs.get("frac"), "e2e", d["e2e"]["value"], "cpu", d.get("cpu_baseline",{}).get("value"))
    for k,v in list(d["kernels"].items())[:14]: print(f'  {k:24s} {v["launches_per_step"]:6.1f} {v["ms_mean"]*1000:9.1f} {v["share"]:.3f}')
except Exception as e: print("parse fail", e)
PY
  i=$((i+1))
done
