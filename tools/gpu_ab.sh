#!/bin/bash
# A/B bench lines under environment settings: gpu_ab.sh <tag> "<pytest -k expr|ALL|NONE>" "ENV=1 ENV2=x;ENV3=y;..."
# (each ';'-separated entry is one bench run with those variables set; an empty entry = defaults)
set -u
TAG=$1; KEXPR=${2:-NONE}; VARIANTS=${3:-}; BARGS=${4:-}
O=gpurun_out
mkdir -p $O
if [ "$KEXPR" = "ALL" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
  tail -5 $O/${TAG}_pytest_gpu.log
elif [ "$KEXPR" != "NONE" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
  tail -5 $O/${TAG}_pytest_gpu.log
fi
IFS=';' read -ra VA <<< "$VARIANTS"
i=0
for v in "${VA[@]}"; do
  env $v timeout 900 python bench.py $BARGS > $O/${TAG}_ab$i.json 2> $O/${TAG}_ab$i.err; echo "bench [$v] rc=$?"
  tail -2 $O/${TAG}_ab$i.err
  python - <<PY
import json
try:
    d=json.loads(open("$O/${TAG}_ab$i.json").read().strip().splitlines()[-1])
    r=d.get("roofline",{}); rs=d.get("roofline_step",{})
    print("value", round(d["value"]), "ms", round(d["ms_per_step"],4), "kfrac", round(r.get("frac",0),3), "stepfrac", round(rs.get("frac",0),3), "e2e", d["e2e"]["value"])
    for k,v in list(d["kernels"].items())[:8]: print(f'  {k:24s} {v["launches_per_step"]:6.1f} {v["ms_mean"]*1000:9.1f} {v["share"]:.3f}')
except Exception as e: print("parse fail", e)
PY
  i=$((i+1))
done
