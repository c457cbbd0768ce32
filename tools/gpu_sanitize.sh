#!/bin/bash
# compute-sanitizer on smoke() and tools/sanitize_run.py (every round-2 kernel too) -> gpurun_out/<tag>_sanitizer_*.txt
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
      > $O/${TAG}_sanitizer_${tool}_smoke.txt 2>&1; echo "$tool smoke rc=$?"; tail -2 $O/${TAG}_sanitizer_${tool}_smoke.txt
  timeout 1800 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py \
      > $O/${TAG}_sanitizer_${tool}_run.txt 2>&1; echo "$tool run rc=$?"; tail -2 $O/${TAG}_sanitizer_${tool}_run.txt
done
