#!/bin/bash
# Round-end evidence: bench lines of every config, the reference arm, the A/B of the pipeline count, the
# fig:s_bub-d study and the ncu captures at HEAD. -> gpurun_out/<tag>_*
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/${TAG}_gpu.txt 2>&1
run() {   # name, args...
  local name=$1; shift
  timeout 1500 python bench.py "$@" > $O/${TAG}_bench_${name}.json 2> $O/${TAG}_bench_${name}.err
  echo "bench $name rc=$? $(tail -c 300 $O/${TAG}_bench_${name}.json | head -c 120)"
}
run c2
REGEN_PIPES=2 run c2_pipes2 --no-cpu-baseline
run c2_nv12 --input nv12 --no-cpu-baseline
run c2_u8out --out u8 --no-cpu-baseline
run c1 --config c1 --no-cpu-baseline
run c3 --config c3 --steps 5 --warmup 3 --no-cpu-baseline
run c4g --config c4g --steps 5 --warmup 3 --no-cpu-baseline
run c4 --config c4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2
for r in 5 10 15 20 25 35 50; do
  run c5_r$r --config c5 --ratio $r --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err
echo "reference rc=$? $(head -c 200 $O/${TAG}_bench_reference.json)"
if [ "${SBUBD:-0}" = "1" ]; then   # the packing study (packer unchanged since profiles/r02_sbubd_study.*)
  timeout 1500 python tools/sbubd_study.py --shuffles 1000 > $O/${TAG}_sbubd.log 2>&1; echo "sbubd rc=$?"
fi
bash tools/gpu_profile.sh $TAG
