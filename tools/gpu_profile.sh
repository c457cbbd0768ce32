#!/bin/bash
# Evidence for profiles/: ncu launch lists (C2 and one C4 group) and `ncu --set full` captures of the
# hot kernels at HEAD, plus compute-sanitizer runs. Everything lands in gpurun_out/<tag>_*.
#   gpurun --timeout 3000 -- bash tools/gpu_profile.sh r02
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
B="python bench.py --steps 1 --warmup 1 --no-graph --no-cpu-baseline --e2e-steps 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c2.csv \
    $B > $O/${TAG}_ncu_launch_c2.log 2>&1; echo "launches c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c4g.csv \
    $B --config c4g > $O/${TAG}_ncu_launch_c4g.log 2>&1; echo "launches c4g rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'resblock' -c 2 -o $O/${TAG}_prof_rb -f \
    $B > $O/${TAG}_ncu_full_rb.log 2>&1; echo "full rb rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"conv_tc|bilinear|stitch|pack_kernel|select_kernel|ccl_kernel|box_write|sort_bitonic" -c 14 \
    -o $O/${TAG}_prof -f $B > $O/${TAG}_ncu_full.log 2>&1; echo "full rc=$?"
for r in ${TAG}_prof_rb ${TAG}_prof; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
done
# per-kernel source pages (SASS + stall samples) of the multi-kernel capture, then drop its report
# (gpurun copies back at most 64 MiB)
for k in stitch_band bilinear_kernel conv_tc_kernel; do
  ncu -i $O/${TAG}_prof.ncu-rep --page source --csv --print-source sass -k regex:$k > $O/${TAG}_src_$k.csv 2>/dev/null
done
rm -f $O/${TAG}_prof.ncu-rep
ls -la $O | grep $TAG
