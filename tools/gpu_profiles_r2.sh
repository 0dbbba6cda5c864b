#!/bin/bash
# Round-2 final evidence: ncu --set full of one bench step's kernels (2 x 4096^2 u8), of the
# C5 k_tc2 kernels and of one 4096^2 tile's pruning; launch list of a short bench run.
TAG=${1:-r02e}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 6 -c 6 -o gpurun_out/${TAG}_step \
  python tools/prof_run.py --batch 2 > gpurun_out/${TAG}_step.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_step.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tc2" -s 6 -c 3 -o gpurun_out/${TAG}_c5 \
  python tools/c5_time.py > gpurun_out/${TAG}_c5.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --batch 16 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/${TAG}_launch.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_nms26|k_nms_gather4" -s 2 -c 2 -o gpurun_out/${TAG}_nms26 \
  python tools/prof_run.py --batch 2 --nms 26 > gpurun_out/${TAG}_nms26.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_nms26.log
