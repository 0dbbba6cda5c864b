#!/bin/bash
# second A/B of the NMS count pass (lane-distributed segment counters in k_nms_roll),
# plus a launch list of the NMS-stage kernels under each variant
mkdir -p gpurun_out
MHFD_NMS_ROLL=8 timeout 600 python -m pytest tests -m gpu -x -q -k "nms or parity or band" > gpurun_out/nms_ab2_tests_8.log 2>&1
echo "exit $?" >> gpurun_out/nms_ab2_tests_8.log
for rep in 1 2; do
  for v in 0 4 8; do
    MHFD_NMS_ROLL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-configs > gpurun_out/nms_ab2_bench_${v}_$rep.json 2>/dev/null
  done
done
for v in 0 4 8; do
  MHFD_NMS_ROLL=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_nms|k_seg_scan" -c 6 --csv python tools/prof_run.py --batch 16 > gpurun_out/nms_ab2_ncu_$v.csv 2>&1
done
