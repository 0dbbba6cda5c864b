#!/bin/bash
# A/B of the Eq. 3 NMS count pass: k_nms_rows (default) vs k_nms_roll<4>/<8>
# (MHFD_NMS_ROLL): parity tests under each variant, then bench stage times.
mkdir -p gpurun_out
for v in 4 8; do
  MHFD_NMS_ROLL=$v timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/nms_ab_tests_$v.log 2>&1
  echo "variant $v tests exit $?" >> gpurun_out/nms_ab_tests_$v.log
done
for rep in 1 2; do
  for v in 0 4 8; do
    MHFD_NMS_ROLL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-configs > gpurun_out/nms_ab_bench_${v}_$rep.json 2>/dev/null
  done
done
