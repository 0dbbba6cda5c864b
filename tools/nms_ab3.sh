#!/bin/bash
# k_nms_roll<4> with the column-max predicate (default) vs k_nms_rows: full GPU suite on
# the default path, then bench stage times of both
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/nms_ab3_tests.log 2>&1
echo "exit $?" >> gpurun_out/nms_ab3_tests.log
for rep in 1 2; do
  for v in 0 4 8; do
    MHFD_NMS_ROLL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-configs > gpurun_out/nms_ab3_bench_${v}_$rep.json 2>/dev/null
  done
done
