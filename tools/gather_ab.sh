#!/bin/bash
# k_nms_gather4 (default) vs k_nms_gather (MHFD_NMS_GATHER1): GPU suite on the default,
# then bench stage times of both
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gather_tests.log 2>&1
echo "exit $?" >> gpurun_out/gather_tests.log
for rep in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-configs > gpurun_out/gather_bench_4_$rep.json 2>/dev/null
  MHFD_NMS_GATHER1=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-configs > gpurun_out/gather_bench_1_$rep.json 2>/dev/null
done
