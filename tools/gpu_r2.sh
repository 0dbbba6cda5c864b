#!/bin/bash
# Round-2 GPU session: smoke, GPU tests, default bench, ncu launch list.
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest.log 2>&1; rc=$?; echo "pytest_rc=$rc" >> gpurun_out/${TAG}_pytest.log
timeout 400 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench_rc=$?" >> gpurun_out/${TAG}_bench.err
[ "${NO_NCU:-0}" = "1" ] && exit 0
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --batch 16 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu_launch_rc=$?" >> gpurun_out/${TAG}_ncu_launch.log
