#!/bin/bash
# One GPU session: GPU tests, default bench, ncu launch list of a short bench, one
# `ncu --set full` capture of the hot kernel.  Outputs land in gpurun_out/$TAG*.
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench_rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --batch 16 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu_launch_rc=$?" >> gpurun_out/${TAG}_ncu_launch.log
python tools/prof_run.py --batch 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_band -s 1 -c 1 -o gpurun_out/${TAG}_band \
  python tools/prof_run.py --batch 2 > gpurun_out/${TAG}_prof_ncu.log 2>&1
echo "ncu_full_rc=$?" >> gpurun_out/${TAG}_prof_ncu.log
