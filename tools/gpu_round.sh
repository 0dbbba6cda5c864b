#!/bin/bash
# One GPU session: a quick multi-tile run (stop on failure), smoke, GPU tests, default
# bench, ncu launch list of a short bench, one `ncu --set full` capture of the hot
# kernel.  Outputs land in gpurun_out/$TAG*.
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 90 python tools/prof_run.py --batch 2 > gpurun_out/${TAG}_prof_plain.log 2>&1
rc=$?; echo "prof_plain_rc=$rc" >> gpurun_out/${TAG}_prof_plain.log
if [ $rc -ne 0 ]; then echo "multi-tile run failed, stopping"; exit 1; fi
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; rc=$?; echo "pytest_rc=$rc" >> gpurun_out/${TAG}_pytest.log
if [ $rc -ne 0 ]; then echo "gpu tests failed, stopping"; exit 1; fi
timeout 300 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench_rc=$?" >> gpurun_out/${TAG}_bench.err
[ "${NO_NCU:-0}" = "1" ] && exit 0
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --batch 16 --no-e2e --no-cpu-baseline --no-configs > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu_launch_rc=$?" >> gpurun_out/${TAG}_ncu_launch.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_tc|k_prune|k_nms_rows|k_hist" -s 5 -c 5 -o gpurun_out/${TAG}_tc \
  python tools/prof_run.py --batch 2 > gpurun_out/${TAG}_prof_ncu.log 2>&1
echo "ncu_full_rc=$?" >> gpurun_out/${TAG}_prof_ncu.log
