timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tc1_smoke.log 2>&1; echo rc=$? >> gpurun_out/tc1_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tc1_pytest.log 2>&1; echo rc=$? >> gpurun_out/tc1_pytest.log
timeout 300 python bench.py --batch 16 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tc1_bench.json 2> gpurun_out/tc1_bench.err; echo rc=$? >> gpurun_out/tc1_bench.err
