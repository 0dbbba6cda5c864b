#!/bin/bash
# Quick GPU check of a kernel change: timing A/B (tools/tc_exp.py) then the GPU parity suite
# (PYTEST_K: a pytest -k expression).
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 300 python tools/tc_exp.py "$@" paper_2108_12050_b200/libmhfd.so > gpurun_out/${TAG}_time.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${TAG}_pytest.log
