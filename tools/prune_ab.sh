#!/bin/bash
# A/B of pruning-kernel builds: single-tile stage times and the 16-image batch rate.
for L in "$@"; do
  echo "== $L"
  MHFD_LIB=$L python tools/latency_split.py 1024 4096 2>&1 | grep "overlap 0.5"
  python tools/tc_exp.py $L 2>&1 | tail -1
done
