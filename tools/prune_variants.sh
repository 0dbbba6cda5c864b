#!/bin/bash
# pruning kernel register caps: stage times at batch 16 for library variants in build/
for v in "" build/lib_p4.so build/lib_p6.so; do
  echo "== ${v:-default}"
  MHFD_LIB=$v timeout 200 python tools/stage_split.py 16 2>&1 | head -1
done
