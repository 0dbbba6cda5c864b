#!/bin/bash
for k in 1 2 4 8; do
  echo "== MHFD_PRUNE_CTAS_PER_SM=$k"
  MHFD_PRUNE_CTAS_PER_SM=$k timeout 200 python tools/stage_split.py 1 2>&1 | head -1
  MHFD_PRUNE_CTAS_PER_SM=$k timeout 200 python tools/stage_split.py 4 2>&1 | head -1
done
