#!/bin/bash
# pruning grid size sweep: device bench (batch 64) and e2e for CTAs/SM in {1,2,4,8}
for k in 1 2 4 8; do
  echo "== MHFD_PRUNE_CTAS_PER_SM=$k"
  MHFD_PRUNE_CTAS_PER_SM=$k timeout 200 python tools/stage_split.py 16 2>&1 | head -1
  MHFD_PRUNE_CTAS_PER_SM=$k timeout 300 python tools/e2e_chunks.py 2>&1 | grep "chunk  8"
done
