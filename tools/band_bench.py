"""bench.py's single-image band measurements (C3 on k_tc, C5 on k_tc2) alone: per G the
slowest band's mhfd_detect_band, the replicated pruning, and the sharded pruning
(band + halo, mhfd_prune_band)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
print(json.dumps({"C3": bench.band_times(dev), "C5": bench.band_times(dev, c5=True)}, indent=1))
