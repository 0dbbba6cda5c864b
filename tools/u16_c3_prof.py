"""One 4096^2 u16 tile (sigma 1-10, 10 scales) and its LoG variant (u8) through the pair
kernels, for an ncu launch list (2 warm calls, then the profiled ones)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

img = synth.em_tile(4096, 4096, 1000, defocus=0.0, dose=300.0, bits=16, device="cuda")
img16 = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16)).cuda().unsqueeze(0)
img8 = synth.em_tile(4096, 4096, 1000, defocus=0.0, dose=300.0, device="cuda").unsqueeze(0)
d16 = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09)
dlog = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.1, response="log")
for _ in range(3):
    d16.focus_score(img16)
    dlog.focus_score(img8)
torch.cuda.synchronize()
