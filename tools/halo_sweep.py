"""How many bands certify (mhfd_prune_band) for halos (r + 1) D, r = 1..6: C3 (4096^2 u8)
and C5 (8192^2 u16, sigma 1-30) tiles cut into 8 bands."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402
from paper_2108_12050_b200.dist import band_rows  # noqa: E402

for name, size in (("C3", 4096), ("C5", 8192)):
    for seed, dfc in ((1000, 0.0), (1001, 2.0)):
        if name == "C3":
            img = synth.em_tile(size, size, seed, defocus=dfc, dose=300.0, device="cuda")
            det = mhfd.Detector(size, size, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
        else:
            a = synth.em_tile(size, size, seed, defocus=dfc, dose=300.0, bits=16, device="cuda")
            img = torch.from_numpy(a.to(torch.int32).cpu().numpy().astype(np.uint16)).cuda()
            det = mhfd.Detector(size, size, 1.0, 30.0, 20, threshold=0.145, overlap=0.5)
        D = det.interaction_radius()
        row = []
        for r in range(1, 7):
            h = (r + 1) * D
            ok = 0
            for k in range(8):
                y0, y1 = band_rows(size, 8, k)
                e0, e1 = max(0, y0 - h), min(size, y1 + h)
                c, n = det.detect_band(img, e0, e1)
                ok += int(det.prune_band(c, int(n), e0, e1, y0, y1)[1][0])
            row.append(ok)
        print(name, "defocus", dfc, "D", D, "certified of 8 for rounds 1..6:", row, flush=True)
