"""k_tc2 on u16 4096^2 tiles (sigma 1-10, 10 scales): per-stage device times for 1 and 8
images, for an ncu launch list of the two-pass kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

n = 4096
img = synth.em_tile(n, n, 1000, defocus=0.0, dose=300.0, bits=16, device="cuda")
img = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16)).cuda()
for B in (1, 8):
    imgs = img.unsqueeze(0).repeat(B, 1, 1).contiguous()
    det = mhfd.Detector(n, n, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
    for _ in range(3):
        det.focus_score(imgs)
    torch.cuda.synchronize()
    det.timing_enable(10)
    for _ in range(10):
        det.focus_score(imgs)
    torch.cuda.synchronize()
    t = det.timing_read()
    avg = [sum(r[i] for r in t) / len(t) / B for i in range(4)]
    print(f"{B} x {n}^2 u16 {det.schedule('u16')}: per image stages " + " ".join(f"{a:.4f}" for a in avg))
