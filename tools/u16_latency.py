"""Per-stage device times (percentiles, blur, NMS, pruning) of one 4096^2 u16 tile and of
C5 (8192^2 u16, sigma 1-30, 20 scales) on k_tc2, periodic and reflect."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

for n, sig, ns, seed in ((4096, (1.0, 10.0), 10, 1000), (8192, (1.0, 30.0), 20, 7)):
    img = synth.em_tile(n, n, seed, defocus=0.0, dose=300.0, bits=16, device="cuda")
    img = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16)).cuda().unsqueeze(0)
    for bd in ("periodic", "reflect"):
        det = mhfd.Detector(n, n, sig[0], sig[1], ns, threshold=0.1 * (sig[1] - sig[0]) / ns, overlap=0.5, boundary=bd)
        for _ in range(3):
            s = det.focus_score(img)
        torch.cuda.synchronize()
        det.timing_enable(10)
        for _ in range(10):
            s = det.focus_score(img)
        torch.cuda.synchronize()
        t = det.timing_read()
        avg = [sum(r[i] for r in t) / len(t) for i in range(4)]
        print(f"{n}^2 u16 {bd:8s} {det.schedule('u16')}: stages (ms) " + " ".join(f"{a:.4f}" for a in avg) +
              f"  total {sum(avg):.4f}  score {float(s[0])}")
