"""C3 (one 4096^2 u8 tile and a batch of 8, sigma 1-10, 10 scales) in both NMS modes:
per-stage device ms (percentiles, blur, NMS, pruning) per image."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * b, dose=300.0, device="cuda") for b in range(8)])
for B in (1, 8):
    x = imgs[:B].contiguous()
    for nms in ("paper", "26"):
        det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=0.5, nms=nms)
        for _ in range(3):
            s = det.focus_score(x)
        torch.cuda.synchronize()
        det.timing_enable(10)
        for _ in range(10):
            s = det.focus_score(x)
        torch.cuda.synchronize()
        t = det.timing_read()
        avg = [sum(r[i] for r in t) / len(t) / B for i in range(4)]
        print(f"B {B} nms {nms:5s}: per image (ms) " + " ".join(f"{a:.4f}" for a in avg) +
              f"  total {sum(avg):.4f}  mean score {float(s.float().mean()):.0f}")
