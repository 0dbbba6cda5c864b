"""Small driver for ncu: one warm-up and `--calls` focus_score calls on a batch of
4096^2 synthetic tiles (the bench configuration, fewer images)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--size", type=int, default=4096)
ap.add_argument("--calls", type=int, default=1)
ap.add_argument("--nms", default="paper")
a = ap.parse_args()
imgs = torch.stack([synth.em_tile(a.size, a.size, 1000 + b, defocus=0.5 * b, dose=300.0, device="cuda")
                    for b in range(a.batch)])
det = mhfd.Detector(a.size, a.size, 1.0, 10.0, 10, threshold=0.09, overlap=0.5, nms=a.nms)
det.focus_score(imgs)
torch.cuda.synchronize()
for _ in range(a.calls):
    s = det.focus_score(imgs)
torch.cuda.synchronize()
print("scores", s.tolist())
