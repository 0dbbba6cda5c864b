"""Per-stage device times of one focus_score call on a single 1024^2 u8 tile (config C2,
sigma 1-10, 10 scales): where the single-image latency goes (stages: percentiles,
blur+DoG+argmax, NMS+compaction, pruning)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

for n in (1024, 2048):
    img = synth.em_tile(n, n, 11, defocus=0.0, dose=300.0, device="cuda").unsqueeze(0)
    det = mhfd.Detector(n, n, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
    for _ in range(3):
        det.focus_score(img)
    torch.cuda.synchronize()
    det.timing_enable(20)
    for _ in range(20):
        s = det.focus_score(img)
    torch.cuda.synchronize()
    t = det.timing_read()
    avg = [sum(r[i] for r in t) / len(t) for i in range(4)]
    print(f"{n}^2: stages (ms) " + " ".join(f"{a:.4f}" for a in avg) + f"  total {sum(avg):.4f}  score {float(s[0])}")
