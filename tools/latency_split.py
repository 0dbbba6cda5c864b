"""Per-stage device times of one focus_score call on a single u8 tile (C2 1024^2, C3
4096^2; sigma 1-10, 10 scales) and, with --launches, nothing else (for an ncu launch
list): where the single-image latency goes (percentiles, blur+DoG+argmax, NMS+compaction,
pruning)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

sizes = [int(a) for a in sys.argv[1:] if a.isdigit()] or [1024, 4096]
for n in sizes:
    img = synth.em_tile(n, n, 11, defocus=0.0, dose=300.0, device="cuda").unsqueeze(0)
    for ov in (0.5, 1.0):
        det = mhfd.Detector(n, n, 1.0, 10.0, 10, threshold=0.09, overlap=ov)
        for _ in range(3):
            det.focus_score(img)
        torch.cuda.synchronize()
        det.timing_enable(20)
        for _ in range(20):
            s = det.focus_score(img)
        torch.cuda.synchronize()
        t = det.timing_read()
        avg = [sum(r[i] for r in t) / len(t) for i in range(4)]
        print(f"{n}^2 overlap {ov}: stages (ms) " + " ".join(f"{a:.4f}" for a in avg) +
              f"  total {sum(avg):.4f}  score {float(s[0])}")
