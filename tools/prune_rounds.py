"""Decision rounds of the pruning kernel (MHFD_PRUNE_TRACE) and prune-stage device time
for a single 1024^2 tile (C2) and a 16 x 4096^2 batch, overlap 0.5 vs 1.0 (no rounds)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

for n, B in ((1024, 1), (4096, 16)):
    imgs = torch.stack([synth.em_tile(n, n, 11 + b, defocus=0.5 * (b % 9), dose=300.0, device="cuda") for b in range(B)])
    for ov in (0.5, 1.0):
        det = mhfd.Detector(n, n, 1.0, 10.0, 10, threshold=0.09, overlap=ov)
        for _ in range(3):
            det.focus_score(imgs)
        torch.cuda.synchronize()
        os.environ["MHFD_PRUNE_TRACE"] = "1"
        det.focus_score(imgs)
        torch.cuda.synchronize()
        os.environ.pop("MHFD_PRUNE_TRACE")
        det.timing_enable(10)
        for _ in range(10):
            det.focus_score(imgs)
        torch.cuda.synchronize()
        t = det.timing_read()
        avg = [sum(r[i] for r in t) / len(t) for i in range(4)]
        print(f"{B} x {n}^2 overlap {ov}: stages ms " + " ".join(f"{a:.4f}" for a in avg), flush=True)
