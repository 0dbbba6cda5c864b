"""Per-stage device times of focus_score on a 4096^2 batch for several overlap values
(overlap 1 skips the pruning rounds and the row-block index): where pruning time goes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * (b % 9), dose=300.0, device="cuda")
                    for b in range(B)])
for ov in (0.5, 0.1, 1.0):
    det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=ov)
    for _ in range(2):
        det.focus_score(imgs)
    torch.cuda.synchronize()
    det.timing_enable(5)
    for _ in range(5):
        s = det.focus_score(imgs)
    torch.cuda.synchronize()
    t = det.timing_read()
    avg = [sum(r[i] for r in t) / len(t) for i in range(4)]
    print(f"overlap {ov}: stages ms {['%.3f' % a for a in avg]} mean score {float(s.mean()):.1f}")
