"""Device time of one focus_score call against the batch size B (4096^2 u8, sigma 1-10,
n 10): the per-call overhead that the e2e chunk plan pays per chunk."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * (b % 9), dose=300.0, device="cuda")
                    for b in range(32)])
det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for B in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32):
    x = imgs[:B].contiguous()
    for _ in range(3):
        det.focus_score(x)
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        e0.record()
        det.focus_score(x)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    m = statistics.median(ms)
    det.timing_enable(10)
    for _ in range(10):
        det.focus_score(x)
    torch.cuda.synchronize()
    t = det.timing_read()
    st = [sum(r[i] for r in t) / len(t) for i in range(4)]
    print(f"B {B:3d}: {m:.3f} ms  {m / B:.4f} ms/image  overhead vs 0.3025*B: {m - 0.3025 * B:+.3f} ms  "
          f"stages/image (pct, blur, nms, prune) " + " ".join(f"{a / B:.4f}" for a in st))
