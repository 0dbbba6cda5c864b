"""e2e (pinned host batch -> scores) time of focus_score_host for several chunk sizes."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

B = 64
imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * (b % 9), dose=300.0, device="cuda")
                    for b in range(B)])
host = imgs.cpu().pin_memory()
det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
dev = det.focus_score(imgs)
torch.cuda.synchronize()
for chunk in (1, 2, 4, 8, 16):
    for _ in range(2):
        det.focus_score_host(host, chunk=chunk)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(5):
        hs = det.focus_score_host(host, chunk=chunk)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 5
    assert torch.equal(hs, dev.cpu())
    print(f"chunk {chunk:2d}: {ms:.2f} ms/step, {B * 4096 * 4096 / ms / 1e3:.0f} MPix/s")
