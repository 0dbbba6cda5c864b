"""Per-chunk device stage times inside one focus_score_host call (64 x 4096^2 u8, chunks
of 8): are the chunks slower than the device-resident run (interference), or are there
gaps (waiting on copies)?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

B = 64
imgs = torch.stack([synth.em_tile(4096, 4096, 1000 + b, defocus=0.5 * (b % 9), dose=300.0, device="cuda")
                    for b in range(B)])
host = imgs.cpu().pin_memory()
det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
for _ in range(2):
    det.focus_score_host(host, chunk=8)
    det.focus_score(imgs[:8].contiguous())
torch.cuda.synchronize()
det.timing_enable(16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
det.focus_score_host(host, chunk=8)
e1.record()
torch.cuda.synchronize()
t = det.timing_read()
tot = [sum(r) for r in t]
print(f"wall (events) {e0.elapsed_time(e1):.2f} ms; chunks {len(t)}; sum of chunk device times {sum(tot):.2f} ms")
for i, r in enumerate(t):
    print(i, " ".join(f"{x:.3f}" for x in r), f"= {sum(r):.3f}")
det.timing_enable(4)
x = imgs[:8].contiguous()
for _ in range(4):
    det.focus_score(x)
torch.cuda.synchronize()
t = det.timing_read()
print("device-resident B=8:", [round(sum(r), 3) for r in t])
