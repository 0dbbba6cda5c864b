"""C3 (one 4096^2 u8 tile, sigma 1-10, 10 scales) with the LoG response on both
schedules (k_tc2 default, the CUDA-core pair kernels with schedule="band"): device ms."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

img = synth.em_tile(4096, 4096, 1000, defocus=0.0, dose=300.0, device="cuda").unsqueeze(0)
for sch in (None, "band"):
    det = mhfd.Detector(4096, 4096, 1.0, 10.0, 10, threshold=0.1, overlap=0.5, response="log", schedule=sch)
    for _ in range(3):
        s = det.focus_score(img)
    torch.cuda.synchronize()
    det.timing_enable(10)
    for _ in range(10):
        s = det.focus_score(img)
    torch.cuda.synchronize()
    t = det.timing_read()
    avg = [sum(r[i] for r in t) / len(t) for i in range(4)]
    print(f"LoG {det.schedule('u8'):32s} stages (ms) " + " ".join(f"{a:.4f}" for a in avg) +
          f"  total {sum(avg):.4f}  score {float(s[0])}")
