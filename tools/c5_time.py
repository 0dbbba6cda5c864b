"""Device time of one 8192^2 u16 tile, sigma 1-30, 20 scales (config C5), per schedule knob."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

img = synth.em_tile(8192, 8192, 7, defocus=0.0, dose=300.0, bits=16, device="cuda")
img = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16)).cuda().unsqueeze(0)
det = mhfd.Detector(8192, 8192, 1.0, 30.0, 20, threshold=0.145, overlap=0.5)
for _ in range(2):
    s = det.focus_score(img)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(5):
    e0.record()
    s = det.focus_score(img)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
print(f"C5 {os.environ.get('MHFD_NO_BH384') and 'BH<=256' or 'auto'}: {statistics.median(ms):.2f} ms, score {float(s[0])}")
