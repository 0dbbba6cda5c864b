"""Device time of one focus_score call on u16 tiles (C2/C3 sizes, sigma 1-10, 10 scales)
for the fused generic schedule (MHFD_SCHEDULE=generic) vs the default two-pass pair schedule.
Measured (B200): 1024^2 0.381 vs 0.222 ms; 4096^2 2.31 vs 1.51 ms; 8 x 4096^2 15.3 vs 10.8 ms."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

for n, B in ((1024, 1), (4096, 1), (4096, 8)):
    img = synth.em_tile(n, n, 1000, defocus=0.0, dose=300.0, bits=16, device="cuda")
    img = torch.from_numpy(img.to(torch.int32).cpu().numpy().astype(np.uint16)).cuda()
    imgs = img.unsqueeze(0).repeat(B, 1, 1).contiguous()
    for sched in ("generic", None):
        det = mhfd.Detector(n, n, 1.0, 10.0, 10, threshold=0.09, overlap=0.5, schedule=sched)
        for _ in range(3):
            det.focus_score(imgs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(7):
            e0.record()
            s = det.focus_score(imgs)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        print(f"{B} x {n}^2 u16 {det.schedule('u16'):28s} {statistics.median(ms):8.3f} ms  score {float(s[0])}",
              flush=True)
