"""DoG error of the CUDA path against the oracle relative to the peak P (the parity
tolerance is 1e-4 P): one 1024^2 u8 tile, sigma 1-10, 10 scales, defocus 0 and 2.
Run with MHFD_LIB pointing at an experiment build to see what a numerics change costs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402

for dfc in (0.0, 2.0):
    a = synth.em_tile_np(1024, 1024, 1000, defocus=dfc, dose=300.0, bits=8)
    det = mhfd.Detector(1024, 1024, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
    d = det.debug_dump(torch.from_numpy(a), dog=True, cands=False)
    torch.cuda.synchronize()
    ref = oracle.detect(a, 1.0, 10.0, 10, 0.09, 0.5, dump=True)
    D = ref["D"]
    P = float(D.max())
    e = np.abs(d["dog"][0].cpu().numpy().astype(np.float64) - D)
    per = [float(e[i].max()) / P for i in range(e.shape[0])]
    print(f"{os.path.basename(os.environ.get('MHFD_LIB', 'libmhfd.so'))} defocus {dfc}: max err/P {max(per):.2e}  "
          f"per plane " + " ".join(f"{x:.1e}" for x in per) + f"  schedule {det.schedule('u8')}")
