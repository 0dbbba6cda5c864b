"""Quick k_tc2 check: v / argmax of the two-pass tensor-core schedule against the CUDA-core
pair kernels (schedule="band") on u16 tiles, then device times of one 4096^2 u16 tile
(sigma 1-10, 10 scales) and the C5 tile (8192^2 u16, sigma 1-30, 20 scales)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402


def u16(t):
    return torch.from_numpy(t.to(torch.int32).cpu().numpy().astype(np.uint16)).cuda()


def timeit(fn, n=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(n):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


for (size, sig, n) in ((512, (1.0, 5.0), 5), (1024, (1.0, 10.0), 10)):
    img = u16(synth.em_tile(size, size, 1000, defocus=0.0, dose=300.0, bits=16, device="cuda"))
    tau = 0.1 * (sig[1] - sig[0]) / n
    a = mhfd.Detector(size, size, sig[0], sig[1], n, threshold=tau)
    b = mhfd.Detector(size, size, sig[0], sig[1], n, threshold=tau, schedule="band")
    da, db = a.debug_dump(img, dog=False, cands=False), b.debug_dump(img, dog=False, cands=False)
    torch.cuda.synchronize()
    dv = float((da["v"] - db["v"]).abs().max())
    mism = float((da["idx"] != db["idx"]).float().mean())
    print(f"{size}^2 {a.schedule('u16')} vs {b.schedule('u16')}: max|dv| {dv:.3e} (max v {float(db['v'].max()):.3f}),"
          f" argmax mismatch {mism:.2e}, scores {float(a.focus_score(img)[0])} {float(b.focus_score(img)[0])}",
          flush=True)
for (size, sig, n, tau) in ((4096, (1.0, 10.0), 10, 0.09), (8192, (1.0, 30.0), 20, 0.145)):
    img = u16(synth.em_tile(size, size, 7, defocus=0.0, dose=300.0, bits=16, device="cuda")).unsqueeze(0)
    a = mhfd.Detector(size, size, sig[0], sig[1], n, threshold=tau)
    a.timing_enable(8)
    t = timeit(lambda: a.focus_score(img))
    st = a.timing_read()[-1]
    print(f"{size}^2 u16 sigma {sig} n {n}: {a.schedule('u16')} {t:.3f} ms (stages {[round(x, 3) for x in st]})",
          flush=True)
