"""Single-image latency through a CUDA graph: one focus_score call (C2 1024^2 / C3 4096^2
u8) captured once with torch.cuda.graph and replayed (the call is stream-ordered, no host
synchronisation, so it captures whole), against the eager call.  Device time by CUDA
events; host-visible = wall time of replay + synchronize."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12050_b200 as mhfd  # noqa: E402
import synth  # noqa: E402


def ev(fn, n=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    d, w = [], []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        w.append((time.perf_counter() - t0) * 1e3)
        d.append(e0.elapsed_time(e1))
    return statistics.median(d), statistics.median(w)


for n in (1024, 4096):
    img = synth.em_tile(n, n, 11, defocus=0.0, dose=300.0, device="cuda").unsqueeze(0).contiguous()
    det = mhfd.Detector(n, n, 1.0, 10.0, 10, threshold=0.09, overlap=0.5)
    ref = float(det.focus_score(img)[0])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        det.focus_score(img)   # workspace allocated outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = det.focus_score(img)
    g.replay()
    torch.cuda.synchronize()
    assert float(out[0]) == ref, (float(out[0]), ref)
    de, we = ev(lambda: det.focus_score(img))
    dg, wg = ev(lambda: g.replay())
    print(f"{n}^2: eager device {de:.4f} ms host-visible {we:.4f} ms | graph device {dg:.4f} ms host-visible "
          f"{wg:.4f} ms | score {ref}", flush=True)
