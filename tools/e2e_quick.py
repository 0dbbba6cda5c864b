"""End-to-end (pinned host batch -> scores) time of 64 x 4096^2 u8 through
mhfd_focus_score_host with bench.py's chunk size, against the device-resident call."""
import os
import statistics
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, n=5):
    for _ in range(2):
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


ch = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = t(lambda: det.focus_score(imgs))
e2e = t(lambda: det.focus_score_host(host, chunk=ch))


def five():   # five back-to-back calls, no synchronisation between them (bench.py's e2e loop)
    for _ in range(5):
        det.focus_score_host(host, chunk=ch)


e2e5 = t(five, 3) / 5
cp = t(lambda: imgs.copy_(host, non_blocking=True))
print(f"device {dev:.2f} ms, e2e chunk {ch}: one call {e2e:.2f} ms ({B * 16.777216 / e2e * 1e3:.0f} MPix/s), "
      f"5 back-to-back calls {e2e5:.2f} ms per call ({B * 16.777216 / e2e5 * 1e3:.0f} MPix/s), "
      f"plain H2D copy {cp:.2f} ms ({B * 16.777216 / cp:.1f} GB/s)")
